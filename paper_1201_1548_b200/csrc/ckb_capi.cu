#include <cstdlib>
#include <algorithm>
// C-ABI boundary of the B200 modular symbolic engine (declared in
// include/curvekit_b200.h).  Plain pointers and sizes only; every host buffer
// is caller-owned and never retained; device memory is owned by a
// process-global context; calls are serialised by a mutex.  Return value:
// 0 ok, > 0 recoverable (see CKB_STATUS_*), < 0 CUDA/usage failure with the
// message in ckb_last_error().
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <chrono>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/curvekit_b200.h"
#include "ckb_kernels.cuh"
#include <dlfcn.h>
#include <nccl.h>

using namespace ckb;

namespace {

thread_local std::string g_err;

int fail(const std::string& msg, int code = -1) {
  g_err = msg;
  return code;
}

#define CK(call)                                                                          \
  do {                                                                                    \
    cudaError_t e_ = (call);                                                              \
    if (e_ != cudaSuccess)                                                                \
      return fail(std::string(#call) + ": " + cudaGetErrorString(e_) + " @" + __FILE__ + \
                  ":" + std::to_string(__LINE__));                                        \
  } while (0)

struct Buf {
  void* p = nullptr;
  size_t n = 0;
};

struct CrtEntry {
  std::vector<uint32_t> primes;
  int LW = 0;
  Prime* d_primes = nullptr;
  void* d_blob = nullptr;  // p, c, cc, pinvd, Mi, Ml, Mh
  void* d_bt = nullptr;    // tensor-core byte table
  CrtTables t;
  uint64_t last_use = 0;
};

struct Ctx {
  bool ready = false;
  int device = -1;
  cudaStream_t stream = nullptr;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  std::map<std::string, Buf> dev;
  std::map<std::string, Buf> host;  // pinned staging
  std::vector<CrtEntry> crt;
  uint64_t tick = 0;
  uint64_t launches = 0;
  bool timing = false;
  cudaEvent_t sev[8] = {};
  int nsev = 0;
  uint64_t epoch = 0;  // bumped whenever a buffer or table a captured graph may reference is freed
  bool graphs = true;  // CKB_NO_GRAPHS=1 disables graph replay
  std::string ns;      // buffer-name prefix: each problem of a batch owns its buffers
  cudaStream_t bst[4] = {};  // streams of the batched entry (created on first use)
  const uint32_t* last_fail = nullptr;  // fallback counter of the last pipeline call (device)
  cudaStream_t last_stream = nullptr;   // ... and the stream that call ran on
  uint64_t last_images = 0;
  cudaEvent_t bev[4] = {};
};

// One context per device (index = position in the device list of
// ckb_init_devices; ckb_init(device) sets up context 0 only).  Every entry point
// works on context 0 unless the multi-device call has switched g_ci.
constexpr int kMaxCtx = 8;
Ctx g_ctxs[kMaxCtx];
float g_host_times[2] = {0.f, 0.f};
int g_ci = 0;     // current context
int g_nctx = 0;   // contexts initialised by ckb_init_devices (1 after ckb_init)
#define g (g_ctxs[g_ci])
std::mutex g_mu;
// dynamic shared memory a per-problem kernel may ask for; beyond it the
// operands live in a global scratch slice per problem (L2-resident in practice)
constexpr size_t kSmemLimit = 200 * 1024;
}  // namespace
namespace ckb {
bool g_pdl = true;
}
namespace {

// ---- Descartes sign-variation test ------------------------------------------
// A handle holds one polynomial's residues modulo a prefix of PRIMES30-style
// primes and the per-(primes, n) plan; each test then needs only the interval.
struct DescHandle {
  bool used = false;
  int n = 0, K = 0;
  std::vector<uint32_t> primes, gens;
  void* blob = nullptr;  // residues [K][n+1] then the plan tables
  DescPlan pl;
  uint32_t* d_res = nullptr;
  Prime* d_primes = nullptr;
};
std::vector<DescHandle> g_desc;

// CKB_POISON=1 (checking runs; also disables graphs): every scratch buffer is
// filled with a poison byte each time a call fetches it (alternating 0xA5 /
// 0xFF between fetches), so a kernel reading scratch no earlier kernel of the
// same call wrote changes the result and fails the parity tests
int poison_mode() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("CKB_POISON");
    v = (e && e[0] == '1') ? 1 : 0;
  }
  return v;
}

int dev_buf(const char* name, size_t bytes, void** out) {
  Buf& b = g.dev[g.ns + name];
  if (b.n < bytes) {
    if (b.p) cudaFree(b.p);
    ++g.epoch;
    b.p = nullptr;
    b.n = 0;
    size_t want = bytes + bytes / 4 + 256;
    CK(cudaMalloc(&b.p, want));
    b.n = want;
  }
  if (poison_mode()) {
    static unsigned n = 0;
    CK(cudaStreamSynchronize(g.stream));
    CK(cudaMemset(b.p, (n++ & 1) ? 0xFF : 0xA5, b.n));
    CK(cudaDeviceSynchronize());
  }
  *out = b.p;
  return 0;
}

int host_buf(const char* name, size_t bytes, void** out) {
  Buf& b = g.host[g.ns + name];
  if (b.n < bytes) {
    if (b.p) cudaFreeHost(b.p);
    ++g.epoch;
    b.p = nullptr;
    b.n = 0;
    size_t want = bytes + bytes / 4 + 256;
    // portable: every device's copy engine may read / write it (multi-device calls)
    CK(cudaHostAlloc(&b.p, want, cudaHostAllocPortable));
    b.n = want;
  }
  *out = b.p;
  return 0;
}

template <typename T>
int dbuf(const char* name, size_t count, T** out) {
  void* p;
  int rc = dev_buf(name, count * sizeof(T) + 16, &p);
  *out = (T*)p;
  return rc;
}

// ---- host arithmetic for the tables ----------------------------------------
uint32_t h_inv32(uint32_t p) {
  uint32_t x = p;
  for (int i = 0; i < 5; ++i) x *= 2u - p * x;
  return x;
}
uint32_t h_powmod(uint64_t a, uint64_t e, uint32_t p) {
  uint64_t r = 1 % p;
  a %= p;
  while (e) {
    if (e & 1) r = r * a % p;
    a = a * a % p;
    e >>= 1;
  }
  return (uint32_t)r;
}
Prime h_prime(uint32_t p) {
  Prime P;
  P.p = p;
  P.pinv = h_inv32(p);
  uint64_t r1 = (1ull << 32) % p;
  P.r2 = (uint32_t)(r1 * r1 % p);
  return P;
}
uint32_t h_mont(uint64_t x, uint32_t p) { return (uint32_t)(((x % p) << 32) % p); }

int check_primes(const uint32_t* primes, int K) {
  for (int i = 0; i < K; ++i) {
    uint32_t p = primes[i];
    if (p < 3 || !(p & 1u) || p >= 0x80000000u) return fail("prime out of range (odd, 3 <= p < 2^31): " + std::to_string(p), -2);
  }
  return 0;
}

int upload_primes(const uint32_t* primes, int K, Prime** d_out) {
  Prime* hp;
  void* hv;
  int rc = host_buf("primes", sizeof(Prime) * K, &hv);
  if (rc) return rc;
  hp = (Prime*)hv;
  for (int i = 0; i < K; ++i) hp[i] = h_prime(primes[i]);
  Prime* d;
  if ((rc = dbuf("primes", K, &d))) return rc;
  CK(cudaMemcpyAsync(d, hp, sizeof(Prime) * K, cudaMemcpyHostToDevice, g.stream));
  *d_out = d;
  return 0;
}

int get_crt(const uint32_t* primes, int K, int LW, CrtEntry** out) {
  // the u8 tensor-core product accumulates 4K * 255^2 per s32 entry
  if (K > 8192) return fail("CRT over more than 8192 primes is not supported (s32 accumulation bound)", -2);
  for (auto& e : g.crt) {
    if ((int)e.primes.size() == K && e.LW == LW && !memcmp(e.primes.data(), primes, 4 * (size_t)K)) {
      e.last_use = ++g.tick;
      *out = &e;
      return 0;
    }
  }
  if (g.crt.size() >= 64) {  // evict least recently used (an entry is ~1-25 MB)
    size_t v = 0;
    for (size_t i = 1; i < g.crt.size(); ++i)
      if (g.crt[i].last_use < g.crt[v].last_use) v = i;
    CrtEntry& e = g.crt[v];
    cudaFree(e.d_primes);
    cudaFree(e.d_blob);
    cudaFree(e.d_bt);
    g.crt.erase(g.crt.begin() + v);
    ++g.epoch;
  }
  CrtEntry e;
  e.primes.assign(primes, primes + K);
  e.LW = LW;
  std::vector<Prime> hp(K);
  for (int i = 0; i < K; ++i) hp[i] = h_prime(primes[i]);
  // M = prod p_i as LW limbs
  std::vector<uint32_t> M(LW + 1, 0);
  M[0] = 1;
  for (int j = 0; j < K; ++j) {
    uint64_t carry = 0;
    for (int l = 0; l <= LW; ++l) {
      uint64_t t = (uint64_t)M[l] * primes[j] + carry;
      M[l] = (uint32_t)t;
      carry = t >> 32;
    }
  }
  if (M[LW]) return fail("CRT output width too small for the prime product", -2);
  std::vector<uint32_t> Mh(LW);
  std::vector<double> pinvd(K);
  for (int i = 0; i < K; ++i) pinvd[i] = 1.0 / (double)primes[i];
  {
    uint32_t carry = 0;
    for (int l = LW - 1; l >= 0; --l) {
      Mh[l] = (M[l] >> 1) | (carry << 31);
      carry = M[l] & 1u;
    }
  }
  const size_t nb = 4 * (size_t)K * 3 + 8 * (size_t)K + 4 * (size_t)K * LW + 8 * (size_t)LW + 64;
  CK(cudaMalloc(&e.d_primes, sizeof(Prime) * K));
  CK(cudaMalloc(&e.d_blob, nb + 16));
  uint8_t* b = (uint8_t*)e.d_blob;
  double* d_pinvd = (double*)b;  // 8-byte aligned first
  uint32_t* d_p = (uint32_t*)(b + 8 * (size_t)K);
  uint32_t* d_c = d_p + K;
  uint32_t* d_cc = d_c + K;
  uint32_t* d_Mi = d_cc + K;
  uint32_t* d_Ml = d_Mi + (size_t)K * LW;
  uint32_t* d_Mh = d_Ml + LW;
  uint32_t* d_bad = d_Mh + LW;  // one flag word (in the blob's spare bytes)
  CK(cudaMemcpy(e.d_primes, hp.data(), sizeof(Prime) * K, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(d_pinvd, pinvd.data(), 8 * (size_t)K, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(d_p, primes, 4 * (size_t)K, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(d_Ml, M.data(), 4 * (size_t)LW, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(d_Mh, Mh.data(), 4 * (size_t)LW, cudaMemcpyHostToDevice));
  CK(cudaMemset(d_bad, 0, 4));
  // M / p_i and (M / p_i)^-1 mod p_i on the device (one thread per prime)
  launch_crt_tables(d_p, K, d_Ml, LW, d_Mi, d_c, d_cc, d_bad, g.stream);
  CK(cudaGetLastError());
  uint32_t hbad = 0;
  CK(cudaMemcpyAsync(&hbad, d_bad, 4, cudaMemcpyDeviceToHost, g.stream));
  CK(cudaStreamSynchronize(g.stream));
  if (hbad) {
    cudaFree(e.d_primes);
    cudaFree(e.d_blob);
    return fail("CRT primes are not pairwise distinct", -2);
  }
  e.t.K = K;
  e.t.LW = LW;
  e.t.p = d_p;
  e.t.c = d_c;
  e.t.cc = d_cc;
  e.t.pinvd = d_pinvd;
  e.t.Mi = d_Mi;
  e.t.Ml = d_Ml;
  e.t.Mh = d_Mh;
  CK(cudaMalloc(&e.d_bt, crt_btable_bytes(K, LW)));
  launch_crt_btable(K, LW, d_Mi, (uint32_t*)e.d_bt, g.stream);
  CK(cudaGetLastError());
  CK(cudaStreamSynchronize(g.stream));
  e.t.Bt = (const uint8_t*)e.d_bt;
  e.last_use = ++g.tick;
  g.crt.push_back(e);
  *out = &g.crt.back();
  return 0;
}

bool is_pinned(const void* p) {
  cudaPointerAttributes at;
  if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return at.type == cudaMemoryTypeHost;
}

void* pinned_alloc(size_t bytes) {
  void* p = nullptr;
  return cudaMallocHost(&p, bytes) == cudaSuccess ? p : nullptr;
}

void stage_mark(cudaStream_t st) {
  if (g.timing && g.nsev < 8) cudaEventRecord(g.sev[g.nsev++], st);
}

struct PrimeEntry {
  std::vector<uint32_t> primes;
  Prime* d = nullptr;
};
std::vector<PrimeEntry> g_pcache_[kMaxCtx];
#define g_pcache (g_pcache_[g_ci])

int get_primes_dev(const uint32_t* primes, int K, Prime** out) {
  for (auto& e : g_pcache)
    if ((int)e.primes.size() == K && !memcmp(e.primes.data(), primes, 4 * (size_t)K)) {
      *out = e.d;
      return 0;
    }
  if (g_pcache.size() >= 16) {
    cudaFree(g_pcache.front().d);
    g_pcache.erase(g_pcache.begin());
    ++g.epoch;
  }
  PrimeEntry e;
  e.primes.assign(primes, primes + K);
  std::vector<Prime> hp(K);
  for (int i = 0; i < K; ++i) hp[i] = h_prime(primes[i]);
  CK(cudaMalloc(&e.d, sizeof(Prime) * K));
  CK(cudaMemcpy(e.d, hp.data(), sizeof(Prime) * K, cudaMemcpyHostToDevice));
  g_pcache.push_back(e);
  *out = g_pcache.back().d;
  return 0;
}

int ensure_ready() {
  if (!g.ready) return fail("ckb_init() has not been called", -3);
  CK(cudaSetDevice(g.device));
  return 0;
}

cudaStream_t pick_stream(void* s) { return s ? (cudaStream_t)s : g.stream; }

// ---- interpolation plans, cached per (primes, generators, N) -----------------
struct PlanEntry {
  std::vector<uint32_t> primes, gens;
  int N = 0, S = 1;
  InterpPlan pl;
  void* blob = nullptr;
  void* ab = nullptr;  // tensor-core interpolation matrix (polyphase plans), or nullptr
  size_t bytes = 0;
  uint64_t last_use = 0;
};
std::vector<PlanEntry> g_plans_[kMaxCtx];
// plans are input independent (like FFT plans) and rebuilt cold in 5-40 ms: a
// Bisolve-style caller with many distinct (primes, N) keeps up to kPlanMax of
// them, within kPlanBytes of HBM per device (a cfg4 plan is ~40 MB)
constexpr size_t kPlanMax = 32;
constexpr size_t kPlanBytes = (size_t)8 << 30;
#define g_plans (g_plans_[g_ci])

// Nfull points per prime, polyphase factor S (1 or 8): the interpolation plan
// has M = ceil(Nfull / S) points with ratio g^S
int get_plan(const uint32_t* primes, const uint32_t* gens, int K, int Nfull, int S, InterpPlan* out) {
  for (auto& e : g_plans)
    if (e.N == Nfull && e.S == S && (int)e.primes.size() == K && !memcmp(e.primes.data(), primes, 4 * (size_t)K) &&
        !memcmp(e.gens.data(), gens, 4 * (size_t)K)) {
      e.last_use = ++g.tick;
      *out = e.pl;
      return 0;
    }
  const int N = (Nfull + S - 1) / S;
  int logL = 0;
  while ((1 << logL) < 2 * N - 1) ++logL;
  if (logL > 14) return fail("interpolation supports N <= 8192 points (NTT length <= 2^14)", -2);
  const uint32_t L = 1u << logL;
  for (int i = 0; i < K; ++i)
    if ((primes[i] - 1) % L) return fail("pipeline primes must be 1 mod the NTT length (use PRIMES30)", -2);
  auto plan_bytes = [&]() {
    size_t t = 0;
    for (auto& e : g_plans) t += e.bytes;
    return t;
  };
  while (!g_plans.empty() && (g_plans.size() >= kPlanMax || plan_bytes() > kPlanBytes)) {
    size_t v = 0;
    for (size_t i = 1; i < g_plans.size(); ++i)
      if (g_plans[i].last_use < g_plans[v].last_use) v = i;
    cudaFree(g_plans[v].blob);
    if (g_plans[v].ab) cudaFree(g_plans[v].ab);
    g_plans.erase(g_plans.begin() + v);
    ++g.epoch;
  }
  PlanEntry e;
  e.primes.assign(primes, primes + K);
  e.gens.assign(gens, gens + K);
  e.N = Nfull;
  e.S = S;
  InterpPlan& pl = e.pl;
  pl.N = N;
  pl.K = K;
  pl.S = S;
  pl.Nfull = Nfull;
  pl.L = (int)L;
  pl.logL = logL;
  const size_t kn = (size_t)K * N, kn1 = (size_t)K * (N + 1), kl = (size_t)K * L, kh = kl / 2;
  const size_t words =
      kn * 10 + kn1 * 3 + kh * 4 + kl * 4 + (size_t)K * 5 + (size_t)K * 4 * S + (S > 1 ? 2 * (size_t)S * kn : 0) + 256;
  CK(cudaMalloc(&e.blob, 4 * words));
  e.bytes = 4 * words;
  uint32_t* b = (uint32_t*)e.blob;
  // every table 16-byte aligned (the interpolation stages them with 16-byte cp.async)
  auto take = [&](size_t n) { uint32_t* r = b; b += (n + 3) & ~(size_t)3; return r; };
  pl.yq = take(kn);
  pl.yqi = take(kn);
  pl.om = take((size_t)K * 4 * S);
  pl.xq = take(kn);
  pl.hC = take(2 * kn);
  pl.hCinv = take(kn);
  pl.z = take(kn);
  pl.zc = take(kn);
  pl.sS = take(kn);
  pl.sSc = take(kn);
  pl.Mt = take(kn1);
  pl.phi = take(kn1);
  pl.iphi = take(kn1);
  pl.W = take(kh);
  pl.Wc = take(kh);
  pl.Wi = take(kh);
  pl.Wic = take(kh);
  pl.Hf = take(kl);
  pl.Hfc = take(kl);
  pl.Mf = take(kl);
  pl.Mfc = take(kl);
  pl.Linv = take(K);
  pl.zr = S > 1 ? take((size_t)S * kn) : nullptr;
  pl.zrc = S > 1 ? take((size_t)S * kn) : nullptr;
  uint32_t* d_gens = take(K);
  Prime* d_primes = reinterpret_cast<Prime*>(take((size_t)K * 3));
  std::vector<Prime> hp(K);
  for (int i = 0; i < K; ++i) hp[i] = h_prime(primes[i]);
  CK(cudaMemcpy(d_gens, gens, 4 * (size_t)K, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(d_primes, hp.data(), sizeof(Prime) * K, cudaMemcpyHostToDevice));
  launch_plan_base(d_primes, d_gens, pl, g.stream);
  launch_plan_ntt(d_primes, d_gens, pl, g.stream);
  pl.Ab = nullptr;
  {
    // the interpolation as a tensor-core product: the per-prime inverse
    // Vandermonde in bytes (input independent), when it is small enough
    // (cfg4: 37 MB; <= 16 K-steps of 32 bytes for the kernel's shared memory).  At cfg5 (1.3 GB of
    // matrix bytes) the NTT path measured faster: 546 vs 601 us.  CKB_INTERP_MMA=0 disables.
    const char* env = getenv("CKB_INTERP_MMA");
    int kch, mt;
    const size_t ab = interp_mma_bytes(K, N, &kch, &mt);
    if (S > 1 && !(env && env[0] == '0') && kch <= 16 && ab <= ((size_t)512 << 20)) {
      CK(cudaMalloc(&e.ab, ab));
      e.bytes += ab;
      pl.Ab = (uint8_t*)e.ab;
      launch_interp_lagrange(d_primes, pl, pl.Ab, g.stream);
    }
  }
  CK(cudaGetLastError());
  CK(cudaStreamSynchronize(g.stream));
  e.last_use = ++g.tick;
  g_plans.push_back(e);
  *out = pl;
  return 0;
}

// the modular part of the pipeline on device buffers:
// limbs -> residues -> choose c -> images -> interpolated coefficients [K][N]
// ---- CUDA graphs of a call's launch sequence --------------------------------
// The device work of a pipeline call depends only on its shapes, primes,
// degrees and buffer addresses.  The first call with a key runs eagerly (it
// builds the cached plan and tables); the second is captured into a graph;
// later ones replay it with one launch.  A graph is dropped when any buffer or
// table it may reference is freed (g.epoch), and a key whose capture fails
// (an allocation or a synchronising call inside) stays eager.
struct GraphEntry {
  std::vector<uint64_t> key;
  uint64_t epoch = 0;
  cudaGraphExec_t exec = nullptr;
  uint64_t launches = 0;  // kernels per replay (for ckb_launch_count)
  int seen = 0;           // < 0: not capturable
  uint64_t last_use = 0;
};
std::vector<GraphEntry> g_graphs_[kMaxCtx];
#define g_graphs (g_graphs_[g_ci])

void drop_graphs() {
  for (auto& e : g_graphs)
    if (e.exec) cudaGraphExecDestroy(e.exec);
  g_graphs.clear();
}

template <class F>
int graphed(const std::vector<uint64_t>& key, cudaStream_t st, F&& body) {
  if (g.timing || !g.graphs) return body();
  GraphEntry* ge = nullptr;
  for (auto& e : g_graphs)
    if (e.key == key) ge = &e;
  if (ge && ge->epoch != g.epoch) {
    if (ge->exec) cudaGraphExecDestroy(ge->exec);
    ge->exec = nullptr;
    ge->seen = ge->seen < 0 ? ge->seen : 0;
    ge->epoch = g.epoch;
  }
  if (!ge) {
    if (g_graphs.size() >= 64) {
      size_t v = 0;
      for (size_t i = 1; i < g_graphs.size(); ++i)
        if (g_graphs[i].last_use < g_graphs[v].last_use) v = i;
      if (g_graphs[v].exec) cudaGraphExecDestroy(g_graphs[v].exec);
      g_graphs.erase(g_graphs.begin() + v);
    }
    GraphEntry e;
    e.key = key;
    e.epoch = g.epoch;
    g_graphs.push_back(e);
    ge = &g_graphs.back();
  }
  ge->last_use = ++g.tick;
  if (ge->exec) {
    CK(cudaGraphLaunch(ge->exec, st));
    g.launches += ge->launches;
    return 0;
  }
  if (ge->seen < 0 || ge->seen++ == 0) return body();
  const uint64_t l0 = g.launches, ep = g.epoch;
  CK(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
  const int rc = body();
  cudaGraph_t graph = nullptr;
  const cudaError_t ce = cudaStreamEndCapture(st, &graph);
  cudaGraphExec_t exec = nullptr;
  bool ok = rc == 0 && ce == cudaSuccess && graph != nullptr && g.epoch == ep;
  if (ok) ok = cudaGraphInstantiate(&exec, graph, 0) == cudaSuccess;
  if (graph) cudaGraphDestroy(graph);
  if (!ok) {
    cudaGetLastError();  // clear capture errors; run this call eagerly, never capture the key again
    for (auto& e : g_graphs)
      if (e.key == key) e.seen = -1;
    g.launches = l0;
    return body();
  }
  for (auto& e : g_graphs)
    if (e.key == key) {
      e.exec = exec;
      e.launches = g.launches - l0;
      e.epoch = g.epoch;
    }
  CK(cudaGraphLaunch(exec, st));
  return 0;
}

void key_push(std::vector<uint64_t>& k, const void* p, size_t bytes) {
  const uint8_t* b = (const uint8_t*)p;
  for (size_t i = 0; i < bytes; i += 8) {
    uint64_t w = 0;
    memcpy(&w, b + i, bytes - i < 8 ? bytes - i : 8);
    k.push_back(w);
  }
}

// structured inputs: a y-coefficient strictly inside the degree range vanishes identically (as in
// F(x, y^2)), so the remainder sequences of (almost) all images drop the degree by more than one --
// the subresultant coefficients vanish identically, for every point and shift.  Such inputs run the
// register kernel's any-degree elimination directly (CKB_STRUCTURED=0/1 forces the choice).
bool structured_input(const int16_t* h_degs, int m, int n) {
  static int force = -2;
  if (force == -2) {
    const char* e = getenv("CKB_STRUCTURED");
    force = e ? atoi(e) : -1;
  }
  if (force >= 0) return force != 0;
  for (int j = 1; j < m; ++j)
    if (h_degs[j] < 0) return true;
  for (int j = 1; j < n; ++j)
    if (h_degs[m + 1 + j] < 0) return true;
  return false;
}

int modular_stage(const uint32_t* d_limbs, int C, int L, const int16_t* d_degs, const int16_t* h_degs, int m,
                  int n, int dfx, int dgx, const Prime* d_primes, const uint32_t* h_primes, const uint32_t* h_gens,
                  int K, int N, uint32_t* d_coeffs, uint32_t* d_status, cudaStream_t st,
                  const CrtTables* crt = nullptr, const PeerOut* po = nullptr) {
  // with crt: the output rows are the explicit CRT's y = coeff (M/p_i)^-1 mod p_i
  for (int i = 0; i < K; ++i)
    if (h_primes[i] >= (1u << 30)) return fail("pipeline primes must be below 2^30", -2);
  uint32_t *d_red, *d_vals, *d_cval;
  int rc;
  InterpPlan pl;
  constexpr int S = 8;  // polyphase cosets (the images kernel's 8-lane groups)
  if ((rc = get_plan(h_primes, h_gens, K, N, S, &pl))) return rc;
  const int NI = S * pl.N;  // images per prime (>= N)
  // y-degrees above the register kernel's buckets, or tables too large for its
  // shared memory: every image goes through the general warp kernel
  const bool general = !images_fast_ok(m, n, dfx, dgx, NI, K);
  if ((rc = dbuf("red", (size_t)K * C, &d_red))) return rc;
  uint32_t* d_tab = nullptr;
  if (!general && (rc = dbuf("tab", (size_t)K * images_tab_words(m, n, dfx, dgx), &d_tab))) return rc;
  if ((rc = dbuf("vals", (size_t)K * NI, &d_vals))) return rc;
  if ((rc = dbuf("cval", (size_t)K, &d_cval))) return rc;
  uint32_t* d_fail;
  if ((rc = dbuf("fail", (size_t)K * NI + 1, &d_fail))) return rc;
  // the fail counter is zeroed by K1 (the images kernel runs after K1 completes)
  stage_mark(st);
  const int lcf_off = m * (dfx + 1), lcg_off = (m + 1) * (dfx + 1) + n * (dgx + 1);
  const bool merged = !general && reduce_tab_chooses(h_degs[m], h_degs[m + 1 + n]);
  if (general)
    launch_reduce(d_limbs, C, L, d_primes, K, d_red, st);
  else if (merged)  // K1 and the point scales in one launch
    launch_reduce_tab(d_limbs, C, L, d_primes, K, m, n, dfx, dgx, d_red, d_tab, st, &pl, lcf_off, h_degs[m],
                      lcg_off, h_degs[m + 1 + n], d_cval, d_status, d_fail + (size_t)K * NI);
  else
    launch_reduce_tab(d_limbs, C, L, d_primes, K, m, n, dfx, dgx, d_red, d_tab, st, nullptr, 0, 0, 0, 0, nullptr,
                      nullptr, d_fail + (size_t)K * NI);
  stage_mark(st);
  if (!merged)
    launch_choose_c(d_primes, pl, d_red, C, lcf_off, h_degs[m], lcg_off, h_degs[m + 1 + n], d_cval, d_status, st);
  stage_mark(st);
  ImageArgs a;
  a.red = d_red;
  a.tab = d_tab;
  a.degs = d_degs;
  a.yq = pl.yq;
  a.om = pl.om;
  a.cval = d_cval;
  a.primes = d_primes;
  a.C = C;
  a.m = m;
  a.n = n;
  a.dfx = dfx;
  a.dgx = dgx;
  a.N = NI;
  a.M = pl.N;
  a.K = K;
  a.values = d_vals;
  a.status = d_status;
  a.fail_list = d_fail;
  a.fail_count = a.fail_list + (size_t)K * NI;
  g.last_fail = general ? nullptr : a.fail_count;
  g.last_stream = st;
  g.last_images = (uint64_t)K * NI;
  if (general)
    launch_images_general(a, st);
  else
    launch_images(a, st, structured_input(h_degs, m, n));
  stage_mark(st);
  launch_interp(pl, d_primes, d_vals, d_cval, d_coeffs, st, crt ? crt->c : nullptr, crt ? crt->cc : nullptr, po);
  stage_mark(st);
  // reduce (+ choose when merged), [choose], images (general: iota + warp kernel), fallback, interpolation
  g.launches += general ? 5 : (merged ? 4 : 5);
  CK(cudaGetLastError());
  return 0;
}

// ---- per-device contexts -----------------------------------------------------
struct CtxSwitch {  // restores context 0 when a multi-device call returns
  ~CtxSwitch() {
    g_ci = 0;
    if (g_ctxs[0].ready) cudaSetDevice(g_ctxs[0].device);
  }
};

int init_ctx(int idx, int device) {
  g_ci = idx;
  int n = 0;
  CK(cudaGetDeviceCount(&n));
  if (device < 0 || device >= n) return fail("ckb_init: no such CUDA device " + std::to_string(device), -3);
  CK(cudaSetDevice(device));
  CK(cudaStreamCreateWithFlags(&g.stream, cudaStreamNonBlocking));
  CK(cudaEventCreate(&g.ev0));
  CK(cudaEventCreate(&g.ev1));
  for (int i = 0; i < 8; ++i) CK(cudaEventCreate(&g.sev[i]));
  g.device = device;
  {
    const char* e = getenv("CKB_NO_GRAPHS");
    g.graphs = !(e && e[0] == '1') && !poison_mode();
    const char* q = getenv("CKB_NO_PDL");
    ckb::g_pdl = !(q && q[0] == '1');
  }
  g.ready = true;
  return 0;
}

void shutdown_ctx() {
  if (!g.ready) return;
  cudaSetDevice(g.device);
  cudaStreamSynchronize(g.stream);
  drop_graphs();
  ++g.epoch;
  if (g_ci == 0) {
    for (auto& d : g_desc)
      if (d.blob) cudaFree(d.blob);
    g_desc.clear();
  }
  for (auto& kv : g.dev) cudaFree(kv.second.p);
  for (auto& kv : g.host) cudaFreeHost(kv.second.p);
  for (auto& e : g.crt) {
    cudaFree(e.d_primes);
    cudaFree(e.d_blob);
    cudaFree(e.d_bt);
  }
  for (auto& e : g_pcache) cudaFree(e.d);
  g_pcache.clear();
  for (auto& e : g_plans) {
    cudaFree(e.blob);
    if (e.ab) cudaFree(e.ab);
  }
  g_plans.clear();
  g.dev.clear();
  g.host.clear();
  g.crt.clear();
  cudaEventDestroy(g.ev0);
  cudaEventDestroy(g.ev1);
  for (int i = 0; i < 8; ++i) cudaEventDestroy(g.sev[i]);
  for (int i = 0; i < 4; ++i) {
    if (g.bst[i]) cudaStreamDestroy(g.bst[i]);
    if (g.bev[i]) cudaEventDestroy(g.bev[i]);
  }
  cudaStreamDestroy(g.stream);
  g = Ctx();
}

// ---- the residue exchange between device contexts --------------
// Default: folded into the interpolation (PeerOut): every context stores its
// residues straight into the owning context's CRT input -- over NVLink peer
// access between distinct devices, plainly when contexts share a device -- and
// each CRT waits on the other contexts' events.  Without peer access (or with
// CKB_EXCHANGE=nccl|copy) a separate step: NCCL point-to-point (ncclCommInitAll:
// one communicator per device in this process, loaded with dlopen so the
// library has no NCCL dependency on single-GPU hosts) or peer copies ordered by
// events.
struct NcclApi {
  void* h = nullptr;
  ncclResult_t (*CommInitAll)(ncclComm_t*, int, const int*) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};
struct Exchange {
  bool nccl = false;
  NcclApi api;
  ncclComm_t comms[kMaxCtx] = {};
  int n = 0;
  cudaEvent_t ready[kMaxCtx] = {};  // phase 1 done on context d (peer-copy / peer-store exchange)
  bool peer_all = false;             // every context can store into every other context's memory
};
Exchange g_x;
int g_last_exchange = 0;  // last multi-device call: 0 one context, 1 peer stores, 2 NCCL, 3 peer copies

bool load_nccl(NcclApi& a) {
  const char* names[] = {"libnccl.so.2", "libnccl.so"};
  for (const char* nm : names)
    if ((a.h = dlopen(nm, RTLD_NOW | RTLD_GLOBAL))) break;
  if (!a.h) return false;
  a.CommInitAll = (decltype(a.CommInitAll))dlsym(a.h, "ncclCommInitAll");
  a.CommDestroy = (decltype(a.CommDestroy))dlsym(a.h, "ncclCommDestroy");
  a.GroupStart = (decltype(a.GroupStart))dlsym(a.h, "ncclGroupStart");
  a.GroupEnd = (decltype(a.GroupEnd))dlsym(a.h, "ncclGroupEnd");
  a.Send = (decltype(a.Send))dlsym(a.h, "ncclSend");
  a.Recv = (decltype(a.Recv))dlsym(a.h, "ncclRecv");
  a.GetErrorString = (decltype(a.GetErrorString))dlsym(a.h, "ncclGetErrorString");
  return a.CommInitAll && a.CommDestroy && a.GroupStart && a.GroupEnd && a.Send && a.Recv && a.GetErrorString;
}

#define NC(call)                                                                                 \
  do {                                                                                           \
    ncclResult_t r_ = (call);                                                                    \
    if (r_ != ncclSuccess) return fail(std::string(#call) + ": " + g_x.api.GetErrorString(r_)); \
  } while (0)

int setup_exchange(int n, const int* devices) {
  if (g_x.n == n) return 0;
  g_x.n = n;
  for (int i = 0; i < n; ++i) {
    g_ci = i;
    CK(cudaSetDevice(g.device));
    if (!g_x.ready[i]) CK(cudaEventCreateWithFlags(&g_x.ready[i], cudaEventDisableTiming));
  }
  bool distinct = n > 1;
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < i; ++j)
      if (devices[i] == devices[j]) distinct = false;
  // NVLink peer access both ways between distinct devices (the peer-store / peer-copy
  // exchange); contexts sharing a device reach each other's memory directly
  g_x.peer_all = true;
  for (int i = 0; i < n; ++i) {
    CK(cudaSetDevice(devices[i]));
    for (int j = 0; j < n; ++j) {
      if (devices[i] == devices[j]) continue;
      int can = 0;
      if (cudaDeviceCanAccessPeer(&can, devices[i], devices[j]) == cudaSuccess && can) {
        const cudaError_t e = cudaDeviceEnablePeerAccess(devices[j], 0);
        if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) CK(e);
        cudaGetLastError();
      } else {
        cudaGetLastError();
        g_x.peer_all = false;
      }
    }
  }
  if (!distinct) return 0;
  const char* off = getenv("CKB_NO_NCCL");
  if (!(off && off[0] == '1') && load_nccl(g_x.api)) {
    NC(g_x.api.CommInitAll(g_x.comms, n, devices));
    g_x.nccl = true;
  }
  return 0;
}

void teardown_exchange() {
  if (g_x.nccl)
    for (int i = 0; i < g_x.n; ++i)
      if (g_x.comms[i]) g_x.api.CommDestroy(g_x.comms[i]);
  for (int i = 0; i < kMaxCtx; ++i)
    if (g_x.ready[i]) {
      if (g_ctxs[i].ready) cudaSetDevice(g_ctxs[i].device);
      cudaEventDestroy(g_x.ready[i]);
    }
  NcclApi api = g_x.api;
  g_x = Exchange();
  g_x.api = api;  // the dlopen handle stays (NCCL does not support unloading cleanly)
}

}  // namespace

extern "C" {

int ckb_abi_version(void) { return CKB_ABI_VERSION; }

const char* ckb_last_error(void) { return g_err.c_str(); }

int ckb_init(int device) {
  std::lock_guard<std::mutex> lk(g_mu);
  g_ci = 0;
  if (g.ready) {
    if (device == g.device) return 0;
    return fail("ckb_init: already initialised on another device", -3);
  }
  int rc = init_ctx(0, device);
  if (rc == 0 && g_nctx < 1) g_nctx = 1;
  return rc;
}

int ckb_init_devices(int n, const int* devices) {
  std::lock_guard<std::mutex> lk(g_mu);
  CtxSwitch cs;
  if (n < 1 || n > kMaxCtx) return fail("ckb_init_devices: 1 to 8 devices", -2);
  if (g_nctx > 1 && n != g_nctx) return fail("ckb_init_devices: already initialised with another device list", -3);
  int rc;
  for (int i = 0; i < n; ++i) {
    g_ci = i;
    if (g.ready) {
      if (g.device != devices[i]) return fail("ckb_init_devices: context " + std::to_string(i) + " is on another device", -3);
      continue;
    }
    if ((rc = init_ctx(i, devices[i]))) return rc;
  }
  g_nctx = n;
  return setup_exchange(n, devices);
}

int ckb_devices(int* n_contexts, int* nccl) {
  std::lock_guard<std::mutex> lk(g_mu);
  if (n_contexts) *n_contexts = g_nctx;
  if (nccl) *nccl = g_x.nccl ? 1 : 0;
  return 0;
}

int ckb_shutdown(void) {
  std::lock_guard<std::mutex> lk(g_mu);
  teardown_exchange();
  for (int i = kMaxCtx - 1; i >= 0; --i) {
    g_ci = i;
    shutdown_ctx();
  }
  g_ci = 0;
  g_nctx = 0;
  return 0;
}

int ckb_last_exchange(void) { return g_last_exchange; }

int ckb_last_fallback(unsigned long long* fallback, unsigned long long* images) {
  // images of the last pipeline call (context 0) that the register kernel handed
  // to the general warp kernel (non-generic remainder sequences), and all images
  std::lock_guard<std::mutex> lk(g_mu);
  int rc;
  if ((rc = ensure_ready())) return rc;
  uint32_t c = 0;
  if (g.last_fail) {
    CK(cudaStreamSynchronize(g.last_stream ? g.last_stream : g.stream));
    CK(cudaMemcpy(&c, g.last_fail, 4, cudaMemcpyDeviceToHost));
  } else if (g.last_images) {
    c = (uint32_t)g.last_images;  // the general path: every image went to the warp kernel
  }
  if (fallback) *fallback = c;
  if (images) *images = g.last_images;
  return 0;
}

unsigned long long ckb_launch_count(void) {
  unsigned long long t = 0;
  for (int i = 0; i < kMaxCtx; ++i) t += g_ctxs[i].launches;
  return t;
}

}  // extern "C"

namespace {

// one res_y pipeline enqueued on a stream; finished by res_finish
struct ResPending {
  uint32_t* out;
  uint8_t* ho;
  size_t words;
  bool out_direct;
};

bool zero_copy_on() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("CKB_ZERO_COPY");
    v = (e && e[0] == '0') ? 0 : 1;
  }
  return v == 1;
}

int res_enqueue(const uint32_t* limbs, int C, int L, const int16_t* degs, int m, int n, int dfx, int dgx,
                const uint32_t* primes, const uint32_t* gens, int K, int N, int LW, uint32_t* out, cudaStream_t st,
                int slot, ResPending* pd) {
  int rc;
  if (m < 1 || n < 1 || K < 1 || N < 1 || L < 1 || LW < 1) return fail("ckb_biv_resultant: bad sizes", -2);
  if (C != (m + 1) * (dfx + 1) + (n + 1) * (dgx + 1)) return fail("ckb_biv_resultant: C mismatch", -2);
  if ((rc = check_primes(primes, K))) return rc;
  // stage inputs in pinned memory, then one async copy each
  const size_t nl = (size_t)C * L, nd = (size_t)(m + n + 2);
  void *h_in, *h_out;
  if ((rc = host_buf("in", 4 * nl + 2 * nd + 4 * (size_t)K + 64, &h_in))) return rc;
  if ((rc = host_buf("out", 4 * (size_t)N * LW + 64, &h_out))) return rc;
  // page-locked caller buffers are copied to / from directly (no staging memcpy)
  const bool in_direct = is_pinned(limbs), out_direct = is_pinned(out);
  uint8_t* hb = (uint8_t*)h_in;
  if (!in_direct) memcpy(hb, limbs, 4 * nl);
  memcpy(hb + 4 * nl, gens, 4 * (size_t)K);
  memcpy(hb + 4 * nl + 4 * (size_t)K, degs, 2 * nd);
  const void* src_limbs = in_direct ? (const void*)limbs : (const void*)hb;
  uint32_t *d_limbs, *d_coeffs, *d_out, *d_status;
  int16_t* d_degs;
  if ((rc = dbuf("limbs", nl, &d_limbs))) return rc;
  if ((rc = dbuf("degs", nd, &d_degs))) return rc;
  if ((rc = dbuf("coeffs", std::max((size_t)K * N, crt_a_words(K, N)), &d_coeffs))) return rc;
  if ((rc = dbuf("out", (size_t)N * LW, &d_out))) return rc;
  if ((rc = dbuf("status", 4, &d_status))) return rc;
  CrtEntry* ce;
  if ((rc = get_crt(primes, K, LW, &ce))) return rc;
  uint32_t* d_crtS;
  if ((rc = dbuf("crtS", crt_scratch_words(K, N, LW), &d_crtS))) return rc;
  uint8_t* ho = (uint8_t*)h_out;
  void* dst_out = out_direct ? (void*)out : (void*)ho;
  // zero copy: the carry kernel writes the limbs (and the status word) straight
  // into the page-locked destination, overlapping the transfer with the carry
  // instead of a 1 MB copy after it (CKB_ZERO_COPY=0: the copies).  Results
  // above 4 MB go through the copy engine: the kernel's stores drain slower
  // than its DMA (cfg5, 36 MB: e2e 11.46 -> 11.51 ms zero-copy; cfg4 0.346 ->
  // 0.335 ms, cfg2 0.086 -> 0.077 ms)
  uint32_t *z_out = nullptr, *z_status = nullptr;
  if (zero_copy_on() && 4 * (size_t)N * LW <= ((size_t)4 << 20)) {
    void *a = nullptr, *b = nullptr;
    if (cudaHostGetDevicePointer(&a, dst_out, 0) == cudaSuccess &&
        cudaHostGetDevicePointer(&b, ho + 4 * (size_t)N * LW, 0) == cudaSuccess) {
      z_out = (uint32_t*)a;
      z_status = (uint32_t*)b;
    } else {
      cudaGetLastError();
    }
  }
  std::vector<uint64_t> key = {2, (uint64_t)C, (uint64_t)L, (uint64_t)m, (uint64_t)n, (uint64_t)dfx, (uint64_t)dgx,
                               (uint64_t)K, (uint64_t)N, (uint64_t)LW, (uint64_t)src_limbs, (uint64_t)dst_out,
                               (uint64_t)slot};
  key_push(key, degs, 2 * nd);
  key_push(key, primes, 4 * (size_t)K);
  key_push(key, gens, 4 * (size_t)K);
  rc = graphed(key, st, [&]() -> int {
    int r;
    CK(cudaMemcpyAsync(d_limbs, src_limbs, 4 * nl, cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(d_degs, hb + 4 * nl + 4 * (size_t)K, 2 * nd, cudaMemcpyHostToDevice, st));
    CK(cudaMemsetAsync(d_status, 0, 4, st));
    g.nsev = 0;
    if ((r = modular_stage(d_limbs, C, L, d_degs, degs, m, n, dfx, dgx, ce->d_primes, primes, gens, K, N, d_coeffs,
                           d_status, st, &ce->t)))
      return r;
    if (z_out) {
      g.launches += launch_crt(ce->t, d_coeffs, N, z_out, d_crtS, st, true, d_status, z_status);
      stage_mark(st);
      CK(cudaGetLastError());
      return 0;
    }
    g.launches += launch_crt(ce->t, d_coeffs, N, d_out, d_crtS, st, true);
    stage_mark(st);
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(dst_out, d_out, 4 * (size_t)N * LW, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(ho + 4 * (size_t)N * LW, d_status, 4, cudaMemcpyDeviceToHost, st));
    return 0;
  });
  if (rc) return rc;
  pd->out = out;
  pd->ho = ho;
  pd->words = (size_t)N * LW;
  pd->out_direct = out_direct;
  return 0;
}

// spin on an event: a blocking synchronise adds a thread wake-up to every
// call's latency (a cfg4 call is ~0.4 ms end to end)
int spin_event(cudaEvent_t ev) {
  for (;;) {
    const cudaError_t q = cudaEventQuery(ev);
    if (q == cudaSuccess) return 0;
    if (q != cudaErrorNotReady) CK(q);
  }
}

uint32_t res_finish(const ResPending& pd) {
  if (!pd.out_direct) memcpy(pd.out, pd.ho, 4 * pd.words);
  uint32_t s;
  memcpy(&s, pd.ho + 4 * pd.words, 4);
  return s;
}

}  // namespace

extern "C" {

int ckb_biv_resultant(const uint32_t* limbs, int C, int L, const int16_t* degs, int m, int n, int dfx, int dgx,
                      const uint32_t* primes, const uint32_t* gens, int K, int N, int LW, uint32_t* out,
                      uint32_t* status, float* device_ms) {
  const auto t0 = std::chrono::steady_clock::now();
  std::lock_guard<std::mutex> lk(g_mu);
  int rc;
  if ((rc = ensure_ready())) return rc;
  cudaStream_t st = g.stream;
  ResPending pd;
  CK(cudaEventRecord(g.ev0, st));
  if ((rc = res_enqueue(limbs, C, L, degs, m, n, dfx, dgx, primes, gens, K, N, LW, out, st, 0, &pd))) return rc;
  CK(cudaEventRecord(g.ev1, st));
  const auto t1 = std::chrono::steady_clock::now();
  if ((rc = spin_event(g.ev1))) return rc;
  const auto t2 = std::chrono::steady_clock::now();
  g_host_times[0] = std::chrono::duration<float, std::micro>(t1 - t0).count();
  g_host_times[1] = std::chrono::duration<float, std::micro>(t2 - t1).count();
  const uint32_t s = res_finish(pd);
  if (status) *status = s;
  if (device_ms) CK(cudaEventElapsedTime(device_ms, g.ev0, g.ev1));
  return s ? CKB_STATUS_REPLAN : 0;
}

int ckb_biv_resultant_batch(int P, const uint32_t* const* limbs, const int* C, const int* L,
                            const int16_t* const* degs, const int* m, const int* n, const int* dfx, const int* dgx,
                            const uint32_t* const* primes, const uint32_t* const* gens, const int* K, const int* N,
                            const int* LW, uint32_t* const* out, uint32_t* status) {
  std::lock_guard<std::mutex> lk(g_mu);
  int rc;
  if ((rc = ensure_ready())) return rc;
  if (P < 1 || P > 4) return fail("ckb_biv_resultant_batch: 1 to 4 problems", -2);
  for (int i = 0; i < P; ++i) {
    if (!g.bst[i]) {
      CK(cudaStreamCreateWithFlags(&g.bst[i], cudaStreamNonBlocking));
      CK(cudaEventCreateWithFlags(&g.bev[i], cudaEventDisableTiming));
    }
  }
  // cached tables first (built on the context stream, which get_plan / get_crt
  // synchronise), so that enqueueing one problem cannot evict another's
  for (int i = 0; i < P; ++i) {
    InterpPlan pl;
    CrtEntry* ce;
    if (m[i] < 1 || n[i] < 1 || K[i] < 1) return fail("ckb_biv_resultant_batch: bad sizes", -2);
    if ((rc = check_primes(primes[i], K[i]))) return rc;
    if ((rc = get_plan(primes[i], gens[i], K[i], N[i], 8, &pl))) return rc;
    if ((rc = get_crt(primes[i], K[i], LW[i], &ce))) return rc;
  }
  CK(cudaStreamSynchronize(g.stream));
  // (with at most 4 problems every plan / CRT entry stays cached during the
  // enqueue pass; buffers are per problem, so no problem's setup can free
  // memory another problem's enqueued work uses)
  ResPending pd[4];
  const bool timing = g.timing;
  g.timing = false;
  for (int i = 0; i < P && rc == 0; ++i) {
    g.ns = "b" + std::to_string(i) + ".";
    rc = res_enqueue(limbs[i], C[i], L[i], degs[i], m[i], n[i], dfx[i], dgx[i], primes[i], gens[i], K[i], N[i],
                     LW[i], out[i], g.bst[i], 1 + i, &pd[i]);
    if (rc == 0 && cudaEventRecord(g.bev[i], g.bst[i]) != cudaSuccess) rc = fail("cudaEventRecord", -1);
  }
  g.ns.clear();
  g.timing = timing;
  for (int i = 0; i < P; ++i) cudaStreamSynchronize(g.bst[i]);
  if (rc) return rc;
  uint32_t any = 0;
  for (int i = 0; i < P; ++i) {
    status[i] = res_finish(pd[i]);
    any |= status[i];
  }
  return any ? CKB_STATUS_REPLAN : 0;
}

int ckb_biv_resultant_multi(const uint32_t* limbs, int C, int L, const int16_t* degs, int m, int n, int dfx, int dgx,
                            const uint32_t* primes, const uint32_t* gens, int K, int N, int LW, int G, uint32_t* out,
                            uint32_t* status, float* device_ms) {
  // res_y over G device contexts (option B):
  //   phase 1, context d: its contiguous block of primes [k0_d, k0_d + K_d) through
  //            reduce -> point scales -> images -> interpolation, giving the
  //            residues [K_d][N]; column block s (coefficients [a_s, a_s + w_s))
  //            packed contiguously for context s;
  //   exchange: every context receives ALL K residues of its coefficient block
  //            (NCCL send/recv over NVLink, or peer copies);
  //   phase 3, context s: CRT of its w_s coefficients with all K primes, limbs
  //            straight into the caller's rows [a_s, a_s + w_s).
  std::lock_guard<std::mutex> lk(g_mu);
  CtxSwitch cs;
  int rc;
  g_ci = 0;
  if ((rc = ensure_ready())) return rc;
  if (G < 1 || G > g_nctx) return fail("ckb_biv_resultant_multi: G must be 1 .. ckb_init_devices' count", -2);
  if (m < 1 || n < 1 || K < G || N < G || L < 1 || LW < 1) return fail("ckb_biv_resultant_multi: bad sizes", -2);
  if (C != (m + 1) * (dfx + 1) + (n + 1) * (dgx + 1)) return fail("ckb_biv_resultant_multi: C mismatch", -2);
  if ((rc = check_primes(primes, K))) return rc;
  int k0[kMaxCtx + 1], a0[kMaxCtx + 1];
  for (int d = 0; d <= G; ++d) {
    k0[d] = (int)((int64_t)K * d / G);  // balanced contiguous prime blocks
    const int nc = (N + G - 1) / G;
    a0[d] = std::min(N, d * nc);        // coefficient blocks of ceil(N / G)
  }
  // host staging in context 0's portable pinned memory (every device DMAs from it)
  const size_t nl = (size_t)C * L, nd = (size_t)(m + n + 2);
  void *h_in, *h_out;
  if ((rc = host_buf("m.in", 4 * nl + 2 * nd + 64, &h_in))) return rc;
  if ((rc = host_buf("m.out", 4 * (size_t)N * LW + 4 * kMaxCtx + 64, &h_out))) return rc;
  const bool in_direct = is_pinned(limbs), out_direct = is_pinned(out);
  uint8_t* hb = (uint8_t*)h_in;
  if (!in_direct) memcpy(hb, limbs, 4 * nl);
  memcpy(hb + 4 * nl, degs, 2 * nd);
  const void* src_limbs = in_direct ? (const void*)limbs : (const void*)hb;
  uint8_t* ho = (uint8_t*)h_out;
  uint32_t* dst_out = out_direct ? out : (uint32_t*)ho;
  uint32_t* h_status = (uint32_t*)(ho + 4 * (size_t)N * LW);
  struct Dev {
    uint32_t *limbs, *coeffs, *send, *recv, *out, *status, *crtS;
    int16_t* degs;
    Prime* primes;
    CrtEntry* ce;
  } dv[kMaxCtx];
  // per-context buffers and cached tables (plans, CRT tables) first: building
  // them synchronises the context's stream
  for (int d = 0; d < G; ++d) {
    g_ci = d;
    if ((rc = ensure_ready())) return rc;
    const int kd = k0[d + 1] - k0[d], wd = a0[d + 1] - a0[d];
    Dev& v = dv[d];
    if ((rc = dbuf("m.limbs", nl, &v.limbs))) return rc;
    if ((rc = dbuf("m.degs", nd, &v.degs))) return rc;
    if ((rc = dbuf("m.coeffs", (size_t)kd * N, &v.coeffs))) return rc;
    if ((rc = dbuf("m.send", (size_t)kd * N, &v.send))) return rc;
    if ((rc = dbuf("m.recv", std::max((size_t)K * wd, crt_a_words(K, wd)), &v.recv))) return rc;
    if ((rc = dbuf("m.out", (size_t)wd * LW, &v.out))) return rc;
    if ((rc = dbuf("m.status", 4, &v.status))) return rc;
    if ((rc = dbuf("m.crtS", crt_scratch_words(K, wd, LW), &v.crtS))) return rc;
    if ((rc = get_primes_dev(primes + k0[d], kd, &v.primes))) return rc;
    if ((rc = get_crt(primes, K, LW, &v.ce))) return rc;
    InterpPlan pl;
    if ((rc = get_plan(primes + k0[d], gens + k0[d], kd, N, 8, &pl))) return rc;
  }
  // the exchange: folded into the interpolation's stores when every context can
  // reach every other's memory (CKB_EXCHANGE=nccl / copy: the separate step)
  const char* xm = getenv("CKB_EXCHANGE");
  const bool fused = G > 1 && g_x.peer_all && !(xm && (strcmp(xm, "nccl") == 0 || strcmp(xm, "copy") == 0));
  g_last_exchange = G < 2 ? 0 : fused ? 1 : g_x.nccl ? 2 : 3;
  // phase 1 (each context's launches replayed as one CUDA graph after the first calls)
  for (int d = 0; d < G; ++d) {
    g_ci = d;
    CK(cudaSetDevice(g.device));
    cudaStream_t st = g.stream;
    const int kd = k0[d + 1] - k0[d];
    Dev& v = dv[d];
    CK(cudaEventRecord(g.ev0, st));
    std::vector<uint64_t> key = {5, (uint64_t)G, (uint64_t)C, (uint64_t)L, (uint64_t)m, (uint64_t)n, (uint64_t)dfx,
                                 (uint64_t)dgx, (uint64_t)K, (uint64_t)N, (uint64_t)LW, (uint64_t)src_limbs,
                                 (uint64_t)hb};
    key_push(key, degs, 2 * nd);
    key_push(key, primes + k0[d], 4 * (size_t)kd);
    key_push(key, gens + k0[d], 4 * (size_t)kd);
    PeerOut po{};
    CrtTables ct = v.ce->t;  // this context's rows of the CRT premultipliers
    if (fused) {
      po.G = G;
      po.nc = (N + G - 1) / G;
      po.KC = (K + 31) / 32;
      po.k0 = k0[d];
      for (int s2 = 0; s2 < G; ++s2) po.dst[s2] = dv[s2].recv;
      ct.c += k0[d];
      ct.cc += k0[d];
    }
    key.push_back(fused ? 1u : 0u);
    for (int s2 = 0; s2 < G && fused; ++s2) key.push_back((uint64_t)po.dst[s2]);
    rc = graphed(key, st, [&]() -> int {
      int r;
      CK(cudaMemcpyAsync(v.limbs, src_limbs, 4 * nl, cudaMemcpyHostToDevice, st));
      CK(cudaMemcpyAsync(v.degs, hb + 4 * nl, 2 * nd, cudaMemcpyHostToDevice, st));
      CK(cudaMemsetAsync(v.status, 0, 4, st));
      g.nsev = 0;
      if ((r = modular_stage(v.limbs, C, L, v.degs, degs, m, n, dfx, dgx, v.primes, primes + k0[d], gens + k0[d], kd,
                             N, v.coeffs, v.status, st, fused ? &ct : nullptr, fused ? &po : nullptr)))
        return r;
      if (fused) return 0;  // the y values are already in every context's CRT input
      for (int s2 = 0; s2 < G; ++s2) {  // column block s2 -> contiguous [K_d][w_s2] at K_d a_s2
        const int ws = a0[s2 + 1] - a0[s2];
        if (ws > 0)
          CK(cudaMemcpy2DAsync(v.send + (size_t)kd * a0[s2], 4 * (size_t)ws, v.coeffs + a0[s2], 4 * (size_t)N,
                               4 * (size_t)ws, kd, cudaMemcpyDeviceToDevice, st));
      }
      return 0;
    });
    if (rc) return rc;
    if (fused || !g_x.nccl) CK(cudaEventRecord(g_x.ready[d], st));
  }
  // the exchange
  if (fused) {
    for (int s2 = 0; s2 < G; ++s2) {  // each CRT waits for every context's stores into its input
      g_ci = s2;
      CK(cudaSetDevice(g.device));
      for (int d = 0; d < G; ++d)
        if (d != s2) CK(cudaStreamWaitEvent(g.stream, g_x.ready[d], 0));
    }
  } else if (g_x.nccl) {
    NC(g_x.api.GroupStart());
    for (int d = 0; d < G; ++d) {
      const int kd = k0[d + 1] - k0[d], wd = a0[d + 1] - a0[d];
      for (int s2 = 0; s2 < G; ++s2) {
        const int ks = k0[s2 + 1] - k0[s2], ws = a0[s2 + 1] - a0[s2];
        if (ws > 0)
          NC(g_x.api.Send(dv[d].send + (size_t)kd * a0[s2], (size_t)kd * ws, ncclUint32, s2, g_x.comms[d],
                          g_ctxs[d].stream));
        if (wd > 0)
          NC(g_x.api.Recv(dv[d].recv + (size_t)k0[s2] * wd, (size_t)ks * wd, ncclUint32, s2, g_x.comms[d],
                          g_ctxs[d].stream));
      }
    }
    NC(g_x.api.GroupEnd());
  } else {
    for (int s2 = 0; s2 < G; ++s2) {
      g_ci = s2;
      CK(cudaSetDevice(g.device));
      const int ws = a0[s2 + 1] - a0[s2];
      for (int d = 0; d < G; ++d) {
        const int kd = k0[d + 1] - k0[d];
        CK(cudaStreamWaitEvent(g.stream, g_x.ready[d], 0));
        if (ws > 0)
          CK(cudaMemcpyPeerAsync(dv[s2].recv + (size_t)k0[d] * ws, g.device, dv[d].send + (size_t)kd * a0[s2],
                                 g_ctxs[d].device, 4 * (size_t)kd * ws, g.stream));
      }
    }
  }
  // phase 3: CRT of each context's coefficient block, limbs to the caller's rows
  for (int s2 = 0; s2 < G; ++s2) {
    g_ci = s2;
    CK(cudaSetDevice(g.device));
    cudaStream_t st = g.stream;
    const int ws = a0[s2 + 1] - a0[s2];
    Dev& v = dv[s2];
    std::vector<uint64_t> key = {6, (uint64_t)G, (uint64_t)K, (uint64_t)N, (uint64_t)LW, (uint64_t)dst_out,
                                 (uint64_t)h_status, fused ? 1u : 0u};
    key_push(key, primes, 4 * (size_t)K);
    // zero copy as in ckb_biv_resultant: the carry kernel writes this block's rows and the status
    // word straight into the page-locked destination (blocks <= 4 MB)
    uint32_t *z_out = nullptr, *z_status = nullptr;
    if (ws > 0 && zero_copy_on() && 4 * (size_t)ws * LW <= ((size_t)4 << 20)) {
      void *zo = nullptr, *zs = nullptr;
      if (cudaHostGetDevicePointer(&zo, dst_out + (size_t)a0[s2] * LW, 0) == cudaSuccess &&
          cudaHostGetDevicePointer(&zs, h_status + s2, 0) == cudaSuccess) {
        z_out = (uint32_t*)zo;
        z_status = (uint32_t*)zs;
      } else {
        cudaGetLastError();
      }
    }
    key.push_back(z_out ? 1u : 0u);
    rc = graphed(key, st, [&]() -> int {
      if (z_out) {  // fused: the input is y already
        g.launches += launch_crt(v.ce->t, v.recv, ws, z_out, v.crtS, st, fused, v.status, z_status);
        CK(cudaGetLastError());
        return 0;
      }
      if (ws > 0) {
        g.launches += launch_crt(v.ce->t, v.recv, ws, v.out, v.crtS, st, fused);
        CK(cudaGetLastError());
        CK(cudaMemcpyAsync(dst_out + (size_t)a0[s2] * LW, v.out, 4 * (size_t)ws * LW, cudaMemcpyDeviceToHost, st));
      }
      CK(cudaMemcpyAsync(h_status + s2, v.status, 4, cudaMemcpyDeviceToHost, st));
      return 0;
    });
    if (rc) return rc;
    CK(cudaEventRecord(g.ev1, st));
  }
  float worst = 0.f;
  uint32_t any = 0;
  for (int d = 0; d < G; ++d) {
    g_ci = d;
    CK(cudaSetDevice(g.device));
    if ((rc = spin_event(g.ev1))) return rc;
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, g.ev0, g.ev1));
    worst = std::max(worst, ms);
    any |= h_status[d];
  }
  if (!out_direct) memcpy(out, ho, 4 * (size_t)N * LW);
  if (status) *status = any;
  if (device_ms) *device_ms = worst;
  return any ? CKB_STATUS_REPLAN : 0;
}

int ckb_reduce(const uint32_t* limbs, int C, int L, const uint32_t* primes, int K, uint32_t* out) {
  std::lock_guard<std::mutex> lk(g_mu);
  int rc;
  if ((rc = ensure_ready())) return rc;
  if ((rc = check_primes(primes, K))) return rc;
  cudaStream_t st = g.stream;
  uint32_t *d_limbs, *d_out;
  Prime* d_primes;
  if ((rc = dbuf("r.limbs", (size_t)C * L, &d_limbs))) return rc;
  if ((rc = dbuf("r.out", (size_t)K * C, &d_out))) return rc;
  if ((rc = upload_primes(primes, K, &d_primes))) return rc;
  CK(cudaMemcpyAsync(d_limbs, limbs, 4 * (size_t)C * L, cudaMemcpyHostToDevice, st));
  launch_reduce(d_limbs, C, L, d_primes, K, d_out, st);
  g.launches += 1;
  CK(cudaGetLastError());
  CK(cudaMemcpyAsync(out, d_out, 4 * (size_t)K * C, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  return 0;
}

int ckb_uni_resultant_batch(const uint32_t* fa, const int32_t* da, const uint32_t* gb, const int32_t* db, int W,
                            const uint32_t* primes, int P, const int32_t* pidx, int B, uint32_t* out) {
  std::lock_guard<std::mutex> lk(g_mu);
  int rc;
  if ((rc = ensure_ready())) return rc;
  if ((rc = check_primes(primes, P))) return rc;
  if (W < 1) return fail("ckb_uni_resultant_batch: need W >= 1", -2);
  if (B == 0) return 0;
  cudaStream_t st = g.stream;
  uint32_t *d_fa, *d_gb, *d_out;
  int32_t *d_da, *d_db, *d_pi;
  Prime* d_primes;
  if ((rc = dbuf("u.fa", (size_t)B * W, &d_fa))) return rc;
  if ((rc = dbuf("u.gb", (size_t)B * W, &d_gb))) return rc;
  if ((rc = dbuf("u.da", (size_t)B, &d_da))) return rc;
  if ((rc = dbuf("u.db", (size_t)B, &d_db))) return rc;
  if ((rc = dbuf("u.pi", (size_t)B, &d_pi))) return rc;
  if ((rc = dbuf("u.out", (size_t)B, &d_out))) return rc;
  if ((rc = upload_primes(primes, P, &d_primes))) return rc;
  CK(cudaMemcpyAsync(d_fa, fa, 4 * (size_t)B * W, cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(d_gb, gb, 4 * (size_t)B * W, cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(d_da, da, 4 * (size_t)B, cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(d_db, db, 4 * (size_t)B, cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(d_pi, pidx, 4 * (size_t)B, cudaMemcpyHostToDevice, st));
  uint32_t* d_gs = nullptr;  // operands beyond shared memory: a global slice per pair
  if ((size_t)3 * W * 4 > kSmemLimit && (rc = dbuf("u.gs", (size_t)B * 3 * W, &d_gs))) return rc;
  launch_uni_resultant(d_fa, d_da, d_gb, d_db, W, d_primes, d_pi, B, d_out, d_gs, st);
  g.launches += 1;
  CK(cudaGetLastError());
  CK(cudaMemcpyAsync(out, d_out, 4 * (size_t)B, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  return 0;
}

int ckb_crt_lift(const uint32_t* residues, int K, int N, const uint32_t* primes, int LW, uint32_t* out) {
  std::lock_guard<std::mutex> lk(g_mu);
  int rc;
  if ((rc = ensure_ready())) return rc;
  if ((rc = check_primes(primes, K))) return rc;
  cudaStream_t st = g.stream;
  CrtEntry* ce;
  if ((rc = get_crt(primes, K, LW, &ce))) return rc;
  uint32_t *d_res, *d_out;
  if ((rc = dbuf("c.res", (size_t)K * N, &d_res))) return rc;
  if ((rc = dbuf("c.out", (size_t)N * LW, &d_out))) return rc;
  CK(cudaMemcpyAsync(d_res, residues, 4 * (size_t)K * N, cudaMemcpyHostToDevice, st));
  uint32_t* d_crtS;
  if ((rc = dbuf("crtS", crt_scratch_words(K, N, LW), &d_crtS))) return rc;
  g.launches += launch_crt(ce->t, d_res, N, d_out, d_crtS, st);
  CK(cudaGetLastError());
  CK(cudaMemcpyAsync(out, d_out, 4 * (size_t)N * LW, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  return 0;
}

int ckb_interp_plan_points(const uint32_t* primes, const uint32_t* gens, int K, int N, uint32_t* xpts) {
  // the planned evaluation points for constant leading coefficients (c = 1): x_t = q^t
  std::lock_guard<std::mutex> lk(g_mu);
  int rc;
  if ((rc = ensure_ready())) return rc;
  if ((rc = check_primes(primes, K))) return rc;
  InterpPlan pl;
  if ((rc = get_plan(primes, gens, K, N, 1, &pl))) return rc;
  CK(cudaMemcpy(xpts, pl.xq, 4 * (size_t)K * N, cudaMemcpyDeviceToHost));
  return 0;
}

int ckb_interp_geometric(const uint32_t* values, const uint32_t* primes, const uint32_t* gens, int K, int N,
                         uint32_t* coeffs) {
  // interpolate values given at the planned points x_t = q^t (c = 1)
  std::lock_guard<std::mutex> lk(g_mu);
  int rc;
  if ((rc = ensure_ready())) return rc;
  if ((rc = check_primes(primes, K))) return rc;
  cudaStream_t st = g.stream;
  InterpPlan pl;
  if ((rc = get_plan(primes, gens, K, N, 1, &pl))) return rc;
  Prime* d_primes;
  uint32_t *d_vals, *d_coeffs, *d_cval;
  if ((rc = get_primes_dev(primes, K, &d_primes))) return rc;
  if ((rc = dbuf("i.vals", (size_t)K * N, &d_vals))) return rc;
  if ((rc = dbuf("i.coeffs", (size_t)K * N, &d_coeffs))) return rc;
  if ((rc = dbuf("i.cval", (size_t)K, &d_cval))) return rc;
  std::vector<uint32_t> ones((size_t)K, 1u);
  CK(cudaMemcpyAsync(d_cval, ones.data(), 4 * (size_t)K, cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(d_vals, values, 4 * (size_t)K * N, cudaMemcpyHostToDevice, st));
  launch_interp(pl, d_primes, d_vals, d_cval, d_coeffs, st);
  g.launches += 1;
  CK(cudaGetLastError());
  CK(cudaMemcpyAsync(coeffs, d_coeffs, 4 * (size_t)K * N, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  return 0;
}

int ckb_gcd_mod_batch(const uint32_t* fa, const int32_t* da, int Wf, const uint32_t* gb, const int32_t* db, int Wg,
                      const uint32_t* primes, int P, const int32_t* pidx, int B, uint32_t* out, int Wo,
                      int32_t* odeg) {
  std::lock_guard<std::mutex> lk(g_mu);
  int rc;
  if ((rc = ensure_ready())) return rc;
  if ((rc = check_primes(primes, P))) return rc;
  if (B == 0) return 0;
  cudaStream_t st = g.stream;
  uint32_t *d_fa, *d_gb, *d_out;
  int32_t *d_da, *d_db, *d_pi, *d_odeg;
  Prime* d_primes;
  if ((rc = dbuf("g.fa", (size_t)B * Wf, &d_fa))) return rc;
  if ((rc = dbuf("g.gb", (size_t)B * Wg, &d_gb))) return rc;
  if ((rc = dbuf("g.da", (size_t)B, &d_da))) return rc;
  if ((rc = dbuf("g.db", (size_t)B, &d_db))) return rc;
  if ((rc = dbuf("g.pi", (size_t)B, &d_pi))) return rc;
  if ((rc = dbuf("g.out", (size_t)B * Wo, &d_out))) return rc;
  if ((rc = dbuf("g.odeg", (size_t)B, &d_odeg))) return rc;
  if ((rc = upload_primes(primes, P, &d_primes))) return rc;
  CK(cudaMemcpyAsync(d_fa, fa, 4 * (size_t)B * Wf, cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(d_gb, gb, 4 * (size_t)B * Wg, cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(d_da, da, 4 * (size_t)B, cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(d_db, db, 4 * (size_t)B, cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(d_pi, pidx, 4 * (size_t)B, cudaMemcpyHostToDevice, st));
  uint32_t* d_gs = nullptr;
  const size_t gw = (size_t)2 * (Wf > Wg ? Wf : Wg);
  if (gw * 4 > kSmemLimit && (rc = dbuf("g.gs", (size_t)B * gw, &d_gs))) return rc;
  launch_gcd_mod(d_fa, d_da, Wf, d_gb, d_db, Wg, d_primes, d_pi, B, d_out, Wo, d_odeg, d_gs, st);
  g.launches += 1;
  CK(cudaGetLastError());
  CK(cudaMemcpyAsync(out, d_out, 4 * (size_t)B * Wo, cudaMemcpyDeviceToHost, st));
  CK(cudaMemcpyAsync(odeg, d_odeg, 4 * (size_t)B, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  return 0;
}

int ckb_interp_points(const uint32_t* xs, const uint32_t* vs, const int32_t* ns, int W, const uint32_t* primes, int P,
                      const int32_t* pidx, int B, uint32_t* out) {
  std::lock_guard<std::mutex> lk(g_mu);
  int rc;
  if ((rc = ensure_ready())) return rc;
  if ((rc = check_primes(primes, P))) return rc;
  if (B == 0) return 0;
  cudaStream_t st = g.stream;
  uint32_t *d_xs, *d_vs, *d_out;
  int32_t *d_ns, *d_pi;
  Prime* d_primes;
  if ((rc = dbuf("ip.xs", (size_t)B * W, &d_xs))) return rc;
  if ((rc = dbuf("ip.vs", (size_t)B * W, &d_vs))) return rc;
  if ((rc = dbuf("ip.ns", (size_t)B, &d_ns))) return rc;
  if ((rc = dbuf("ip.pi", (size_t)B, &d_pi))) return rc;
  if ((rc = dbuf("ip.out", (size_t)B * W, &d_out))) return rc;
  if ((rc = upload_primes(primes, P, &d_primes))) return rc;
  CK(cudaMemcpyAsync(d_xs, xs, 4 * (size_t)B * W, cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(d_vs, vs, 4 * (size_t)B * W, cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(d_ns, ns, 4 * (size_t)B, cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(d_pi, pidx, 4 * (size_t)B, cudaMemcpyHostToDevice, st));
  uint32_t* d_gs = nullptr;
  if ((size_t)(4 * W + 2) * 4 > kSmemLimit && (rc = dbuf("ip.gs", (size_t)B * (4 * W + 2), &d_gs))) return rc;
  launch_interp_points(d_xs, d_vs, d_ns, W, d_primes, d_pi, B, d_out, d_gs, st);
  g.launches += 1;
  CK(cudaGetLastError());
  CK(cudaMemcpyAsync(out, d_out, 4 * (size_t)B * W, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  return 0;
}

int ckb_biv_gcd_images(const uint32_t* limbs, int C, int L, const int16_t* degs, int m, int n, int dax, int dbx,
                       int dgam, const uint32_t* primes, int K, int NP, uint32_t* out, int Wo, int32_t* odeg) {
  std::lock_guard<std::mutex> lk(g_mu);
  int rc;
  if ((rc = ensure_ready())) return rc;
  if ((rc = check_primes(primes, K))) return rc;
  if (K == 0 || NP == 0) return 0;
  if (m < n || n < 0 || dax < 0 || dbx < 0 || dgam < 0) return fail("ckb_biv_gcd_images: need m >= n >= 0", -2);
  if (C != (m + 1) * (dax + 1) + (n + 1) * (dbx + 1) + dgam + 1) return fail("ckb_biv_gcd_images: bad C", -2);
  if (Wo < m + 1) return fail("ckb_biv_gcd_images: Wo < m + 1", -2);
  if ((size_t)8 * (m + 1) * 4 > 200 * 1024) return fail("ckb_biv_gcd_images: y-degree too large", -2);
  cudaStream_t st = g.stream;
  uint32_t *d_limbs, *d_res, *d_out;
  int16_t* d_degs;
  int32_t* d_odeg;
  Prime* d_primes;
  const size_t B = (size_t)K * NP;
  if ((rc = dbuf("bg.limbs", (size_t)C * L, &d_limbs))) return rc;
  if ((rc = dbuf("bg.res", (size_t)K * C, &d_res))) return rc;
  if ((rc = dbuf("bg.degs", (size_t)(m + n + 2), &d_degs))) return rc;
  if ((rc = dbuf("bg.out", B * Wo, &d_out))) return rc;
  if ((rc = dbuf("bg.odeg", B, &d_odeg))) return rc;
  if ((rc = upload_primes(primes, K, &d_primes))) return rc;
  CK(cudaMemcpyAsync(d_limbs, limbs, 4 * (size_t)C * L, cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(d_degs, degs, 2 * (size_t)(m + n + 2), cudaMemcpyHostToDevice, st));
  launch_reduce(d_limbs, C, L, d_primes, K, d_res, st);
  launch_biv_gcd_images(d_res, C, d_degs, m, n, dax, dbx, dgam, d_primes, K, NP, d_out, Wo, d_odeg, st);
  g.launches += 2;
  CK(cudaGetLastError());
  CK(cudaMemcpyAsync(out, d_out, 4 * B * Wo, cudaMemcpyDeviceToHost, st));
  CK(cudaMemcpyAsync(odeg, d_odeg, 4 * B, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  return 0;
}

int ckb_psc_values(const uint32_t* fres, const int16_t* fdeg, int m, int dfx, const uint32_t* gres,
                   const int16_t* gdeg, int n, int dgx, uint32_t p, int ncand, uint32_t* out, uint8_t* valid) {
  std::lock_guard<std::mutex> lk(g_mu);
  int rc;
  if ((rc = ensure_ready())) return rc;
  if ((rc = check_primes(&p, 1))) return rc;
  if (m < 0 || n < 0 || m < n || ncand < 1) return fail("ckb_psc_values: bad sizes (need m >= n >= 0)", -2);
  if (!psc_fits(m, n)) return fail("ckb_psc_values: degree too large", -2);
  cudaStream_t st = g.stream;
  const size_t nf = (size_t)(m + 1) * (dfx + 1), ng = (size_t)(n + 1) * (dgx + 1);
  uint32_t *d_f, *d_g, *d_out;
  int16_t *d_fd, *d_gd;
  uint8_t* d_valid;
  if ((rc = dbuf("s.f", nf, &d_f))) return rc;
  if ((rc = dbuf("s.g", ng, &d_g))) return rc;
  if ((rc = dbuf("s.fd", (size_t)m + 1, &d_fd))) return rc;
  if ((rc = dbuf("s.gd", (size_t)n + 1, &d_gd))) return rc;
  const int nrow = n > 0 ? n : 1;
  if ((rc = dbuf("s.out", (size_t)nrow * ncand, &d_out))) return rc;
  if ((rc = dbuf("s.valid", (size_t)ncand, &d_valid))) return rc;
  CK(cudaMemcpyAsync(d_f, fres, 4 * nf, cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(d_g, gres, 4 * ng, cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(d_fd, fdeg, 2 * ((size_t)m + 1), cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(d_gd, gdeg, 2 * ((size_t)n + 1), cudaMemcpyHostToDevice, st));
  launch_psc(d_f, d_fd, m, dfx, d_g, d_gd, n, dgx, h_prime(p), nullptr, ncand, d_out, d_valid, st);
  g.launches += 1;
  CK(cudaGetLastError());
  if (n > 0) CK(cudaMemcpyAsync(out, d_out, 4 * (size_t)n * ncand, cudaMemcpyDeviceToHost, st));
  CK(cudaMemcpyAsync(valid, d_valid, (size_t)ncand, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  return 0;
}

int ckb_subres_profile(const uint32_t* fres, const int16_t* fdeg, int m, int dfx, const uint32_t* gres,
                       const int16_t* gdeg, int n, int dgx, const uint32_t* rmod, int rlen, int rlen_int, int dmax,
                       uint32_t p, int32_t* chain) {
  std::lock_guard<std::mutex> lk(g_mu);
  int rc;
  if ((rc = ensure_ready())) return rc;
  if ((rc = check_primes(&p, 1))) return rc;
  if (m < 1 || n < 1 || m < n || dmax < 0 || rlen < 1 || rlen_int < 1)
    return fail("ckb_subres_profile: bad sizes (need m >= n >= 1, rstar nonzero)", -2);
  if (!psc_fits(m, n)) return fail("ckb_subres_profile: degree too large", -2);
  const int need = (m + n - 2) * dmax + 1;  // modpoly.py:447
  const int W = need;
  if (!gcd_chain_fits(rlen, W)) return fail("ckb_subres_profile: chain degrees too large", -2);
  // candidates: need plus a margin for the skipped t (re-run with more if a
  // leading coefficient vanishes unusually often); t never reaches p
  const int64_t lim = (int64_t)p;
  cudaStream_t st = g.stream;
  const size_t nf = (size_t)(m + 1) * (dfx + 1), ng = (size_t)(n + 1) * (dgx + 1);
  uint32_t *d_f, *d_g, *d_sel, *d_vals, *d_sr, *d_r, *d_status;
  int16_t *d_fd, *d_gd;
  int *d_count, *d_cnt, *d_chain;
  int32_t *d_ns, *d_pi;
  Prime* d_prime;
  if ((rc = dbuf("sp.f", nf, &d_f))) return rc;
  if ((rc = dbuf("sp.g", ng, &d_g))) return rc;
  if ((rc = dbuf("sp.fd", (size_t)m + 1, &d_fd))) return rc;
  if ((rc = dbuf("sp.gd", (size_t)n + 1, &d_gd))) return rc;
  if ((rc = dbuf("sp.sel", (size_t)need, &d_sel))) return rc;
  if ((rc = dbuf("sp.vals", (size_t)n * need, &d_vals))) return rc;
  if ((rc = dbuf("sp.sr", (size_t)n * W, &d_sr))) return rc;
  if ((rc = dbuf("sp.r", (size_t)rlen, &d_r))) return rc;
  if ((rc = dbuf("sp.status", 4, &d_status))) return rc;
  if ((rc = dbuf("sp.count", 1, &d_count))) return rc;
  if ((rc = dbuf("sp.cnt", (size_t)n, &d_cnt))) return rc;
  if ((rc = dbuf("sp.chain", (size_t)n + 1, &d_chain))) return rc;
  if ((rc = dbuf("sp.ns", (size_t)n, &d_ns))) return rc;
  if ((rc = dbuf("sp.pi", (size_t)n, &d_pi))) return rc;
  if ((rc = upload_primes(&p, 1, &d_prime))) return rc;
  std::vector<int32_t> cnt(n), zeros(n, 0);
  for (int i = 1; i <= n; ++i) cnt[i - 1] = (m + n - 2 * i) * dmax + 1;  // modpoly.py:466
  CK(cudaMemcpyAsync(d_f, fres, 4 * nf, cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(d_g, gres, 4 * ng, cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(d_fd, fdeg, 2 * ((size_t)m + 1), cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(d_gd, gdeg, 2 * ((size_t)n + 1), cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(d_r, rmod, 4 * (size_t)rlen, cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(d_cnt, cnt.data(), 4 * (size_t)n, cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(d_ns, cnt.data(), 4 * (size_t)n, cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(d_pi, zeros.data(), 4 * (size_t)n, cudaMemcpyHostToDevice, st));
  CK(cudaMemsetAsync(d_status, 0, 4, st));
  const Prime P = h_prime(p);
  const uint32_t* lcf = d_f + (size_t)m * (dfx + 1);
  const uint32_t* lcg = d_g + (size_t)n * (dgx + 1);
  int64_t ncand = need + 64;
  for (;;) {
    if (ncand > lim) ncand = lim;
    launch_psc_points(lcf, fdeg[m], lcg, gdeg[n], P, (int)ncand, need, d_sel, d_count, st);
    int count = 0;
    CK(cudaMemcpyAsync(&count, d_count, 4, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    g.launches += 1;
    if (count >= need) break;
    if (ncand >= lim) return CKB_STATUS_UNLUCKY;  // modpoly.py:450-451: t reached p
    ncand *= 2;
  }
  launch_psc(d_f, d_fd, m, dfx, d_g, d_gd, n, dgx, P, d_sel, need, d_vals, nullptr, st);
  uint32_t* d_gs = nullptr;  // every psc_i interpolated from its first cnt_i points, one launch
  if ((size_t)(4 * W + 2) * 4 > kSmemLimit && (rc = dbuf("sp.gs", (size_t)n * (4 * W + 2), &d_gs))) return rc;
  launch_interp_points(d_sel, d_vals, d_ns, W, d_prime, d_pi, n, d_sr, d_gs, st, 0);
  launch_gcd_chain(d_r, rlen, rlen_int, d_sr, d_cnt, W, n, P, d_chain, d_status, st);
  g.launches += 3;
  CK(cudaGetLastError());
  uint32_t status = 0;
  CK(cudaMemcpyAsync(chain, d_chain, 4 * ((size_t)n + 1), cudaMemcpyDeviceToHost, st));
  CK(cudaMemcpyAsync(&status, d_status, 4, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  return status ? CKB_STATUS_UNLUCKY : 0;
}

// ---- device-pointer entry points for the multi-GPU driver -------------------
int ckb_dev_modular_images(const uint32_t* d_limbs, int C, int L, const int16_t* d_degs, const int16_t* h_degs, int m,
                           int n, int dfx, int dgx, const uint32_t* primes, const uint32_t* gens, int K, int N,
                           uint32_t* d_coeffs, uint32_t* d_status, void* stream) {
  std::lock_guard<std::mutex> lk(g_mu);
  int rc;
  if ((rc = ensure_ready())) return rc;
  if ((rc = check_primes(primes, K))) return rc;
  cudaStream_t st = pick_stream(stream);
  Prime* d_primes;
  if ((rc = get_primes_dev(primes, K, &d_primes))) return rc;
  std::vector<uint64_t> key = {3, (uint64_t)C, (uint64_t)L, (uint64_t)m, (uint64_t)n, (uint64_t)dfx, (uint64_t)dgx,
                               (uint64_t)K, (uint64_t)N, (uint64_t)d_limbs, (uint64_t)d_degs, (uint64_t)d_coeffs,
                               (uint64_t)d_status, (uint64_t)st, (uint64_t)d_primes};
  key_push(key, h_degs, 2 * (size_t)(m + n + 2));
  key_push(key, primes, 4 * (size_t)K);
  key_push(key, gens, 4 * (size_t)K);
  return graphed(key, st, [&]() -> int {
    g.nsev = 0;
    return modular_stage(d_limbs, C, L, d_degs, h_degs, m, n, dfx, dgx, d_primes, primes, gens, K, N, d_coeffs,
                         d_status, st);
  });
}

int ckb_dev_crt(const uint32_t* d_coeffs, int K, int N, const uint32_t* primes, int LW, uint32_t* d_out,
                void* stream) {
  std::lock_guard<std::mutex> lk(g_mu);
  int rc;
  if ((rc = ensure_ready())) return rc;
  if ((rc = check_primes(primes, K))) return rc;
  cudaStream_t st = pick_stream(stream);
  CrtEntry* ce;
  if ((rc = get_crt(primes, K, LW, &ce))) return rc;
  uint32_t* d_crtS;
  if ((rc = dbuf("crtS", crt_scratch_words(K, N, LW), &d_crtS))) return rc;
  std::vector<uint64_t> key = {4, (uint64_t)K, (uint64_t)N, (uint64_t)LW, (uint64_t)d_coeffs, (uint64_t)d_out,
                               (uint64_t)st};
  key_push(key, primes, 4 * (size_t)K);
  return graphed(key, st, [&]() -> int {
    g.launches += launch_crt(ce->t, d_coeffs, N, d_out, d_crtS, st);
    CK(cudaGetLastError());
    return 0;
  });
}

int ckb_dev_biv_resultant(const uint32_t* d_limbs, int C, int L, const int16_t* d_degs, const int16_t* h_degs, int m,
                          int n, int dfx, int dgx, const uint32_t* primes, const uint32_t* gens, int K, int N, int LW,
                          uint32_t* d_out, uint32_t* d_status, void* stream) {
  std::lock_guard<std::mutex> lk(g_mu);
  int rc;
  if ((rc = ensure_ready())) return rc;
  if (m < 1 || n < 1 || K < 1 || N < 1 || L < 1 || LW < 1) return fail("ckb_dev_biv_resultant: bad sizes", -2);
  if ((rc = check_primes(primes, K))) return rc;
  cudaStream_t st = pick_stream(stream);
  CrtEntry* ce;
  if ((rc = get_crt(primes, K, LW, &ce))) return rc;
  uint32_t* d_coeffs;
  if ((rc = dbuf("coeffs", std::max((size_t)K * N, crt_a_words(K, N)), &d_coeffs))) return rc;
  uint32_t* d_crtS;
  if ((rc = dbuf("crtS", crt_scratch_words(K, N, LW), &d_crtS))) return rc;
  std::vector<uint64_t> key = {1, (uint64_t)C, (uint64_t)L, (uint64_t)m, (uint64_t)n, (uint64_t)dfx, (uint64_t)dgx,
                               (uint64_t)K, (uint64_t)N, (uint64_t)LW, (uint64_t)d_limbs, (uint64_t)d_degs,
                               (uint64_t)d_out, (uint64_t)d_status, (uint64_t)st};
  key_push(key, h_degs, 2 * (size_t)(m + n + 2));
  key_push(key, primes, 4 * (size_t)K);
  key_push(key, gens, 4 * (size_t)K);
  return graphed(key, st, [&]() -> int {
    int r;
    g.nsev = 0;
    if ((r = modular_stage(d_limbs, C, L, d_degs, h_degs, m, n, dfx, dgx, ce->d_primes, primes, gens, K, N,
                           d_coeffs, d_status, st, &ce->t)))
      return r;
    g.launches += launch_crt(ce->t, d_coeffs, N, d_out, d_crtS, st, true);
    stage_mark(st);
    CK(cudaGetLastError());
    return 0;
  });
}


int ckb_descartes_prepare(const uint32_t* limbs, int n, int L, const uint32_t* primes, const uint32_t* gens, int K) {
  std::lock_guard<std::mutex> lk(g_mu);
  int rc;
  if ((rc = ensure_ready())) return rc;
  if (n < 1 || L < 1 || K < 1 || K > 8192) return fail("ckb_descartes_prepare: bad sizes", -2);
  if ((rc = check_primes(primes, K))) return rc;
  int logL = 0;
  while ((1 << logL) < 2 * n + 1) ++logL;
  // degrees whose correlation length exceeds the primes' 2^14 roots of unity: direct O(n^2) correlations
  const char* fd = getenv("CKB_DESC_DIRECT");  // force the direct mode (parity tests of that path at small n)
  const bool direct = logL > DESC_NTT_LOG2_MAX || (fd && fd[0] == '1');
  for (int i = 0; i < K; ++i)
    if (primes[i] >= (1u << 30) || (!direct && (primes[i] - 1) % (1u << logL)))
      return fail("ckb_descartes_prepare: primes must be < 2^30 and 1 mod the NTT length (PRIMES30)", -2);
  int h = -1;
  for (size_t i = 0; i < g_desc.size(); ++i)
    if (!g_desc[i].used) h = (int)i;
  if (h < 0) {
    if (g_desc.size() >= 64) return fail("ckb_descartes_prepare: too many live handles", -2);
    g_desc.emplace_back();
    h = (int)g_desc.size() - 1;
  }
  DescHandle d;  // committed to the slot only once everything succeeded
  d.n = n;
  d.K = K;
  d.primes.assign(primes, primes + K);
  d.gens.assign(gens, gens + K);
  const int Lt = direct ? n + 1 : 1 << logL;
  const size_t n1 = (size_t)n + 1, kh = direct ? 0 : (size_t)K * (Lt / 2), kl = (size_t)K * Lt;
  const size_t words = (size_t)K * n1 * 3 + kh * 4 + kl * (direct ? 1 : 2) + (size_t)K * 5 + 64;
  auto bail = [&](int code) {
    if (d.blob) cudaFree(d.blob);
    return code;
  };
  {
    cudaError_t e = cudaMalloc(&d.blob, 4 * words);
    if (e != cudaSuccess) {
      d.blob = nullptr;
      return fail(std::string("ckb_descartes_prepare: cudaMalloc: ") + cudaGetErrorString(e));
    }
  }
  uint32_t* b = (uint32_t*)d.blob;
  auto take = [&](size_t m) { uint32_t* r = b; b += m; return r; };
  d.d_res = take((size_t)K * n1);
  DescPlan& pl = d.pl;
  pl.K = K;
  pl.n = n;
  pl.L = Lt;
  pl.logL = direct ? 0 : logL;
  pl.direct = direct ? 1 : 0;
  pl.fact = take((size_t)K * n1);
  pl.ifact = take((size_t)K * n1);
  pl.W = take(kh);
  pl.Wc = take(kh);
  pl.Wi = take(kh);
  pl.Wic = take(kh);
  pl.Vf = take(kl);
  pl.Vfc = direct ? nullptr : take(kl);
  pl.Linv = take(K);
  uint32_t* d_gens = take(K);
  d.d_primes = reinterpret_cast<Prime*>(take((size_t)K * 3));
  std::vector<Prime> hp(K);
  for (int i = 0; i < K; ++i) hp[i] = h_prime(primes[i]);
  cudaStream_t st = g.stream;
  uint32_t* d_limbs;
  if ((rc = dbuf("desc.limbs", n1 * L, &d_limbs))) return bail(rc);
  cudaError_t e = cudaMemcpyAsync(d.d_primes, hp.data(), sizeof(Prime) * K, cudaMemcpyHostToDevice, st);
  if (e == cudaSuccess) e = cudaMemcpyAsync(d_gens, gens, 4 * (size_t)K, cudaMemcpyHostToDevice, st);
  if (e == cudaSuccess) e = cudaMemcpyAsync(d_limbs, limbs, 4 * n1 * L, cudaMemcpyHostToDevice, st);
  if (e == cudaSuccess) {
    launch_reduce(d_limbs, (int)n1, L, d.d_primes, K, d.d_res, st);
    launch_desc_plan(d.d_primes, d_gens, pl, st);
    g.launches += 2;
    e = cudaGetLastError();
  }
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) return bail(fail(std::string("ckb_descartes_prepare: ") + cudaGetErrorString(e)));
  d.used = true;
  g_desc[h] = d;
  return h;
}

int ckb_descartes_variations_batch(int handle, const uint32_t* aw, int AL, const int32_t* ld, int B, int K, int LW,
                                   int32_t* variations) {
  std::lock_guard<std::mutex> lk(g_mu);
  int rc;
  if ((rc = ensure_ready())) return rc;
  if (handle < 0 || handle >= (int)g_desc.size() || !g_desc[handle].used)
    return fail("ckb_descartes_variations: bad handle", -2);
  DescHandle& d = g_desc[handle];
  if (K < 1 || K > d.K || AL < 1 || LW < 1 || B < 1 || B > 4096) return fail("ckb_descartes_variations: bad sizes", -2);
  for (int b = 0; b < B; ++b)
    if (ld[b] < 0) return fail("ckb_descartes_variations: negative ld", -2);
  cudaStream_t st = g.stream;
  const int N = d.n + 1;
  CrtEntry* ce;
  if ((rc = get_crt(d.primes.data(), K, LW, &ce))) return rc;
  uint32_t *d_aw, *d_c, *d_out, *d_crtS;
  int32_t *d_v, *d_ld;
  const size_t NB = (size_t)N * B;  // every interval's coefficients side by side: one CRT
  if ((rc = dbuf("desc.aw", 2 * (size_t)AL * B, &d_aw))) return rc;
  if ((rc = dbuf("desc.ld", (size_t)B, &d_ld))) return rc;
  if ((rc = dbuf("desc.c", (size_t)K * NB, &d_c))) return rc;
  if ((rc = dbuf("desc.out", NB * LW, &d_out))) return rc;
  if ((rc = dbuf("desc.v", (size_t)B, &d_v))) return rc;
  if ((rc = dbuf("crtS", crt_scratch_words(K, (int)NB, LW), &d_crtS))) return rc;
  CK(cudaMemcpyAsync(d_aw, aw, 8 * (size_t)AL * B, cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(d_ld, ld, 4 * (size_t)B, cudaMemcpyHostToDevice, st));
  DescPlan pl = d.pl;
  pl.K = K;  // the first K primes of the prepared set
  uint32_t* d_dscr = nullptr;
  if (pl.direct && (rc = dbuf("desc.direct", desc_direct_scratch_words(K, d.n, B), &d_dscr))) return rc;
  launch_desc_shift(d.d_primes, pl, d.d_res, d_aw, AL, d_ld, B, d_c, d_dscr, st);
  g.launches += launch_crt(ce->t, d_c, (int)NB, d_out, d_crtS, st);
  launch_desc_signs(d_out, N, LW, B, d_v, st);
  g.launches += pl.direct ? 4 : 2;  // the shift (3 direct kernels or 1), the sign count
  CK(cudaGetLastError());
  CK(cudaMemcpyAsync(variations, d_v, 4 * (size_t)B, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  return 0;
}

int ckb_descartes_variations(int handle, const uint32_t* aw, int AL, int ld, int K, int LW, int32_t* variations) {
  return ckb_descartes_variations_batch(handle, aw, AL, &ld, 1, K, LW, variations);
}

int ckb_descartes_release(int handle) {
  std::lock_guard<std::mutex> lk(g_mu);
  if (handle < 0 || handle >= (int)g_desc.size() || !g_desc[handle].used) return 0;
  DescHandle& d = g_desc[handle];
  cudaStreamSynchronize(g.stream);
  cudaFree(d.blob);
  d = DescHandle();
  return 0;
}

void* ckb_host_alloc(unsigned long long bytes) {
  std::lock_guard<std::mutex> lk(g_mu);
  if (ensure_ready()) return nullptr;
  void* p = pinned_alloc((size_t)bytes);
  if (!p) fail("ckb_host_alloc: cudaMallocHost failed", -1);
  return p;
}

int ckb_host_free(void* p) {
  std::lock_guard<std::mutex> lk(g_mu);
  if (p) CK(cudaFreeHost(p));
  return 0;
}

int ckb_set_graphs(int on) {
  std::lock_guard<std::mutex> lk(g_mu);
  const char* e = getenv("CKB_NO_GRAPHS");
  g.graphs = on != 0 && !(e && e[0] == '1') && !poison_mode();
  return 0;
}

int ckb_host_times(float* us, int max) {
  // diagnostics of the last ckb_biv_resultant call: host microseconds from entry
  // to the work enqueued (checks, staging, graph launch), and waiting for it
  std::lock_guard<std::mutex> lk(g_mu);
  for (int i = 0; i < max && i < 2; ++i) us[i] = g_host_times[i];
  return 2;
}

int ckb_set_timing(int on) {
  std::lock_guard<std::mutex> lk(g_mu);
  g.timing = on != 0;
  g.nsev = 0;
  return 0;
}

int ckb_stage_times(float* ms, int max) {
  // durations between consecutive stage marks of the last pipeline call:
  // reduce, plan, images, interpolation, crt
  std::lock_guard<std::mutex> lk(g_mu);
  int rc;
  if ((rc = ensure_ready())) return rc;
  if (g.nsev < 2) return 0;
  CK(cudaEventSynchronize(g.sev[g.nsev - 1]));
  int n = 0;
  for (int i = 1; i < g.nsev && n < max; ++i, ++n) CK(cudaEventElapsedTime(&ms[n], g.sev[i - 1], g.sev[i]));
  return n;
}

}  // extern "C"
