/* CPU oracle: a plain-C restatement of the reference's modular loops.
 *
 * TEST INFRASTRUCTURE ONLY.  Imported by tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs as the checker and the CPU
 * reference timing -- never by the product path (paper_1201_1548_b200/).
 *
 * Every function follows pkg/src/curvekit/modpoly.py line by line, including
 * the reference's algorithmic choices (Euclidean remainder sequence with a
 * Fermat inverse per division, Newton interpolation with a Fermat inverse
 * inside the O(N^2) loop, points t = 0, 1, 2, ... skipping zeros of the
 * leading coefficients).  Residues are < p < 2^31, so products fit in 64 bits.
 * Pinned against the reference's golden vectors in tests/test_oracle.py.
 */
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef uint64_t u64;
typedef int64_t i64;

static u64 powmod(u64 a, u64 e, u64 p) { /* Python pow(a, e, p) */
  u64 r = 1 % p;
  a %= p;
  while (e) {
    if (e & 1) r = r * a % p;
    a = a * a % p;
    e >>= 1;
  }
  return r;
}

static int trim(const u64* c, int len) { /* _zp_trim: returns new length */
  while (len > 0 && c[len - 1] == 0) --len;
  return len;
}

/* _zp_rem (modpoly.py:102-112): r = a rem b; returns len(r); r has room for la */
static int zp_rem(u64* r, const u64* a, int la, const u64* b, int lb, u64 p) {
  memcpy(r, a, sizeof(u64) * (size_t)la);
  int lr = la;
  u64 inv = powmod(b[lb - 1], p - 2, p);
  while (lr >= lb) {
    u64 c = r[lr - 1] * inv % p;
    if (c) {
      int k = lr - lb;
      for (int j = 0; j < lb; ++j) r[k + j] = (r[k + j] + p - c * b[j] % p) % p;
    }
    lr -= 1; /* r.pop() */
  }
  return trim(r, lr);
}

/* _zp_resultant (modpoly.py:132-153); a, b low-first residues */
u64 ck_zp_resultant(const u64* a0, int la, const u64* b0, int lb, u64 p) {
  la = trim(a0, la);
  lb = trim(b0, lb);
  if (!la || !lb) return 0;
  int W = (la > lb ? la : lb) + 1;
  u64* A = (u64*)malloc(sizeof(u64) * W);
  u64* B = (u64*)malloc(sizeof(u64) * W);
  u64* R = (u64*)malloc(sizeof(u64) * W);
  memcpy(A, a0, sizeof(u64) * la);
  memcpy(B, b0, sizeof(u64) * lb);
  u64 res = 1;
  if (la < lb) {
    if ((u64)(la - 1) * (u64)(lb - 1) % 2) res = p - 1;
    u64* t = A; A = B; B = t;
    int tl = la; la = lb; lb = tl;
  }
  for (;;) {
    int da = la - 1, db = lb - 1;
    if (db == 0) {
      res = res * powmod(B[0], (u64)da, p) % p;
      break;
    }
    int lr = zp_rem(R, A, la, B, lb, p);
    if (!lr) {
      res = 0;
      break;
    }
    int dr = lr - 1;
    if ((u64)da * (u64)db % 2) res = (p - res) % p;
    res = res * powmod(B[lb - 1], (u64)(da - dr), p) % p;
    u64* t = A; A = B; B = R; R = t; /* a, b = b, r */
    la = lb;
    lb = lr;
  }
  free(A);
  free(B);
  free(R);
  return res;
}

/* _zp_eval (modpoly.py:125-129) */
static u64 zp_eval(const u64* c, int len, u64 t, u64 p) {
  u64 acc = 0;
  for (int i = len - 1; i >= 0; --i) acc = (acc * t + c[i]) % p;
  return acc;
}

/* _zp_interp (modpoly.py:164-185); returns the trimmed length, out has n+1 room */
int ck_zp_interp(const i64* points, const u64* values, int n, u64 p, u64* out) {
  u64* c = (u64*)malloc(sizeof(u64) * (size_t)(n ? n : 1));
  u64* nxt = (u64*)malloc(sizeof(u64) * (size_t)(n + 2));
  memcpy(c, values, sizeof(u64) * (size_t)n);
  for (int j = 1; j < n; ++j)
    for (int i = n - 1; i >= j; --i) {
      u64 d = (u64)(((points[i] - points[i - j]) % (i64)p + (i64)p) % (i64)p);
      c[i] = ((c[i] + p - c[i - 1]) % p) * powmod(d, p - 2, p) % p;
    }
  int lo = 1;
  out[0] = 0;
  for (int i = n - 1; i >= 0; --i) {
    u64 pt = (u64)((points[i] % (i64)p + (i64)p) % (i64)p);
    for (int k = 0; k <= lo; ++k) nxt[k] = 0;
    for (int k = 0; k < lo; ++k) {
      nxt[k] = (nxt[k] + p - out[k] * pt % p) % p;
      nxt[k + 1] = (nxt[k + 1] + out[k]) % p;
    }
    nxt[0] = (nxt[0] + c[i]) % p;
    lo += 1;
    memcpy(out, nxt, sizeof(u64) * (size_t)lo);
  }
  free(c);
  free(nxt);
  return trim(out, lo);
}

/* _zp_gcd (modpoly.py:115-122); returns len of the monic gcd in out (room max(la,lb)) */
int ck_zp_gcd(const u64* a0, int la, const u64* b0, int lb, u64 p, u64* out) {
  int W = (la > lb ? la : lb) + 1;
  u64* A = (u64*)malloc(sizeof(u64) * W);
  u64* B = (u64*)malloc(sizeof(u64) * W);
  u64* R = (u64*)malloc(sizeof(u64) * W);
  memcpy(A, a0, sizeof(u64) * la);
  memcpy(B, b0, sizeof(u64) * lb);
  la = trim(A, la);
  lb = trim(B, lb);
  while (lb) {
    int lr = zp_rem(R, A, la, B, lb, p);
    u64* t = A; A = B; B = R; R = t;
    la = lb;
    lb = lr;
  }
  if (la) {
    u64 inv = powmod(A[la - 1], p - 2, p);
    for (int i = 0; i < la; ++i) out[i] = A[i] * inv % p;
  }
  free(A);
  free(B);
  free(R);
  return la;
}

/* One prime of biv_resultant's loop body (modpoly.py:376-391) on residues.
 * fres: (m+1) rows of (dfx+1) residues; gres likewise; lens = trimmed row lengths.
 * Produces the interpolated polynomial mod p in out (room npts+1); returns its
 * trimmed length, or -1 if a leading coefficient collapses (unlucky prime),
 * -2 if p is too small for the points. */
int ck_prime_image(const u64* fres, const int* flen, int m, int dfx, const u64* gres, const int* glen, int n,
                   int dgx, int npts, u64 p, u64* out) {
  const u64* lcf = fres + (size_t)m * (dfx + 1);
  const u64* lcg = gres + (size_t)n * (dgx + 1);
  if (!trim(lcf, flen[m]) || !trim(lcg, glen[n])) return -1;
  i64* pts = (i64*)malloc(sizeof(i64) * (size_t)npts);
  u64* vals = (u64*)malloc(sizeof(u64) * (size_t)npts);
  u64* fu = (u64*)malloc(sizeof(u64) * (size_t)(m + 1));
  u64* gu = (u64*)malloc(sizeof(u64) * (size_t)(n + 1));
  int cnt = 0;
  u64 t = 0;
  int rc = 0;
  while (cnt < npts) {
    if (t >= p) {
      rc = -2;
      break;
    }
    if (zp_eval(lcf, flen[m], t, p) && zp_eval(lcg, glen[n], t, p)) {
      for (int j = 0; j <= m; ++j) fu[j] = zp_eval(fres + (size_t)j * (dfx + 1), flen[j], t, p);
      for (int j = 0; j <= n; ++j) gu[j] = zp_eval(gres + (size_t)j * (dgx + 1), glen[j], t, p);
      pts[cnt] = (i64)t;
      vals[cnt] = ck_zp_resultant(fu, m + 1, gu, n + 1, p);
      ++cnt;
    }
    ++t;
  }
  if (!rc) rc = ck_zp_interp(pts, vals, npts, p, out);
  free(pts);
  free(vals);
  free(fu);
  free(gu);
  return rc;
}

/* Many primes in parallel (SPEC.md:269-270 permits concurrent primes). */
typedef struct {
  const u64* fres;  /* [K][(m+1)(dfx+1)] */
  const int* flen;
  int m, dfx;
  const u64* gres;  /* [K][(n+1)(dgx+1)] */
  const int* glen;
  int n, dgx, npts;
  const u64* primes;
  u64* out;         /* [K][npts+1] */
  int* rcs;         /* [K] */
  int K, next;
  pthread_mutex_t mu;
} Job;

static void* worker(void* arg) {
  Job* J = (Job*)arg;
  for (;;) {
    pthread_mutex_lock(&J->mu);
    int k = J->next++;
    pthread_mutex_unlock(&J->mu);
    if (k >= J->K) break;
    J->rcs[k] = ck_prime_image(J->fres + (size_t)k * (J->m + 1) * (J->dfx + 1), J->flen, J->m, J->dfx,
                               J->gres + (size_t)k * (J->n + 1) * (J->dgx + 1), J->glen, J->n, J->dgx, J->npts,
                               J->primes[k], J->out + (size_t)k * (J->npts + 1));
  }
  return NULL;
}

int ck_prime_images(const u64* fres, const int* flen, int m, int dfx, const u64* gres, const int* glen, int n, int dgx,
                    int npts, const u64* primes, int K, int threads, u64* out, int* rcs) {
  Job J;
  J.fres = fres; J.flen = flen; J.m = m; J.dfx = dfx;
  J.gres = gres; J.glen = glen; J.n = n; J.dgx = dgx; J.npts = npts;
  J.primes = primes; J.out = out; J.rcs = rcs; J.K = K; J.next = 0;
  pthread_mutex_init(&J.mu, NULL);
  if (threads < 1) threads = 1;
  if (threads > 256) threads = 256;
  pthread_t th[256];
  for (int i = 0; i < threads; ++i) pthread_create(&th[i], NULL, worker, &J);
  for (int i = 0; i < threads; ++i) pthread_join(th[i], NULL);
  pthread_mutex_destroy(&J.mu);
  return 0;
}
