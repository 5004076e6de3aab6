// Principal subresultant coefficients psc_i(t) mod p at many points, one warp
// per (point, i) -- the data-parallel core of modular_subres_profile
// (pkg/src/curvekit/modpoly.py:428-474, GeoTop's N^- test).
//
// For each candidate point t the warp evaluates the y-coefficients of f and g
// at t (modpoly.py:459-460), builds the (m+n-2i)-square matrix of _psc_det
// (:477-501) in shared memory and runs _zp_det (:504-526) -- Gaussian
// elimination with the first nonzero pivot, the determinant being the product
// of the pivots with a sign per row swap -- with the row updates spread over
// the lanes.  Lane 0 of the i = 1 warp also reports whether t annihilates a
// leading coefficient, so the host can select the reference's points.
#include "ckb_kernels.cuh"

namespace ckb {

__global__ void k_psc(const uint32_t* __restrict__ fres, const int16_t* __restrict__ fdeg, int m, int dfx,
                      const uint32_t* __restrict__ gres, const int16_t* __restrict__ gdeg, int n, int dgx, Prime P,
                      int ncand, int smax, uint32_t* __restrict__ out, uint8_t* __restrict__ valid) {
  extern __shared__ uint32_t sm[];
  const int cand = blockIdx.x, i = blockIdx.y + 1, lane = threadIdx.x;
  const uint32_t p = P.p;
  uint32_t* fu = sm;
  uint32_t* gu = sm + (m + 1);
  uint32_t* mat = gu + (n + 1);
  const uint32_t t = (uint32_t)cand % p;
  const uint32_t tc = shoup_comp(t, P);
  for (int j = lane; j <= m + n + 1; j += 32) {
    const bool isf = j <= m;
    const int jj = isf ? j : j - m - 1;
    const uint32_t* c = isf ? fres + j * (dfx + 1) : gres + jj * (dgx + 1);
    const int deg = isf ? fdeg[j] : gdeg[jj];
    uint32_t acc = 0;
    for (int e = deg; e >= 0; --e) acc = add_mod(shoup(acc, t, tc, p), c[e], p);
    (isf ? fu : gu)[jj] = acc;
  }
  __syncwarp();
  if (i == 1 && lane == 0) valid[cand] = (fu[m] != 0u && gu[n] != 0u);
  const int s = m + n - 2 * i;
  uint32_t det;
  if (s <= 0) {
    det = 1u % p;
  } else {
    // rows of _psc_det: n-i rows from a (= fu), m-i rows from b (= gu)
    for (int e = lane; e < s * s; e += 32) {
      const int r = e / s, col = e % s;
      int k;
      uint32_t v;
      if (r < n - i) {
        k = (col < s - 1) ? (m - col + r) : (2 * i - n + 1 + r);
        v = (k >= 0 && k <= m) ? fu[k] : 0u;
      } else {
        const int rr = r - (n - i);
        k = (col < s - 1) ? (n - col + rr) : (2 * i - m + 1 + rr);
        v = (k >= 0 && k <= n) ? gu[k] : 0u;
      }
      mat[e] = v;
    }
    __syncwarp();
    det = 1u % p;
    bool neg = false;
    for (int col = 0; col < s; ++col) {
      int sel = -1;
      for (int r0 = col; r0 < s && sel < 0; r0 += 32) {
        const int r = r0 + lane;
        const unsigned b = __ballot_sync(0xffffffffu, r < s && mat[r * s + col] != 0u);
        if (b) sel = r0 + __ffs(b) - 1;
      }
      if (sel < 0) {
        det = 0u;
        break;
      }
      if (sel != col) {
        for (int c = lane; c < s; c += 32) {
          const uint32_t a = mat[col * s + c];
          mat[col * s + c] = mat[sel * s + c];
          mat[sel * s + c] = a;
        }
        neg = !neg;
        __syncwarp();
      }
      const uint32_t pv = mat[col * s + col];
      det = mul_mod(det, pv, P);
      const uint32_t inv = inv_mod(pv, P);
      for (int r = col + 1; r < s; ++r) {
        const uint32_t f = mul_mod(mat[r * s + col], inv, P);
        __syncwarp();  // every lane has read mat[r][col] before lane 0 overwrites it
        if (f) {
          const uint32_t nf = p - f, nfc = shoup_comp(nf, P);
          for (int c = col + lane; c < s; c += 32)
            mat[r * s + c] = add_mod(mat[r * s + c], shoup(mat[col * s + c], nf, nfc, p), p);
        }
        __syncwarp();
      }
    }
    if (neg) det = neg_mod(det, p);
  }
  if (lane == 0) out[(size_t)(i - 1) * ncand + cand] = det;
}

void launch_psc(const uint32_t* fres, const int16_t* fdeg, int m, int dfx, const uint32_t* gres,
                const int16_t* gdeg, int n, int dgx, const Prime& P, int ncand, uint32_t* out, uint8_t* valid,
                cudaStream_t st) {
  const int smax = m + n - 2 > 0 ? m + n - 2 : 0;
  const size_t smem = (size_t)(m + n + 2 + smax * smax) * 4;
  if (smem > 48 * 1024) cudaFuncSetAttribute(k_psc, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  k_psc<<<dim3(ncand, n > 0 ? n : 1), 32, smem, st>>>(fres, fdeg, m, dfx, gres, gdeg, n, dgx, P, ncand, smax, out,
                                                      valid);
}

}  // namespace ckb
