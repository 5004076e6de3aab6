// Helpers of the images kernels (ckb_images.cu): the polyphase factor, the
// staged table layout and the mbarrier / bulk-copy primitives of the table staging.
#pragma once
#include <cstdint>

namespace ckb {

constexpr int POLY = 8;  // polyphase factor S: one 8-lane group per coset {w^j y_u}

__device__ __forceinline__ uint32_t img_smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void img_mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(bar), "r"(count));
}
__device__ __forceinline__ void img_mbar_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void img_mbar_wait(uint32_t bar, uint32_t parity) {
  uint32_t done = 0;
  do {
    asm volatile(
        "{\n .reg .pred P;\n mbarrier.try_wait.parity.shared::cta.b64 P, [%1], %2;\n selp.u32 %0, 1, 0, P;\n}\n"
        : "=r"(done)
        : "r"(bar), "r"(parity)
        : "memory");
  } while (!done);
}
__device__ __forceinline__ void img_bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(dst),
               "l"(src), "r"(bytes), "r"(bar)
               : "memory");
}

// shared-memory row width of the transposed, top-aligned residue tables.  An
// odd number of 16-byte chunks per row makes the 8 rows read by one lane
// group (x-powers r + 8e', r < 8) fall in disjoint banks.
template <int MAXD>
struct ImgLayout {
  static constexpr int NCH = (MAXD + 4) / 4;                   // chunks of 4 registers
  static constexpr int SW = ((NCH & 1) ? NCH : NCH + 1) * 4;   // words per x-power row
};


}  // namespace ckb
