// Shared pieces of the sm_100a attention kernels (attention_fwd.cu, attention_bwd.cu):
// 128 x 128 bf16 tiles stored as two 64-column SWIZZLE_128B atoms, their tcgen05 smem
// descriptors, and the TMEM store / exp2 helpers.
#pragma once

#include "dm_common.cuh"
#include "dm_internal.h"

namespace dm {

constexpr int AT_D = 128;                               // head dim
constexpr int AT_BM = 128;                              // query rows per CTA (= TMEM lanes)
constexpr int AT_BN = 128;                              // keys per KV tile
constexpr uint32_t AT_TILE = AT_BM * AT_D * 2;          // 32 KiB: one Q, K, V or P tile
constexpr uint32_t AT_ATOM = AT_BM * 128;               // 16 KiB: 128 rows x 64 bf16 (SWIZZLE_128B)

__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};"
      :: "r"(taddr), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]),
         "r"(r[7]), "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]),
         "r"(r[15])
      : "memory");
}
__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
// K-major [128 rows x 128] bf16 tile stored as two 64-column SWIZZLE_128B atoms: k16 step kk.
__device__ __forceinline__ uint64_t at_kmajor(uint32_t base, int kk) {
  return make_sdesc_sw128(base + (kk >> 2) * AT_ATOM + (kk & 3) * 32, 16, 1024);
}
// V as the MN-major B operand of P·V: [128 keys (K) x 128 d (N)], two 64-d atoms.
__device__ __forceinline__ uint64_t at_mnmajor(uint32_t base, int kk) {
  return make_sdesc_sw128(base + kk * 2048, AT_ATOM, 1024);
}

}  // namespace dm
