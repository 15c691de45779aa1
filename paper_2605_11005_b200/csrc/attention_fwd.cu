// Causal GQA flash-attention forward on 5th-gen tensor cores (sm_100a): the A-side
// attention of SURVEY.md §8f row 3, whose cost the reference only models,
// C_a = b·(s·H²·(2+2/g) + 4·s²·H) (pkg/src/afpipe/costs.py:84-87).
//
// One CTA = one (sequence, query head, 128-query tile); head_dim 128. Warp roles:
//   warp 0   TMA producer: the Q tile once, then K_j / V_j tiles through a 2-stage ring
//   warp 1   MMA issuer (one thread): S_j = Q·K_jᵀ into one of two TMEM S buffers, then
//            O += P_{j-1}·V_{j-1} into the TMEM O accumulator (P from smem, V MN-major)
//   warp 2   TMEM allocator
//   warps 4-7 softmax: thread r owns query row r (= TMEM lane r): reads its S row with
//            tcgen05.ld, online softmax in the exp2 domain (running max m, sum l), rescales
//            its O row in TMEM (tcgen05.ld/st) when the max moved, writes its P row (bf16)
//            into the SWIZZLE_128B smem tile the next MMA reads; final O / l and the
//            natural-log LSE go to global memory.
// S_{j+1} is issued before PV_j, so the exponentials of tile j+1 overlap the P·V MMA of
// tile j; the causal diagonal tile masks key > query. Query tiles run heaviest first.
#include "dm_common.cuh"
#include "dm_internal.h"

namespace dm {

constexpr int AT_D = 128;                               // head dim
constexpr int AT_BM = 128;                              // query rows per CTA (= TMEM lanes)
constexpr int AT_BN = 128;                              // keys per KV tile
constexpr int AT_STAGES = 2;
constexpr uint32_t AT_TILE = AT_BM * AT_D * 2;          // 32 KiB: one Q, K, V or P tile
constexpr uint32_t AT_ATOM = AT_BM * 128;               // 16 KiB: 128 rows x 64 bf16 (SWIZZLE_128B)
constexpr int AT_THREADS = 256;
constexpr size_t AT_SMEM = 1024 + (size_t)AT_TILE * (2 + 2 * AT_STAGES) + 256;

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

// K-major [128 rows x 128] bf16 tile stored as two 64-column SWIZZLE_128B atoms: k16 step kk.
__device__ __forceinline__ uint64_t at_kmajor(uint32_t base, int kk) {
  return make_sdesc_sw128(base + (kk >> 2) * AT_ATOM + (kk & 3) * 32, 16, 1024);
}
// V as the MN-major B operand of P·V: [128 keys (K) x 128 d (N)], two 64-d atoms.
__device__ __forceinline__ uint64_t at_mnmajor(uint32_t base, int kk) {
  return make_sdesc_sw128(base + kk * 2048, AT_ATOM, 1024);
}

__global__ void __launch_bounds__(AT_THREADS, 1)
attn_fwd_kernel(const __grid_constant__ CUtensorMap tm, int seq_len, int nh, int nkv, int ld_out,
                __nv_bfloat16* __restrict__ out, float* __restrict__ lse, float scale_log2) {
  extern __shared__ uint8_t smem_raw[];
  const uint32_t pad = (1024u - (smem_u32(smem_raw) & 1023u)) & 1023u;
  uint8_t* smem = smem_raw + pad;
  uint8_t* sQ = smem;
  uint8_t* sP = smem + AT_TILE;
  uint8_t* sKV = smem + 2 * AT_TILE;                    // stage s: K at +2s·TILE, V at +(2s+1)·TILE
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + (size_t)AT_TILE * (2 + 2 * AT_STAGES));
  uint64_t* q_full = bars;
  uint64_t* kv_full = bars + 1;                         // [AT_STAGES]
  uint64_t* kv_empty = bars + 1 + AT_STAGES;            // [AT_STAGES]
  uint64_t* s_full = bars + 1 + 2 * AT_STAGES;          // [2]
  uint64_t* s_free = bars + 3 + 2 * AT_STAGES;          // [2]
  uint64_t* p_full = bars + 5 + 2 * AT_STAGES;
  uint64_t* pv_done = bars + 6 + 2 * AT_STAGES;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 8 + 2 * AT_STAGES);

  const int n_qt = seq_len / AT_BM;
  const int qt = n_qt - 1 - (int)blockIdx.x;            // longest causal rows first
  const int h = blockIdx.y, b = blockIdx.z;
  const int hk = h / (nh / nkv);
  const int row0 = b * seq_len;
  const int n_kv = qt + 1;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    mbar_init(q_full, 1);
    for (int s = 0; s < AT_STAGES; ++s) { mbar_init(&kv_full[s], 1); mbar_init(&kv_empty[s], 1); }
    for (int i = 0; i < 2; ++i) { mbar_init(&s_full[i], 1); mbar_init(&s_free[i], AT_BM); }
    mbar_init(p_full, AT_BM);
    mbar_init(pv_done, 1);
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc(tmem_slot, 512);            // S0 [0,128) S1 [128,256) O [256,384)
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      tma_prefetch_desc(&tm);
      const int qcol = h * AT_D, kcol = (nh + hk) * AT_D, vcol = (nh + nkv + hk) * AT_D;
      mbar_expect_tx(q_full, AT_TILE);
      tma_load_2d(sQ, &tm, q_full, qcol, row0 + qt * AT_BM);
      tma_load_2d(sQ + AT_ATOM, &tm, q_full, qcol + 64, row0 + qt * AT_BM);
      for (int j = 0; j < n_kv; ++j) {
        const int s = j % AT_STAGES;
        mbar_wait(&kv_empty[s], ((j / AT_STAGES) & 1) ^ 1);
        uint8_t* k = sKV + (size_t)s * 2 * AT_TILE;
        uint8_t* v = k + AT_TILE;
        const int r = row0 + j * AT_BN;
        mbar_expect_tx(&kv_full[s], 2 * AT_TILE);
        tma_load_2d(k, &tm, &kv_full[s], kcol, r);
        tma_load_2d(k + AT_ATOM, &tm, &kv_full[s], kcol + 64, r);
        tma_load_2d(v, &tm, &kv_full[s], vcol, r);
        tma_load_2d(v + AT_ATOM, &tm, &kv_full[s], vcol + 64, r);
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idesc_s = make_idesc_bf16(AT_BM, AT_BN, 0, 0);   // Q K-major, K K-major
      constexpr uint32_t idesc_o = make_idesc_bf16(AT_BM, AT_D, 0, 1);    // P K-major, V MN-major
      const uint32_t qa = smem_u32(sQ), pa = smem_u32(sP);
      mbar_wait(q_full, 0);
      tc_fence_after();
      for (int j = 0; j <= n_kv; ++j) {
        if (j < n_kv) {
          const int s = j % AT_STAGES, sb = j & 1;
          mbar_wait(&kv_full[s], (j / AT_STAGES) & 1);
          if (j >= 2) mbar_wait(&s_free[sb], ((j - 2) >> 1) & 1);
          tc_fence_after();
          const uint32_t ka = smem_u32(sKV + (size_t)s * 2 * AT_TILE);
#pragma unroll
          for (int kk = 0; kk < AT_D / 16; ++kk)
            umma_bf16_ss(tmem + sb * AT_BN, at_kmajor(qa, kk), at_kmajor(ka, kk), idesc_s, kk > 0 ? 1u : 0u);
          umma_commit(&s_full[sb]);
        }
        if (j >= 1) {
          const int jj = j - 1, s = jj % AT_STAGES;
          mbar_wait(p_full, jj & 1);
          tc_fence_after();
          const uint32_t va = smem_u32(sKV + (size_t)s * 2 * AT_TILE + AT_TILE);
#pragma unroll
          for (int kk = 0; kk < AT_BN / 16; ++kk)
            umma_bf16_ss(tmem + 2 * AT_BN, at_kmajor(pa, kk), at_mnmajor(va, kk), idesc_o,
                         (jj | kk) != 0 ? 1u : 0u);
          umma_commit(pv_done);
          umma_commit(&kv_empty[s]);
        }
      }
    }
    __syncwarp();
  } else if (warp >= 4) {
    const int q4 = warp & 3;
    const int r = q4 * 32 + lane;                       // query row in the tile = TMEM lane
    const uint32_t trow = tmem + (static_cast<uint32_t>(q4 * 32) << 16);
    const uint32_t prow = smem_u32(sP);
    float m = -INFINITY, l = 0.0f;
    for (int j = 0; j < n_kv; ++j) {
      const int sb = j & 1;
      mbar_wait(&s_full[sb], (j >> 1) & 1);
      tc_fence_after();
      uint32_t sv[AT_BN];
#pragma unroll
      for (int c = 0; c < AT_BN / 16; ++c)
        tmem_ld16(trow + sb * AT_BN + c * 16, *reinterpret_cast<uint32_t(*)[16]>(sv + c * 16));
      tmem_wait_ld();
      tc_fence_before();
      mbar_arrive(&s_free[sb]);                         // the MMA may overwrite this S buffer
      if (j == qt) {                                    // diagonal tile: key > query is masked
#pragma unroll
        for (int c = 0; c < AT_BN; ++c)
          if (c > r) sv[c] = __float_as_uint(-INFINITY);
      }
      float mx = -INFINITY;
#pragma unroll
      for (int c = 0; c < AT_BN; ++c) mx = fmaxf(mx, __uint_as_float(sv[c]));
      const float m_new = fmaxf(m, mx * scale_log2);
      const float alpha = exp2f(m - m_new);             // 0 on the first tile
      float sum = 0.0f;
      uint32_t pk[AT_BN / 2];
#pragma unroll
      for (int c = 0; c < AT_BN / 2; ++c) {
        const float p0 = exp2f(__fmaf_rn(__uint_as_float(sv[2 * c]), scale_log2, -m_new));
        const float p1 = exp2f(__fmaf_rn(__uint_as_float(sv[2 * c + 1]), scale_log2, -m_new));
        sum += p0 + p1;
        pk[c] = pack_bf16(p0, p1);
      }
      l = __fmaf_rn(l, alpha, sum);
      m = m_new;
      if (j >= 1) {
        mbar_wait(pv_done, (j - 1) & 1);                // O holds tiles < j; P buffer is free
        tc_fence_after();
        if (__any_sync(0xffffffffu, alpha != 1.0f)) {
#pragma unroll 1
          for (int c = 0; c < AT_D / 16; ++c) {
            uint32_t o[16];
            tmem_ld16(trow + 2 * AT_BN + c * 16, o);
            tmem_wait_ld();
#pragma unroll
            for (int i = 0; i < 16; ++i) o[i] = __float_as_uint(__uint_as_float(o[i]) * alpha);
            tmem_st16(trow + 2 * AT_BN + c * 16, o);
          }
          tmem_wait_st();
        }
      }
#pragma unroll
      for (int a = 0; a < 2; ++a)
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          const uint32_t* q = pk + a * 32 + c * 4;
          st_shared_v4(prow + a * AT_ATOM + sw128(r, c), q[0], q[1], q[2], q[3]);
        }
      fence_proxy_async_smem();                         // generic-proxy P writes -> tensor core
      tc_fence_before();
      mbar_arrive(p_full);
    }
    mbar_wait(pv_done, (n_kv - 1) & 1);
    tc_fence_after();
    const float inv = 1.0f / l;
    __nv_bfloat16* orow = out + (size_t)(row0 + qt * AT_BM + r) * ld_out + (size_t)h * AT_D;
#pragma unroll 1
    for (int c = 0; c < AT_D / 16; ++c) {
      uint32_t o[16];
      tmem_ld16(trow + 2 * AT_BN + c * 16, o);
      tmem_wait_ld();
      uint32_t w[8];
#pragma unroll
      for (int i = 0; i < 8; ++i)
        w[i] = pack_bf16(__uint_as_float(o[2 * i]) * inv, __uint_as_float(o[2 * i + 1]) * inv);
      int4* dst = reinterpret_cast<int4*>(orow + c * 16);
      dst[0] = make_int4((int)w[0], (int)w[1], (int)w[2], (int)w[3]);
      dst[1] = make_int4((int)w[4], (int)w[5], (int)w[6], (int)w[7]);
    }
    lse[((size_t)b * nh + h) * seq_len + qt * AT_BM + r] = (m + log2f(l)) * 0.69314718055994531f;
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 2) tmem_dealloc(tmem, 512);
}

}  // namespace dm

using namespace dm;

int dm_attention_fwd(const void* qkv, int T, int seq_len, int nh, int nkv, int head_dim, void* out, float* lse,
                     void* stream) {
  if (head_dim != AT_D) return set_error(DM_ERR_SHAPE, "attention_fwd: head_dim %d (only 128)", head_dim);
  if (T < 1 || seq_len < AT_BM || seq_len % AT_BM || T % seq_len)
    return set_error(DM_ERR_SHAPE, "attention_fwd: seq_len %d must be a multiple of 128 dividing T=%d", seq_len, T);
  if (nh < 1 || nkv < 1 || nh % nkv) return set_error(DM_ERR_SHAPE, "attention_fwd: %d heads, %d kv heads", nh, nkv);
  if ((reinterpret_cast<uintptr_t>(qkv) & 15) || (reinterpret_cast<uintptr_t>(out) & 15))
    return set_error(DM_ERR_ALIGN, "attention_fwd: qkv/out not 16-byte aligned");
  PFN_cuTensorMapEncodeTiled_v12000 enc = tensor_map_encoder();
  if (!enc) return set_error(DM_ERR_DRIVER, "cuTensorMapEncodeTiled entry point unavailable");
  const uint64_t cols = (uint64_t)(nh + 2 * nkv) * AT_D;
  CUtensorMap tm;
  cuuint64_t dims[2] = {cols, (cuuint64_t)T};
  cuuint64_t strides[1] = {cols * 2};
  cuuint32_t box[2] = {64, AT_BM};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(qkv), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return set_error(DM_ERR_DRIVER, "attention_fwd: cuTensorMapEncodeTiled failed (%d)", (int)r);
  static bool configured = false;
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(attn_fwd_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)AT_SMEM);
    if (e != cudaSuccess) return set_cuda_error(e, "cudaFuncSetAttribute(attn_fwd)");
    configured = true;
  }
  const float scale_log2 = 1.4426950408889634f / sqrtf((float)AT_D);
  dim3 grid(seq_len / AT_BM, nh, T / seq_len);
  attn_fwd_kernel<<<grid, AT_THREADS, AT_SMEM, (cudaStream_t)stream>>>(
      tm, seq_len, nh, nkv, nh * AT_D, reinterpret_cast<__nv_bfloat16*>(out), lse, scale_log2);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return set_cuda_error(e, "attention_fwd launch");
  note_launch();
  return DM_OK;
}
