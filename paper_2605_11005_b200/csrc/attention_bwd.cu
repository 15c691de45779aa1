// Causal GQA flash-attention backward on 5th-gen tensor cores (sm_100a): the backward of
// dm_attention_fwd (attention_fwd.cu), the A-side attention of SURVEY.md §8f row 3 whose
// cost the reference models as C_a's backward share (pkg/src/afpipe/costs.py:84-87,
// backward_scale costs.py:146-150).
//
// Given qkv [T, (nh + 2 nkv)·128], O, dO [T, nh·128] bf16 and the forward's natural-log
// LSE [b, nh, s], with S = scale·Q Kᵀ, P = exp(S - LSE), D = rowsum(dO ∘ O):
//   dV = Pᵀ dO,  dP = dO Vᵀ,  dS = P ∘ (dP - D),  dQ = scale·dS K,  dK = scale·dSᵀ Q.
// Three launches, all deterministic (no atomics):
//   attn_bwd_dot_kernel   D (warp per (token, head))
//   attn_bwd_dkdv_kernel  CTA per (128-key tile j, KV head, sequence): dK_j, dV_j accumulate in
//                         TMEM over the group's g query heads and the 64-query tiles at or past
//                         the diagonal: Sᵀ = K_j Q_iᵀ and dPᵀ = V_j dO_iᵀ (M = 128 keys, N = 64),
//                         the elementwise warps form Pᵀ and dSᵀ rows in bf16 (SWIZZLE_128B smem),
//                         then dV += Pᵀ dO_i, dK += dSᵀ Q_i with dO_i / Q_i re-read as MN-major
//                         B operands of the same smem tiles
//   attn_bwd_dq_kernel    CTA per (128-query tile i, query head, sequence): S = Q_i K_jᵀ and
//                         dP = dO_i V_jᵀ over the 64-key tiles j up to the diagonal, dS rows,
//                         dQ += dS K_j
// Both main kernels are software-pipelined: the S/dP accumulators are double-buffered in TMEM
// (2 x 2 x 64 columns) and the P/dS tiles in smem, the streamed operand (Q/dO, resp. K/V) has a
// 3-deep TMA ring, and the single MMA thread issues S(it+1), dP(it+1) before the dV/dK (dQ)
// MMAs of step it — so the tensor core works on the next step while the elementwise warps turn
// step it's S/dP rows into P/dS. Warp roles (384 threads): warp 0 TMA, warp 1 MMA issuer (one
// thread), warp 2 TMEM allocator, warps 4-11 elementwise (warp w: TMEM lanes 32·(w%4).., 32 of
// the 64 columns by (w-4)/4).
#include <map>

#include "attention_common.cuh"

namespace dm {

constexpr int AB_THREADS = 384;
constexpr float AB_LOG2E = 1.4426950408889634f;
constexpr int AB_EW = 8;                                  // elementwise warps
constexpr int AB_T = 64;                                  // streamed tile rows (queries / keys)
constexpr int AB_STAGES = 3;                              // TMA ring depth of the streamed tiles
constexpr uint32_t AB_ATOM64 = AB_T * 128;                // 8 KiB: 64 rows x 64 bf16 (SWIZZLE_128B)
constexpr uint32_t AB_TILE64 = 2 * AB_ATOM64;             // 16 KiB: 64 rows x 128 d
constexpr uint32_t AB_PT = AT_BM * 128;                   // 16 KiB: 128 rows x 64 bf16 (P / dS)

// K-major [64 rows x 128] tile (two 8 KiB atoms): k16 step kk of the 128-deep reduction
__device__ __forceinline__ uint64_t ab_kmajor64(uint32_t base, int kk) {
  return make_sdesc_sw128(base + (kk >> 2) * AB_ATOM64 + (kk & 3) * 32, 16, 1024);
}
// the same [64 rows x 128 d] tile as an MN-major B operand: K = its 64 rows, N = d
__device__ __forceinline__ uint64_t ab_mnmajor64(uint32_t base, int kk) {
  return make_sdesc_sw128(base + kk * 2048, AB_ATOM64, 1024);
}
// [128 rows x 64] single-atom tile (P / dS) as a K-major A operand: K = its 64 columns
__device__ __forceinline__ uint64_t ab_kmajor_p(uint32_t base, int kk) {
  return make_sdesc_sw128(base + kk * 32, 16, 1024);
}

// D[b][h][s] = sum_d dO[t, h, d] * O[t, h, d] (fp32) and the log2-domain LSE lse2 = LSE·log2(e)
// into the workspace [2][b][h][s] (D, then lse2): warp per (token, head)
__global__ void __launch_bounds__(256)
attn_bwd_dot_kernel(const __nv_bfloat16* __restrict__ o, const __nv_bfloat16* __restrict__ dout,
                    const float* __restrict__ lse, int T, int seq_len, int nh, float* __restrict__ dl) {
  const int lane = threadIdx.x & 31;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  for (int q = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; q < T * nh; q += nw) {
    const int t = q / nh, h = q % nh;
    const size_t off = (size_t)t * nh * AT_D + (size_t)h * AT_D + lane * 4;
    const uint2 a = *reinterpret_cast<const uint2*>(o + off), b = *reinterpret_cast<const uint2*>(dout + off);
    float s = bf16lo(a.x) * bf16lo(b.x);
    s = __fmaf_rn(bf16hi(a.x), bf16hi(b.x), s);
    s = __fmaf_rn(bf16lo(a.y), bf16lo(b.y), s);
    s = __fmaf_rn(bf16hi(a.y), bf16hi(b.y), s);
    s = warp_sum_butterfly(s);
    if (lane == 0) {
      const size_t q2 = ((size_t)(t / seq_len) * nh + h) * seq_len + t % seq_len;
      dl[q2] = s;
      dl[(size_t)T * nh + q2] = lse[q2] * AB_LOG2E;
    }
  }
}

// Elementwise step of one thread = one accumulator row r (TMEM lane) over 32 columns
// [c0, c0 + 32) of the 64-column S / dP buffers: bf16 P and dS into the row's four 16-byte
// chunks c0/8 .. c0/8+3 of a [128 x 64] SWIZZLE_128B tile. Key-major kernel (COLS_ARE_QUERIES):
// row = key, column = query, lse2c / ddc per column (smem, 16-byte aligned); query-major: row =
// query, one lse2r / ddr. MASK (diagonal tiles only): causal key > query, i.e. (row - col > off)
// key-major, (col - row > off) query-major, off = the tiles' position difference.
template <bool COLS_ARE_QUERIES, bool MASK>
__device__ __forceinline__ void ab_row32(uint32_t tS, uint32_t tP, uint32_t sPt, uint32_t sDS, int r, int c0, int off,
                                         const float* lse2c, const float* ddc, float lse2r, float ddr,
                                         float scale_log2) {
  uint32_t s32[32], d32[32];
  tmem_ld16(tS + c0, *reinterpret_cast<uint32_t(*)[16]>(s32));
  tmem_ld16(tS + c0 + 16, *reinterpret_cast<uint32_t(*)[16]>(s32 + 16));
  tmem_ld16(tP + c0, *reinterpret_cast<uint32_t(*)[16]>(d32));
  tmem_ld16(tP + c0 + 16, *reinterpret_cast<uint32_t(*)[16]>(d32 + 16));
  float l2v[COLS_ARE_QUERIES ? 32 : 1], ddv[COLS_ARE_QUERIES ? 32 : 1];
  if constexpr (COLS_ARE_QUERIES) {
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const float4 a = reinterpret_cast<const float4*>(lse2c + c0)[q], b = reinterpret_cast<const float4*>(ddc + c0)[q];
      l2v[4 * q] = a.x; l2v[4 * q + 1] = a.y; l2v[4 * q + 2] = a.z; l2v[4 * q + 3] = a.w;
      ddv[4 * q] = b.x; ddv[4 * q + 1] = b.y; ddv[4 * q + 2] = b.z; ddv[4 * q + 3] = b.w;
    }
  }
  tmem_wait_ld();
  uint32_t pw[16], dw[16];
#pragma unroll
  for (int q = 0; q < 16; ++q) {
    float p2[2], ds2[2];
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const int cc = 2 * q + u, c = c0 + cc;
      const float l2 = COLS_ARE_QUERIES ? l2v[cc] : lse2r;
      const float dv = COLS_ARE_QUERIES ? ddv[cc] : ddr;
      float p = ex2(__fmaf_rn(__uint_as_float(s32[cc]), scale_log2, -l2));
      if constexpr (MASK) p = (COLS_ARE_QUERIES ? (r - c > off) : (c - r > off)) ? 0.f : p;
      p2[u] = p;
      ds2[u] = p * (__uint_as_float(d32[cc]) - dv);
    }
    pw[q] = pack_bf16(p2[0], p2[1]);
    dw[q] = pack_bf16(ds2[0], ds2[1]);
  }
  const int ch = c0 >> 3;
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    if (sPt) st_shared_v4(sPt + sw128(r, ch + q), pw[4 * q], pw[4 * q + 1], pw[4 * q + 2], pw[4 * q + 3]);
    st_shared_v4(sDS + sw128(r, ch + q), dw[4 * q], dw[4 * q + 1], dw[4 * q + 2], dw[4 * q + 3]);
  }
}

// Accumulator rows r of a [128 x 128] fp32 TMEM block, columns [c0, c0 + 64) -> bf16 * sc
__device__ __forceinline__ void ab_store_acc(uint32_t tacc, int c0, float sc, bool zero, __nv_bfloat16* dst) {
#pragma unroll 1
  for (int c = c0; c < c0 + 64; c += 16) {
    uint32_t v[16];
    tmem_ld16(tacc + c, v);
    tmem_wait_ld();
    uint32_t w8[8];
#pragma unroll
    for (int q = 0; q < 8; ++q)
      w8[q] = zero ? 0u : pack_bf16(__uint_as_float(v[2 * q]) * sc, __uint_as_float(v[2 * q + 1]) * sc);
    int4* o4 = reinterpret_cast<int4*>(dst + c);
    o4[0] = make_int4((int)w8[0], (int)w8[1], (int)w8[2], (int)w8[3]);
    o4[1] = make_int4((int)w8[4], (int)w8[5], (int)w8[6], (int)w8[7]);
  }
}

// smem carve-up shared by both kernels' host sizing
constexpr size_t AB_SMEM_DKDV = 1024 + 2 * (size_t)AT_TILE + AB_STAGES * 2 * (size_t)AB_TILE64 + 4 * (size_t)AB_PT +
                                AB_STAGES * 2 * AB_T * sizeof(float) + 256;
constexpr size_t AB_SMEM_DQ = 1024 + 2 * (size_t)AT_TILE + AB_STAGES * 2 * (size_t)AB_TILE64 + 2 * (size_t)AB_PT + 256;

// smem descriptor + a byte offset (the 14-bit address field holds addr >> 4; tiles sit below
// 256 KiB, so the add never carries out of it)
__device__ __forceinline__ uint64_t dsc(uint64_t d, uint32_t bytes) { return d + (bytes >> 4); }

// dK_j, dV_j: CTA (128-key tile j = blockIdx.x (heaviest first), KV head, sequence)
__global__ void __launch_bounds__(AB_THREADS, 1)
attn_bwd_dkdv_kernel(const __grid_constant__ CUtensorMap tmkv, const __grid_constant__ CUtensorMap tmq,
                     const __grid_constant__ CUtensorMap tmdo, const float* __restrict__ lse2,
                     const float* __restrict__ dl, int seq_len, int nh, int nkv, float scale_log2, float scale,
                     __nv_bfloat16* __restrict__ dqkv) {
  extern __shared__ uint8_t smem_raw[];
  const uint32_t pad = (1024u - (smem_u32(smem_raw) & 1023u)) & 1023u;
  uint8_t* smem = smem_raw + pad;
  uint8_t* sK = smem;
  uint8_t* sV = sK + AT_TILE;
  uint8_t* sQ = sV + AT_TILE;                                   // [AB_STAGES] x 16 KiB
  uint8_t* sDO = sQ + AB_STAGES * AB_TILE64;                    // [AB_STAGES] x 16 KiB
  uint8_t* sPt = sDO + AB_STAGES * AB_TILE64;                   // [2] x 16 KiB
  uint8_t* sDSt = sPt + 2 * AB_PT;                              // [2] x 16 KiB
  float* s_lse = reinterpret_cast<float*>(sDSt + 2 * AB_PT);    // [AB_STAGES][64] log2-domain LSE of Q_i's rows
  float* s_dd = s_lse + AB_STAGES * AB_T;                       // [AB_STAGES][64] D of Q_i's rows
  uint64_t* bars = reinterpret_cast<uint64_t*>(s_dd + AB_STAGES * AB_T);
  uint64_t* kv_full = bars;
  uint64_t* ld_full = bars + 1;                  // [AB_STAGES] Q_i, dO_i, lse2, D landed
  uint64_t* ld_empty = ld_full + AB_STAGES;      // [AB_STAGES]
  uint64_t* st_full = ld_empty + AB_STAGES;      // [2] S^T / dP^T buffer b computed
  uint64_t* tm_empty = st_full + 2;              // [2] ... read out of TMEM
  uint64_t* p_full = tm_empty + 2;               // [2] P^T / dS^T smem buffer b written
  uint64_t* ps_empty = p_full + 2;               // [2] ... consumed by the dV / dK MMAs
  uint64_t* acc_done = ps_empty + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_done + 1);

  const int j = blockIdx.x, kvh = blockIdx.y, b = blockIdx.z;
  const int n_q = seq_len / AB_T, g = nh / nkv;
  const int per_head = n_q - 2 * j, n_it = g * per_head;
  const int row0 = b * seq_len;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    mbar_init(kv_full, 1);
    for (int s = 0; s < AB_STAGES; ++s) {
      mbar_init(&ld_full[s], 1);
      mbar_init(&ld_empty[s], 1);
    }
    for (int q = 0; q < 2; ++q) {
      mbar_init(&st_full[q], 1);
      mbar_init(&tm_empty[q], AB_EW);
      mbar_init(&p_full[q], AB_EW * 32);
      mbar_init(&ps_empty[q], 1);
    }
    mbar_init(acc_done, 1);
    fence_mbar_init();
  }
  // TMEM: S^T / dP^T buffer q at [128q, 128q + 64) / [128q + 64, 128q + 128); dV [256, 384), dK [384, 512)
  if (warp == 2) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      tma_prefetch_desc(&tmkv);
      tma_prefetch_desc(&tmq);
      tma_prefetch_desc(&tmdo);
      const int kcol = (nh + kvh) * AT_D, vcol = (nh + nkv + kvh) * AT_D, krow = row0 + j * AT_BN;
      mbar_expect_tx(kv_full, 2 * AT_TILE);
      tma_load_2d(sK, &tmkv, kv_full, kcol, krow);
      tma_load_2d(sK + AT_ATOM, &tmkv, kv_full, kcol + 64, krow);
      tma_load_2d(sV, &tmkv, kv_full, vcol, krow);
      tma_load_2d(sV + AT_ATOM, &tmkv, kv_full, vcol + 64, krow);
      for (int it = 0; it < n_it; ++it) {
        const int s = it % AB_STAGES;
        if (it >= AB_STAGES) mbar_wait(&ld_empty[s], (uint32_t)((it / AB_STAGES - 1) & 1));
        const int qh = kvh * g + it / per_head, i = 2 * j + it % per_head;
        const int qrow = row0 + i * AB_T;
        const size_t lrow = ((size_t)b * nh + qh) * seq_len + (size_t)i * AB_T;
        uint8_t* q = sQ + s * AB_TILE64;
        uint8_t* d = sDO + s * AB_TILE64;
        mbar_expect_tx(&ld_full[s], 2 * AB_TILE64 + 2 * AB_T * sizeof(float));
        tma_load_2d(q, &tmq, &ld_full[s], qh * AT_D, qrow);
        tma_load_2d(q + AB_ATOM64, &tmq, &ld_full[s], qh * AT_D + 64, qrow);
        tma_load_2d(d, &tmdo, &ld_full[s], qh * AT_D, qrow);
        tma_load_2d(d + AB_ATOM64, &tmdo, &ld_full[s], qh * AT_D + 64, qrow);
        bulk_load_1d(s_lse + s * AB_T, lse2 + lrow, AB_T * sizeof(float), &ld_full[s]);
        bulk_load_1d(s_dd + s * AB_T, dl + lrow, AB_T * sizeof(float), &ld_full[s]);
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idesc_s = make_idesc_bf16(AT_BN, AB_T, 0, 0);   // M = 128 keys, N = 64 queries
      constexpr uint32_t idesc_a = make_idesc_bf16(AT_BN, AT_D, 0, 1);   // M = 128 keys, N = d, B MN-major
      const uint64_t dk0 = at_kmajor(smem_u32(sK), 0), dv0 = at_kmajor(smem_u32(sV), 0);
      const uint64_t dq0 = ab_kmajor64(smem_u32(sQ), 0), ddo0 = ab_kmajor64(smem_u32(sDO), 0);
      const uint64_t mq0 = ab_mnmajor64(smem_u32(sQ), 0), mdo0 = ab_mnmajor64(smem_u32(sDO), 0);
      const uint64_t dp0 = ab_kmajor_p(smem_u32(sPt), 0), dds0 = ab_kmajor_p(smem_u32(sDSt), 0);
      auto dvdk = [&](int q) {   // dV += P^T dO_q, dK += dS^T Q_q
        const int s = q % AB_STAGES, pb = q & 1;
        mbar_wait(&p_full[pb], (uint32_t)((q >> 1) & 1));
        tc_fence_after();
        const uint64_t pa = dsc(dp0, pb * AB_PT), dsa = dsc(dds0, pb * AB_PT);
        const uint64_t qb = dsc(mq0, s * AB_TILE64), db = dsc(mdo0, s * AB_TILE64);
#pragma unroll
        for (int kk = 0; kk < AB_T / 16; ++kk)
          umma_bf16_ss(tmem + 256, dsc(pa, kk * 32), dsc(db, kk * 2048), idesc_a, (q | kk) ? 1u : 0u);
#pragma unroll
        for (int kk = 0; kk < AB_T / 16; ++kk)
          umma_bf16_ss(tmem + 384, dsc(dsa, kk * 32), dsc(qb, kk * 2048), idesc_a, (q | kk) ? 1u : 0u);
        umma_commit(&ld_empty[s]);
        umma_commit(&ps_empty[pb]);
      };
      mbar_wait(kv_full, 0);
      for (int it = 0; it < n_it; ++it) {
        const int s = it % AB_STAGES, tb = it & 1;
        mbar_wait(&ld_full[s], (uint32_t)((it / AB_STAGES) & 1));
        if (it >= 2) mbar_wait(&tm_empty[tb], (uint32_t)(((it >> 1) - 1) & 1));
        tc_fence_after();
        const uint64_t qa = dsc(dq0, s * AB_TILE64), da = dsc(ddo0, s * AB_TILE64);
        const uint32_t ts = tmem + tb * 128;
#pragma unroll
        for (int kk = 0; kk < AT_D / 16; ++kk) {                           // S^T = K_j Q_i^T
          const uint32_t ko = (kk >> 2) * AT_ATOM + (kk & 3) * 32, qo = (kk >> 2) * AB_ATOM64 + (kk & 3) * 32;
          umma_bf16_ss(ts, dsc(dk0, ko), dsc(qa, qo), idesc_s, kk > 0 ? 1u : 0u);
        }
#pragma unroll
        for (int kk = 0; kk < AT_D / 16; ++kk) {                           // dP^T = V_j dO_i^T
          const uint32_t ko = (kk >> 2) * AT_ATOM + (kk & 3) * 32, qo = (kk >> 2) * AB_ATOM64 + (kk & 3) * 32;
          umma_bf16_ss(ts + 64, dsc(dv0, ko), dsc(da, qo), idesc_s, kk > 0 ? 1u : 0u);
        }
        umma_commit(&st_full[tb]);
        if (it >= 1) dvdk(it - 1);
      }
      if (n_it > 0) dvdk(n_it - 1);
      umma_commit(acc_done);
    }
    __syncwarp();
  } else if (warp >= 4) {
    const int q4 = warp & 3, half = (warp - 4) >> 2;
    const int r = q4 * 32 + lane;                                           // key row = TMEM lane
    const uint32_t trow = tmem + (static_cast<uint32_t>(q4 * 32) << 16);
    for (int it = 0; it < n_it; ++it) {
      const int i = 2 * j + it % per_head;
      const int tb = it & 1, s = it % AB_STAGES;
      mbar_wait(&st_full[tb], (uint32_t)((it >> 1) & 1));                  // (implies ld_full of stage s)
      tc_fence_after();
      if (it >= 2) mbar_wait(&ps_empty[tb], (uint32_t)(((it >> 1) - 1) & 1));   // P^T / dS^T smem free
      const int off = i * AB_T - j * AT_BN;                                 // query tile start - key tile start
      const uint32_t tS = trow + tb * 128, pP = smem_u32(sPt + tb * AB_PT), pD = smem_u32(sDSt + tb * AB_PT);
      if (off < AT_BN)
        ab_row32<true, true>(tS, tS + 64, pP, pD, r, half * 32, off, s_lse + s * AB_T, s_dd + s * AB_T, 0.f, 0.f,
                             scale_log2);
      else
        ab_row32<true, false>(tS, tS + 64, pP, pD, r, half * 32, off, s_lse + s * AB_T, s_dd + s * AB_T, 0.f, 0.f,
                              scale_log2);
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tm_empty[tb]);
      fence_proxy_async_smem();
      mbar_arrive(&p_full[tb]);
    }
    // dV and dK rows of key r -> bf16 (dK scaled by the softmax scale)
    mbar_wait(acc_done, 0);
    tc_fence_after();
    const int ld = (nh + 2 * nkv) * AT_D;
    __nv_bfloat16* drow = dqkv + (size_t)(row0 + j * AT_BN + r) * ld;
    ab_store_acc(trow + 256, half * 64, 1.0f, n_it == 0, drow + (size_t)(nh + nkv + kvh) * AT_D);
    ab_store_acc(trow + 384, half * 64, scale, n_it == 0, drow + (size_t)(nh + kvh) * AT_D);
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 2) tmem_dealloc(tmem, 512);
}

// dQ_i: CTA (128-query tile i = n_t-1-blockIdx.x (heaviest first), query head, sequence)
__global__ void __launch_bounds__(AB_THREADS, 1)
attn_bwd_dq_kernel(const __grid_constant__ CUtensorMap tmq, const __grid_constant__ CUtensorMap tmdo,
                   const __grid_constant__ CUtensorMap tmkv, const float* __restrict__ lse2,
                   const float* __restrict__ dl, int seq_len, int nh, int nkv, float scale_log2, float scale,
                   __nv_bfloat16* __restrict__ dqkv) {
  extern __shared__ uint8_t smem_raw[];
  const uint32_t pad = (1024u - (smem_u32(smem_raw) & 1023u)) & 1023u;
  uint8_t* smem = smem_raw + pad;
  uint8_t* sQ = smem;
  uint8_t* sDO = sQ + AT_TILE;
  uint8_t* sK = sDO + AT_TILE;                                  // [AB_STAGES] x 16 KiB
  uint8_t* sV = sK + AB_STAGES * AB_TILE64;                     // [AB_STAGES] x 16 KiB
  uint8_t* sDS = sV + AB_STAGES * AB_TILE64;                    // [2] x 16 KiB
  uint64_t* bars = reinterpret_cast<uint64_t*>(sDS + 2 * AB_PT);
  uint64_t* q_full = bars;
  uint64_t* kv_full = bars + 1;                  // [AB_STAGES]
  uint64_t* kv_empty = kv_full + AB_STAGES;      // [AB_STAGES]
  uint64_t* s_full = kv_empty + AB_STAGES;       // [2]
  uint64_t* tm_empty = s_full + 2;               // [2]
  uint64_t* p_full = tm_empty + 2;               // [2]
  uint64_t* ds_empty = p_full + 2;               // [2]
  uint64_t* acc_done = ds_empty + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_done + 1);

  const int n_t = seq_len / AT_BM;
  const int i = n_t - 1 - (int)blockIdx.x, h = blockIdx.y, b = blockIdx.z;
  const int g = nh / nkv, kvh = h / g, nj = 2 * i + 2;          // 64-key tiles up to the diagonal
  const int row0 = b * seq_len;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    mbar_init(q_full, 1);
    for (int s = 0; s < AB_STAGES; ++s) {
      mbar_init(&kv_full[s], 1);
      mbar_init(&kv_empty[s], 1);
    }
    for (int q = 0; q < 2; ++q) {
      mbar_init(&s_full[q], 1);
      mbar_init(&tm_empty[q], AB_EW);
      mbar_init(&p_full[q], AB_EW * 32);
      mbar_init(&ds_empty[q], 1);
    }
    mbar_init(acc_done, 1);
    fence_mbar_init();
  }
  // TMEM: S / dP buffer q at [128q, 128q + 64) / [128q + 64, 128q + 128); dQ [256, 384)
  if (warp == 2) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      tma_prefetch_desc(&tmq);
      tma_prefetch_desc(&tmdo);
      tma_prefetch_desc(&tmkv);
      const int qrow = row0 + i * AT_BM;
      mbar_expect_tx(q_full, 2 * AT_TILE);
      tma_load_2d(sQ, &tmq, q_full, h * AT_D, qrow);
      tma_load_2d(sQ + AT_ATOM, &tmq, q_full, h * AT_D + 64, qrow);
      tma_load_2d(sDO, &tmdo, q_full, h * AT_D, qrow);
      tma_load_2d(sDO + AT_ATOM, &tmdo, q_full, h * AT_D + 64, qrow);
      const int kcol = (nh + kvh) * AT_D, vcol = (nh + nkv + kvh) * AT_D;
      for (int jt = 0; jt < nj; ++jt) {
        const int s = jt % AB_STAGES;
        if (jt >= AB_STAGES) mbar_wait(&kv_empty[s], (uint32_t)((jt / AB_STAGES - 1) & 1));
        const int krow = row0 + jt * AB_T;
        uint8_t* k = sK + s * AB_TILE64;
        uint8_t* v = sV + s * AB_TILE64;
        mbar_expect_tx(&kv_full[s], 2 * AB_TILE64);
        tma_load_2d(k, &tmkv, &kv_full[s], kcol, krow);
        tma_load_2d(k + AB_ATOM64, &tmkv, &kv_full[s], kcol + 64, krow);
        tma_load_2d(v, &tmkv, &kv_full[s], vcol, krow);
        tma_load_2d(v + AB_ATOM64, &tmkv, &kv_full[s], vcol + 64, krow);
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idesc_s = make_idesc_bf16(AT_BM, AB_T, 0, 0);   // M = 128 queries, N = 64 keys
      constexpr uint32_t idesc_a = make_idesc_bf16(AT_BM, AT_D, 0, 1);   // dQ: N = d, B (K_j) MN-major
      const uint64_t dq0 = at_kmajor(smem_u32(sQ), 0), ddo0 = at_kmajor(smem_u32(sDO), 0);
      const uint64_t dk0 = ab_kmajor64(smem_u32(sK), 0), dv0 = ab_kmajor64(smem_u32(sV), 0);
      const uint64_t mk0 = ab_mnmajor64(smem_u32(sK), 0), dds0 = ab_kmajor_p(smem_u32(sDS), 0);
      auto dq_step = [&](int q) {   // dQ += dS K_q
        const int s = q % AB_STAGES, pb = q & 1;
        mbar_wait(&p_full[pb], (uint32_t)((q >> 1) & 1));
        tc_fence_after();
        const uint64_t dsa = dsc(dds0, pb * AB_PT), kb = dsc(mk0, s * AB_TILE64);
#pragma unroll
        for (int kk = 0; kk < AB_T / 16; ++kk)
          umma_bf16_ss(tmem + 256, dsc(dsa, kk * 32), dsc(kb, kk * 2048), idesc_a, (q | kk) ? 1u : 0u);
        umma_commit(&kv_empty[s]);
        umma_commit(&ds_empty[pb]);
      };
      mbar_wait(q_full, 0);
      for (int jt = 0; jt < nj; ++jt) {
        const int s = jt % AB_STAGES, tb = jt & 1;
        mbar_wait(&kv_full[s], (uint32_t)((jt / AB_STAGES) & 1));
        if (jt >= 2) mbar_wait(&tm_empty[tb], (uint32_t)(((jt >> 1) - 1) & 1));
        tc_fence_after();
        const uint64_t ka = dsc(dk0, s * AB_TILE64), va = dsc(dv0, s * AB_TILE64);
        const uint32_t ts = tmem + tb * 128;
#pragma unroll
        for (int kk = 0; kk < AT_D / 16; ++kk) {                           // S = Q_i K_j^T
          const uint32_t qo = (kk >> 2) * AT_ATOM + (kk & 3) * 32, ko = (kk >> 2) * AB_ATOM64 + (kk & 3) * 32;
          umma_bf16_ss(ts, dsc(dq0, qo), dsc(ka, ko), idesc_s, kk > 0 ? 1u : 0u);
        }
#pragma unroll
        for (int kk = 0; kk < AT_D / 16; ++kk) {                           // dP = dO_i V_j^T
          const uint32_t qo = (kk >> 2) * AT_ATOM + (kk & 3) * 32, ko = (kk >> 2) * AB_ATOM64 + (kk & 3) * 32;
          umma_bf16_ss(ts + 64, dsc(ddo0, qo), dsc(va, ko), idesc_s, kk > 0 ? 1u : 0u);
        }
        umma_commit(&s_full[tb]);
        if (jt >= 1) dq_step(jt - 1);
      }
      dq_step(nj - 1);
      umma_commit(acc_done);
    }
    __syncwarp();
  } else if (warp >= 4) {
    const int q4 = warp & 3, half = (warp - 4) >> 2;
    const int r = q4 * 32 + lane;                                           // query row = TMEM lane
    const uint32_t trow = tmem + (static_cast<uint32_t>(q4 * 32) << 16);
    const size_t lrow = ((size_t)b * nh + h) * seq_len + (size_t)i * AT_BM + r;
    const float l2 = lse2[lrow], dd = dl[lrow];
    for (int jt = 0; jt < nj; ++jt) {
      const int tb = jt & 1;
      mbar_wait(&s_full[tb], (uint32_t)((jt >> 1) & 1));
      tc_fence_after();
      if (jt >= 2) mbar_wait(&ds_empty[tb], (uint32_t)(((jt >> 1) - 1) & 1));   // dS smem free
      const int off = i * AT_BM - jt * AB_T;                                // query tile start - key tile start
      const uint32_t tS = trow + tb * 128, pD = smem_u32(sDS + tb * AB_PT);
      if (off < AB_T)
        ab_row32<false, true>(tS, tS + 64, 0u, pD, r, half * 32, off, nullptr, nullptr, l2, dd, scale_log2);
      else
        ab_row32<false, false>(tS, tS + 64, 0u, pD, r, half * 32, off, nullptr, nullptr, l2, dd, scale_log2);
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tm_empty[tb]);
      fence_proxy_async_smem();
      mbar_arrive(&p_full[tb]);
    }
    mbar_wait(acc_done, 0);
    tc_fence_after();
    const int ld = (nh + 2 * nkv) * AT_D;
    ab_store_acc(trow + 256, half * 64, scale, false, dqkv + (size_t)(row0 + i * AT_BM + r) * ld + (size_t)h * AT_D);
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 2) tmem_dealloc(tmem, 512);
}

static int ab_map(CUtensorMap* tm, const void* base, uint64_t cols, uint64_t rows, uint32_t box_rows) {
  PFN_cuTensorMapEncodeTiled_v12000 enc = tensor_map_encoder();
  if (!enc) return set_error(DM_ERR_DRIVER, "cuTensorMapEncodeTiled entry point unavailable");
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {cols * 2};
  cuuint32_t box[2] = {64, box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return set_error(DM_ERR_DRIVER, "attention_bwd: cuTensorMapEncodeTiled failed (%d)", (int)r);
  return DM_OK;
}

}  // namespace dm

using namespace dm;

extern "C" {

int dm_attention_bwd(const void* qkv, const void* out, const void* dout, const float* lse, int T, int seq_len,
                     int nh, int nkv, int head_dim, float* dl_ws, void* dqkv, void* stream) {
  if (head_dim != AT_D) return set_error(DM_ERR_SHAPE, "attention_bwd: head_dim %d (only 128)", head_dim);
  if (nh < 1 || nkv < 1 || nh % nkv) return set_error(DM_ERR_SHAPE, "attention_bwd: %d heads, %d kv heads", nh, nkv);
  if (T < 1 || seq_len < AT_BM || seq_len % AT_BM || T % seq_len)
    return set_error(DM_ERR_SHAPE, "attention_bwd: seq_len %d must be a multiple of %d dividing T=%d", seq_len, AT_BM,
                     T);
  if ((reinterpret_cast<uintptr_t>(qkv) | reinterpret_cast<uintptr_t>(out) | reinterpret_cast<uintptr_t>(dout) |
       reinterpret_cast<uintptr_t>(dqkv)) & 15)
    return set_error(DM_ERR_ALIGN, "attention_bwd: operands not 16-byte aligned");
  cudaStream_t st = (cudaStream_t)stream;
  const int nb = T / seq_len, n_t = seq_len / AT_BM;
  const uint64_t qkv_cols = (uint64_t)(nh + 2 * nkv) * AT_D;
  CUtensorMap tm128, tm64, tmdo128, tmdo64;
  int rc;
  if ((rc = ab_map(&tm128, qkv, qkv_cols, (uint64_t)T, AT_BM))) return rc;
  if ((rc = ab_map(&tm64, qkv, qkv_cols, (uint64_t)T, AB_T))) return rc;
  if ((rc = ab_map(&tmdo128, dout, (uint64_t)nh * AT_D, (uint64_t)T, AT_BM))) return rc;
  if ((rc = ab_map(&tmdo64, dout, (uint64_t)nh * AT_D, (uint64_t)T, AB_T))) return rc;
  int blocks = (T * nh + 7) / 8;
  if (blocks > num_sms_current() * 8) blocks = num_sms_current() * 8;
  attn_bwd_dot_kernel<<<blocks, 256, 0, st>>>(reinterpret_cast<const __nv_bfloat16*>(out),
                                              reinterpret_cast<const __nv_bfloat16*>(dout), lse, T, seq_len, nh, dl_ws);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return set_cuda_error(e, "attention_bwd dot launch");
  note_launch();
  const float scale = 1.0f / sqrtf((float)AT_D), scale_log2 = AB_LOG2E * scale;
  const float* lse2 = dl_ws + (size_t)T * nh;   // written by the dot kernel
  if ((rc = ensure_smem_attr((const void*)attn_bwd_dkdv_kernel, (int)AB_SMEM_DKDV, "cudaFuncSetAttribute(attn_bwd_dkdv)")))
    return rc;
  if ((rc = ensure_smem_attr((const void*)attn_bwd_dq_kernel, (int)AB_SMEM_DQ, "cudaFuncSetAttribute(attn_bwd_dq)")))
    return rc;
  __nv_bfloat16* d = reinterpret_cast<__nv_bfloat16*>(dqkv);
  // dK/dV and dQ are independent: dQ runs on a side stream (per host thread and device) forked
  // from and joined back into the caller's stream, so each kernel's last partial wave is filled
  // by the other's CTAs (stream capture records the fork / join as graph edges)
  int dev = 0;
  if ((e = cudaGetDevice(&dev)) != cudaSuccess) return set_cuda_error(e, "attention_bwd cudaGetDevice");
  thread_local std::map<int, cudaStream_t> side_streams;
  cudaStream_t side = side_streams[dev];
  if (!side) {
    if ((e = cudaStreamCreateWithFlags(&side, cudaStreamNonBlocking)) != cudaSuccess)
      return set_cuda_error(e, "attention_bwd side stream");
    side_streams[dev] = side;
  }
  cudaEvent_t fork, join;
  if ((e = cudaEventCreateWithFlags(&fork, cudaEventDisableTiming)) != cudaSuccess ||
      (e = cudaEventCreateWithFlags(&join, cudaEventDisableTiming)) != cudaSuccess)
    return set_cuda_error(e, "attention_bwd events");
  cudaEventRecord(fork, st);
  cudaStreamWaitEvent(side, fork, 0);
  attn_bwd_dq_kernel<<<dim3(n_t, nh, nb), AB_THREADS, AB_SMEM_DQ, side>>>(tm128, tmdo128, tm64, lse2, dl_ws, seq_len,
                                                                           nh, nkv, scale_log2, scale, d);
  if ((e = cudaGetLastError()) != cudaSuccess) return set_cuda_error(e, "attention_bwd dq launch");
  note_launch();
  attn_bwd_dkdv_kernel<<<dim3(n_t, nkv, nb), AB_THREADS, AB_SMEM_DKDV, st>>>(tm128, tm64, tmdo64, lse2, dl_ws, seq_len,
                                                                              nh, nkv, scale_log2, scale, d);
  if ((e = cudaGetLastError()) != cudaSuccess) return set_cuda_error(e, "attention_bwd dkdv launch");
  note_launch();
  cudaEventRecord(join, side);
  cudaStreamWaitEvent(st, join, 0);
  cudaEventDestroy(fork);   // destruction is deferred until the recorded work completes
  cudaEventDestroy(join);
  return DM_OK;
}

}  // extern "C"
