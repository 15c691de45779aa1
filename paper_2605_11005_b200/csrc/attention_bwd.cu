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
//   attn_bwd_dkdv_kernel  CTA per (key tile j, KV head, sequence): dK_j, dV_j accumulate in
//                         TMEM over the group's g query heads and the query tiles i >= j:
//                         Sᵀ = K_j Q_iᵀ and dPᵀ = V_j dO_iᵀ (tcgen05, M = keys), the
//                         elementwise warps (thread = key row = TMEM lane) form Pᵀ and dSᵀ
//                         rows in bf16 (SWIZZLE_128B smem), then dV += Pᵀ dO_i, dK += dSᵀ Q_i
//                         with dO_i / Q_i re-read as MN-major B operands of the same tiles
//   attn_bwd_dq_kernel    CTA per (query tile i, query head, sequence): S = Q_i K_jᵀ and
//                         dP = dO_i V_jᵀ, dS rows, dQ += dS K_j for the key tiles j <= i
// Warp roles (256 threads): warp 0 TMA, warp 1 MMA issuer (one thread), warp 2 TMEM
// allocator, warps 4-7 elementwise (thread r = tile row r). Tiles 128 x 128, head_dim 128.
#include "attention_common.cuh"

namespace dm {

constexpr int AB_THREADS = 256;
constexpr float AB_LOG2E = 1.4426950408889634f;

// D[b][h][s] = sum_d dO[t, h, d] * O[t, h, d] (fp32): warp per (token, head)
__global__ void __launch_bounds__(256)
attn_bwd_dot_kernel(const __nv_bfloat16* __restrict__ o, const __nv_bfloat16* __restrict__ dout, int T, int seq_len,
                    int nh, float* __restrict__ dl) {
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
    if (lane == 0) dl[((size_t)(t / seq_len) * nh + h) * seq_len + t % seq_len] = s;
  }
}

// Write 32 bf16-pair words (64 values, columns c0..c0+63 of row r) into a 128 x 128 bf16
// SWIZZLE_128B tile (two 64-column atoms).
__device__ __forceinline__ void ab_store_row64(uint32_t tile, int r, int c0, const uint32_t (&v)[32]) {
  const uint32_t atom = tile + (c0 >> 6) * AT_ATOM;
#pragma unroll
  for (int c = 0; c < 8; ++c) st_shared_v4(atom + sw128(r, c), v[4 * c], v[4 * c + 1], v[4 * c + 2], v[4 * c + 3]);
}

// Elementwise step of one row: 128 (S, dP) accumulator columns in TMEM -> bf16 P and dS rows in
// smem. lse2[c] / dd[c] give the per-column (key-major kernel) or per-row (query-major kernel,
// uniform) log2-LSE and D; masked columns (causal) produce P = dS = 0.
template <bool COLS_ARE_QUERIES>
__device__ __forceinline__ void ab_row(uint32_t tS, uint32_t tP, uint32_t sPt, uint32_t sDSt, int r, bool diag,
                                       const float* lse2c, const float* ddc, float lse2r, float ddr,
                                       float scale_log2) {
#pragma unroll 1
  for (int c0 = 0; c0 < AT_BN; c0 += 64) {
    uint32_t pw[32], dw[32];
#pragma unroll
    for (int half = 0; half < 2; ++half) {
      uint32_t s32[32], d32[32];
      tmem_ld16(tS + c0 + half * 32, *reinterpret_cast<uint32_t(*)[16]>(s32));
      tmem_ld16(tS + c0 + half * 32 + 16, *reinterpret_cast<uint32_t(*)[16]>(s32 + 16));
      tmem_ld16(tP + c0 + half * 32, *reinterpret_cast<uint32_t(*)[16]>(d32));
      tmem_ld16(tP + c0 + half * 32 + 16, *reinterpret_cast<uint32_t(*)[16]>(d32 + 16));
      tmem_wait_ld();
#pragma unroll
      for (int q = 0; q < 16; ++q) {
        float p2[2], ds2[2];
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          const int c = c0 + half * 32 + 2 * q + u;
          const float l2 = COLS_ARE_QUERIES ? lse2c[c] : lse2r;
          const float dv = COLS_ARE_QUERIES ? ddc[c] : ddr;
          // causal: key > query is masked (key tile j == query tile i on the diagonal)
          const bool masked = diag && (COLS_ARE_QUERIES ? (r > c) : (c > r));
          const float p = masked ? 0.f : ex2(__fmaf_rn(__uint_as_float(s32[2 * q + u]), scale_log2, -l2));
          p2[u] = p;
          ds2[u] = p * (__uint_as_float(d32[2 * q + u]) - dv);
        }
        pw[half * 16 + q] = pack_bf16(p2[0], p2[1]);
        dw[half * 16 + q] = pack_bf16(ds2[0], ds2[1]);
      }
    }
    if (sPt) ab_store_row64(sPt, r, c0, pw);
    ab_store_row64(sDSt, r, c0, dw);
  }
}

// dK_j, dV_j: CTA (key tile j = blockIdx.x, KV head = blockIdx.y, sequence = blockIdx.z)
__global__ void __launch_bounds__(AB_THREADS, 1)
attn_bwd_dkdv_kernel(const __grid_constant__ CUtensorMap tmq, const __grid_constant__ CUtensorMap tmdo,
                     const float* __restrict__ lse, const float* __restrict__ dl, int seq_len, int nh, int nkv,
                     float scale_log2, float scale, __nv_bfloat16* __restrict__ dqkv) {
  extern __shared__ uint8_t smem_raw[];
  const uint32_t pad = (1024u - (smem_u32(smem_raw) & 1023u)) & 1023u;
  uint8_t* smem = smem_raw + pad;
  uint8_t* sK = smem;
  uint8_t* sV = smem + AT_TILE;
  uint8_t* sQ = smem + 2 * AT_TILE;
  uint8_t* sDO = smem + 3 * AT_TILE;
  uint8_t* sPt = smem + 4 * AT_TILE;
  uint8_t* sDSt = smem + 5 * AT_TILE;
  float* s_lse = reinterpret_cast<float*>(smem + 6 * AT_TILE);   // [2][128] (parity double buffer)
  float* s_dd = s_lse + 2 * AT_BM;                               // [2][128]
  uint64_t* bars = reinterpret_cast<uint64_t*>(s_dd + 2 * AT_BM);
  uint64_t* kv_full = bars;
  uint64_t* ld_full = bars + 1;
  uint64_t* st_full = bars + 2;
  uint64_t* p_full = bars + 3;
  uint64_t* acc_done = bars + 4;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 5);

  const int j = blockIdx.x, kvh = blockIdx.y, b = blockIdx.z;
  const int n_t = seq_len / AT_BM, g = nh / nkv;
  const int per_head = n_t - j, n_it = g * per_head;
  const int row0 = b * seq_len;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    mbar_init(kv_full, 1);
    mbar_init(ld_full, 1);
    mbar_init(st_full, 1);
    mbar_init(p_full, AT_BM);
    mbar_init(acc_done, 1);
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc(tmem_slot, 512);   // S^T [0,128) dP^T [128,256) dV [256,384) dK [384,512)
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      tma_prefetch_desc(&tmq);
      tma_prefetch_desc(&tmdo);
      const int kcol = (nh + kvh) * AT_D, vcol = (nh + nkv + kvh) * AT_D, krow = row0 + j * AT_BN;
      mbar_expect_tx(kv_full, 2 * AT_TILE);
      tma_load_2d(sK, &tmq, kv_full, kcol, krow);
      tma_load_2d(sK + AT_ATOM, &tmq, kv_full, kcol + 64, krow);
      tma_load_2d(sV, &tmq, kv_full, vcol, krow);
      tma_load_2d(sV + AT_ATOM, &tmq, kv_full, vcol + 64, krow);
      for (int it = 0; it < n_it; ++it) {
        const int qh = kvh * g + it / per_head, i = j + it % per_head;
        if (it > 0) mbar_wait(acc_done, (it - 1) & 1);   // the previous Q_i / dO_i are read out
        const int qrow = row0 + i * AT_BM;
        mbar_expect_tx(ld_full, 2 * AT_TILE);
        tma_load_2d(sQ, &tmq, ld_full, qh * AT_D, qrow);
        tma_load_2d(sQ + AT_ATOM, &tmq, ld_full, qh * AT_D + 64, qrow);
        tma_load_2d(sDO, &tmdo, ld_full, qh * AT_D, qrow);
        tma_load_2d(sDO + AT_ATOM, &tmdo, ld_full, qh * AT_D + 64, qrow);
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idesc_kk = make_idesc_bf16(AT_BM, AT_BN, 0, 0);   // both operands K-major
      constexpr uint32_t idesc_km = make_idesc_bf16(AT_BM, AT_D, 0, 1);    // A K-major, B MN-major
      const uint32_t ka = smem_u32(sK), va = smem_u32(sV), qa = smem_u32(sQ), da = smem_u32(sDO);
      const uint32_t pa = smem_u32(sPt), dsa = smem_u32(sDSt);
      mbar_wait(kv_full, 0);
      for (int it = 0; it < n_it; ++it) {
        mbar_wait(ld_full, it & 1);
        tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < AT_D / 16; ++kk)                             // S^T = K_j Q_i^T
          umma_bf16_ss(tmem, at_kmajor(ka, kk), at_kmajor(qa, kk), idesc_kk, kk > 0 ? 1u : 0u);
#pragma unroll
        for (int kk = 0; kk < AT_D / 16; ++kk)                             // dP^T = V_j dO_i^T
          umma_bf16_ss(tmem + AT_BN, at_kmajor(va, kk), at_kmajor(da, kk), idesc_kk, kk > 0 ? 1u : 0u);
        umma_commit(st_full);
        mbar_wait(p_full, it & 1);
        tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < AT_BM / 16; ++kk)                            // dV += P^T dO_i
          umma_bf16_ss(tmem + 2 * AT_BN, at_kmajor(pa, kk), at_mnmajor(da, kk), idesc_km, (it | kk) ? 1u : 0u);
#pragma unroll
        for (int kk = 0; kk < AT_BM / 16; ++kk)                            // dK += dS^T Q_i
          umma_bf16_ss(tmem + 3 * AT_BN, at_kmajor(dsa, kk), at_mnmajor(qa, kk), idesc_km, (it | kk) ? 1u : 0u);
        umma_commit(acc_done);
      }
    }
    __syncwarp();
  } else if (warp >= 4) {
    const int q4 = warp & 3;
    const int r = q4 * 32 + lane;                                           // key row = TMEM lane
    const uint32_t trow = tmem + (static_cast<uint32_t>(q4 * 32) << 16);
    for (int it = 0; it < n_it; ++it) {
      const int qh = kvh * g + it / per_head, i = j + it % per_head;
      float* l2 = s_lse + (it & 1) * AT_BM;
      float* dd = s_dd + (it & 1) * AT_BM;
      const size_t lrow = ((size_t)b * nh + qh) * seq_len + (size_t)i * AT_BM + r;
      l2[r] = lse[lrow] * AB_LOG2E;                                        // query r of tile i
      dd[r] = dl[lrow];
      asm volatile("bar.sync 1, 128;" ::: "memory");
      mbar_wait(st_full, it & 1);
      tc_fence_after();
      if (it > 0) mbar_wait(acc_done, (it - 1) & 1);                       // P^T / dS^T smem free
      ab_row<true>(trow, trow + AT_BN, smem_u32(sPt), smem_u32(sDSt), r, i == j, l2, dd, 0.f, 0.f, scale_log2);
      fence_proxy_async_smem();
      tc_fence_before();
      mbar_arrive(p_full);
    }
    // dV and dK rows of key r -> bf16 (dK scaled by the softmax scale)
    if (n_it > 0) mbar_wait(acc_done, (n_it - 1) & 1);
    tc_fence_after();
    const int ld = (nh + 2 * nkv) * AT_D;
    __nv_bfloat16* drow = dqkv + (size_t)(row0 + j * AT_BN + r) * ld;
#pragma unroll 1
    for (int which = 0; which < 2; ++which) {                               // 0: dV, 1: dK
      const uint32_t tacc = trow + (2 + which) * AT_BN;
      const float sc = which ? scale : 1.0f;
      __nv_bfloat16* dst = drow + (size_t)(which ? (nh + kvh) : (nh + nkv + kvh)) * AT_D;
#pragma unroll 1
      for (int c = 0; c < AT_D; c += 16) {
        uint32_t v[16];
        tmem_ld16(tacc + c, v);
        tmem_wait_ld();
        uint32_t w8[8];
#pragma unroll
        for (int q = 0; q < 8; ++q)
          w8[q] = n_it > 0 ? pack_bf16(__uint_as_float(v[2 * q]) * sc, __uint_as_float(v[2 * q + 1]) * sc) : 0u;
        int4* o4 = reinterpret_cast<int4*>(dst + c);
        o4[0] = make_int4((int)w8[0], (int)w8[1], (int)w8[2], (int)w8[3]);
        o4[1] = make_int4((int)w8[4], (int)w8[5], (int)w8[6], (int)w8[7]);
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 2) tmem_dealloc(tmem, 512);
}

// dQ_i: CTA (query tile i = n_t-1-blockIdx.x (heaviest first), query head, sequence)
__global__ void __launch_bounds__(AB_THREADS, 1)
attn_bwd_dq_kernel(const __grid_constant__ CUtensorMap tmq, const __grid_constant__ CUtensorMap tmdo,
                   const float* __restrict__ lse, const float* __restrict__ dl, int seq_len, int nh, int nkv,
                   float scale_log2, float scale, __nv_bfloat16* __restrict__ dqkv) {
  extern __shared__ uint8_t smem_raw[];
  const uint32_t pad = (1024u - (smem_u32(smem_raw) & 1023u)) & 1023u;
  uint8_t* smem = smem_raw + pad;
  uint8_t* sQ = smem;
  uint8_t* sDO = smem + AT_TILE;
  uint8_t* sK = smem + 2 * AT_TILE;
  uint8_t* sV = smem + 3 * AT_TILE;
  uint8_t* sDS = smem + 4 * AT_TILE;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + 5 * AT_TILE);
  uint64_t* q_full = bars;
  uint64_t* kv_full = bars + 1;
  uint64_t* s_full = bars + 2;
  uint64_t* p_full = bars + 3;
  uint64_t* acc_done = bars + 4;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 5);

  const int n_t = seq_len / AT_BM;
  const int i = n_t - 1 - (int)blockIdx.x, h = blockIdx.y, b = blockIdx.z;
  const int g = nh / nkv, kvh = h / g, nj = i + 1;
  const int row0 = b * seq_len;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    mbar_init(q_full, 1);
    mbar_init(kv_full, 1);
    mbar_init(s_full, 1);
    mbar_init(p_full, AT_BM);
    mbar_init(acc_done, 1);
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc(tmem_slot, 512);   // S [0,128) dP [128,256) dQ [256,384)
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      tma_prefetch_desc(&tmq);
      tma_prefetch_desc(&tmdo);
      const int qrow = row0 + i * AT_BM;
      mbar_expect_tx(q_full, 2 * AT_TILE);
      tma_load_2d(sQ, &tmq, q_full, h * AT_D, qrow);
      tma_load_2d(sQ + AT_ATOM, &tmq, q_full, h * AT_D + 64, qrow);
      tma_load_2d(sDO, &tmdo, q_full, h * AT_D, qrow);
      tma_load_2d(sDO + AT_ATOM, &tmdo, q_full, h * AT_D + 64, qrow);
      const int kcol = (nh + kvh) * AT_D, vcol = (nh + nkv + kvh) * AT_D;
      for (int jj = 0; jj < nj; ++jj) {
        if (jj > 0) mbar_wait(acc_done, (jj - 1) & 1);   // the previous K_j / V_j are read out
        const int krow = row0 + jj * AT_BN;
        mbar_expect_tx(kv_full, 2 * AT_TILE);
        tma_load_2d(sK, &tmq, kv_full, kcol, krow);
        tma_load_2d(sK + AT_ATOM, &tmq, kv_full, kcol + 64, krow);
        tma_load_2d(sV, &tmq, kv_full, vcol, krow);
        tma_load_2d(sV + AT_ATOM, &tmq, kv_full, vcol + 64, krow);
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idesc_kk = make_idesc_bf16(AT_BM, AT_BN, 0, 0);
      constexpr uint32_t idesc_km = make_idesc_bf16(AT_BM, AT_D, 0, 1);
      const uint32_t qa = smem_u32(sQ), da = smem_u32(sDO), ka = smem_u32(sK), va = smem_u32(sV);
      const uint32_t dsa = smem_u32(sDS);
      mbar_wait(q_full, 0);
      for (int jj = 0; jj < nj; ++jj) {
        mbar_wait(kv_full, jj & 1);
        tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < AT_D / 16; ++kk)                             // S = Q_i K_j^T
          umma_bf16_ss(tmem, at_kmajor(qa, kk), at_kmajor(ka, kk), idesc_kk, kk > 0 ? 1u : 0u);
#pragma unroll
        for (int kk = 0; kk < AT_D / 16; ++kk)                             // dP = dO_i V_j^T
          umma_bf16_ss(tmem + AT_BN, at_kmajor(da, kk), at_kmajor(va, kk), idesc_kk, kk > 0 ? 1u : 0u);
        umma_commit(s_full);
        mbar_wait(p_full, jj & 1);
        tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < AT_BN / 16; ++kk)                            // dQ += dS K_j
          umma_bf16_ss(tmem + 2 * AT_BN, at_kmajor(dsa, kk), at_mnmajor(ka, kk), idesc_km, (jj | kk) ? 1u : 0u);
        umma_commit(acc_done);
      }
    }
    __syncwarp();
  } else if (warp >= 4) {
    const int q4 = warp & 3;
    const int r = q4 * 32 + lane;                                           // query row = TMEM lane
    const uint32_t trow = tmem + (static_cast<uint32_t>(q4 * 32) << 16);
    const size_t lrow = ((size_t)b * nh + h) * seq_len + (size_t)i * AT_BM + r;
    const float l2 = lse[lrow] * AB_LOG2E, dd = dl[lrow];
    for (int jj = 0; jj < nj; ++jj) {
      mbar_wait(s_full, jj & 1);
      tc_fence_after();
      if (jj > 0) mbar_wait(acc_done, (jj - 1) & 1);                       // dS smem free
      ab_row<false>(trow, trow + AT_BN, 0u, smem_u32(sDS), r, jj == i, nullptr, nullptr, l2, dd, scale_log2);
      fence_proxy_async_smem();
      tc_fence_before();
      mbar_arrive(p_full);
    }
    mbar_wait(acc_done, (nj - 1) & 1);
    tc_fence_after();
    const int ld = (nh + 2 * nkv) * AT_D;
    __nv_bfloat16* dst = dqkv + (size_t)(row0 + i * AT_BM + r) * ld + (size_t)h * AT_D;
#pragma unroll 1
    for (int c = 0; c < AT_D; c += 16) {
      uint32_t v[16];
      tmem_ld16(trow + 2 * AT_BN + c, v);
      tmem_wait_ld();
      uint32_t w8[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) w8[q] = pack_bf16(__uint_as_float(v[2 * q]) * scale, __uint_as_float(v[2 * q + 1]) * scale);
      int4* o4 = reinterpret_cast<int4*>(dst + c);
      o4[0] = make_int4((int)w8[0], (int)w8[1], (int)w8[2], (int)w8[3]);
      o4[1] = make_int4((int)w8[4], (int)w8[5], (int)w8[6], (int)w8[7]);
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 2) tmem_dealloc(tmem, 512);
}

static int ab_map(CUtensorMap* tm, const void* base, uint64_t cols, uint64_t rows) {
  PFN_cuTensorMapEncodeTiled_v12000 enc = tensor_map_encoder();
  if (!enc) return set_error(DM_ERR_DRIVER, "cuTensorMapEncodeTiled entry point unavailable");
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {cols * 2};
  cuuint32_t box[2] = {64, AT_BM};
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
  CUtensorMap tmq, tmdo;
  int rc;
  if ((rc = ab_map(&tmq, qkv, (uint64_t)(nh + 2 * nkv) * AT_D, (uint64_t)T))) return rc;
  if ((rc = ab_map(&tmdo, dout, (uint64_t)nh * AT_D, (uint64_t)T))) return rc;
  int blocks = (T * nh + 7) / 8;
  if (blocks > num_sms_current() * 8) blocks = num_sms_current() * 8;
  attn_bwd_dot_kernel<<<blocks, 256, 0, st>>>(reinterpret_cast<const __nv_bfloat16*>(out),
                                              reinterpret_cast<const __nv_bfloat16*>(dout), T, seq_len, nh, dl_ws);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return set_cuda_error(e, "attention_bwd dot launch");
  note_launch();
  const float scale = 1.0f / sqrtf((float)AT_D), scale_log2 = AB_LOG2E * scale;
  const size_t smem_kv = 1024 + 6 * (size_t)AT_TILE + 4 * AT_BM * sizeof(float) + 64;
  const size_t smem_q = 1024 + 5 * (size_t)AT_TILE + 64;
  if ((rc = ensure_smem_attr((const void*)attn_bwd_dkdv_kernel, (int)smem_kv, "cudaFuncSetAttribute(attn_bwd_dkdv)")))
    return rc;
  if ((rc = ensure_smem_attr((const void*)attn_bwd_dq_kernel, (int)smem_q, "cudaFuncSetAttribute(attn_bwd_dq)")))
    return rc;
  __nv_bfloat16* d = reinterpret_cast<__nv_bfloat16*>(dqkv);
  attn_bwd_dkdv_kernel<<<dim3(n_t, nkv, nb), AB_THREADS, smem_kv, st>>>(tmq, tmdo, lse, dl_ws, seq_len, nh, nkv,
                                                                       scale_log2, scale, d);
  if ((e = cudaGetLastError()) != cudaSuccess) return set_cuda_error(e, "attention_bwd dkdv launch");
  note_launch();
  attn_bwd_dq_kernel<<<dim3(n_t, nh, nb), AB_THREADS, smem_q, st>>>(tmq, tmdo, lse, dl_ws, seq_len, nh, nkv, scale_log2,
                                                                   scale, d);
  if ((e = cudaGetLastError()) != cudaSuccess) return set_cuda_error(e, "attention_bwd dq launch");
  note_launch();
  return DM_OK;
}

}  // extern "C"
