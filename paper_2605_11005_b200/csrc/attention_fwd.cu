// Causal GQA flash-attention forward on 5th-gen tensor cores (sm_100a): the A-side
// attention of SURVEY.md §8f row 3, whose cost the reference only models,
// C_a = b·(s·H²·(2+2/g) + 4·s²·H) (pkg/src/afpipe/costs.py:84-87).
//
// Persistent CTAs (one per SM) walk work items of two 128-query tiles A and B; head_dim 128.
// Warp roles:
//   warp 0    TMA: the item's two Q tiles, then K_j through a 2-stage ring
//   warp 3    TMA: V_j (one stage; V_j is consumed by both tiles' P·V)
//   warp 1    MMA issuer (one thread), per KV tile j: S_A(j) = Q_A·K_jᵀ, S_B(j) = Q_B·K_jᵀ,
//             O_A += P_A(j-1)·V_{j-1}, O_B += P_B(j-1)·V_{j-1}: each tile's softmax of KV tile j
//             overlaps the other MMAs of the step, so the tensor core works for one tile
//             while the other tile's softmax runs
//   warp 2    TMEM allocator (S_A, S_B, O_A, O_B: 4 x 128 fp32 columns)
//   warps 4-7 / 8-11  softmax of tile A / B: thread r owns query row r (= TMEM lane r),
//             reads its S row with tcgen05.ld, online softmax in the exp2 domain with a lazy
//             running max, rescales its O row in TMEM (tcgen05.ld/st) when the max moved, and
//             writes its P row (bf16) into the SWIZZLE_128B smem tile the P·V MMA reads; the
//             final O / l and the natural-log LSE go to global memory.
// Tiles A and B are two query heads of one KV group on the same rows (GQA with an even
// group size: each K/V tile serves both) or two adjacent row tiles of one head. Causal:
// each tile stops at its diagonal KV tile (masked key > query). Items run heaviest first.
#include "attention_common.cuh"

namespace dm {

constexpr int AT_STAGES = 2;
constexpr int AT_THREADS = 384;
// Q_A, Q_B | P_A, P_B | K ring (AT_STAGES) | V
constexpr size_t AT_SMEM = 1024 + (size_t)AT_TILE * (5 + AT_STAGES) + 256;

// Packed fp32 pairs (FADD2) and three-input max (FMNMX3): the softmax warps are issue-bound
// (an FMA-pipe exp2 polynomial for part of the row measured slower), so the row reductions
// and the exp2 argument FMAs run two elements per instruction.
__device__ __forceinline__ float2 fadd2(float2 a, float2 b) {
  unsigned long long ra, rb, rc;
  asm("mov.b64 %0, {%1, %2};" : "=l"(ra) : "f"(a.x), "f"(a.y));
  asm("mov.b64 %0, {%1, %2};" : "=l"(rb) : "f"(b.x), "f"(b.y));
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(rc) : "l"(ra), "l"(rb));
  float2 d;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(d.x), "=f"(d.y) : "l"(rc));
  return d;
}
__device__ __forceinline__ float fmax3(float a, float b, float c) {
  float d;
  asm("max.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c));
  return d;
}
// The running max only moves when a row's new max exceeds it by more than 2^8 (log2
// domain): P entries stay <= 256 (exact in fp32, representable in bf16) and the O rescale
// (tcgen05.ld/st of the whole O row) is skipped on most tiles; m, l and O stay consistent.
constexpr float AT_RESCALE_LOG2 = 8.0f;

// One work item = two 128-query tiles (A, B): two query heads of one KV group on the same
// rows (GQA with an even group: each K/V tile serves both) or two adjacent row tiles of one
// head. Items are numbered heaviest (longest causal rows) first.
struct AtItem {
  int qtA, qtB, hA, hB, b;
};
__device__ __forceinline__ AtItem at_item(int i, int head_pairs, int n_qt, int nh, int nb) {
  AtItem it;
  if (head_pairs) {
    const int per = (nh / 2) * nb, rt = i / per, rem = i % per;
    it.qtA = it.qtB = n_qt - 1 - rt;
    it.hA = 2 * (rem % (nh / 2));
    it.hB = it.hA + 1;
    it.b = rem / (nh / 2);
  } else {
    const int per = nh * nb, rt = i / per, rem = i % per;
    it.qtA = 2 * (n_qt / 2 - 1 - rt);
    it.qtB = it.qtA + 1;
    it.hA = it.hB = rem % nh;
    it.b = rem / nh;
  }
  return it;
}

// Round r of the persistent walk: CTA k takes item r·G + k on even rounds and r·G + G-1-k on
// odd ones (snake order over the heaviest-first list, so every CTA's total work is close to
// the mean); -1 when the last, partial round has nothing for this CTA.
__device__ __forceinline__ int at_snake(int r, int n_items) {
  const int G = gridDim.x, k = blockIdx.x;
  const int i = r * G + ((r & 1) ? G - 1 - k : k);
  return i < n_items ? i : -1;
}

// Persistent: one CTA per SM walks the items in snake order (at_snake); TMEM, barriers
// and the K/V rings live across items (phases from running counters), the next item's Q
// load waits only for the last S MMAs of the previous one, and its first P·V waits for the
// previous epilogue to drain O — prologue and epilogue overlap the neighbouring items.
__global__ void __launch_bounds__(AT_THREADS, 1)
attn_fwd_kernel(const __grid_constant__ CUtensorMap tm, int seq_len, int nh, int nkv, int ld_out,
                __nv_bfloat16* __restrict__ out, float* __restrict__ lse, float scale_log2, int head_pairs,
                int nb) {
  extern __shared__ uint8_t smem_raw[];
  const uint32_t pad = (1024u - (smem_u32(smem_raw) & 1023u)) & 1023u;
  uint8_t* smem = smem_raw + pad;
  uint8_t* sQ = smem;                                   // tile t at +t·TILE
  uint8_t* sP = smem + 2 * AT_TILE;                     // tile t at +t·TILE
  uint8_t* sK = smem + 4 * AT_TILE;                     // stage s at +s·TILE
  uint8_t* sV = smem + (4 + AT_STAGES) * AT_TILE;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + (size_t)AT_TILE * (5 + AT_STAGES));
  uint64_t* q_full = bars;
  uint64_t* k_full = bars + 1;                          // [AT_STAGES]
  uint64_t* k_empty = bars + 1 + AT_STAGES;             // [AT_STAGES]
  uint64_t* v_full = bars + 1 + 2 * AT_STAGES;
  uint64_t* v_empty = bars + 2 + 2 * AT_STAGES;
  uint64_t* s_full = bars + 3 + 2 * AT_STAGES;          // [2] per tile
  uint64_t* s_free = bars + 5 + 2 * AT_STAGES;          // [2]
  uint64_t* p_full = bars + 7 + 2 * AT_STAGES;          // [2]
  uint64_t* pv_done = bars + 9 + 2 * AT_STAGES;         // [2]
  uint64_t* o_free = bars + 11 + 2 * AT_STAGES;         // [2] epilogue drained O
  uint64_t* q_empty = bars + 13 + 2 * AT_STAGES;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 14 + 2 * AT_STAGES);

  const int n_qt = seq_len / AT_BM;
  const int n_items = head_pairs ? n_qt * (nh / 2) * nb : (n_qt / 2) * nh * nb;
  const int g = nh / nkv;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    mbar_init(q_full, 1);
    mbar_init(q_empty, 1);
    for (int s = 0; s < AT_STAGES; ++s) { mbar_init(&k_full[s], 1); mbar_init(&k_empty[s], 1); }
    mbar_init(v_full, 1);
    mbar_init(v_empty, 1);
    for (int t = 0; t < 2; ++t) {
      mbar_init(&s_full[t], 1); mbar_init(&s_free[t], AT_BM);
      mbar_init(&p_full[t], AT_BM); mbar_init(&pv_done[t], 1);
      mbar_init(&o_free[t], AT_BM);
    }
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc(tmem_slot, 512);            // S_A [0,128) S_B [128,256) O_A [256,384) O_B [384,512)
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      tma_prefetch_desc(&tm);
      int gk = 0, it = 0;
      for (int rd = 0; rd * (int)gridDim.x < n_items; ++rd) {
        const int i = at_snake(rd, n_items);
        if (i < 0) continue;
        const AtItem w = at_item(i, head_pairs, n_qt, nh, nb);
        const int row0 = w.b * seq_len, kcol = (nh + w.hA / g) * AT_D, nB = w.qtB + 1;
        if (it > 0) mbar_wait(q_empty, (it - 1) & 1);   // previous item's S MMAs are done with Q
        mbar_expect_tx(q_full, 2 * AT_TILE);
        for (int t = 0; t < 2; ++t) {
          const int r = row0 + (t ? w.qtB : w.qtA) * AT_BM, qcol = (t ? w.hB : w.hA) * AT_D;
          tma_load_2d(sQ + t * AT_TILE, &tm, q_full, qcol, r);
          tma_load_2d(sQ + t * AT_TILE + AT_ATOM, &tm, q_full, qcol + 64, r);
        }
        for (int j = 0; j < nB; ++j, ++gk) {
          const int s = gk % AT_STAGES;
          mbar_wait(&k_empty[s], ((gk / AT_STAGES) & 1) ^ 1);
          uint8_t* k = sK + (size_t)s * AT_TILE;
          mbar_expect_tx(&k_full[s], AT_TILE);
          tma_load_2d(k, &tm, &k_full[s], kcol, row0 + j * AT_BN);
          tma_load_2d(k + AT_ATOM, &tm, &k_full[s], kcol + 64, row0 + j * AT_BN);
        }
        ++it;
      }
    }
    __syncwarp();
  } else if (warp == 3) {
    if (lane == 0) {
      int gv = 0;
      for (int rd = 0; rd * (int)gridDim.x < n_items; ++rd) {
        const int i = at_snake(rd, n_items);
        if (i < 0) continue;
        const AtItem w = at_item(i, head_pairs, n_qt, nh, nb);
        const int row0 = w.b * seq_len, vcol = (nh + nkv + w.hA / g) * AT_D, nB = w.qtB + 1;
        for (int j = 0; j < nB; ++j, ++gv) {
          mbar_wait(v_empty, (gv & 1) ^ 1);
          mbar_expect_tx(v_full, AT_TILE);
          tma_load_2d(sV, &tm, v_full, vcol, row0 + j * AT_BN);
          tma_load_2d(sV + AT_ATOM, &tm, v_full, vcol + 64, row0 + j * AT_BN);
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idesc_s = make_idesc_bf16(AT_BM, AT_BN, 0, 0);   // Q K-major, K K-major
      constexpr uint32_t idesc_o = make_idesc_bf16(AT_BM, AT_D, 0, 1);    // P K-major, V MN-major
      const uint32_t qa = smem_u32(sQ), pa = smem_u32(sP), va = smem_u32(sV);
      int gk = 0, gv = 0, it = 0;
      int gs[2] = {0, 0}, gp[2] = {0, 0};
      for (int rd = 0; rd * (int)gridDim.x < n_items; ++rd) {
        const int i = at_snake(rd, n_items);
        if (i < 0) continue;
        const AtItem w = at_item(i, head_pairs, n_qt, nh, nb);
        const int nA = w.qtA + 1, nB = w.qtB + 1;
        mbar_wait(q_full, it & 1);
        // step j: S_A(j), S_B(j), then O_A += P_A(j-1)·V_{j-1}, O_B += P_B(j-1)·V_{j-1}: each
        // tile's softmax hides behind the other MMAs of the step and V_j has two S MMAs of slack
        for (int j = 0; j <= nB; ++j) {
          if (j < nB) {
            const int s = gk % AT_STAGES;
            const uint32_t ka = smem_u32(sK + (size_t)s * AT_TILE);
            mbar_wait(&k_full[s], (gk / AT_STAGES) & 1);
            for (int t = 0; t < 2; ++t) {
              if (t == 0 && j >= nA) continue;
              if (gs[t] >= 1) mbar_wait(&s_free[t], (gs[t] - 1) & 1);
              tc_fence_after();
#pragma unroll
              for (int kk = 0; kk < AT_D / 16; ++kk)
                umma_bf16_ss(tmem + t * AT_BN, at_kmajor(qa + t * AT_TILE, kk), at_kmajor(ka, kk), idesc_s,
                             kk > 0 ? 1u : 0u);
              umma_commit(&s_full[t]);
              ++gs[t];
            }
            umma_commit(&k_empty[s]);
            ++gk;
            if (j == nB - 1) umma_commit(q_empty);      // this item's Q is no longer read
          }
          if (j >= 1) {
            const int jj = j - 1;
            mbar_wait(v_full, gv & 1);
            for (int t = 0; t < 2; ++t) {
              if (t == 0 && jj >= nA) continue;
              if (jj == 0 && it > 0) mbar_wait(&o_free[t], (it - 1) & 1);   // previous O drained
              mbar_wait(&p_full[t], gp[t] & 1);
              tc_fence_after();
#pragma unroll
              for (int kk = 0; kk < AT_BN / 16; ++kk)
                umma_bf16_ss(tmem + (2 + t) * AT_BN, at_kmajor(pa + t * AT_TILE, kk), at_mnmajor(va, kk), idesc_o,
                             (jj | kk) != 0 ? 1u : 0u);
              umma_commit(&pv_done[t]);
              ++gp[t];
            }
            umma_commit(v_empty);
            ++gv;
          }
        }
        ++it;
      }
    }
    __syncwarp();
  } else if (warp >= 4) {
    const int t = (warp - 4) >> 2;                      // 0: tile A, 1: tile B
    const int q4 = warp & 3;
    const int r = q4 * 32 + lane;                       // query row in the tile = TMEM lane
    const uint32_t trow = tmem + (static_cast<uint32_t>(q4 * 32) << 16);
    const uint32_t tS = trow + t * AT_BN, tO = trow + (2 + t) * AT_BN;
    const uint32_t prow = smem_u32(sP) + t * AT_TILE;
    int base = 0;                                       // S / P·V count of this tile before the item
    for (int rd = 0; rd * (int)gridDim.x < n_items; ++rd) {
      const int i = at_snake(rd, n_items);
      if (i < 0) continue;
      const AtItem w = at_item(i, head_pairs, n_qt, nh, nb);
      const int qt = t ? w.qtB : w.qtA, n = qt + 1, h = t ? w.hB : w.hA;
      float m = -INFINITY, l = 0.0f;
      for (int j = 0; j < n; ++j) {
        mbar_wait(&s_full[t], (base + j) & 1);
        tc_fence_after();
        uint32_t sv[AT_BN];
#pragma unroll
        for (int c = 0; c < AT_BN / 16; ++c)
          tmem_ld16(tS + c * 16, *reinterpret_cast<uint32_t(*)[16]>(sv + c * 16));
        tmem_wait_ld();
        tc_fence_before();
        mbar_arrive(&s_free[t]);                        // the MMA may overwrite this S buffer
        if (j == qt) {                                  // diagonal tile: key > query is masked
#pragma unroll
          for (int c = 0; c < AT_BN; ++c)
            if (c > r) sv[c] = __float_as_uint(-INFINITY);
        }
        float mx4[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
#pragma unroll
        for (int c = 0; c < AT_BN / 2; ++c)
          mx4[c & 3] = fmax3(mx4[c & 3], __uint_as_float(sv[2 * c]), __uint_as_float(sv[2 * c + 1]));
        const float mx = fmax3(mx4[0], mx4[1], fmaxf(mx4[2], mx4[3])) * scale_log2;
        const bool move = mx > m + AT_RESCALE_LOG2;     // always on the first tile (m = -inf)
        const float m_new = move ? mx : m;
        const float alpha = move ? ex2(m - m_new) : 1.0f;
        float2 sum2[4] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f),
                          make_float2(0.f, 0.f)};
        const float2 sc2 = make_float2(scale_log2, scale_log2), nm2 = make_float2(-m_new, -m_new);
#pragma unroll
        for (int c = 0; c < AT_BN / 2; ++c) {           // P packed in place: sv[c] = bf16x2(p_2c, p_2c+1)
          const float2 x = ffma2(make_float2(__uint_as_float(sv[2 * c]), __uint_as_float(sv[2 * c + 1])), sc2, nm2);
          const float2 pp = make_float2(ex2(x.x), ex2(x.y));
          sum2[c & 3] = fadd2(sum2[c & 3], pp);
          sv[c] = pack_bf16(pp.x, pp.y);
        }
        const float2 s01 = fadd2(fadd2(sum2[0], sum2[1]), fadd2(sum2[2], sum2[3]));
        l = __fmaf_rn(l, alpha, s01.x + s01.y);
        m = m_new;
        if (j >= 1) {
          mbar_wait(&pv_done[t], (base + j - 1) & 1);   // O holds tiles < j; P buffer is free
          tc_fence_after();
          if (__any_sync(0xffffffffu, alpha != 1.0f)) {
#pragma unroll 1
            for (int c = 0; c < AT_D / 16; ++c) {
              uint32_t o[16];
              tmem_ld16(tO + c * 16, o);
              tmem_wait_ld();
#pragma unroll
              for (int q = 0; q < 16; ++q) o[q] = __float_as_uint(__uint_as_float(o[q]) * alpha);
              tmem_st16(tO + c * 16, o);
            }
            tmem_wait_st();
          }
        }
#pragma unroll
        for (int a = 0; a < 2; ++a)
#pragma unroll
          for (int c = 0; c < 8; ++c) {
            const uint32_t* q = sv + a * 32 + c * 4;
            st_shared_v4(prow + a * AT_ATOM + sw128(r, c), q[0], q[1], q[2], q[3]);
          }
        fence_proxy_async_smem();                       // generic-proxy P writes -> tensor core
        tc_fence_before();
        mbar_arrive(&p_full[t]);
      }
      mbar_wait(&pv_done[t], (base + n - 1) & 1);
      tc_fence_after();
      base += n;
      const float inv = 1.0f / l;
      const int row0 = w.b * seq_len;
      __nv_bfloat16* orow = out + (size_t)(row0 + qt * AT_BM + r) * ld_out + (size_t)h * AT_D;
#pragma unroll 1
      for (int c = 0; c < AT_D / 16; ++c) {
        uint32_t o[16];
        tmem_ld16(tO + c * 16, o);
        tmem_wait_ld();
        uint32_t v8[8];
#pragma unroll
        for (int q = 0; q < 8; ++q)
          v8[q] = pack_bf16(__uint_as_float(o[2 * q]) * inv, __uint_as_float(o[2 * q + 1]) * inv);
        int4* dst = reinterpret_cast<int4*>(orow + c * 16);
        dst[0] = make_int4((int)v8[0], (int)v8[1], (int)v8[2], (int)v8[3]);
        dst[1] = make_int4((int)v8[4], (int)v8[5], (int)v8[6], (int)v8[7]);
      }
      tc_fence_before();
      mbar_arrive(&o_free[t]);                          // the next item's first P·V may overwrite O
      lse[((size_t)w.b * nh + h) * seq_len + qt * AT_BM + r] = (m + log2f(l)) * 0.69314718055994531f;
    }
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
  if (nh < 1 || nkv < 1 || nh % nkv) return set_error(DM_ERR_SHAPE, "attention_fwd: %d heads, %d kv heads", nh, nkv);
  const int row_tile = (nh / nkv) % 2 == 0 ? AT_BM : 2 * AT_BM;   // head pairs vs adjacent row tiles
  if (T < 1 || seq_len < row_tile || seq_len % row_tile || T % seq_len)
    return set_error(DM_ERR_SHAPE, "attention_fwd: seq_len %d must be a multiple of %d dividing T=%d", seq_len,
                     row_tile, T);
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
  if (int rc = ensure_smem_attr((const void*)attn_fwd_kernel, (int)AT_SMEM, "cudaFuncSetAttribute(attn_fwd)")) return rc;
  const float scale_log2 = 1.4426950408889634f / sqrtf((float)AT_D);
  const int head_pairs = (nh / nkv) % 2 == 0, nb = T / seq_len;
  const int n_items = head_pairs ? (seq_len / AT_BM) * (nh / 2) * nb : (seq_len / (2 * AT_BM)) * nh * nb;
  const int grid = n_items < num_sms_current() ? n_items : num_sms_current();
  attn_fwd_kernel<<<grid, AT_THREADS, AT_SMEM, (cudaStream_t)stream>>>(
      tm, seq_len, nh, nkv, nh * AT_D, reinterpret_cast<__nv_bfloat16*>(out), lse, scale_log2, head_pairs, nb);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return set_cuda_error(e, "attention_fwd launch");
  note_launch();
  return DM_OK;
}
