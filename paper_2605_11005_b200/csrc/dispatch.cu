// Dispatch side of the MoE hot path (attention/A ranks): router logits with a
// fixed, documented fp32 reduction order, top-k gating, per-chunk expert
// histograms, a deterministic scan to 128-aligned expert offsets, and the
// stable counting-sort permutation into expert-contiguous buffers.
//
// Reference counterpart: none in code. The semantics come from the paper's
// gating sentence ("trainable gate network to select the top-k
// experts"); the reference only models this stage's exchange volume,
// m2n_comm_bytes V = e*b*s*k*H (pkg/src/afpipe/costs.py:95-103). The CPU oracle
// (oracle/moe_oracle.c) restates the exact same order, so expert ids,
// permutation indices and counts are bit-exact.
//
// Canonical logit order (shared with oracle/moe_oracle.c:dm_oracle_router_logits):
//   partial[p][s], lane p in [0,32), parity s in {0,1}: fmaf chain over the
//   8-element chunks c with c % 32 == p (c ascending) and the elements j of each
//   chunk with j % 2 == s (ascending); v[p] = partial[p][0] + partial[p][1]; then
//   an xor butterfly 16,8,4,2,1 of round-to-nearest fp32 adds. Two chains per
//   lane map onto packed fp32x2 FMAs (FFMA2), bit-identical to scalar fmaf.
#include "dm_common.cuh"
#include "dm_internal.h"

namespace dm {

constexpr int ROUTER_NT = 4;        // tokens per warp per pass
constexpr int ROUTER_WARPS = 8;
constexpr int ROUTER_ER = 8;        // experts per register tile
constexpr int ROUTER_SMEM_BUDGET = 160 * 1024;

__global__ void __launch_bounds__(ROUTER_WARPS * 32)
router_logits_kernel(const __nv_bfloat16* __restrict__ x, const float* __restrict__ wg,
                     float* __restrict__ logits, int T, int H, int E, int ec) {
  extern __shared__ float4 sw4[];
  float* sw = reinterpret_cast<float*>(sw4);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nch = H >> 3;
  for (int e0 = 0; e0 < E; e0 += ec) {
    const int ecur = min(ec, E - e0);
    __syncthreads();
    const float4* src = reinterpret_cast<const float4*>(wg + (size_t)e0 * H);
    for (int i = threadIdx.x; i < ecur * H / 4; i += blockDim.x) sw4[i] = src[i];
    __syncthreads();
    for (int tg = (blockIdx.x * ROUTER_WARPS + warp) * ROUTER_NT; tg < T;
         tg += gridDim.x * ROUTER_WARPS * ROUTER_NT) {
      for (int er = 0; er < ecur; er += ROUTER_ER) {
        float2 acc[ROUTER_NT][ROUTER_ER];   // {even-element chain, odd-element chain}
#pragma unroll
        for (int t = 0; t < ROUTER_NT; ++t)
#pragma unroll
          for (int e = 0; e < ROUTER_ER; ++e) acc[t][e] = make_float2(0.f, 0.f);
        for (int c = lane; c < nch; c += 32) {
          int4 xv[ROUTER_NT];
#pragma unroll
          for (int t = 0; t < ROUTER_NT; ++t)
            xv[t] = (tg + t < T) ? ld_nc_v4(x + (size_t)(tg + t) * H + c * 8) : make_int4(0, 0, 0, 0);
#pragma unroll
          for (int e = 0; e < ROUTER_ER; ++e) {
            if (er + e < ecur) {
              const float4* wp = reinterpret_cast<const float4*>(sw + (size_t)(er + e) * H + c * 8);
              const float4 w0 = wp[0], w1 = wp[1];
#pragma unroll
              for (int t = 0; t < ROUTER_NT; ++t) {
                const uint32_t* xp = reinterpret_cast<const uint32_t*>(&xv[t]);
                float2 a = acc[t][e];
                a = ffma2(make_float2(bf16lo(xp[0]), bf16hi(xp[0])), make_float2(w0.x, w0.y), a);
                a = ffma2(make_float2(bf16lo(xp[1]), bf16hi(xp[1])), make_float2(w0.z, w0.w), a);
                a = ffma2(make_float2(bf16lo(xp[2]), bf16hi(xp[2])), make_float2(w1.x, w1.y), a);
                a = ffma2(make_float2(bf16lo(xp[3]), bf16hi(xp[3])), make_float2(w1.z, w1.w), a);
                acc[t][e] = a;
              }
            }
          }
        }
#pragma unroll
        for (int t = 0; t < ROUTER_NT; ++t) {
#pragma unroll
          for (int e = 0; e < ROUTER_ER; ++e) {
            const float v = warp_sum_butterfly(__fadd_rn(acc[t][e].x, acc[t][e].y));
            if (lane == e && er + e < ecur && tg + t < T)
              logits[(size_t)(tg + t) * E + e0 + er + e] = v;
          }
        }
      }
    }
  }
}

// Stable within-chunk ranks (warp 0): sel[] holds the chunk's expert ids in
// token-major (t, j) order; rank[s] = number of earlier slots of the chunk that
// chose the same expert. run[] (E ints, zeroed) ends as the chunk histogram.
__device__ __forceinline__ void chunk_ranks(const int* sel, int nslots, int* run, int32_t* rank_out, int lane) {
  for (int base = 0; base < nslots; base += 32) {
    const int s = base + lane;
    const bool valid = s < nslots;
    const int e = valid ? sel[s] : -1 - lane;
    const unsigned peers = __match_any_sync(0xffffffffu, e);
    const int r = __popc(peers & ((1u << lane) - 1u));
    const int prior = valid ? run[e] : 0;
    __syncwarp();
    if (valid) {
      rank_out[s] = prior + r;
      if (r == 0) run[e] = prior + __popc(peers);
    }
    __syncwarp();
  }
}

// Fused router for E <= EM (Mixtral-class gates): one pass over x computes the
// canonical-order logits, top-k, softmax weights, the within-chunk ranks and
// the chunk histogram. CTA = one 32-token chunk per pass (16 warps x 2 tokens; 8 warps
// x 4 tokens halves the smem reads but measured slower: 28.7 vs 23.5 us, fewer warps),
// persistent over chunks so W_g is staged into smem once per CTA, stored
// lane-interleaved ([e][iteration][half][lane] float4) so each 128-bit smem read
// of a warp is 512 contiguous bytes. The even/odd element chains of the
// canonical order run as packed fp32x2 FMAs (FFMA2) on naturally paired
// registers. W_g rows e >= E are zero-filled, so the hot loop has no E checks.
// x loads are double-buffered two k-tiles deep (unroll 2 beats 4: fewer spills,
// dispatch stage 52.2 -> 50.2 us cold-L2, scripts/dispatch_ab.py).
constexpr int FUSED_UNROLL = 2;
constexpr int FUSED_NT = 2;
constexpr int FUSED_WARPS = DM_CHUNK_TOKENS / FUSED_NT;   // 16

template <int EM>
__global__ void __launch_bounds__(FUSED_WARPS * 32)
router_fused_kernel(const __nv_bfloat16* __restrict__ x, const float* __restrict__ wg, int T, int H, int E,
                    int k, float* __restrict__ logits, int32_t* __restrict__ idx, float* __restrict__ w,
                    int32_t* __restrict__ rank, int32_t* __restrict__ chunk_hist) {
  extern __shared__ float4 sw4[];
  __shared__ int sel[DM_CHUNK_TOKENS * DM_MAX_TOPK];
  __shared__ int run[EM];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nch = H >> 3;
  const int NI = (nch + 31) >> 5;
  for (int i = threadIdx.x; i < EM * NI * 64; i += blockDim.x) {
    const int l = i & 31, half = (i >> 5) & 1, rest = i >> 6;
    const int it = rest % NI, e = rest / NI;
    const int c = it * 32 + l;
    sw4[i] = (c < nch && e < E) ? reinterpret_cast<const float4*>(wg + (size_t)e * H + c * 8)[half]
                                : make_float4(0.f, 0.f, 0.f, 0.f);
  }
  const int nchunk = (T + DM_CHUNK_TOKENS - 1) / DM_CHUNK_TOKENS;
  for (int chunk = blockIdx.x; chunk < nchunk; chunk += gridDim.x) {
    if (threadIdx.x < EM) run[threadIdx.x] = 0;
    __syncthreads();   // also orders the W_g fill before first use
    const int t0 = chunk * DM_CHUNK_TOKENS;
    const int tg = t0 + warp * FUSED_NT;
    float2 acc[FUSED_NT][EM];   // {even-element chain, odd-element chain}
#pragma unroll
    for (int t = 0; t < FUSED_NT; ++t)
#pragma unroll
      for (int e = 0; e < EM; ++e) acc[t][e] = make_float2(0.f, 0.f);
    // x k-tiles are double-buffered in registers: the loads of batch i+1 are in flight
    // while batch i is multiplied (the loop is unrolled by two batches).
    int4 xa[FUSED_UNROLL][FUSED_NT], xb[FUSED_UNROLL][FUSED_NT];
    auto load = [&](int4 (&xv)[FUSED_UNROLL][FUSED_NT], int it0) {
#pragma unroll
      for (int u = 0; u < FUSED_UNROLL; ++u)
#pragma unroll
        for (int t = 0; t < FUSED_NT; ++t) {
          const int c = (it0 + u) * 32 + lane;
          xv[u][t] = (it0 + u < NI && c < nch && tg + t < T) ? ld_nc_v4(x + (size_t)(tg + t) * H + c * 8)
                                                            : make_int4(0, 0, 0, 0);
        }
    };
    auto compute = [&](const int4 (&xv)[FUSED_UNROLL][FUSED_NT], int it0) {
#pragma unroll
      for (int u = 0; u < FUSED_UNROLL; ++u) {
        if (it0 + u >= NI) break;
        float2 xp[FUSED_NT][4];
#pragma unroll
        for (int t = 0; t < FUSED_NT; ++t) {
          const uint32_t* q = reinterpret_cast<const uint32_t*>(&xv[u][t]);
#pragma unroll
          for (int i = 0; i < 4; ++i) xp[t][i] = make_float2(bf16lo(q[i]), bf16hi(q[i]));
        }
#pragma unroll
        for (int e = 0; e < EM; ++e) {
          const float4* wp = sw4 + ((size_t)(e * NI + it0 + u) * 2) * 32 + lane;
          const float4 w0 = wp[0], w1 = wp[32];
#pragma unroll
          for (int t = 0; t < FUSED_NT; ++t) {
            float2 a = acc[t][e];
            a = ffma2(xp[t][0], make_float2(w0.x, w0.y), a);
            a = ffma2(xp[t][1], make_float2(w0.z, w0.w), a);
            a = ffma2(xp[t][2], make_float2(w1.x, w1.y), a);
            a = ffma2(xp[t][3], make_float2(w1.z, w1.w), a);
            acc[t][e] = a;
          }
        }
      }
    };
    load(xa, 0);
    for (int it0 = 0; it0 < NI; it0 += 2 * FUSED_UNROLL) {
      if (it0 + FUSED_UNROLL < NI) load(xb, it0 + FUSED_UNROLL);
      compute(xa, it0);
      if (it0 + FUSED_UNROLL >= NI) break;
      if (it0 + 2 * FUSED_UNROLL < NI) load(xa, it0 + 2 * FUSED_UNROLL);
      compute(xb, it0 + FUSED_UNROLL);
    }
#pragma unroll
    for (int t = 0; t < FUSED_NT; ++t) {
      float lg[EM];
#pragma unroll
      for (int e = 0; e < EM; ++e) lg[e] = warp_sum_butterfly(__fadd_rn(acc[t][e].x, acc[t][e].y));
      const int tok = tg + t;
      if (tok >= T) continue;
      if (lane < E) {
        float v = lg[0];
#pragma unroll
        for (int e = 1; e < EM; ++e) v = (lane == e) ? lg[e] : v;
        logits[(size_t)tok * E + lane] = v;
      }
      // top-k over registers (uniform across lanes): ties -> lower expert id
      unsigned taken = 0;
      float sel_v[DM_MAX_TOPK];
      int sel_e[DM_MAX_TOPK];
      for (int j = 0; j < k; ++j) {
        float bv = -INFINITY;
        int be = -1;
#pragma unroll
        for (int e = 0; e < EM; ++e) {
          if (e < E && !((taken >> e) & 1u) && (be < 0 || lg[e] > bv)) { bv = lg[e]; be = e; }
        }
        taken |= 1u << be;
        sel_v[j] = bv;
        sel_e[j] = be;
      }
      float s = 0.0f;
      for (int j = 0; j < k; ++j) s += expf(sel_v[j] - sel_v[0]);
      for (int j = lane; j < k; j += 32) {
        idx[(size_t)tok * k + j] = sel_e[j];
        w[(size_t)tok * k + j] = expf(sel_v[j] - sel_v[0]) / s;
        sel[(tok - t0) * k + j] = sel_e[j];
      }
    }
    __syncthreads();
    if (warp == 0) chunk_ranks(sel, min(DM_CHUNK_TOKENS, T - t0) * k, run, rank + (size_t)t0 * k, lane);
    __syncthreads();
    if (threadIdx.x < E) chunk_hist[(size_t)chunk * E + threadIdx.x] = run[threadIdx.x];
  }
}

// Generic top-k (any E): warp per token over the logits row; ties -> lower expert
// id; weights = softmax over the selected logits. CTA per chunk also produces the
// within-chunk ranks and the chunk histogram.
__global__ void __launch_bounds__(256)
router_topk_kernel(const float* __restrict__ logits, int T, int E, int k, int32_t* __restrict__ idx,
                   float* __restrict__ w, int32_t* __restrict__ rank, int32_t* __restrict__ chunk_hist) {
  extern __shared__ int run[];   // [E]
  __shared__ int sel[DM_CHUNK_TOKENS * DM_MAX_TOPK];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nwarps = blockDim.x >> 5;
  for (int i = threadIdx.x; i < E; i += blockDim.x) run[i] = 0;
  const int t0 = blockIdx.x * DM_CHUNK_TOKENS;
  for (int tt = warp; tt < DM_CHUNK_TOKENS; tt += nwarps) {
    const int t = t0 + tt;
    if (t >= T) break;
    const float* row = logits + (size_t)t * E;
    int sel_e[DM_MAX_TOPK];
    float sel_v[DM_MAX_TOPK];
    for (int j = 0; j < k; ++j) {
      float bv = -INFINITY;
      int be = 0x7fffffff;
      for (int e = lane; e < E; e += 32) {
        bool taken = false;
        for (int q = 0; q < j; ++q) taken |= (sel_e[q] == e);
        const float v = row[e];
        if (!taken && (v > bv || (v == bv && e < be))) { bv = v; be = e; }
      }
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) {
        const float ov = __shfl_xor_sync(0xffffffffu, bv, off);
        const int oe = __shfl_xor_sync(0xffffffffu, be, off);
        if (ov > bv || (ov == bv && oe < be)) { bv = ov; be = oe; }
      }
      sel_e[j] = be;
      sel_v[j] = bv;
    }
    float s = 0.0f;
    for (int j = 0; j < k; ++j) s += expf(sel_v[j] - sel_v[0]);
    if (lane == 0) {
      for (int j = 0; j < k; ++j) {
        idx[(size_t)t * k + j] = sel_e[j];
        w[(size_t)t * k + j] = expf(sel_v[j] - sel_v[0]) / s;
        sel[tt * k + j] = sel_e[j];
      }
    }
  }
  __syncthreads();
  if (warp == 0) chunk_ranks(sel, min(DM_CHUNK_TOKENS, T - t0) * k, run, rank + (size_t)t0 * k, lane);
  __syncthreads();
  for (int i = threadIdx.x; i < E; i += blockDim.x) chunk_hist[(size_t)blockIdx.x * E + i] = run[i];
}

// One CTA, warp per expert: pass 1 sums the expert's chunk counts, thread 0
// turns the totals into DM_ROW_ALIGN-padded block offsets, pass 2 writes the
// exclusive per-chunk bases (warp shuffle scan, chunks in ascending order).
__global__ void __launch_bounds__(1024)
expert_scan_kernel(const int32_t* __restrict__ hist, int nchunk, int E, int32_t* __restrict__ counts,
                   int32_t* __restrict__ pad_off, int32_t* __restrict__ chunk_base) {
  __shared__ int s_off[DM_MAX_EXPERTS + 1];
  __shared__ int s_cnt[DM_MAX_EXPERTS];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nwarps = blockDim.x >> 5;
  for (int e = warp; e < E; e += nwarps) {
    int tot = 0;
    for (int c = lane; c < nchunk; c += 32) tot += hist[(size_t)c * E + e];
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) tot += __shfl_xor_sync(0xffffffffu, tot, off);
    if (lane == 0) { s_cnt[e] = tot; counts[e] = tot; }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    int acc = 0;
    for (int e = 0; e < E; ++e) {
      s_off[e] = acc;
      acc += (s_cnt[e] + DM_ROW_ALIGN - 1) / DM_ROW_ALIGN * DM_ROW_ALIGN;
    }
    s_off[E] = acc;
  }
  __syncthreads();
  for (int e = threadIdx.x; e <= E; e += blockDim.x) pad_off[e] = s_off[e];
  for (int e = warp; e < E; e += nwarps) {
    int runv = s_off[e];
    for (int c0 = 0; c0 < nchunk; c0 += 32) {
      const int c = c0 + lane;
      const int v = c < nchunk ? hist[(size_t)c * E + e] : 0;
      int incl = v;
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) {
        const int o = __shfl_up_sync(0xffffffffu, incl, off);
        if (lane >= off) incl += o;
      }
      if (c < nchunk) chunk_base[(size_t)c * E + e] = runv + incl - v;
      runv += __shfl_sync(0xffffffffu, incl, 31);
    }
  }
}

// Scan for many experts (E >= 64): thread per expert, so every pass over the
// [nchunk][E] histogram is coalesced across threads; the padded per-expert sizes
// are prefix-summed with a block scan (warp shuffles + warp totals).
__global__ void __launch_bounds__(1024)
expert_scan_wide_kernel(const int32_t* __restrict__ hist, int nchunk, int E, int32_t* __restrict__ counts,
                        int32_t* __restrict__ pad_off, int32_t* __restrict__ chunk_base) {
  __shared__ int s_warp[32];
  const int e = threadIdx.x, lane = e & 31, warp = e >> 5;
  int tot = 0;
  if (e < E) {
#pragma unroll 8
    for (int c = 0; c < nchunk; ++c) tot += hist[(size_t)c * E + e];
    counts[e] = tot;
  }
  const int padded = (tot + DM_ROW_ALIGN - 1) / DM_ROW_ALIGN * DM_ROW_ALIGN;
  int incl = padded;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const int o = __shfl_up_sync(0xffffffffu, incl, off);
    if (lane >= off) incl += o;
  }
  if (lane == 31) s_warp[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    const int nw = (blockDim.x + 31) >> 5;
    int w = lane < nw ? s_warp[lane] : 0;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const int o = __shfl_up_sync(0xffffffffu, w, off);
      if (lane >= off) w += o;
    }
    s_warp[lane] = w;   // inclusive prefix of warp totals
  }
  __syncthreads();
  const int excl = incl - padded + (warp > 0 ? s_warp[warp - 1] : 0);
  if (e < E) {
    pad_off[e] = excl;
    if (e == E - 1) pad_off[E] = excl + padded;
    int run = excl;
#pragma unroll 8
    for (int c = 0; c < nchunk; ++c) {
      const int v = hist[(size_t)c * E + e];
      chunk_base[(size_t)c * E + e] = run;
      run += v;
    }
  }
}

// Permute (scatter-copy), warp per token: pos(t, j) = chunk_base[chunk(t), e] +
// rank[t, j]; x[t] is read once with 8-deep 128-bit loads and written to its k
// expert rows. Every warp then helps zero the padding rows (they feed the
// ragged-K wgrad, so they must be finite) and mark them src_token = -1.
template <int KT>
__global__ void __launch_bounds__(256)
permute_kernel(const __nv_bfloat16* __restrict__ x, const int32_t* __restrict__ idx,
               const int32_t* __restrict__ rank, const int32_t* __restrict__ chunk_base,
               const int32_t* __restrict__ counts, const int32_t* __restrict__ pad_off, int T, int H,
               int E, int k_rt, int32_t* __restrict__ row_map, int32_t* __restrict__ src_token,
               __nv_bfloat16* __restrict__ x_perm) {
  const int k = KT ? KT : k_rt;
  const int gwarp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  const int nwarps = (gridDim.x * blockDim.x) >> 5;
  const int nvec = H >> 3;
  for (int t = gwarp; t < T; t += nwarps) {
    const int c = t / DM_CHUNK_TOKENS;
    int p[KT ? KT : DM_MAX_TOPK];
#pragma unroll
    for (int j = 0; j < k; ++j) {
      const int e = idx[(size_t)t * k + j];
      p[j] = chunk_base[(size_t)c * E + e] + rank[(size_t)t * k + j];
    }
    if (lane < k) {
      int pj = p[0];
#pragma unroll
      for (int j = 1; j < k; ++j) pj = (lane == j) ? p[j] : pj;
      row_map[(size_t)t * k + lane] = pj;
      src_token[pj] = t;
    }
    const __nv_bfloat16* src = x + (size_t)t * H;
    int ch = lane;
    for (; ch + 32 * 7 < nvec; ch += 256) {
      int4 v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) v[u] = ld_nc_v4(src + (ch + 32 * u) * 8);
#pragma unroll
      for (int j = 0; j < k; ++j) {
        __nv_bfloat16* dst = x_perm + (size_t)p[j] * H;
#pragma unroll
        for (int u = 0; u < 8; ++u) st_v4(dst + (ch + 32 * u) * 8, v[u]);
      }
    }
    for (; ch < nvec; ch += 32) {
      const int4 v = ld_nc_v4(src + ch * 8);
#pragma unroll
      for (int j = 0; j < k; ++j) st_v4(x_perm + (size_t)p[j] * H + ch * 8, v);
    }
  }
  zero_padding_rows(x_perm, H, counts, pad_off, E, gwarp, nwarps, lane, src_token);
}

// Tiled router logits for large E (DeepSeek-class gates). Same canonical order:
// lane p of a warp owns chunk p of every 256-element k-tile (even/odd element
// chains as one FFMA2 pair) for each of the warp's 8-token x 8-expert outputs,
// and the 32 lane partials are reduced by the xor butterfly at the end. A CTA of
// 8 warps (4 token groups x 2 expert groups) covers 32 tokens x 16 experts; the
// x (bf16) and W_g (fp32) k-tiles are staged L2 -> smem by cp.async (no register
// round trip) through a 3-deep ring. Per k-tile a warp reads 8 x 16 B of x and
// 8 x 32 B of W_g per lane for 256 FFMA2 (8 tokens x 8 experts x 4 pairs), which
// keeps shared-memory reads below the FMA-pipe time.
constexpr int RT_TOK = 32, RT_EXP = 16, RT_THREADS = 256, RT_STAGES = 3;
constexpr int RT_STAGE_INT4 = RT_TOK * 32 + RT_EXP * 2 * 32;  // 16 KB x + 16 KB W_g

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, bool valid) {
  const uint32_t d = static_cast<uint32_t>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(d), "l"(gmem), "r"(valid ? 16 : 0)
               : "memory");
}

__global__ void __launch_bounds__(RT_THREADS, 1)
router_logits_tiled_kernel(const __nv_bfloat16* __restrict__ x, const float* __restrict__ wg,
                           float* __restrict__ logits, int T, int H, int E) {
  extern __shared__ int4 rt_smem[];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int t0 = blockIdx.x * RT_TOK, e0 = blockIdx.y * RT_EXP;
  const int wt = (warp & 3) * 8, we = (warp >> 2) * 8;   // this warp's 8 tokens x 8 experts
  const int nch = H >> 3, nkt = (nch + 31) >> 5;
  // stage layout: xs[tok][lane] int4, then ws[exp][half][lane] float4
  auto xs = [&](int st, int t, int l) -> int4* { return rt_smem + st * RT_STAGE_INT4 + t * 32 + l; };
  auto ws = [&](int st, int e, int h, int l) -> int4* {
    return rt_smem + st * RT_STAGE_INT4 + RT_TOK * 32 + (e * 2 + h) * 32 + l;
  };
  auto issue = [&](int kt) {
    const int st = kt % RT_STAGES;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int f = tid + q * RT_THREADS;            // 32 tokens x 32 chunks
      const int t = f >> 5, l = f & 31, c = kt * 32 + l;
      const bool ok = t0 + t < T && c < nch;
      cp_async16(xs(st, t, l), ok ? (const void*)(x + (size_t)(t0 + t) * H + c * 8) : (const void*)x, ok);
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int f = tid + q * RT_THREADS;            // 16 experts x 32 chunks x 2 halves
      const int e = f >> 6, l = (f >> 1) & 31, h = f & 1, c = kt * 32 + l;
      const bool ok = e0 + e < E && c < nch;
      cp_async16(ws(st, e, h, l), ok ? (const void*)(wg + (size_t)(e0 + e) * H + c * 8 + h * 4) : (const void*)wg,
                 ok);
    }
  };
  float2 acc[8][8];
#pragma unroll
  for (int t = 0; t < 8; ++t)
#pragma unroll
    for (int e = 0; e < 8; ++e) acc[t][e] = make_float2(0.f, 0.f);
#pragma unroll
  for (int kt = 0; kt < RT_STAGES - 1; ++kt) {
    if (kt < nkt) issue(kt);
    asm volatile("cp.async.commit_group;\n" ::: "memory");
  }
  for (int kt = 0; kt < nkt; ++kt) {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(RT_STAGES - 2) : "memory");
    __syncthreads();   // stage kt landed for all threads; stage kt-1 is no longer read
    if (kt + RT_STAGES - 1 < nkt) issue(kt + RT_STAGES - 1);
    asm volatile("cp.async.commit_group;\n" ::: "memory");
    const int st = kt % RT_STAGES;
    float2 w[8][4];
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const float4 a = *reinterpret_cast<const float4*>(ws(st, we + e, 0, lane));
      const float4 b = *reinterpret_cast<const float4*>(ws(st, we + e, 1, lane));
      w[e][0] = make_float2(a.x, a.y);
      w[e][1] = make_float2(a.z, a.w);
      w[e][2] = make_float2(b.x, b.y);
      w[e][3] = make_float2(b.z, b.w);
    }
#pragma unroll
    for (int t = 0; t < 8; ++t) {
      const int4 v = *xs(st, wt + t, lane);
      const uint32_t* q = reinterpret_cast<const uint32_t*>(&v);
      float2 xp[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) xp[i] = make_float2(bf16lo(q[i]), bf16hi(q[i]));
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        float2 a = acc[t][e];
#pragma unroll
        for (int i = 0; i < 4; ++i) a = ffma2(xp[i], w[e][i], a);
        acc[t][e] = a;
      }
    }
  }
  asm volatile("cp.async.wait_group 0;\n" ::: "memory");
  float out0 = 0.0f, out1 = 0.0f;
#pragma unroll
  for (int t = 0; t < 8; ++t)
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const float v = warp_sum_butterfly(__fadd_rn(acc[t][e].x, acc[t][e].y));
      if (lane == (t & 3) * 8 + e) {
        if (t < 4) out0 = v; else out1 = v;
      }
    }
  const int ex = e0 + we + (lane & 7);
  const int tok0 = t0 + wt + (lane >> 3), tok1 = tok0 + 4;
  if (ex < E) {
    if (tok0 < T) logits[(size_t)tok0 * E + ex] = out0;
    if (tok1 < T) logits[(size_t)tok1 * E + ex] = out1;
  }
}

int router_logits_launch(const void* x, const float* wg, float* logits, int T, int H, int E,
                         cudaStream_t stream) {
  if (E > 16) {
    constexpr size_t rt_smem = (size_t)RT_STAGES * RT_STAGE_INT4 * sizeof(int4);
    if (int rc = ensure_smem_attr((const void*)router_logits_tiled_kernel, (int)rt_smem,
                                  "cudaFuncSetAttribute(router_tiled)")) return rc;
    dim3 grid((T + RT_TOK - 1) / RT_TOK, (E + RT_EXP - 1) / RT_EXP);
    router_logits_tiled_kernel<<<grid, RT_THREADS, rt_smem, stream>>>(reinterpret_cast<const __nv_bfloat16*>(x), wg,
                                                                logits, T, H, E);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return set_cuda_error(e, "router_logits_tiled launch");
    note_launch();
    return DM_OK;
  }
  const size_t row_bytes = (size_t)H * sizeof(float);
  int ec = (int)(ROUTER_SMEM_BUDGET / row_bytes);
  if (ec < 1) return set_error(DM_ERR_SHAPE, "router: hidden %d too large for one smem row", H);
  if (ec > E) ec = E;
  const size_t smem = (size_t)ec * row_bytes;
  if (int rc = ensure_smem_attr((const void*)router_logits_kernel, ROUTER_SMEM_BUDGET, "cudaFuncSetAttribute(router)"))
    return rc;
  const int per_cta = ROUTER_WARPS * ROUTER_NT;
  int grid = (T + per_cta - 1) / per_cta;
  const int cap = num_sms_current();
  if (grid > cap) grid = cap;
  if (grid < 1) grid = 1;
  router_logits_kernel<<<grid, ROUTER_WARPS * 32, smem, stream>>>(
      reinterpret_cast<const __nv_bfloat16*>(x), wg, logits, T, H, E, ec);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return set_cuda_error(e, "router_logits launch");
  note_launch();
  return DM_OK;
}

// Returns -1 when the fused router does not apply (E > 16 or W_g over the smem budget).
int router_fused_launch(const void* x, const float* wg, int T, int H, int E, int k, float* logits,
                        int32_t* idx, float* w, int32_t* rank, int32_t* chunk_hist, cudaStream_t stream) {
  const int NI = ((H >> 3) + 31) >> 5;
  const size_t smem = (size_t)(E <= 8 ? 8 : 16) * NI * 64 * sizeof(float4);
  if (E > 16 || smem > (size_t)ROUTER_SMEM_BUDGET) return -1;
  if (reinterpret_cast<uintptr_t>(x) & 15 || reinterpret_cast<uintptr_t>(wg) & 15) return -1;
  if (int rc = ensure_smem_attr((const void*)router_fused_kernel<8>, ROUTER_SMEM_BUDGET,
                                "cudaFuncSetAttribute(router_fused)")) return rc;
  if (int rc = ensure_smem_attr((const void*)router_fused_kernel<16>, ROUTER_SMEM_BUDGET,
                                "cudaFuncSetAttribute(router_fused)")) return rc;
  const int nchunk = dm_num_chunks(T);
  const int grid = nchunk < num_sms_current() ? nchunk : num_sms_current();
  const __nv_bfloat16* xb = reinterpret_cast<const __nv_bfloat16*>(x);
  if (E <= 8)
    router_fused_kernel<8><<<grid, FUSED_WARPS * 32, smem, stream>>>(xb, wg, T, H, E, k, logits, idx, w, rank,
                                                                      chunk_hist);
  else
    router_fused_kernel<16><<<grid, FUSED_WARPS * 32, smem, stream>>>(xb, wg, T, H, E, k, logits, idx, w, rank,
                                                                       chunk_hist);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return set_cuda_error(e, "router_fused launch");
  note_launch();
  return DM_OK;
}

static int token_grid_dispatch(int T) {
  int blocks = (T + 7) / 8;  // 8 warps (tokens) per 256-thread block
  const int cap = num_sms_current() * 8;
  return blocks < cap ? blocks : cap;
}

}  // namespace dm

using namespace dm;

static int check_route_shape(int T, int H, int E, int k) {
  if (T < 1 || H < 8 || E < 1 || k < 1) return set_error(DM_ERR_SHAPE, "bad shape T=%d H=%d E=%d k=%d", T, H, E, k);
  if (H % 8) return set_error(DM_ERR_ALIGN, "hidden %d must be a multiple of 8 (128-bit rows)", H);
  if (E > DM_MAX_EXPERTS) return set_error(DM_ERR_SHAPE, "experts %d > %d", E, DM_MAX_EXPERTS);
  if (k > DM_MAX_TOPK || k > E) return set_error(DM_ERR_SHAPE, "topk %d invalid (max %d, E=%d)", k, DM_MAX_TOPK, E);
  return DM_OK;
}

extern "C" {

int dm_router_logits(const void* x, const float* wg, float* logits, int T, int H, int E, void* stream) {
  int rc = check_route_shape(T, H, E, 1);
  if (rc) return rc;
  if (reinterpret_cast<uintptr_t>(x) & 15 || reinterpret_cast<uintptr_t>(wg) & 15)
    return set_error(DM_ERR_ALIGN, "router operands must be 16-byte aligned");
  return router_logits_launch(x, wg, logits, T, H, E, (cudaStream_t)stream);
}

int dm_router_topk(const float* logits, int T, int E, int k, int32_t* idx, float* w, int32_t* rank,
                   int32_t* chunk_hist, void* stream) {
  int rc = check_route_shape(T, 8, E, k);
  if (rc) return rc;
  const int nchunk = dm_num_chunks(T);
  router_topk_kernel<<<nchunk, 256, E * sizeof(int), (cudaStream_t)stream>>>(logits, T, E, k, idx, w, rank,
                                                                             chunk_hist);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return set_cuda_error(e, "router_topk launch");
  note_launch();
  return DM_OK;
}

int dm_expert_scan(const int32_t* chunk_hist, int T, int E, int32_t* counts, int32_t* pad_off,
                   int32_t* chunk_base, void* stream) {
  int rc = check_route_shape(T, 8, E, 1);
  if (rc) return rc;
  const int nchunk = dm_num_chunks(T);
  if (E >= 64)
    expert_scan_wide_kernel<<<1, (E + 31) / 32 * 32, 0, (cudaStream_t)stream>>>(chunk_hist, nchunk, E, counts,
                                                                                pad_off, chunk_base);
  else
    expert_scan_kernel<<<1, 1024, 0, (cudaStream_t)stream>>>(chunk_hist, nchunk, E, counts, pad_off, chunk_base);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return set_cuda_error(e, "expert_scan launch");
  note_launch();
  return DM_OK;
}

int dm_permute(const void* x, const int32_t* idx, const int32_t* rank, const int32_t* chunk_base,
               const int32_t* counts, const int32_t* pad_off, int T, int H, int E, int k, int32_t* row_map,
               int32_t* src_token, void* x_perm, void* stream) {
  int rc = check_route_shape(T, H, E, k);
  if (rc) return rc;
  if (reinterpret_cast<uintptr_t>(x) & 15 || reinterpret_cast<uintptr_t>(x_perm) & 15)
    return set_error(DM_ERR_ALIGN, "permute rows must be 16-byte aligned");
  const __nv_bfloat16* xb = reinterpret_cast<const __nv_bfloat16*>(x);
  __nv_bfloat16* xp = reinterpret_cast<__nv_bfloat16*>(x_perm);
  const int grid = token_grid_dispatch(T);
  cudaStream_t st = (cudaStream_t)stream;
  switch (k) {
    case 1: permute_kernel<1><<<grid, 256, 0, st>>>(xb, idx, rank, chunk_base, counts, pad_off, T, H, E, k, row_map, src_token, xp); break;
    case 2: permute_kernel<2><<<grid, 256, 0, st>>>(xb, idx, rank, chunk_base, counts, pad_off, T, H, E, k, row_map, src_token, xp); break;
    case 4: permute_kernel<4><<<grid, 256, 0, st>>>(xb, idx, rank, chunk_base, counts, pad_off, T, H, E, k, row_map, src_token, xp); break;
    case 8: permute_kernel<8><<<grid, 256, 0, st>>>(xb, idx, rank, chunk_base, counts, pad_off, T, H, E, k, row_map, src_token, xp); break;
    default: permute_kernel<0><<<grid, 256, 0, st>>>(xb, idx, rank, chunk_base, counts, pad_off, T, H, E, k, row_map, src_token, xp); break;
  }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return set_cuda_error(e, "permute launch");
  note_launch();
  return DM_OK;
}

int dm_route_and_dispatch(const void* x, const float* wg, int T, int H, int E, int k, void* workspace,
                          int32_t* idx, float* w, int32_t* counts, int32_t* pad_off,
                          int32_t* row_map, int32_t* src_token, void* x_perm, void* stream) {
  int rc = check_route_shape(T, H, E, k);
  if (rc) return rc;
  dm_route_ws ws;
  dm_route_workspace_layout(T, H, E, k, workspace, &ws);
  if ((rc = router_fused_launch(x, wg, T, H, E, k, ws.logits, idx, w, ws.rank, ws.chunk_hist,
                                (cudaStream_t)stream)) > 0)
    return rc;
  if (rc < 0) {  // gate too large for the fused kernel: logits pass + top-k pass
    if ((rc = dm_router_logits(x, wg, ws.logits, T, H, E, stream))) return rc;
    if ((rc = dm_router_topk(ws.logits, T, E, k, idx, w, ws.rank, ws.chunk_hist, stream))) return rc;
  }
  if ((rc = dm_expert_scan(ws.chunk_hist, T, E, counts, pad_off, ws.chunk_base, stream))) return rc;
  return dm_permute(x, idx, ws.rank, ws.chunk_base, counts, pad_off, T, H, E, k, row_map, src_token, x_perm, stream);
}

}  // extern "C"
