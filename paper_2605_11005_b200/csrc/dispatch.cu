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
#include <stdlib.h>

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
template <typename SelT, typename RunT = int>
__device__ __forceinline__ void chunk_ranks(const SelT* sel, int nslots, RunT* run, int32_t* rank_out, int lane) {
  for (int base = 0; base < nslots; base += 32) {
    const int s = base + lane;
    const bool valid = s < nslots;
    const int e = valid ? (int)sel[s] : -1 - lane;
    const unsigned peers = __match_any_sync(0xffffffffu, e);
    const int r = __popc(peers & ((1u << lane) - 1u));
    const int prior = valid ? run[e] : 0;
    __syncwarp();
    if (valid) {
      rank_out[s] = prior + r;
      if (r == 0) run[e] = (RunT)(prior + __popc(peers));
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

// ------------------------------------------------------------------------
// Streaming dispatch (E <= 16, H % 256 == 0, k <= 8): dm_route_and_dispatch in ONE
// cooperative launch — route, grid barrier, offset scan, permute. Same canonical-order
// logits, top-k, softmax weights and stable permutation as the three-launch path
// (router_fused_kernel / expert_scan / permute_kernel, kept for other shapes and for A/B
// runs with DM_DISPATCH_LEGACY=1). Shaped by per-CTA globaltimer timelines
// (dm_debug_route_profile, scripts/rs_probe.py) of four designs:
//   * work unit = RS_NT = DM_ROUTE_UNIT_TOKENS tokens (one warp); CTA b owns the contiguous
//     units [b*upc, (b+1)*upc), so T = 4096 keeps all 148 SMs busy (7 units each) where
//     32-token chunks left 20 SMs idle;
//   * W_g (fp32, the whole [E, H] gate) arrives by TMA in SWIZZLE_128B boxes: a lane's 32-byte
//     chunk of a 1 KB k-tile sits at granules (2(l&3)+h) ^ (l>>2) of 128-byte row l>>2, which
//     makes the lane-strided 128-bit reads conflict-free without a transposing fill (register
//     / cp.async fills took 5.8 / 9.8 us of L2 latency per CTA; the TMA fill 1.3-1.8 us);
//   * x is read straight from global memory into registers two k-tiles ahead, so all 8 warps
//     compute at once (a bulk-copy ring next to W_g held 3 units: 3 warps, 2-3x slower), with
//     an L2 evict_last policy so the permute phase re-reads x from L2 (scripts/rs_probe.py:
//     45 -> 41 us; an up-front cp.async.bulk.prefetch.L2 of the CTA's rows bought nothing more);
//   * 4 tokens per warp share every W_g read; the k-tile's W_g pairs are loaded before its
//     FFMA2s, which run element pair j outermost (independent chains back to back). The
//     route phase is fp32-FMA bound (T*E*H FMAs in the canonical fmaf order: 128 FFMA2 per
//     16 LDS.128 per k-tile in SASS; ~12.6 us for Mixtral's 134 M FMAs vs the 7.4 us FMA-pipe
//     floor at 64 FMA/clk/SM), not HBM bound;
//   * histogram offsets: each CTA prefix-sums its own units in smem, publishes its totals,
//     and after a grid barrier (fire-and-forget reductions on a monotonic counter: returning
//     same-address atomics from 148 SMs serialise to ~10 us) every CTA scans the CTA totals
//     (~1.2k ints) itself — no serial last-CTA tail;
//   * permute: each CTA copies its own token rows (x L2-resident) to their k expert rows,
//     warp per row with the whole row's loads in flight, and zeroes a share of the padding
//     rows. It runs at the write rate of a dirty L2 (the state every real step and the cold-L2
//     measurement leave): scripts/probes/permute_copy.cu copies 64 MB in 17.4 us with any copy
//     structure (pipelined rows, quarter rows, smem + bulk stores) against 15.3 us for a pure
//     64 MB write. Moving the copy onto TMA (one thread: bulk row loads into a ring in the freed
//     W_g smem, k bulk stores each) was slower, 30 us.
constexpr int RS_NT = DM_ROUTE_UNIT_TOKENS;
constexpr int RS_WARPS = 8;
constexpr int RS_THREADS = RS_WARPS * 32;
constexpr int RS_MAX_UPC = 64;                      // units per CTA (grid grows past #SMs beyond)
constexpr int RS_SMEM_BUDGET = 227 * 1024;

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
// optional per-CTA timeline (dm_debug_route_profile): [cta][0..63] globaltimer ns
__device__ unsigned long long* g_rs_prof = nullptr;

template <int EM>
__global__ void __launch_bounds__(RS_THREADS, 1)
dispatch_stream_kernel(const __grid_constant__ CUtensorMap tmW, const __nv_bfloat16* __restrict__ x, int T, int H,
                       int E, int k, int upc, int w_boxes, int w_box_rows, int32_t* __restrict__ idx,
                       float* __restrict__ w, int32_t* __restrict__ rank, int32_t* __restrict__ cta_tot,
                       uint32_t* __restrict__ gbar, int32_t* __restrict__ counts, int32_t* __restrict__ pad_off,
                       int32_t* __restrict__ row_map, int32_t* __restrict__ src_token,
                       __nv_bfloat16* __restrict__ x_perm) {
  extern __shared__ uint8_t rs_raw[];
  __shared__ uint64_t wbar;
  __shared__ int8_t sel[RS_WARPS][RS_NT * 8];              // expert ids < 16; RS_NT * k <= 32
  __shared__ int16_t run[RS_WARPS][EM];
  __shared__ int16_t s_uh[RS_MAX_UPC][EM];                 // unit histograms -> within-CTA bases
  __shared__ int s_pad[EM + 1], s_cnt[EM];
  __shared__ unsigned long long s_target;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int NI = H >> 8;                                    // 256-element k-tiles (H % 256 == 0)
  const uint32_t pad = (1024u - (smem_u32(rs_raw) & 1023u)) & 1023u;
  uint8_t* sW = rs_raw + pad;                               // [EM][H] fp32, SWIZZLE_128B rows
  const int nunit = (T + RS_NT - 1) / RS_NT;
  const int ub = blockIdx.x * upc;
  const int nmine = max(0, min(upc, nunit - ub));
  unsigned long long* prof = g_rs_prof ? g_rs_prof + (size_t)blockIdx.x * 64 : nullptr;
  if (prof && tid == 0) prof[0] = gtimer();
  if (tid == 0) {
    // grid barrier target: the arrival counter's value once every CTA of THIS launch arrived
    s_target = *reinterpret_cast<volatile unsigned long long*>(gbar + 32) + gridDim.x;
    mbar_init(&wbar, 1);
    fence_mbar_init();
    tma_prefetch_desc(&tmW);
    mbar_expect_tx(&wbar, (uint32_t)(w_boxes * w_box_rows * 128));
    for (int b = 0; b < w_boxes; ++b) tma_load_2d(sW + (size_t)b * w_box_rows * 128, &tmW, &wbar, 0, b * w_box_rows);
  }
  {   // W_g rows e >= E are zero (the hot loop has no E checks)
    const int4 z = make_int4(0, 0, 0, 0);
    for (size_t o = (size_t)E * H * 4 + tid * 16; o < (size_t)EM * H * 4; o += RS_THREADS * 16)
      *reinterpret_cast<int4*>(sW + o) = z;
  }
  __syncthreads();
  // this lane's two 16-byte W_g granules inside every 1 KB k-tile (see the header comment)
  const uint32_t wrow = (uint32_t)(lane >> 2) * 128u;
  const uint32_t wof0 = wrow + ((((uint32_t)(lane & 3) << 1) ^ (uint32_t)(lane >> 2)) << 4);
  const uint32_t wof1 = wrow + (((((uint32_t)(lane & 3) << 1) | 1u) ^ (uint32_t)(lane >> 2)) << 4);
  const uint32_t sWa = smem_u32(sW);
  bool w_ready = false;
  for (int i = warp; i < nmine; i += RS_WARPS) {
    const int u = ub + i;
    const int t0 = u * RS_NT;
    // this unit's token rows (rows past T read row T-1; their results are dropped)
    const __nv_bfloat16* xr[RS_NT];
#pragma unroll
    for (int t = 0; t < RS_NT; ++t) xr[t] = x + (size_t)min(t0 + t, T - 1) * H + lane * 8;
    auto ldx = [&](int it, int4 (&xv)[RS_NT]) {
#pragma unroll
      for (int t = 0; t < RS_NT; ++t)
        xv[t] = it < NI ? ld_nc_v4_hint(xr[t] + it * 256, L2_EVICT_LAST) : make_int4(0, 0, 0, 0);
    };
    int4 x0[RS_NT], x1[RS_NT];
    ldx(0, x0);
    ldx(1, x1);
    if (!w_ready) {
      mbar_wait(&wbar, 0);
      w_ready = true;
      if (prof && tid == 0) prof[1] = gtimer();
    }
    float2 acc[RS_NT][EM];   // {even-element chain, odd-element chain}
#pragma unroll
    for (int t = 0; t < RS_NT; ++t)
#pragma unroll
      for (int e = 0; e < EM; ++e) acc[t][e] = make_float2(0.f, 0.f);
#pragma unroll 1
    for (int it = 0; it < NI; ++it) {
      int4 x2[RS_NT];
      ldx(it + 2, x2);   // two k-tiles ahead
      float4 wv[EM][2];
#pragma unroll
      for (int e = 0; e < EM; ++e) {
        const uint32_t tb = sWa + (uint32_t)((size_t)e * H * 4) + (uint32_t)it * 1024u;
        const int4 a = ld_shared_v4(tb + wof0), b = ld_shared_v4(tb + wof1);
        wv[e][0] = make_float4(__int_as_float(a.x), __int_as_float(a.y), __int_as_float(a.z), __int_as_float(a.w));
        wv[e][1] = make_float4(__int_as_float(b.x), __int_as_float(b.y), __int_as_float(b.z), __int_as_float(b.w));
      }
      // element pair j outermost: each chain (t, e) still takes its pairs in ascending order
      // (the canonical order); consecutive FFMA2s are independent
#pragma unroll
      for (int jj = 0; jj < 4; ++jj) {
        float2 xp[RS_NT];
#pragma unroll
        for (int t = 0; t < RS_NT; ++t) {
          const uint32_t q = reinterpret_cast<const uint32_t*>(&x0[t])[jj];
          xp[t] = make_float2(bf16lo(q), bf16hi(q));
        }
#pragma unroll
        for (int e = 0; e < EM; ++e) {
          const float4 wq = wv[e][jj >> 1];
          const float2 wj = (jj & 1) ? make_float2(wq.z, wq.w) : make_float2(wq.x, wq.y);
#pragma unroll
          for (int t = 0; t < RS_NT; ++t) acc[t][e] = ffma2(xp[t], wj, acc[t][e]);
        }
      }
#pragma unroll
      for (int t = 0; t < RS_NT; ++t) { x0[t] = x1[t]; x1[t] = x2[t]; }
    }
    if (prof && lane == 0 && i < 24) prof[16 + i] = gtimer();
    // butterflies of the RS_NT x EM logits (independent shuffle chains interleave)
    float lgs[RS_NT][EM];
#pragma unroll
    for (int t = 0; t < RS_NT; ++t)
#pragma unroll
      for (int e = 0; e < EM; ++e) lgs[t][e] = __fadd_rn(acc[t][e].x, acc[t][e].y);
#pragma unroll
    for (int off = 16; off > 0; off >>= 1)
#pragma unroll
      for (int t = 0; t < RS_NT; ++t)
#pragma unroll
        for (int e = 0; e < EM; ++e) lgs[t][e] = __fadd_rn(lgs[t][e], __shfl_xor_sync(0xffffffffu, lgs[t][e], off));
    // top-k: lane (t, j) = (lane / k, lane % k) produces pick j of token t; ties -> lower
    // expert id
    {
      const int t = lane / k, j = lane - t * k;
      const bool act = lane < RS_NT * k && t0 + t < T;
      float lgt[EM];
#pragma unroll
      for (int e = 0; e < EM; ++e) {
        float v = lgs[0][e];
#pragma unroll
        for (int tt = 1; tt < RS_NT; ++tt) v = (t == tt) ? lgs[tt][e] : v;
        lgt[e] = v;
      }
      // the k sequential arg-max passes of router_fused_kernel, run by each lane for its
      // own token, keeping pick j (same results for any input, NaN included)
      unsigned taken = 0;
      int mine = -1;
      float v0 = 0.f, vsel = 0.f, ssum = 0.f;
      for (int jj = 0; jj < k; ++jj) {
        float bv = -INFINITY;
        int be = -1;
#pragma unroll
        for (int e = 0; e < EM; ++e)
          if (e < E && !((taken >> e) & 1u) && (be < 0 || lgt[e] > bv)) { bv = lgt[e]; be = e; }
        taken |= 1u << be;
        if (jj == 0) v0 = bv;
        ssum += expf(bv - v0);
        if (jj == j) { mine = be; vsel = bv; }
      }
      const float vmax = v0;
      if (act) {
        const int tok = t0 + t;
        idx[(size_t)tok * k + j] = mine;
        w[(size_t)tok * k + j] = expf(vsel - vmax) / ssum;
        sel[warp][t * k + j] = (int8_t)mine;
      }
    }
    if (lane < EM) run[warp][lane] = 0;
    __syncwarp();
    chunk_ranks(sel[warp], min(RS_NT, T - t0) * k, run[warp], rank + (size_t)t0 * k, lane);
    __syncwarp();
    if (lane < EM) s_uh[i][lane] = run[warp][lane];
    __syncwarp();
  }
  if (prof && tid == 0) prof[2] = gtimer();
  // within-CTA exclusive prefix over the units (thread e walks expert e), CTA totals out
  __syncthreads();
  if (tid < E) {
    int acc = 0;
    for (int i = 0; i < nmine; ++i) {
      const int v = s_uh[i][tid];
      s_uh[i][tid] = (int16_t)acc;
      acc += v;
    }
    cta_tot[(size_t)blockIdx.x * E + tid] = acc;
  }
  // ------------------------------------------------------------ grid barrier
  // (cooperative launch: all CTAs are resident). Arrivals are fire-and-forget reductions on a
  // monotonic 64-bit counter (no returning atomics: 148 returning same-address atomics
  // serialise to ~10 us); each CTA spins until the counter reaches this launch's target;
  // CTA 0 then publishes the next launch's base.
  __syncthreads();
  if (tid == 0) {
    unsigned long long* ctr = reinterpret_cast<unsigned long long*>(gbar);
    fence_acq_rel_gpu();
    asm volatile("red.release.gpu.global.add.u64 [%0], 1;" :: "l"(ctr) : "memory");
    unsigned long long v;
    do {
      asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(ctr) : "memory");
      if (v < s_target) __nanosleep(32);
    } while (v < s_target);
    if (blockIdx.x == 0) *reinterpret_cast<volatile unsigned long long*>(gbar + 32) = s_target;
  }
  __syncthreads();
  fence_acq_rel_gpu();
  if (prof && tid == 0) prof[3] = gtimer();
  // ------------------------------------------------- scan of the CTA totals
  // every CTA: s_base [nb][E] (exclusive over CTAs, in the dynamic smem), s_cnt, s_pad
  const int nb = gridDim.x;
  const int row_bytes = H * 2;
  int* s_base = reinterpret_cast<int*>(rs_raw);
  for (int q = tid; q < nb * E; q += RS_THREADS) s_base[q] = __ldcg(cta_tot + q);
  __syncthreads();
  for (int e = warp; e < E; e += RS_WARPS) {
    int carry = 0;
    for (int b0 = 0; b0 < nb; b0 += 32) {
      const int b = b0 + lane;
      const int v = b < nb ? s_base[b * E + e] : 0;
      int incl = v;
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) {
        const int o = __shfl_up_sync(0xffffffffu, incl, off);
        if (lane >= off) incl += o;
      }
      if (b < nb) s_base[b * E + e] = carry + incl - v;
      carry += __shfl_sync(0xffffffffu, incl, 31);
    }
    if (lane == 0) s_cnt[e] = carry;
  }
  __syncthreads();
  if (tid == 0) {
    int acc = 0;
    for (int e = 0; e < E; ++e) {
      s_pad[e] = acc;
      acc += (s_cnt[e] + DM_ROW_ALIGN - 1) / DM_ROW_ALIGN * DM_ROW_ALIGN;
    }
    s_pad[E] = acc;
    if (blockIdx.x == 0) {
      for (int e = 0; e < E; ++e) { counts[e] = s_cnt[e]; pad_off[e] = s_pad[e]; }
      pad_off[E] = acc;
    }
  }
  __syncthreads();
  // ------------------------------------------------------- permute (scatter)
  // positions of this CTA's (token, slot)s: row_map, src_token, and a smem copy
  const int tok0 = ub * RS_NT;
  const int ntok = max(0, min(nmine * RS_NT, T - tok0));
  const int myb = blockIdx.x;
  int* s_posn = s_base + nb * E;                            // [ntok * k]
  for (int q = tid; q < ntok * k; q += RS_THREADS) {
    const int t = tok0 + q / k;
    const int e = idx[(size_t)t * k + q % k];
    const int pos = s_pad[e] + s_base[myb * E + e] + s_uh[(t / RS_NT) - ub][e] + rank[(size_t)t * k + q % k];
    s_posn[q] = pos;
    row_map[(size_t)t * k + q % k] = pos;
    src_token[pos] = t;
  }
  __syncthreads();
  // copy: warp per token row (x just streamed through L2 by the route phase), the whole row
  // in flight per warp (16 x 16 B per lane at H = 4096), k stores per vector; then the
  // padding rows [s_pad[e] + s_cnt[e], s_pad[e+1]) are zeroed (they feed the ragged-K wgrad)
  // and marked src_token = -1, spread over every CTA's warps
  {
    const int nvec = H >> 3;
    for (int r = warp; r < ntok; r += RS_WARPS) {
      const __nv_bfloat16* src = x + (size_t)(tok0 + r) * H;
      int pj[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) pj[j] = j < k ? s_posn[r * k + j] : 0;
      for (int c0 = lane; c0 < nvec; c0 += 32 * 16) {
        int4 v[16];
#pragma unroll
        for (int q = 0; q < 16; ++q) {
          const int c = c0 + 32 * q;
          v[q] = c < nvec ? ld_nc_v4(src + c * 8) : make_int4(0, 0, 0, 0);
        }
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          if (j >= k) break;
          __nv_bfloat16* dst = x_perm + (size_t)pj[j] * H;
#pragma unroll
          for (int q = 0; q < 16; ++q) {
            const int c = c0 + 32 * q;
            if (c < nvec) st_v4(dst + c * 8, v[q]);
          }
        }
      }
    }
    const int end = s_pad[E];
    const int4 z = make_int4(0, 0, 0, 0);
    for (int r = myb * RS_WARPS + warp; r < end; r += nb * RS_WARPS) {
      int lo = 0, hi = E;   // largest e with s_pad[e] <= r
      while (hi - lo > 1) {
        const int mid = (lo + hi) >> 1;
        if (s_pad[mid] <= r) lo = mid; else hi = mid;
      }
      if (r < s_pad[lo] + s_cnt[lo]) continue;
      if (lane == 0) src_token[r] = -1;
      __nv_bfloat16* row = x_perm + (size_t)r * H;
      for (int c = lane; c < nvec; c += 32) st_v4(row + c * 8, z);
    }
  }
  if (prof && tid == 0) prof[4] = gtimer();
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
               int E, int k_rt, int chunk_tokens, int rel_base, const int32_t* __restrict__ cta_base, int upc,
               int32_t* __restrict__ row_map, int32_t* __restrict__ src_token, __nv_bfloat16* __restrict__ x_perm) {
  const int k = KT ? KT : k_rt;
  const int gwarp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  const int nwarps = (gridDim.x * blockDim.x) >> 5;
  const int nvec = H >> 3;
  for (int t = gwarp; t < T; t += nwarps) {
    const int c = t / chunk_tokens;
    int p[KT ? KT : DM_MAX_TOPK];
#pragma unroll
    for (int j = 0; j < k; ++j) {
      const int e = idx[(size_t)t * k + j];
      p[j] = chunk_base[(size_t)c * E + e] + rank[(size_t)t * k + j] + (rel_base ? pad_off[e] : 0) +
             (cta_base ? cta_base[(size_t)(c / upc) * E + e] : 0);
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

static int permute_launch(const void* x, const int32_t* idx, const int32_t* rank, const int32_t* chunk_base,
                          const int32_t* counts, const int32_t* pad_off, int T, int H, int E, int k,
                          int chunk_tokens, int rel_base, const int32_t* cta_base, int upc, int32_t* row_map,
                          int32_t* src_token, void* x_perm, cudaStream_t st) {
  const __nv_bfloat16* xb = reinterpret_cast<const __nv_bfloat16*>(x);
  __nv_bfloat16* xp = reinterpret_cast<__nv_bfloat16*>(x_perm);
  const int grid = token_grid_dispatch(T);
#define DM_PERM(KTV) permute_kernel<KTV><<<grid, 256, 0, st>>>(xb, idx, rank, chunk_base, counts, pad_off, T, H, E, k, \
                                                                 chunk_tokens, rel_base, cta_base, upc, row_map, src_token, xp)
  switch (k) {
    case 1: DM_PERM(1); break;
    case 2: DM_PERM(2); break;
    case 4: DM_PERM(4); break;
    case 8: DM_PERM(8); break;
    default: DM_PERM(0); break;
  }
#undef DM_PERM
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return set_cuda_error(e, "permute launch");
  note_launch();
  return DM_OK;
}

// Returns -1 when the streaming dispatch does not apply (E > 16, H % 256 != 0, k > 8, W_g
// over the shared-memory budget, more than RS_MAX_UPC units per resident CTA, or no
// cooperative launch). One cooperative launch: route, grid barrier, scan, permute.
static int dispatch_stream_launch(const void* x, const float* wg, int T, int H, int E, int k, int32_t* idx, float* w,
                                  int32_t* rank, int32_t* cta_tot, uint32_t* gbar, int32_t* counts, int32_t* pad_off,
                                  int32_t* row_map, int32_t* src_token, void* x_perm, cudaStream_t stream) {
  if (E > 16 || H % 256 || RS_NT * k > 32) return -1;   // one lane per (token, slot) in the top-k
  if (reinterpret_cast<uintptr_t>(x) & 15 || reinterpret_cast<uintptr_t>(wg) & 15 ||
      reinterpret_cast<uintptr_t>(x_perm) & 15) return -1;
  const int EM = E <= 8 ? 8 : 16;
  const size_t smem = 1024 /* alignment slack */ + (size_t)EM * H * 4;
  if (smem + 4096 /* static */ > (size_t)RS_SMEM_BUDGET) return -1;
  const int nunit = (T + RS_NT - 1) / RS_NT;
  const void* kern = EM == 8 ? (const void*)dispatch_stream_kernel<8> : (const void*)dispatch_stream_kernel<16>;
  if (int rc = ensure_smem_attr(kern, (int)smem, "cudaFuncSetAttribute(dispatch_stream)")) return rc;
  const int resident = num_sms_current() * max_active_blocks(kern, RS_THREADS, smem);
  int grid = nunit < resident ? nunit : resident;
  const int upc = (nunit + grid - 1) / grid;
  if (upc > RS_MAX_UPC) return -1;
  grid = (nunit + upc - 1) / upc;
  // phase 2/3 scratch in the dynamic smem: CTA-total table, positions
  const size_t scratch = (((size_t)grid * E + (size_t)upc * RS_NT * k) * 4 + 1023) & ~(size_t)1023;
  if (scratch > (size_t)EM * H * 4) return -1;
  // W_g as [E*H/32, 32] fp32 rows of 128 B, SWIZZLE_128B boxes of w_box_rows rows
  const int rows_per_expert = H / 32;
  int w_box_rows = 8;
  for (int r = 256; r >= 8; r -= 8)
    if (rows_per_expert % r == 0) { w_box_rows = r; break; }
  const int w_boxes = E * rows_per_expert / w_box_rows;
  CUtensorMap tmW;
  {
    PFN_cuTensorMapEncodeTiled_v12000 enc = tensor_map_encoder();
    if (!enc) return set_error(DM_ERR_DRIVER, "cuTensorMapEncodeTiled entry point unavailable");
    cuuint64_t dims[2] = {32, (cuuint64_t)E * rows_per_expert};
    cuuint64_t strides[1] = {128};
    cuuint32_t box[2] = {32, (cuuint32_t)w_box_rows};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = enc(&tmW, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(wg), dims, strides, box, estr,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return set_error(DM_ERR_DRIVER, "cuTensorMapEncodeTiled(W_g) failed (%d)", (int)r);
  }
  const __nv_bfloat16* xb = reinterpret_cast<const __nv_bfloat16*>(x);
  __nv_bfloat16* xp = reinterpret_cast<__nv_bfloat16*>(x_perm);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(RS_THREADS);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;   // the grid barrier needs every CTA resident
  attr[0].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaError_t e;
  if (EM == 8)
    e = cudaLaunchKernelEx(&cfg, dispatch_stream_kernel<8>, tmW, xb, T, H, E, k, upc, w_boxes, w_box_rows, idx, w, rank,
                           cta_tot, gbar, counts, pad_off, row_map, src_token, xp);
  else
    e = cudaLaunchKernelEx(&cfg, dispatch_stream_kernel<16>, tmW, xb, T, H, E, k, upc, w_boxes, w_box_rows, idx, w,
                           rank, cta_tot, gbar, counts, pad_off, row_map, src_token, xp);
  if (e != cudaSuccess) return set_cuda_error(e, "dispatch_stream launch");
  note_launch();
  return DM_OK;
}

// Group row ranges over n micro-batches stacked cap rows apart, micro-batch i's expert-e block
// [i*cap + pad_off[i][e], i*cap + pad_off[i][e+1]): expert-major (group e*n + i) or
// micro-batch-major (group i*E + e).
__global__ void batch_group_ranges_kernel(const int32_t* __restrict__ pad_off, int n, int E, int cap,
                                          int expert_major, int32_t* __restrict__ start,
                                          int32_t* __restrict__ end) {
  for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < n * E; q += gridDim.x * blockDim.x) {
    const int e = expert_major ? q / n : q % E, i = expert_major ? q % n : q / E;
    start[q] = i * cap + pad_off[i * (E + 1) + e];
    end[q] = i * cap + pad_off[i * (E + 1) + e + 1];
  }
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

/* Debug/profiling hook: when `buf` (device, >= 64 u64 per CTA, zeroed) is non-NULL the
 * streaming router records a per-CTA globaltimer timeline: [0..7] start, W_g staged,
 * warp 0's units done, local prefix, group ticket, ticket, scan done, all units done;
 * [8+i] unit i issued (i < 8); [16+2i], [17+2i] unit i data ready / math done (i < 24). */
int dm_debug_route_profile(void* buf) {
  cudaError_t e = cudaMemcpyToSymbol(g_rs_prof, &buf, sizeof(buf));
  return e == cudaSuccess ? DM_OK : set_cuda_error(e, "cudaMemcpyToSymbol(g_rs_prof)");
}

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
  return permute_launch(x, idx, rank, chunk_base, counts, pad_off, T, H, E, k, DM_CHUNK_TOKENS, 0, nullptr, 1,
                        row_map, src_token, x_perm, (cudaStream_t)stream);
}

int dm_route_and_dispatch(const void* x, const float* wg, int T, int H, int E, int k, void* workspace,
                          int32_t* idx, float* w, int32_t* counts, int32_t* pad_off,
                          int32_t* row_map, int32_t* src_token, void* x_perm, void* stream) {
  int rc = check_route_shape(T, H, E, k);
  if (rc) return rc;
  dm_route_ws ws;
  dm_route_workspace_layout(T, H, E, k, workspace, &ws);
  if (reinterpret_cast<uintptr_t>(x_perm) & 15) return set_error(DM_ERR_ALIGN, "x_perm must be 16-byte aligned");
  // streaming dispatch: ONE cooperative launch (route, grid barrier, scan, permute).
  // Workspace: CTA totals in chunk_hist, grid-barrier counters in done.
  // (DM_DISPATCH_LEGACY=1: the three-launch router_fused / scan / permute path, for A/B runs)
  static const bool legacy = [] {
    const char* e = getenv("DM_DISPATCH_LEGACY");
    return e && e[0] == '1';
  }();
  if (!legacy && (rc = dispatch_stream_launch(x, wg, T, H, E, k, idx, w, ws.rank, ws.chunk_hist, ws.done, counts, pad_off,
                                   row_map, src_token, x_perm, (cudaStream_t)stream)) >= 0)
    return rc;
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

int dm_batch_group_ranges(const int32_t* pad_off, int n, int E, int cap, int expert_major, int32_t* group_start,
                          int32_t* group_end, void* stream) {
  if (n < 1 || E < 1 || cap < 0 || cap % DM_ROW_ALIGN || (long long)n * cap > 0x7fffffffLL)
    return set_error(DM_ERR_SHAPE, "batch_group_ranges: n=%d E=%d cap=%d", n, E, cap);
  const int blocks = (n * E + 255) / 256;
  batch_group_ranges_kernel<<<blocks, 256, 0, (cudaStream_t)stream>>>(pad_off, n, E, cap, expert_major, group_start,
                                                                      group_end);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return set_cuda_error(e, "batch_group_ranges launch");
  note_launch();
  return DM_OK;
}

}  // extern "C"
