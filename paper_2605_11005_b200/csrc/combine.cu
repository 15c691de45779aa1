// Combine side of the MoE hot path (A ranks): gate-weighted unpermute-reduce
// (fwd), its backward (scatter of weighted grads + gate-weight grads, fused
// with the top-k softmax Jacobian), the permutation backward (gather-reduce,
// fused with the router's dx term) and the router weight gradient.
//
// Reference counterpart: "outputs ... reduced by a weighted sum";
// the F->A transfer task of _build_afpipe (pkg/src/afpipe/taskgraph.py:335-339)
// and the backward chain taskgraph.py:343-356 are the reference's stand-ins.
// All kernels are HBM-bound row gathers/scatters: warp per token, 128-bit
// vectors, fp32 accumulation in a fixed j order, no atomics.
#include <stdlib.h>

#include "dm_common.cuh"
#include "dm_internal.h"

namespace dm {

__device__ __forceinline__ void unpack8(const int4& v, float (&f)[8]) {
  const uint32_t* p = reinterpret_cast<const uint32_t*>(&v);
#pragma unroll
  for (int i = 0; i < 4; ++i) { f[2 * i] = bf16lo(p[i]); f[2 * i + 1] = bf16hi(p[i]); }
}
__device__ __forceinline__ int4 pack8(const float (&f)[8]) {
  int4 v;
  uint32_t* p = reinterpret_cast<uint32_t*>(&v);
#pragma unroll
  for (int i = 0; i < 4; ++i) p[i] = pack_bf16(f[2 * i], f[2 * i + 1]);
  return v;
}

// KT = compile-time top-k (1, 2, 4, 8) so the per-token index/weight arrays stay in
// registers and the j loops unroll; KT = 0 is the generic runtime-k version.
#define DM_KT_ARRAY (KT ? KT : DM_MAX_TOPK)
constexpr int DM_TOK_MAX_THREADS = 896;   // 28 warps: <= 73 registers per thread

// y[t] = sum_j w[t,j] * y_perm[row_map[t,j]]
template <int KT>
__global__ void __launch_bounds__(DM_TOK_MAX_THREADS)
combine_fwd_kernel(const __nv_bfloat16* __restrict__ y_perm, const int32_t* __restrict__ row_map,
                   const float* __restrict__ w, int T, int H, int k_rt, const __nv_bfloat16* __restrict__ resid,
                   __nv_bfloat16* __restrict__ y) {
  const int k = KT ? KT : k_rt;
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  const int nwarps = (gridDim.x * blockDim.x) >> 5;
  const int nvec = H >> 3;
  for (int t = warp; t < T; t += nwarps) {
    int pos[DM_KT_ARRAY];
    float wt[DM_KT_ARRAY];
#pragma unroll
    for (int j = 0; j < k; ++j) { pos[j] = row_map[(size_t)t * k + j]; wt[j] = w[(size_t)t * k + j]; }
    if constexpr (KT > 0) {
      // U chunks per lane: every gather of the batch is issued before the first store (a
      // store's memory clobber would otherwise hold the next chunk's loads behind it, leaving
      // one chunk in flight per lane)
      constexpr int U = KT >= 8 ? 1 : 8 / KT;
      for (int c0 = lane; c0 < nvec; c0 += 32 * U) {
        int4 v[U][KT], rv[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int ch = c0 + 32 * u;
          const bool ok = ch < nvec;
#pragma unroll
          for (int j = 0; j < KT; ++j)
            v[u][j] = ok ? ld_nc_v4(y_perm + (size_t)pos[j] * H + ch * 8) : make_int4(0, 0, 0, 0);
          rv[u] = ok && resid ? ld_nc_v4(resid + (size_t)t * H + ch * 8) : make_int4(0, 0, 0, 0);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int ch = c0 + 32 * u;
          if (ch >= nvec) break;
          float acc[8];
          if (resid) {
            unpack8(rv[u], acc);
          } else {
#pragma unroll
            for (int i = 0; i < 8; ++i) acc[i] = 0.0f;
          }
#pragma unroll
          for (int j = 0; j < KT; ++j) {
            float f[8];
            unpack8(v[u][j], f);
#pragma unroll
            for (int i = 0; i < 8; ++i) acc[i] = __fmaf_rn(wt[j], f[i], acc[i]);
          }
          st_v4(y + (size_t)t * H + ch * 8, pack8(acc));
        }
      }
    } else {
      for (int ch = lane; ch < nvec; ch += 32) {
        float acc[8];
        if (resid) {
          unpack8(ld_nc_v4(resid + (size_t)t * H + ch * 8), acc);
        } else {
#pragma unroll
          for (int i = 0; i < 8; ++i) acc[i] = 0.0f;
        }
        for (int j = 0; j < k; ++j) {
          float f[8];
          unpack8(ld_nc_v4(y_perm + (size_t)pos[j] * H + ch * 8), f);
#pragma unroll
          for (int i = 0; i < 8; ++i) acc[i] = __fmaf_rn(wt[j], f[i], acc[i]);
        }
        st_v4(y + (size_t)t * H + ch * 8, pack8(acc));
      }
    }
  }
}

// dy_perm[row_map[t,j]] = w[t,j] * dy[t];  dw[t,j] = <dy[t], y_perm[row_map[t,j]]>;
// dlogit[t,j] = w_j * (dw_j - sum_i w_i dw_i)   (softmax over the selected logits).
template <int KT>
__global__ void __launch_bounds__(DM_TOK_MAX_THREADS)
combine_bwd_kernel(const __nv_bfloat16* __restrict__ dy, const __nv_bfloat16* __restrict__ y_perm,
                   const int32_t* __restrict__ row_map, const float* __restrict__ w,
                   const int32_t* __restrict__ counts, const int32_t* __restrict__ pad_off,
                   int T, int H, int E, int k_rt, __nv_bfloat16* __restrict__ dy_perm,
                   float* __restrict__ dw, float* __restrict__ dlogit, float* __restrict__ dl_perm) {
  const int k = KT ? KT : k_rt;
  const int gwarp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  const int nwarps = (gridDim.x * blockDim.x) >> 5;
  const int nvec = H >> 3;
  for (int t = gwarp; t < T; t += nwarps) {
    int pos[DM_KT_ARRAY];
    float wt[DM_KT_ARRAY], part[DM_KT_ARRAY];
#pragma unroll
    for (int j = 0; j < k; ++j) {
      pos[j] = row_map[(size_t)t * k + j];
      wt[j] = w[(size_t)t * k + j];
      part[j] = 0.0f;
    }
#pragma unroll 4
    for (int ch = lane; ch < nvec; ch += 32) {
      float g[8];
      unpack8(ld_nc_v4(dy + (size_t)t * H + ch * 8), g);
#pragma unroll
      for (int j = 0; j < k; ++j) {
        float f[8], o[8];
        unpack8(ld_nc_v4(y_perm + (size_t)pos[j] * H + ch * 8), f);
        float p = part[j];
#pragma unroll
        for (int i = 0; i < 8; ++i) { p = __fmaf_rn(g[i], f[i], p); o[i] = wt[j] * g[i]; }
        part[j] = p;
        st_v4(dy_perm + (size_t)pos[j] * H + ch * 8, pack8(o));
      }
    }
    float s = 0.0f;
#pragma unroll
    for (int j = 0; j < k; ++j) {
      part[j] = warp_sum_butterfly(part[j]);
      s = __fmaf_rn(wt[j], part[j], s);
    }
    if (lane == 0) {
#pragma unroll
      for (int j = 0; j < k; ++j) {
        dw[(size_t)t * k + j] = part[j];
        dlogit[(size_t)t * k + j] = wt[j] * (part[j] - s);
        if (dl_perm) dl_perm[pos[j]] = wt[j] * (part[j] - s);
      }
    }
  }
  // zero padding rows of dy_perm so the ragged-K wgrad sees exact zeros
  zero_padding_rows(dy_perm, H, counts, pad_off, E, gwarp, nwarps, lane, nullptr);
}

// dx[t] = sum_j dx_perm[row_map[t,j]] + sum_j dlogit[t,j] * W_g[idx[t,j], :]
template <int KT>
__global__ void __launch_bounds__(DM_TOK_MAX_THREADS)
permute_bwd_kernel(const __nv_bfloat16* __restrict__ dx_perm, const int32_t* __restrict__ row_map,
                   const int32_t* __restrict__ idx, const float* __restrict__ dlogit,
                   const float* __restrict__ wg, int T, int H, int k_rt, const __nv_bfloat16* __restrict__ resid,
                   __nv_bfloat16* __restrict__ dx) {
  const int k = KT ? KT : k_rt;
  const int gwarp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  const int nwarps = (gridDim.x * blockDim.x) >> 5;
  const int nvec = H >> 3;
  for (int t = gwarp; t < T; t += nwarps) {
    int pos[DM_KT_ARRAY], ex[DM_KT_ARRAY];
    float dl[DM_KT_ARRAY];
#pragma unroll
    for (int j = 0; j < k; ++j) {
      pos[j] = row_map[(size_t)t * k + j];
      ex[j] = idx[(size_t)t * k + j];
      dl[j] = dlogit ? dlogit[(size_t)t * k + j] : 0.0f;
    }
#pragma unroll 4
    for (int ch = lane; ch < nvec; ch += 32) {
      float acc[8];
      if (resid) {
        unpack8(ld_nc_v4(resid + (size_t)t * H + ch * 8), acc);
      } else {
#pragma unroll
        for (int i = 0; i < 8; ++i) acc[i] = 0.0f;
      }
#pragma unroll
      for (int j = 0; j < k; ++j) {
        float f[8];
        unpack8(ld_nc_v4(dx_perm + (size_t)pos[j] * H + ch * 8), f);
#pragma unroll
        for (int i = 0; i < 8; ++i) acc[i] += f[i];
      }
      if (dlogit) {
#pragma unroll
        for (int j = 0; j < k; ++j) {
          const float4* wr = reinterpret_cast<const float4*>(wg + (size_t)ex[j] * H + ch * 8);
          const float4 a = wr[0], b = wr[1];
          acc[0] = __fmaf_rn(dl[j], a.x, acc[0]); acc[1] = __fmaf_rn(dl[j], a.y, acc[1]);
          acc[2] = __fmaf_rn(dl[j], a.z, acc[2]); acc[3] = __fmaf_rn(dl[j], a.w, acc[3]);
          acc[4] = __fmaf_rn(dl[j], b.x, acc[4]); acc[5] = __fmaf_rn(dl[j], b.y, acc[5]);
          acc[6] = __fmaf_rn(dl[j], b.z, acc[6]); acc[7] = __fmaf_rn(dl[j], b.w, acc[7]);
        }
      }
      st_v4(dx + (size_t)t * H + ch * 8, pack8(acc));
    }
  }
}

// Permute backward for small E: CTA = 8 warps sharing one 256-column chunk whose
// W_g columns ([E][256] fp32, <= 16 KB) sit in smem, so the router dx term
// sum_j dlogit[t,j] * W_g[idx[t,j], :] reads only the k selected rows from smem (the
// per-token W_g reads of the generic kernel were L1-bound; holding all E rows in
// registers cost 64-128 registers and capped occupancy at 25%). Warps stride over
// groups of PBWD_TG tokens; the grid fills the resident CTA slots in one wave.
constexpr int PBWD_TG = 4;
constexpr int PBWD_MAX_E = 16;

template <int KT>
__global__ void __launch_bounds__(256)
permute_bwd_smem_kernel(const __nv_bfloat16* __restrict__ dx_perm, const int32_t* __restrict__ row_map,
                        const int32_t* __restrict__ idx, const float* __restrict__ dlogit,
                        const float* __restrict__ wg, int T, int H, int E, int k_rt,
                        const __nv_bfloat16* __restrict__ resid, __nv_bfloat16* __restrict__ dx) {
  const int k = KT ? KT : k_rt;
  __shared__ float4 ws[PBWD_MAX_E * 64];   // [e][256 columns] as float4
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int col0 = blockIdx.x * 256;
  if (dlogit) {
    for (int i = threadIdx.x; i < E * 64; i += blockDim.x) {
      const int e = i >> 6, c4 = i & 63;
      ws[i] = (col0 + c4 * 4 < H) ? reinterpret_cast<const float4*>(wg + (size_t)e * H + col0)[c4]
                                  : make_float4(0.f, 0.f, 0.f, 0.f);
    }
    __syncthreads();
  }
  const int col = col0 + lane * 8;
  if (col >= H) return;
  const int nw = gridDim.y * 8;
  constexpr int KK = KT ? KT : 1;   // staged gathers per token (runtime k falls back to a loop)
  // a group's indices (row_map, idx, dlogit) are loaded one group ahead, so its row gathers
  // issue without waiting for them
  int npos[PBWD_TG][KK], nex[PBWD_TG][KK];
  float ndl[PBWD_TG][KK];
  auto load_idx = [&](int g0) {
#pragma unroll
    for (int u = 0; u < PBWD_TG; ++u) {
      const int t = min(g0 + u, T - 1);
#pragma unroll
      for (int j = 0; j < KK; ++j) {
        npos[u][j] = KT ? row_map[(size_t)t * k + j] : 0;
        nex[u][j] = KT && dlogit ? idx[(size_t)t * k + j] : 0;
        ndl[u][j] = KT && dlogit ? dlogit[(size_t)t * k + j] : 0.0f;
      }
    }
  };
  const int t_first = (blockIdx.y * 8 + warp) * PBWD_TG;
  if (t_first < T) load_idx(t_first);
  for (int t0 = t_first; t0 < T; t0 += nw * PBWD_TG) {
    // stage 1: all TG * k row gathers of this group in flight at once, then the next group's
    // indices (before this group's stores, whose memory clobber would hold them back)
    int pos[PBWD_TG][KK], ex[PBWD_TG][KK];
    float dlv[PBWD_TG][KK];
    int4 v[PBWD_TG][KK];
    int4 rv[PBWD_TG];
#pragma unroll
    for (int u = 0; u < PBWD_TG; ++u)
#pragma unroll
      for (int j = 0; j < KK; ++j) { pos[u][j] = npos[u][j]; ex[u][j] = nex[u][j]; dlv[u][j] = ndl[u][j]; }
#pragma unroll
    for (int u = 0; u < PBWD_TG; ++u) {
      const int t = min(t0 + u, T - 1);
      rv[u] = resid ? ld_nc_v4(resid + (size_t)t * H + col) : make_int4(0, 0, 0, 0);
#pragma unroll
      for (int j = 0; j < KK; ++j) v[u][j] = KT ? ld_nc_v4(dx_perm + (size_t)pos[u][j] * H + col) : make_int4(0, 0, 0, 0);
    }
    if (t0 + nw * PBWD_TG < T) load_idx(t0 + nw * PBWD_TG);
#pragma unroll
    for (int u = 0; u < PBWD_TG; ++u) {
      const int t = t0 + u;
      if (t >= T) break;
      float acc[8];
      unpack8(rv[u], acc);
      if (KT) {
#pragma unroll
        for (int j = 0; j < KK; ++j) {
          float f[8];
          unpack8(v[u][j], f);
#pragma unroll
          for (int i = 0; i < 8; ++i) acc[i] += f[i];
        }
      } else {
        for (int j = 0; j < k; ++j) {
          float f[8];
          unpack8(ld_nc_v4(dx_perm + (size_t)row_map[(size_t)t * k + j] * H + col), f);
#pragma unroll
          for (int i = 0; i < 8; ++i) acc[i] += f[i];
        }
      }
      if (dlogit) {
        for (int j = 0; j < k; ++j) {
          const int e = KT ? ex[u][KT ? j : 0] : idx[(size_t)t * k + j];
          const float dl = KT ? dlv[u][KT ? j : 0] : dlogit[(size_t)t * k + j];
          const float4 a = ws[e * 64 + lane * 2], b = ws[e * 64 + lane * 2 + 1];
          acc[0] = __fmaf_rn(dl, a.x, acc[0]); acc[1] = __fmaf_rn(dl, a.y, acc[1]);
          acc[2] = __fmaf_rn(dl, a.z, acc[2]); acc[3] = __fmaf_rn(dl, a.w, acc[3]);
          acc[4] = __fmaf_rn(dl, b.x, acc[4]); acc[5] = __fmaf_rn(dl, b.y, acc[5]);
          acc[6] = __fmaf_rn(dl, b.z, acc[6]); acc[7] = __fmaf_rn(dl, b.w, acc[7]);
        }
      }
      st_v4(dx + (size_t)t * H + col, pack8(acc));
    }
  }
}

// Router weight gradient (E <= 16): CTA per (256-column chunk, token block); lane owns 8
// columns and keeps acc[E][8] in registers; every x row is read once (the expert-sorted
// variant gathers it k times). The NW warps take interleaved tokens of the block with
// RWR_DEPTH tokens of x / idx / dlogit in flight per warp (the previous loop kept one),
// are reduced through smem in fixed warp order, and the CTA partial goes to
// partial[tb][E][H]; the last token-block CTA of each column chunk to finish (ticket in
// the workspace) sums the partials in token-block order (+ beta * dW_g) — deterministic,
// one launch. gw[e] = dlogit[t,j] when idx[t,j] == e (each expert at most once per token).
constexpr int RWR_DEPTH = 8;
constexpr int RWR_MAX_TB = 512;   // token-block size bound (its idx / dlogit are staged in smem)

template <int EM, int KT>
__global__ void __launch_bounds__(EM == 8 ? 256 : 128, 2)
router_wgrad_reg_kernel(const __nv_bfloat16* __restrict__ x, const int32_t* __restrict__ idx,
                        const float* __restrict__ dlogit, int T, int H, int E, int k_rt, int tb_tokens,
                        float* __restrict__ partial, unsigned* __restrict__ tickets, float* __restrict__ dwg,
                        float beta) {
  constexpr int NW = EM == 8 ? 8 : 4;
  extern __shared__ float red[];   // [NW][EM][8][32], then the block's idx / dlogit
  __shared__ int s_last;
  const int k = KT ? KT : k_rt;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int col = (blockIdx.x * 32 + lane) * 8;
  const bool live = col < H;
  const int tb = blockIdx.y;
  const int t_beg = tb * tb_tokens, t_end = min(T, t_beg + tb_tokens);
  // ring of RWR_DEPTH prefetched x vectors (tokens warp, warp+NW, ...), issued before the
  // idx / dlogit staging so the two load latencies overlap
  int4 xv[RWR_DEPTH];
#pragma unroll
  for (int d = 0; d < RWR_DEPTH; ++d) {
    const int t = t_beg + warp + d * NW;
    xv[d] = live && t < t_end ? ld_nc_v4(x + (size_t)t * H + col) : make_int4(0, 0, 0, 0);
  }
  // the token block's expert ids and dlogits: one coalesced pass into smem
  int* s_idx = reinterpret_cast<int*>(red + NW * EM * 8 * 32);
  float* s_dl = reinterpret_cast<float*>(s_idx + tb_tokens * k);
  for (int q = threadIdx.x; q < (t_end - t_beg) * k; q += blockDim.x) {
    s_idx[q] = idx[(size_t)t_beg * k + q];
    s_dl[q] = dlogit[(size_t)t_beg * k + q];
  }
  __syncthreads();
  float acc[EM][8];
#pragma unroll
  for (int e = 0; e < EM; ++e)
#pragma unroll
    for (int i = 0; i < 8; ++i) acc[e][i] = 0.0f;
  if (live) {
    for (int t0 = t_beg + warp; t0 < t_end; t0 += RWR_DEPTH * NW) {
#pragma unroll
      for (int d = 0; d < RWR_DEPTH; ++d) {
        const int t = t0 + d * NW;
        if (t >= t_end) break;
        float xf[8];
        unpack8(xv[d], xf);
        const int tn = t + RWR_DEPTH * NW;
        xv[d] = tn < t_end ? ld_nc_v4(x + (size_t)tn * H + col) : make_int4(0, 0, 0, 0);
        // E-wide select-and-FMA: branch-free (branching to the token's k rows measured 2.5x
        // slower — uniform branches and an instruction-cache-bound body)
        float gw[EM];
#pragma unroll
        for (int e = 0; e < EM; ++e) gw[e] = 0.0f;
        const int q0 = (t - t_beg) * k;
        for (int j = 0; j < k; ++j) {
          const int ej = s_idx[q0 + j];
          const float dl = s_dl[q0 + j];
#pragma unroll
          for (int e = 0; e < EM; ++e) gw[e] = (ej == e) ? dl : gw[e];
        }
#pragma unroll
        for (int e = 0; e < EM; ++e)
#pragma unroll
          for (int i = 0; i < 8; ++i) acc[e][i] = __fmaf_rn(gw[e], xf[i], acc[e][i]);
      }
    }
  }
#pragma unroll
  for (int e = 0; e < EM; ++e)
#pragma unroll
    for (int i = 0; i < 8; ++i) red[((warp * EM + e) * 8 + i) * 32 + lane] = acc[e][i];
  __syncthreads();
  // warp w finalises experts w, w+NW, ...: sum over warps 0..NW-1 in order
  for (int e = warp; e < E; e += NW) {
    float o[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      float v = 0.0f;
#pragma unroll
      for (int q = 0; q < NW; ++q) v += red[((q * EM + e) * 8 + i) * 32 + lane];
      o[i] = v;
    }
    if (live) {
      float4* dst = reinterpret_cast<float4*>(partial + ((size_t)tb * E + e) * H + col);
      dst[0] = make_float4(o[0], o[1], o[2], o[3]);
      dst[1] = make_float4(o[4], o[5], o[6], o[7]);
    }
  }
  if (!tickets) return;   // reduced by router_wgrad_reduce_kernel
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) s_last = atomicAdd(tickets + blockIdx.x, 1u) == gridDim.y - 1;
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  if (threadIdx.x == 0) tickets[blockIdx.x] = 0u;   // ready for the next launch
  if (!live) return;
  const int ntb = gridDim.y;
  for (int e = warp; e < E; e += NW) {   // token-block order: router_wgrad_reduce_kernel's sums
    float4 a = make_float4(0.f, 0.f, 0.f, 0.f), b = a;
#pragma unroll 8
    for (int q = 0; q < ntb; ++q) {
      const float4* p = reinterpret_cast<const float4*>(partial + ((size_t)q * E + e) * H + col);
      const float4 pa = __ldcg(p), pb = __ldcg(p + 1);
      a.x += pa.x; a.y += pa.y; a.z += pa.z; a.w += pa.w;
      b.x += pb.x; b.y += pb.y; b.z += pb.z; b.w += pb.w;
    }
    float4* o = reinterpret_cast<float4*>(dwg + (size_t)e * H + col);
    if (beta != 0.0f) {
      const float4 oa = o[0], ob = o[1];
      a.x += beta * oa.x; a.y += beta * oa.y; a.z += beta * oa.z; a.w += beta * oa.w;
      b.x += beta * ob.x; b.y += beta * ob.y; b.z += beta * ob.z; b.w += beta * ob.w;
    }
    o[0] = a;
    o[1] = b;
  }
}

// Router weight gradient, stage 1 (any E): thread per column, accumulators in smem.
__global__ void router_wgrad_partial_kernel(const __nv_bfloat16* __restrict__ x,
                                            const int32_t* __restrict__ idx,
                                            const float* __restrict__ dlogit, int T, int H, int E,
                                            int k, int tb_tokens, float* __restrict__ partial) {
  extern __shared__ float s_acc[];  // [E][blockDim.x]
  const int cw = blockDim.x;
  const int h = blockIdx.x * cw + threadIdx.x;
  const int tb = blockIdx.y;
  const int t_beg = tb * tb_tokens, t_end = min(T, t_beg + tb_tokens);
  for (int e = 0; e < E; ++e) s_acc[e * cw + threadIdx.x] = 0.0f;
  if (h < H) {
    for (int t = t_beg; t < t_end; ++t) {
      const float xv = __bfloat162float(x[(size_t)t * H + h]);
      for (int j = 0; j < k; ++j) {
        const int e = idx[(size_t)t * k + j];
        float* a = &s_acc[e * cw + threadIdx.x];
        *a = __fmaf_rn(dlogit[(size_t)t * k + j], xv, *a);
      }
    }
    for (int e = 0; e < E; ++e) partial[((size_t)tb * E + e) * H + h] = s_acc[e * cw + threadIdx.x];
  }
}

__global__ void router_wgrad_reduce_kernel(const float* __restrict__ partial, int ntb, size_t EH,
                                           float* __restrict__ dwg, float beta) {
  for (size_t i = ((size_t)blockIdx.x * blockDim.x + threadIdx.x) * 4; i < EH;
       i += (size_t)gridDim.x * blockDim.x * 4) {
    float4 s = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll 8
    for (int tb = 0; tb < ntb; ++tb) {
      const float4 v = *reinterpret_cast<const float4*>(partial + (size_t)tb * EH + i);
      s.x += v.x; s.y += v.y; s.z += v.z; s.w += v.w;
    }
    float4* o = reinterpret_cast<float4*>(dwg + i);
    if (beta != 0.0f) {
      const float4 old = *o;
      s.x += beta * old.x; s.y += beta * old.y; s.z += beta * old.z; s.w += beta * old.w;
    }
    *o = s;
  }
}

// Router weight gradient over the expert-sorted rows: the rows of expert e in the
// permuted layout are exactly the (t, j) slots with idx == e in ascending t, so
// dW_g[e, :] = sum over the block of dl_perm[r] * x[src_token[r], :] (dl_perm =
// dlogit scattered to permuted positions by combine_bwd) — R*H FMAs instead of the
// T*E*H of a dense dlogit^T x. CTA per (1024-column chunk, expert, row segment): the
// segment's row indices and weights are staged in smem, then every thread keeps
// RWS_DEPTH x-row gathers (16 B each) in flight — the previous version walked
// src_token -> x dependent loads 8 rows at a time and was latency bound (0.19 of HBM).
// With nseg > 1 each segment writes a partial [seg][E][H]; the last segment CTA of its
// (chunk, expert) to finish (ticket counter in the workspace) sums the partials in
// segment order (+ beta * dW_g): deterministic, and no second launch.
constexpr int RWS_ROWS = 128;    // rows staged per batch
constexpr int RWS_DEPTH = 16;    // x gathers in flight per thread

__global__ void __launch_bounds__(128)
router_wgrad_sorted_kernel(const __nv_bfloat16* __restrict__ x, const int32_t* __restrict__ src_token,
                           const float* __restrict__ dl_perm, const int32_t* __restrict__ counts,
                           const int32_t* __restrict__ pad_off, int H, int E, int nseg, float* __restrict__ partial,
                           unsigned* __restrict__ tickets, float* __restrict__ dwg, float beta) {
  __shared__ int s_t[RWS_ROWS];
  __shared__ float s_d[RWS_ROWS];
  __shared__ int s_last;
  const int e = blockIdx.y, seg = blockIdx.z;
  const int col = (blockIdx.x * blockDim.x + threadIdx.x) * 8;
  const bool live = col < H;
  const int n = counts[e];
  const int r0 = pad_off[e] + (int)((long long)n * seg / nseg);
  const int r1 = pad_off[e] + (int)((long long)n * (seg + 1) / nseg);
  float acc[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) acc[i] = 0.0f;
  for (int rb = r0; rb < r1; rb += RWS_ROWS) {
    const int nr = min(RWS_ROWS, r1 - rb);
    __syncthreads();
    for (int i = threadIdx.x; i < nr; i += blockDim.x) { s_t[i] = src_token[rb + i]; s_d[i] = dl_perm[rb + i]; }
    __syncthreads();
    if (!live) continue;
    for (int i = 0; i < nr; i += RWS_DEPTH) {
      int4 v[RWS_DEPTH];
#pragma unroll
      for (int q = 0; q < RWS_DEPTH; ++q)
        v[q] = i + q < nr ? ld_nc_v4(x + (size_t)s_t[i + q] * H + col) : make_int4(0, 0, 0, 0);
#pragma unroll
      for (int q = 0; q < RWS_DEPTH; ++q) {
        if (i + q >= nr) break;
        const float d = s_d[i + q];
        float f[8];
        unpack8(v[q], f);
#pragma unroll
        for (int c = 0; c < 8; ++c) acc[c] = __fmaf_rn(d, f[c], acc[c]);
      }
    }
  }
  float4 a = make_float4(acc[0], acc[1], acc[2], acc[3]), b = make_float4(acc[4], acc[5], acc[6], acc[7]);
  if (nseg > 1) {
    if (live) {
      float4* o = reinterpret_cast<float4*>(partial + ((size_t)seg * E + e) * H + col);
      o[0] = a;
      o[1] = b;
    }
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) s_last = atomicAdd(tickets + (size_t)blockIdx.x * E + e, 1u) == (unsigned)nseg - 1;
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    if (threadIdx.x == 0) tickets[(size_t)blockIdx.x * E + e] = 0u;   // ready for the next launch
    if (!live) return;
    a = make_float4(0.f, 0.f, 0.f, 0.f);
    b = a;
#pragma unroll 8
    for (int s2 = 0; s2 < nseg; ++s2) {   // segment order: same sums as router_wgrad_reduce_kernel
      const float4* p = reinterpret_cast<const float4*>(partial + ((size_t)s2 * E + e) * H + col);
      const float4 pa = __ldcg(p), pb = __ldcg(p + 1);
      a.x += pa.x; a.y += pa.y; a.z += pa.z; a.w += pa.w;
      b.x += pb.x; b.y += pb.y; b.z += pb.z; b.w += pb.w;
    }
  }
  if (!live) return;
  float4* o = reinterpret_cast<float4*>(dwg + (size_t)e * H + col);
  if (beta != 0.0f) {
    const float4 oa = o[0], ob = o[1];
    a.x += beta * oa.x; a.y += beta * oa.y; a.z += beta * oa.z; a.w += beta * oa.w;
    b.x += beta * ob.x; b.y += beta * ob.y; b.z += beta * ob.z; b.w += beta * ob.w;
  }
  o[0] = a;
  o[1] = b;
}

// Warp-per-token launch shape: 8-warp CTAs over ceil(T/8) blocks, at most 8 per SM. (One
// CTA of ceil(T/#SM) warps per SM — exactly balanced — measured no faster: combine_fwd
// 22.4 -> 24.1 us, combine_bwd 36.4 -> 35.9 us.)
struct TokGrid {
  int blocks, threads;
};
static TokGrid token_grid(int T) {
  int blocks = (T + 7) / 8;
  const int cap = num_sms_current() * 8;
  return {blocks < cap ? blocks : cap, 256};
}

}  // namespace dm

using namespace dm;

extern "C" {

int dm_combine_fwd(const void* y_perm, const int32_t* row_map, const float* w, int T, int H, int k,
                   const void* resid, void* y, void* stream) {
  const TokGrid tg = token_grid(T);

  if (T < 1 || H % 8 || k < 1 || k > DM_MAX_TOPK) return set_error(DM_ERR_SHAPE, "combine_fwd bad shape");
  if (resid && resid == y) return set_error(DM_ERR_SHAPE, "combine_fwd: resid must not alias y");
  const __nv_bfloat16* yp = reinterpret_cast<const __nv_bfloat16*>(y_perm);
  const __nv_bfloat16* rs = reinterpret_cast<const __nv_bfloat16*>(resid);
  __nv_bfloat16* out = reinterpret_cast<__nv_bfloat16*>(y);
  cudaStream_t st = (cudaStream_t)stream;
  switch (k) {
    case 1: combine_fwd_kernel<1><<<tg.blocks, tg.threads, 0, st>>>(yp, row_map, w, T, H, k, rs, out); break;
    case 2: combine_fwd_kernel<2><<<tg.blocks, tg.threads, 0, st>>>(yp, row_map, w, T, H, k, rs, out); break;
    case 4: combine_fwd_kernel<4><<<tg.blocks, tg.threads, 0, st>>>(yp, row_map, w, T, H, k, rs, out); break;
    case 8: combine_fwd_kernel<8><<<tg.blocks, tg.threads, 0, st>>>(yp, row_map, w, T, H, k, rs, out); break;
    default: combine_fwd_kernel<0><<<tg.blocks, tg.threads, 0, st>>>(yp, row_map, w, T, H, k, rs, out); break;
  }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return set_cuda_error(e, "combine_fwd launch");
  note_launch();
  return DM_OK;
}

int dm_combine_bwd(const void* dy, const void* y_perm, const int32_t* row_map, const float* w,
                   const int32_t* counts, const int32_t* pad_off, int T, int H, int E, int k,
                   void* dy_perm, float* dw, float* dlogit, float* dl_perm, void* stream) {
  const TokGrid tg = token_grid(T);

  if (T < 1 || H % 8 || k < 1 || k > DM_MAX_TOPK || E < 1) return set_error(DM_ERR_SHAPE, "combine_bwd bad shape");
  switch (k) {
    case 1: combine_bwd_kernel<1><<<tg.blocks, tg.threads, 0, (cudaStream_t)stream>>>(reinterpret_cast<const __nv_bfloat16*>(dy), reinterpret_cast<const __nv_bfloat16*>(y_perm), row_map, w, counts, pad_off, T, H, E, k, reinterpret_cast<__nv_bfloat16*>(dy_perm), dw, dlogit, dl_perm); break;
    case 2: combine_bwd_kernel<2><<<tg.blocks, tg.threads, 0, (cudaStream_t)stream>>>(reinterpret_cast<const __nv_bfloat16*>(dy), reinterpret_cast<const __nv_bfloat16*>(y_perm), row_map, w, counts, pad_off, T, H, E, k, reinterpret_cast<__nv_bfloat16*>(dy_perm), dw, dlogit, dl_perm); break;
    case 4: combine_bwd_kernel<4><<<tg.blocks, tg.threads, 0, (cudaStream_t)stream>>>(reinterpret_cast<const __nv_bfloat16*>(dy), reinterpret_cast<const __nv_bfloat16*>(y_perm), row_map, w, counts, pad_off, T, H, E, k, reinterpret_cast<__nv_bfloat16*>(dy_perm), dw, dlogit, dl_perm); break;
    case 8: combine_bwd_kernel<8><<<tg.blocks, tg.threads, 0, (cudaStream_t)stream>>>(reinterpret_cast<const __nv_bfloat16*>(dy), reinterpret_cast<const __nv_bfloat16*>(y_perm), row_map, w, counts, pad_off, T, H, E, k, reinterpret_cast<__nv_bfloat16*>(dy_perm), dw, dlogit, dl_perm); break;
    default: combine_bwd_kernel<0><<<tg.blocks, tg.threads, 0, (cudaStream_t)stream>>>(reinterpret_cast<const __nv_bfloat16*>(dy), reinterpret_cast<const __nv_bfloat16*>(y_perm), row_map, w, counts, pad_off, T, H, E, k, reinterpret_cast<__nv_bfloat16*>(dy_perm), dw, dlogit, dl_perm); break;
  }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return set_cuda_error(e, "combine_bwd launch");
  note_launch();
  return DM_OK;
}

int dm_permute_bwd(const void* dx_perm, const int32_t* row_map, const int32_t* idx, const float* dlogit,
                   const float* wg, int T, int H, int E, int k, const void* resid, void* dx, void* stream) {
  const TokGrid tg = token_grid(T);

  if (T < 1 || H % 8 || k < 1 || k > DM_MAX_TOPK || E < 1) return set_error(DM_ERR_SHAPE, "permute_bwd bad shape");
  if (resid && resid == dx) return set_error(DM_ERR_SHAPE, "permute_bwd: resid must not alias dx");
  const __nv_bfloat16* rs = reinterpret_cast<const __nv_bfloat16*>(resid);
  cudaStream_t st = (cudaStream_t)stream;
  const __nv_bfloat16* dxp = reinterpret_cast<const __nv_bfloat16*>(dx_perm);
  __nv_bfloat16* out = reinterpret_cast<__nv_bfloat16*>(dx);
  if (E <= PBWD_MAX_E) {
    const int occ = max_active_blocks((const void*)permute_bwd_smem_kernel<2>, 256, 0);
    const int gx = (H + 255) / 256;
    // exactly one wave: floor, not ceil (ceil left a 3% second wave that doubled the tail)
    int gy = (occ > 0 ? occ : 2) * num_sms_current() / gx;
    if (gy < 1) gy = 1;
    const int groups = (T + 8 * PBWD_TG - 1) / (8 * PBWD_TG);
    if (gy > groups) gy = groups;
    dim3 grid(gx, gy);
#define DM_PBWD(KTV) permute_bwd_smem_kernel<KTV><<<grid, 256, 0, st>>>(dxp, row_map, idx, dlogit, wg, T, H, E, k, rs, out)
    switch (k) { case 1: DM_PBWD(1); break; case 2: DM_PBWD(2); break; case 4: DM_PBWD(4); break;
                 case 8: DM_PBWD(8); break; default: DM_PBWD(0); break; }
#undef DM_PBWD
  } else {
    switch (k) {
      case 1: permute_bwd_kernel<1><<<tg.blocks, tg.threads, 0, st>>>(dxp, row_map, idx, dlogit, wg, T, H, k, rs, out); break;
      case 2: permute_bwd_kernel<2><<<tg.blocks, tg.threads, 0, st>>>(dxp, row_map, idx, dlogit, wg, T, H, k, rs, out); break;
      case 4: permute_bwd_kernel<4><<<tg.blocks, tg.threads, 0, st>>>(dxp, row_map, idx, dlogit, wg, T, H, k, rs, out); break;
      case 8: permute_bwd_kernel<8><<<tg.blocks, tg.threads, 0, st>>>(dxp, row_map, idx, dlogit, wg, T, H, k, rs, out); break;
      default: permute_bwd_kernel<0><<<tg.blocks, tg.threads, 0, st>>>(dxp, row_map, idx, dlogit, wg, T, H, k, rs, out); break;
    }
  }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return set_cuda_error(e, "permute_bwd launch");
  note_launch();
  return DM_OK;
}

int dm_router_wgrad(const void* x, const int32_t* idx, const float* dlogit, int T, int H, int E,
                    int k, float* partial_ws, float* dwg, float beta, void* stream) {
  if (T < 1 || H % 8 || E < 1 || E > DM_MAX_EXPERTS || k < 1 || k > DM_MAX_TOPK)
    return set_error(DM_ERR_SHAPE, "router_wgrad bad shape");
  if (((size_t)E * H) % 4 || reinterpret_cast<uintptr_t>(dwg) & 15 || reinterpret_cast<uintptr_t>(partial_ws) & 15)
    return set_error(DM_ERR_ALIGN, "router_wgrad needs 16-byte aligned fp32 buffers");
  int tbt = dm_router_wgrad_token_block(E);
  int ntb = (T + tbt - 1) / tbt;   // the workspace holds this many partial blocks
  cudaStream_t st = (cudaStream_t)stream;
  if (E <= 16) {
    // segment tickets follow the partial blocks in the workspace (after the sorted kernel's)
    unsigned* tickets = reinterpret_cast<unsigned*>(reinterpret_cast<char*>(partial_ws) + (size_t)ntb * E * H * 4) +
                        (size_t)((H + 1023) / 1024) * E;
    // idx + dlogit of a token block (<= RWR_MAX_TB tokens) after the cross-warp reduction
    // buffer: sized for this k, so two CTAs fit per SM (the DM_MAX_TOPK-sized stage held the
    // kernel to one CTA of 8 warps per SM: latency bound)
    const size_t stage = (size_t)RWR_MAX_TB * k * 8;
    const size_t sm8 = 8 * 8 * 8 * 32 * 4 + stage, sm16 = 4 * 16 * 8 * 32 * 4 + stage;
    const void* k8 = (const void*)router_wgrad_reg_kernel<8, 2>;
    const void* k16 = (const void*)router_wgrad_reg_kernel<16, 2>;
    if (int rc = ensure_smem_attr(E <= 8 ? k8 : k16, (int)(E <= 8 ? sm8 : sm16), "cudaFuncSetAttribute(router_wgrad_reg)"))
      return rc;
    const int occ8 = E <= 8 ? max_active_blocks(k8, 256, sm8) : 1;
    const int occ16 = E <= 8 ? 1 : max_active_blocks(k16, 128, sm16);
    // One wave: as many token blocks as the resident CTA slots allow per column chunk
    // (never more than the workspace's ntb), each a contiguous run of tbt tokens.
    const int gx = (H / 8 + 31) / 32;
    const int slots = (E <= 8 ? occ8 : occ16) * num_sms_current();
    int want = slots / gx;
    if (want < 1) want = 1;
    if (want < ntb) {
      tbt = (T + want - 1) / want;
      tbt = (tbt + 7) & ~7;
      if (tbt > RWR_MAX_TB) tbt = RWR_MAX_TB;   // long sequences: more than one wave of blocks
      ntb = (T + tbt - 1) / tbt;
    }
    if (tbt > RWR_MAX_TB) return set_error(DM_ERR_SHAPE, "router_wgrad token block %d > %d", tbt, RWR_MAX_TB);
    dim3 grid(gx, ntb);
    const __nv_bfloat16* xb = reinterpret_cast<const __nv_bfloat16*>(x);
#define DM_RWR(EMV, KTV, NT, SM)                                                                              \
    do {                                                                                                    \
      if (int rc = ensure_smem_attr((const void*)router_wgrad_reg_kernel<EMV, KTV>, (int)SM,               \
                                    "cudaFuncSetAttribute(router_wgrad_reg)")) return rc;                  \
      router_wgrad_reg_kernel<EMV, KTV><<<grid, NT, SM, st>>>(xb, idx, dlogit, T, H, E, k, tbt, partial_ws, \
                                                              tickets, dwg, beta);                          \
    } while (0)
#define DM_RWR_K(EMV, NT, SM)                                                                \
    switch (k) { case 1: DM_RWR(EMV, 1, NT, SM); break; case 2: DM_RWR(EMV, 2, NT, SM); break;  \
                 case 4: DM_RWR(EMV, 4, NT, SM); break; case 8: DM_RWR(EMV, 8, NT, SM); break;  \
                 default: DM_RWR(EMV, 0, NT, SM); break; }
    if (E <= 8) { DM_RWR_K(8, 256, sm8); } else { DM_RWR_K(16, 128, sm16); }
#undef DM_RWR_K
#undef DM_RWR
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return set_cuda_error(e, "router_wgrad_reg launch");
    note_launch();
    return DM_OK;
  } else {
    int cw = 128;
    while (cw > 32 && (size_t)E * cw * sizeof(float) > 96 * 1024) cw >>= 1;
    const size_t smem = (size_t)E * cw * sizeof(float);
    if (int rc = ensure_smem_attr((const void*)router_wgrad_partial_kernel, 128 * 1024,
                                  "cudaFuncSetAttribute(router_wgrad)")) return rc;
    dim3 grid((H + cw - 1) / cw, ntb);
    router_wgrad_partial_kernel<<<grid, cw, smem, st>>>(reinterpret_cast<const __nv_bfloat16*>(x), idx, dlogit,
                                                       T, H, E, k, tbt, partial_ws);
  }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return set_cuda_error(e, "router_wgrad_partial launch");
  note_launch();
  const size_t EH = (size_t)E * H;
  int rblocks = (int)((EH / 4 + 255) / 256);
  if (rblocks > num_sms_current() * 4) rblocks = num_sms_current() * 4;
  router_wgrad_reduce_kernel<<<rblocks, 256, 0, st>>>(partial_ws, ntb, EH, dwg, beta);
  e = cudaGetLastError();
  if (e != cudaSuccess) return set_cuda_error(e, "router_wgrad_reduce launch");
  note_launch();
  return DM_OK;
}

int dm_router_wgrad_sorted(const void* x, const int32_t* src_token, const float* dl_perm, const int32_t* counts,
                           const int32_t* pad_off, int T, int H, int E, float* partial_ws, float* dwg, float beta,
                           void* stream) {
  if (T < 1 || H % 8 || E < 1 || E > DM_MAX_EXPERTS) return set_error(DM_ERR_SHAPE, "router_wgrad_sorted bad shape");
  if (reinterpret_cast<uintptr_t>(dwg) & 15 || reinterpret_cast<uintptr_t>(partial_ws) & 15)
    return set_error(DM_ERR_ALIGN, "dW_g / workspace must be 16-byte aligned");
  cudaStream_t st = (cudaStream_t)stream;
  const int gx = (H / 8 + 127) / 128;
  // enough row segments for ~4 CTAs per SM, bounded by the workspace's partial blocks
  int nseg = 1;
  if (partial_ws) {
    const int tbt = dm_router_wgrad_token_block(E);
    const int cap_seg = (T + tbt - 1) / tbt;
    nseg = (4 * num_sms_current() + gx * E - 1) / (gx * E);
    if (nseg > cap_seg) nseg = cap_seg;
    if (nseg < 1) nseg = 1;
  }
  dim3 grid(gx, E, nseg);
  // segment tickets follow the partial blocks in the workspace
  const int tbt = dm_router_wgrad_token_block(E);
  unsigned* tickets = partial_ws ? reinterpret_cast<unsigned*>(
      reinterpret_cast<char*>(partial_ws) + (size_t)((T + tbt - 1) / tbt) * E * H * 4) : nullptr;
  router_wgrad_sorted_kernel<<<grid, 128, 0, st>>>(reinterpret_cast<const __nv_bfloat16*>(x), src_token, dl_perm,
                                                   counts, pad_off, H, E, nseg, partial_ws, tickets, dwg, beta);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return set_cuda_error(e, "router_wgrad_sorted launch");
  note_launch();
  return DM_OK;
}

}  // extern "C"
