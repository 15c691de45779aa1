// fp32 mode (experiment bytes_per_element = 4; reference config.py ModelConfig):
// activations, gradients and master weights in fp32 with 1e-4 parity, still on the
// tcgen05 tensor cores. Every fp32 GEMM operand v is split into two bf16 terms,
// v = hi + lo (hi = bf16(v), lo = bf16(v - hi), |v - hi - lo| <= 2^-18 |v|), and a
// product is taken as a.b ~= a_hi.b_hi + a_hi.b_lo + a_lo.b_hi (the dropped
// a_lo.b_lo is ~2^-16 relative). The three terms are ONE bf16 GEMM with a 3x
// longer reduction: activations are stored "split-3" as [hi | hi | lo] along K and
// weights as [hi | lo | hi] (K-major) or stacked [hi; lo; hi] rows (MN-major), so
// A3 . B3 sums exactly those three products in the fp32 TMEM accumulator.
//
// This file holds the fp32-mode A-side kernels (router on fp32 x in the canonical
// order, permute into split-3 rows, combine / combine-bwd / permute-bwd / router
// wgrad on fp32), the SwiGLU elementwise stages between the GEMMs, and the split
// kernel. The GEMMs are dm_grouped_gemm_f32 (grouped_gemm_sm100.cu).
#include "dm_common.cuh"
#include "dm_internal.h"

namespace dm {

__device__ __forceinline__ void split_bf16(float v, __nv_bfloat16& hi, __nv_bfloat16& lo) {
  hi = __float2bfloat16_rn(v);
  lo = __float2bfloat16_rn(v - __bfloat162float(hi));
}

// 8 consecutive fp32 values -> hi and lo int4 (8 bf16 each).
__device__ __forceinline__ void split8(const float (&f)[8], int4& hi, int4& lo) {
  uint32_t* h = reinterpret_cast<uint32_t*>(&hi);
  uint32_t* l = reinterpret_cast<uint32_t*>(&lo);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    __nv_bfloat16 h0, l0, h1, l1;
    split_bf16(f[2 * i], h0, l0);
    split_bf16(f[2 * i + 1], h1, l1);
    h[i] = (uint32_t)__bfloat16_as_ushort(h0) | ((uint32_t)__bfloat16_as_ushort(h1) << 16);
    l[i] = (uint32_t)__bfloat16_as_ushort(l0) | ((uint32_t)__bfloat16_as_ushort(l1) << 16);
  }
}

__device__ __forceinline__ void ld8(const float* p, float (&f)[8]) {
  const float4 a = __ldg(reinterpret_cast<const float4*>(p));
  const float4 b = __ldg(reinterpret_cast<const float4*>(p) + 1);
  f[0] = a.x; f[1] = a.y; f[2] = a.z; f[3] = a.w; f[4] = b.x; f[5] = b.y; f[6] = b.z; f[7] = b.w;
}

__device__ __forceinline__ void st8(float* p, const float (&f)[8]) {
  reinterpret_cast<float4*>(p)[0] = make_float4(f[0], f[1], f[2], f[3]);
  reinterpret_cast<float4*>(p)[1] = make_float4(f[4], f[5], f[6], f[7]);
}

// Split-3 activation row chunk: columns [c, c+8) of [hi | hi | lo] (row width 3K).
__device__ __forceinline__ void st_split3_act(__nv_bfloat16* row, int K, int c, const float (&f)[8]) {
  int4 hi, lo;
  split8(f, hi, lo);
  st_v4(row + c, hi);
  st_v4(row + K + c, hi);
  st_v4(row + 2 * K + c, lo);
}

// ------------------------------------------------------------------ router
// logits = x . W_g^T for fp32 x in the canonical order of dispatch.cu (lane p owns
// the 8-element chunks c = p mod 32, even/odd element chains, xor butterfly).
// Warp per token, W_g rows of an expert block staged in smem.
constexpr int RF_WARPS = 8;
constexpr int RF_EB = 8;    // experts per register block (each x chunk is loaded once per block)

__global__ void __launch_bounds__(RF_WARPS * 32)
router_logits_f32_kernel(const float* __restrict__ x, const float* __restrict__ wg, float* __restrict__ logits,
                         int T, int H, int E, int ec) {
  extern __shared__ float4 rf_sw4[];
  const float* sw = reinterpret_cast<const float*>(rf_sw4);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nch = H >> 3;
  for (int e0 = 0; e0 < E; e0 += ec) {
    const int ecur = min(ec, E - e0);
    __syncthreads();
    const float4* src = reinterpret_cast<const float4*>(wg + (size_t)e0 * H);
    for (int i = threadIdx.x; i < ecur * H / 4; i += blockDim.x) rf_sw4[i] = src[i];
    __syncthreads();
    for (int t = blockIdx.x * RF_WARPS + warp; t < T; t += gridDim.x * RF_WARPS) {
      const float* xr = x + (size_t)t * H;
      for (int eb = 0; eb < ecur; eb += RF_EB) {
        float2 acc[RF_EB];
#pragma unroll
        for (int e = 0; e < RF_EB; ++e) acc[e] = make_float2(0.f, 0.f);
        for (int c = lane; c < nch; c += 32) {
          float xv[8];
          ld8(xr + c * 8, xv);
#pragma unroll
          for (int e = 0; e < RF_EB; ++e) {
            if (eb + e < ecur) {
              const float* wr = sw + (size_t)(eb + e) * H + c * 8;
#pragma unroll
              for (int i = 0; i < 4; ++i) acc[e] = ffma2(make_float2(xv[2 * i], xv[2 * i + 1]),
                                                          make_float2(wr[2 * i], wr[2 * i + 1]), acc[e]);
            }
          }
        }
#pragma unroll
        for (int e = 0; e < RF_EB; ++e) {
          const float v = warp_sum_butterfly(__fadd_rn(acc[e].x, acc[e].y));
          if (lane == 0 && eb + e < ecur) logits[(size_t)t * E + e0 + eb + e] = v;
        }
      }
    }
  }
}

// ------------------------------------------------------------------ permute
// x (fp32 [T,H]) -> x3 (bf16 split-3 rows [cap, 3H]) at the stable counting-sort
// positions; padding rows zeroed, src_token -1 (same contract as dm_permute).
__global__ void __launch_bounds__(256)
permute_f32_kernel(const float* __restrict__ x, const int32_t* __restrict__ idx, const int32_t* __restrict__ rank,
                   const int32_t* __restrict__ chunk_base, const int32_t* __restrict__ counts,
                   const int32_t* __restrict__ pad_off, int T, int H, int E, int k, int32_t* __restrict__ row_map,
                   int32_t* __restrict__ src_token, __nv_bfloat16* __restrict__ x3) {
  const int gwarp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  const int nwarps = (gridDim.x * blockDim.x) >> 5;
  const int nvec = H >> 3;
  for (int t = gwarp; t < T; t += nwarps) {
    const int c = t / DM_CHUNK_TOKENS;
    int p[DM_MAX_TOPK];
    for (int j = 0; j < k; ++j) p[j] = chunk_base[(size_t)c * E + idx[(size_t)t * k + j]] + rank[(size_t)t * k + j];
    if (lane < k) {
      int pj = p[0];
      for (int j = 1; j < k; ++j) pj = (lane == j) ? p[j] : pj;
      row_map[(size_t)t * k + lane] = pj;
      src_token[pj] = t;
    }
    for (int ch = lane; ch < nvec; ch += 32) {
      float f[8];
      ld8(x + (size_t)t * H + ch * 8, f);
      int4 hi, lo;
      split8(f, hi, lo);
      for (int j = 0; j < k; ++j) {
        __nv_bfloat16* row = x3 + (size_t)p[j] * 3 * H;
        st_v4(row + ch * 8, hi);
        st_v4(row + H + ch * 8, hi);
        st_v4(row + 2 * H + ch * 8, lo);
      }
    }
  }
  zero_padding_rows(x3, 3 * H, counts, pad_off, E, gwarp, nwarps, lane, src_token);
}

// ------------------------------------------------------------------ combine
// y[t] = resid[t] + sum_j w[t,j] * y_perm[row_map[t,j]]   (fp32 in / out)
__global__ void __launch_bounds__(256)
combine_fwd_f32_kernel(const float* __restrict__ y_perm, const int32_t* __restrict__ row_map,
                       const float* __restrict__ w, int T, int H, int k, const float* __restrict__ resid,
                       float* __restrict__ y) {
  const int gwarp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  const int nwarps = (gridDim.x * blockDim.x) >> 5;
  const int nvec = H >> 3;
  for (int t = gwarp; t < T; t += nwarps) {
    for (int ch = lane; ch < nvec; ch += 32) {
      float acc[8];
      if (resid) {
        ld8(resid + (size_t)t * H + ch * 8, acc);
      } else {
#pragma unroll
        for (int i = 0; i < 8; ++i) acc[i] = 0.0f;
      }
      for (int j = 0; j < k; ++j) {
        const float wt = w[(size_t)t * k + j];
        float f[8];
        ld8(y_perm + (size_t)row_map[(size_t)t * k + j] * H + ch * 8, f);
#pragma unroll
        for (int i = 0; i < 8; ++i) acc[i] = __fmaf_rn(wt, f[i], acc[i]);
      }
      st8(y + (size_t)t * H + ch * 8, acc);
    }
  }
}

// dy3[row_map[t,j]] = split-3(w[t,j] * dy[t]); dw[t,j] = <dy[t], y_perm[row_map[t,j]]>;
// dlogit[t,j] = w_j (dw_j - sum_i w_i dw_i); dl_perm[row_map[t,j]] = dlogit[t,j].
__global__ void __launch_bounds__(256)
combine_bwd_f32_kernel(const float* __restrict__ dy, const float* __restrict__ y_perm,
                       const int32_t* __restrict__ row_map, const float* __restrict__ w,
                       const int32_t* __restrict__ counts, const int32_t* __restrict__ pad_off, int T, int H,
                       int E, int k, __nv_bfloat16* __restrict__ dy3, float* __restrict__ dw,
                       float* __restrict__ dlogit, float* __restrict__ dl_perm) {
  const int gwarp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  const int nwarps = (gridDim.x * blockDim.x) >> 5;
  const int nvec = H >> 3;
  for (int t = gwarp; t < T; t += nwarps) {
    int pos[DM_MAX_TOPK];
    float wt[DM_MAX_TOPK], part[DM_MAX_TOPK];
    for (int j = 0; j < k; ++j) {
      pos[j] = row_map[(size_t)t * k + j];
      wt[j] = w[(size_t)t * k + j];
      part[j] = 0.0f;
    }
    for (int ch = lane; ch < nvec; ch += 32) {
      float g[8];
      ld8(dy + (size_t)t * H + ch * 8, g);
      for (int j = 0; j < k; ++j) {
        float f[8], s[8];
        ld8(y_perm + (size_t)pos[j] * H + ch * 8, f);
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          part[j] = __fmaf_rn(g[i], f[i], part[j]);
          s[i] = wt[j] * g[i];
        }
        st_split3_act(dy3 + (size_t)pos[j] * 3 * H, H, ch * 8, s);
      }
    }
    for (int j = 0; j < k; ++j) part[j] = warp_sum_butterfly(part[j]);
    if (lane == 0) {
      float sum = 0.0f;
      for (int j = 0; j < k; ++j) sum = __fmaf_rn(wt[j], part[j], sum);
      for (int j = 0; j < k; ++j) {
        const float dl = wt[j] * (part[j] - sum);
        dw[(size_t)t * k + j] = part[j];
        dlogit[(size_t)t * k + j] = dl;
        if (dl_perm) dl_perm[pos[j]] = dl;
      }
    }
  }
  zero_padding_rows(dy3, 3 * H, counts, pad_off, E, gwarp, nwarps, lane, nullptr);
}

// dx[t] = resid[t] + sum_j dx_perm[row_map[t,j]] + sum_j dlogit[t,j] * W_g[idx[t,j]]
__global__ void __launch_bounds__(256)
permute_bwd_f32_kernel(const float* __restrict__ dx_perm, const int32_t* __restrict__ row_map,
                       const int32_t* __restrict__ idx, const float* __restrict__ dlogit,
                       const float* __restrict__ wg, int T, int H, int k, const float* __restrict__ resid,
                       float* __restrict__ dx) {
  const int gwarp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  const int nwarps = (gridDim.x * blockDim.x) >> 5;
  const int nvec = H >> 3;
  for (int t = gwarp; t < T; t += nwarps) {
    for (int ch = lane; ch < nvec; ch += 32) {
      float acc[8];
      if (resid) {
        ld8(resid + (size_t)t * H + ch * 8, acc);
      } else {
#pragma unroll
        for (int i = 0; i < 8; ++i) acc[i] = 0.0f;
      }
      for (int j = 0; j < k; ++j) {
        float f[8];
        ld8(dx_perm + (size_t)row_map[(size_t)t * k + j] * H + ch * 8, f);
#pragma unroll
        for (int i = 0; i < 8; ++i) acc[i] += f[i];
      }
      if (dlogit) {
        for (int j = 0; j < k; ++j) {
          const float dl = dlogit[(size_t)t * k + j];
          float f[8];
          ld8(wg + (size_t)idx[(size_t)t * k + j] * H + ch * 8, f);
#pragma unroll
          for (int i = 0; i < 8; ++i) acc[i] = __fmaf_rn(dl, f[i], acc[i]);
        }
      }
      st8(dx + (size_t)t * H + ch * 8, acc);
    }
  }
}

// dW_g[e,:] = sum over expert e's permuted rows r (ascending) of dl_perm[r] * x[src_token[r], :];
// with nseg > 1 each (expert, row segment) writes a partial reduced in segment order by
// router_wgrad_reduce_f32_kernel (deterministic), as in combine.cu's bf16 version.
__global__ void __launch_bounds__(128)
router_wgrad_sorted_f32_kernel(const float* __restrict__ x, const int32_t* __restrict__ src_token,
                               const float* __restrict__ dl_perm, const int32_t* __restrict__ counts,
                               const int32_t* __restrict__ pad_off, int H, int E, int nseg,
                               float* __restrict__ partial, float* __restrict__ dwg, float beta) {
  const int e = blockIdx.y, seg = blockIdx.z;
  const int col = (blockIdx.x * blockDim.x + threadIdx.x) * 4;
  if (col >= H) return;
  const int n = counts[e];
  const int r0 = pad_off[e] + (int)((long long)n * seg / nseg);
  const int r1 = pad_off[e] + (int)((long long)n * (seg + 1) / nseg);
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll 4
  for (int r = r0; r < r1; ++r) {
    const float d = dl_perm[r];
    const float4 v = __ldg(reinterpret_cast<const float4*>(x + (size_t)src_token[r] * H + col));
    acc.x = __fmaf_rn(d, v.x, acc.x);
    acc.y = __fmaf_rn(d, v.y, acc.y);
    acc.z = __fmaf_rn(d, v.z, acc.z);
    acc.w = __fmaf_rn(d, v.w, acc.w);
  }
  if (nseg > 1) {
    *reinterpret_cast<float4*>(partial + ((size_t)seg * E + e) * H + col) = acc;
    return;
  }
  float4* o = reinterpret_cast<float4*>(dwg + (size_t)e * H + col);
  if (beta != 0.0f) {
    const float4 p = *o;
    acc.x += beta * p.x; acc.y += beta * p.y; acc.z += beta * p.z; acc.w += beta * p.w;
  }
  *o = acc;
}

__global__ void router_wgrad_reduce_f32_kernel(const float* __restrict__ partial, int nseg, size_t EH,
                                               float* __restrict__ dwg, float beta) {
  for (size_t i = ((size_t)blockIdx.x * blockDim.x + threadIdx.x) * 4; i < EH;
       i += (size_t)gridDim.x * blockDim.x * 4) {
    float4 s = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll 8
    for (int q = 0; q < nseg; ++q) {
      const float4 v = *reinterpret_cast<const float4*>(partial + (size_t)q * EH + i);
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

// ------------------------------------------------------------------ SwiGLU
// h13 fp32 [rows, 2De] (DM_GLU_BLOCK-column gate/up blocks, dm_moe.h) -> act3 split-3 [rows, 3De].
__global__ void __launch_bounds__(256)
swiglu_fwd_split_kernel(const float* __restrict__ h13, int rows, int De, __nv_bfloat16* __restrict__ act3) {
  const int per_row = De >> 3;
  const size_t n = (size_t)rows * per_row;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    const int r = (int)(i / per_row), c = (int)(i % per_row) * 8;
    const int blk = c / DM_GLU_BLOCK, off = c % DM_GLU_BLOCK;
    const float* hr = h13 + (size_t)r * 2 * De + blk * 2 * DM_GLU_BLOCK + off;
    float g[8], u[8], a[8];
    ld8(hr, g);
    ld8(hr + DM_GLU_BLOCK, u);
#pragma unroll
    for (int q = 0; q < 8; ++q) a[q] = g[q] / (1.0f + expf(-g[q])) * u[q];
    st_split3_act(act3 + (size_t)r * 3 * De, De, c, a);
  }
}

// d_act fp32 [rows, De], h13 fp32 [rows, 2De] -> dh13_3 split-3 [rows, 6De] of the
// interleaved [dgate | dup] blocks: dg = d_act*u*s*(1+g*(1-s)), du = d_act*g*s.
__global__ void __launch_bounds__(256)
swiglu_bwd_split_kernel(const float* __restrict__ d_act, const float* __restrict__ h13, int rows, int De,
                        __nv_bfloat16* __restrict__ dh13_3) {
  const int per_row = De >> 3;
  const size_t n = (size_t)rows * per_row;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    const int r = (int)(i / per_row), c = (int)(i % per_row) * 8;
    const int blk = c / DM_GLU_BLOCK, off = c % DM_GLU_BLOCK;
    const float* hr = h13 + (size_t)r * 2 * De + blk * 2 * DM_GLU_BLOCK + off;
    float g[8], u[8], d[8], dg[8], du[8];
    ld8(hr, g);
    ld8(hr + DM_GLU_BLOCK, u);
    ld8(d_act + (size_t)r * De + c, d);
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const float s = 1.0f / (1.0f + expf(-g[q]));
      dg[q] = d[q] * u[q] * s * (1.0f + g[q] * (1.0f - s));
      du[q] = d[q] * g[q] * s;
    }
    __nv_bfloat16* row = dh13_3 + (size_t)r * 6 * De;
    st_split3_act(row, 2 * De, blk * 2 * DM_GLU_BLOCK + off, dg);
    st_split3_act(row, 2 * De, blk * 2 * DM_GLU_BLOCK + DM_GLU_BLOCK + off, du);
  }
}

// ------------------------------------------------------------------ split
// src fp32 [groups * rows, cols] -> dst bf16:
//   layout 0 (activation, K-major): row -> [hi | hi | lo]        dst [groups*rows, 3*cols]
//   layout 1 (weight, K-major):     row -> [hi | lo | hi]        dst [groups*rows, 3*cols]
//   layout 2 (weight, MN-major):    group -> rows [hi; lo; hi]  dst [groups*3*rows, cols]
__global__ void __launch_bounds__(256)
split3_kernel(const float* __restrict__ src, long long nrows_total, int rows, int cols, int layout,
              __nv_bfloat16* __restrict__ dst) {
  const int per_row = cols >> 3;
  const long long n = nrows_total * per_row;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const long long r = i / per_row;
    const int c = (int)(i % per_row) * 8;
    float f[8];
    ld8(src + r * cols + c, f);
    int4 hi, lo;
    split8(f, hi, lo);
    if (layout == 2) {
      const long long g = r / rows, rr = r % rows;
      __nv_bfloat16* base = dst + (g * 3 * rows + rr) * cols + c;
      st_v4(base, hi);
      st_v4(base + (long long)rows * cols, lo);
      st_v4(base + 2LL * rows * cols, hi);
    } else {
      __nv_bfloat16* row = dst + r * 3 * cols;
      st_v4(row + c, hi);
      st_v4(row + cols + c, layout == 0 ? hi : lo);
      st_v4(row + 2 * cols + c, layout == 0 ? lo : hi);
    }
  }
}

static int grid_for(long long work, int threads) {
  long long b = (work + threads - 1) / threads;
  const long long cap = (long long)num_sms_current() * 8;
  if (b > cap) b = cap;
  return b < 1 ? 1 : (int)b;
}

static int token_grid_f32(int T) {
  int b = (T + 7) / 8;
  const int cap = num_sms_current() * 8;
  return b < cap ? b : cap;
}

static int finish(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return set_cuda_error(e, what);
  note_launch();
  return DM_OK;
}

}  // namespace dm

using namespace dm;

extern "C" {

int dm_route_and_dispatch_f32(const float* x, const float* wg, int T, int H, int E, int k, void* workspace,
                              int32_t* idx, float* w, int32_t* counts, int32_t* pad_off, int32_t* row_map,
                              int32_t* src_token, void* x3, void* stream) {
  if (T < 1 || H < 8 || H % 8 || E < 1 || E > DM_MAX_EXPERTS || k < 1 || k > DM_MAX_TOPK || k > E)
    return set_error(DM_ERR_SHAPE, "route_and_dispatch_f32 bad shape (T=%d H=%d E=%d k=%d)", T, H, E, k);
  cudaStream_t st = (cudaStream_t)stream;
  dm_route_ws ws;
  dm_route_workspace_layout(T, H, E, k, workspace, &ws);
  const size_t row_bytes = (size_t)H * sizeof(float);
  int ec = (int)((160 * 1024) / row_bytes);
  if (ec < 1) return set_error(DM_ERR_SHAPE, "router_f32: hidden %d too large for one smem row", H);
  if (ec > E) ec = E;
  if (int rc = ensure_smem_attr((const void*)router_logits_f32_kernel, 160 * 1024, "cudaFuncSetAttribute(router_f32)"))
    return rc;
  int grid = (T + RF_WARPS - 1) / RF_WARPS;
  if (grid > num_sms_current()) grid = num_sms_current();
  router_logits_f32_kernel<<<grid, RF_WARPS * 32, (size_t)ec * row_bytes, st>>>(x, wg, ws.logits, T, H, E, ec);
  int rc = finish("router_logits_f32 launch");
  if (rc) return rc;
  if ((rc = dm_router_topk(ws.logits, T, E, k, idx, w, ws.rank, ws.chunk_hist, stream))) return rc;
  if ((rc = dm_expert_scan(ws.chunk_hist, T, E, counts, pad_off, ws.chunk_base, stream))) return rc;
  permute_f32_kernel<<<token_grid_f32(T), 256, 0, st>>>(x, idx, ws.rank, ws.chunk_base, counts, pad_off, T, H, E, k,
                                                         row_map, src_token,
                                                         reinterpret_cast<__nv_bfloat16*>(x3));
  return finish("permute_f32 launch");
}

int dm_combine_fwd_f32(const float* y_perm, const int32_t* row_map, const float* w, int T, int H, int k,
                       const float* resid, float* y, void* stream) {
  if (T < 1 || H % 8 || k < 1 || k > DM_MAX_TOPK) return set_error(DM_ERR_SHAPE, "combine_fwd_f32 bad shape");
  if (resid && resid == y) return set_error(DM_ERR_SHAPE, "combine_fwd_f32: resid must not alias y");
  combine_fwd_f32_kernel<<<token_grid_f32(T), 256, 0, (cudaStream_t)stream>>>(y_perm, row_map, w, T, H, k, resid, y);
  return finish("combine_fwd_f32 launch");
}

int dm_combine_bwd_f32(const float* dy, const float* y_perm, const int32_t* row_map, const float* w,
                       const int32_t* counts, const int32_t* pad_off, int T, int H, int E, int k, void* dy3,
                       float* dw, float* dlogit, float* dl_perm, void* stream) {
  if (T < 1 || H % 8 || k < 1 || k > DM_MAX_TOPK || E < 1) return set_error(DM_ERR_SHAPE, "combine_bwd_f32 bad shape");
  combine_bwd_f32_kernel<<<token_grid_f32(T), 256, 0, (cudaStream_t)stream>>>(
      dy, y_perm, row_map, w, counts, pad_off, T, H, E, k, reinterpret_cast<__nv_bfloat16*>(dy3), dw, dlogit,
      dl_perm);
  return finish("combine_bwd_f32 launch");
}

int dm_permute_bwd_f32(const float* dx_perm, const int32_t* row_map, const int32_t* idx, const float* dlogit,
                       const float* wg, int T, int H, int E, int k, const float* resid, float* dx, void* stream) {
  if (T < 1 || H % 8 || k < 1 || k > DM_MAX_TOPK || E < 1) return set_error(DM_ERR_SHAPE, "permute_bwd_f32 bad shape");
  if (resid && resid == dx) return set_error(DM_ERR_SHAPE, "permute_bwd_f32: resid must not alias dx");
  permute_bwd_f32_kernel<<<token_grid_f32(T), 256, 0, (cudaStream_t)stream>>>(dx_perm, row_map, idx, dlogit, wg, T,
                                                                               H, k, resid, dx);
  return finish("permute_bwd_f32 launch");
}

int dm_router_wgrad_sorted_f32(const float* x, const int32_t* src_token, const float* dl_perm,
                               const int32_t* counts, const int32_t* pad_off, int T, int H, int E,
                               float* partial_ws, float* dwg, float beta, void* stream) {
  if (T < 1 || H % 8 || E < 1 || E > DM_MAX_EXPERTS) return set_error(DM_ERR_SHAPE, "router_wgrad_sorted_f32 bad shape");
  cudaStream_t st = (cudaStream_t)stream;
  const int gx = (H / 4 + 127) / 128;
  int nseg = 1;
  if (partial_ws) {
    const int tbt = dm_router_wgrad_token_block(E);
    const int cap_seg = (T + tbt - 1) / tbt;
    nseg = (4 * num_sms_current() + gx * E - 1) / (gx * E);
    if (nseg > cap_seg) nseg = cap_seg;
    if (nseg < 1) nseg = 1;
  }
  router_wgrad_sorted_f32_kernel<<<dim3(gx, E, nseg), 128, 0, st>>>(x, src_token, dl_perm, counts, pad_off, H, E,
                                                                     nseg, partial_ws, dwg, beta);
  int rc = finish("router_wgrad_sorted_f32 launch");
  if (rc || nseg == 1) return rc;
  const size_t EH = (size_t)E * H;
  router_wgrad_reduce_f32_kernel<<<grid_for((long long)(EH / 4), 64), 64, 0, st>>>(partial_ws, nseg, EH, dwg, beta);
  return finish("router_wgrad_reduce_f32 launch");
}

int dm_swiglu_fwd_split(const float* h13, int rows, int De, void* act3, void* stream) {
  if (rows < 0 || De % 128 || De < 128) return set_error(DM_ERR_SHAPE, "swiglu_fwd_split: D_e %d not a multiple of 128", De);
  static_assert(DM_GLU_BLOCK % 8 == 0 && 128 % DM_GLU_BLOCK == 0, "GLU block must tile 128 columns");
  if (rows == 0) return DM_OK;
  swiglu_fwd_split_kernel<<<grid_for((long long)rows * (De / 8), 256), 256, 0, (cudaStream_t)stream>>>(
      h13, rows, De, reinterpret_cast<__nv_bfloat16*>(act3));
  return finish("swiglu_fwd_split launch");
}

int dm_swiglu_bwd_split(const float* d_act, const float* h13, int rows, int De, void* dh13_3, void* stream) {
  if (rows < 0 || De % 128 || De < 128) return set_error(DM_ERR_SHAPE, "swiglu_bwd_split: D_e %d not a multiple of 128", De);
  if (rows == 0) return DM_OK;
  swiglu_bwd_split_kernel<<<grid_for((long long)rows * (De / 8), 256), 256, 0, (cudaStream_t)stream>>>(
      d_act, h13, rows, De, reinterpret_cast<__nv_bfloat16*>(dh13_3));
  return finish("swiglu_bwd_split launch");
}

int dm_split3(const float* src, int groups, int rows, int cols, int layout, void* dst, void* stream) {
  if (groups < 1 || rows < 1 || cols % 8 || cols < 8 || layout < 0 || layout > 2)
    return set_error(DM_ERR_SHAPE, "split3 bad shape (groups=%d rows=%d cols=%d layout=%d)", groups, rows, cols, layout);
  const long long nrows = (long long)groups * rows;
  split3_kernel<<<grid_for(nrows * (cols / 8), 256), 256, 0, (cudaStream_t)stream>>>(
      src, nrows, rows, cols, layout, reinterpret_cast<__nv_bfloat16*>(dst));
  return finish("split3 launch");
}

}  // extern "C"
