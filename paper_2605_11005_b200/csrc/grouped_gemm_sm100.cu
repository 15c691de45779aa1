// Grouped (per-expert) bf16 GEMMs for the SwiGLU expert FFN, fwd + bwd, on
// 5th-gen tensor cores: TMA -> 4-stage smem ring -> tcgen05.mma (one thread)
// -> fp32 accumulators in TMEM (2 x 128x256 tiles, double buffered) -> fused
// epilogue warps (SwiGLU fwd / SwiGLU bwd / bf16 store / fp32 store+accumulate).
//
// Reference counterpart: the reference only *costs* this stage —
// ffn_flops C_f = 4*b*k*s*H*D_e (pkg/src/afpipe/costs.py:90-92, two GEMMs) and
// backward_scale 2x (costs.py:146-150); the F-side FwdCompute/BwdCompute tasks
// of _build_afpipe (taskgraph.py:333-347) stand for what this file computes.
//
// Two grouping modes, both driven by the 128-aligned per-expert row offsets
// `group_off` produced on device by the dispatch scan (no host sync):
//   ragged-M  (fwd, dgrad): C[rows_e, N] = A[rows_e, K] * B_e^T, tiles over
//             (expert, 128-row m-tile, 256-col n-tile), m fastest so the 8
//             m-tiles of one expert reuse each weight n-tile from L2.
//   ragged-K  (wgrad):      C_e[M, N] = A_tok[rows_e, M]^T * B_tok[rows_e, N],
//             K loop over the expert's (zero-padded) token rows.
#include <stdlib.h>

#include "dm_common.cuh"
#include "dm_internal.h"

namespace dm {

constexpr int GBM = 128, GBN = 256, GBK = 64, GSTAGES = 4;
constexpr uint32_t GA_BYTES = GBM * GBK * 2;   // 16 KiB
constexpr uint32_t GB_BYTES = GBN * GBK * 2;   // 32 KiB
constexpr int GEMM_THREADS = 256;
constexpr int GEMM_MAX_GROUPS = 1024;
constexpr size_t GEMM_SMEM_BYTES =
    1024 /*align slack*/ + GSTAGES * (GA_BYTES + GB_BYTES) + 256 /*barriers*/ +
    2 * (GEMM_MAX_GROUPS + 1) * sizeof(int);

enum { EPI_BF16 = 0, EPI_SWIGLU_FWD = 1, EPI_SWIGLU_BWD = 2, EPI_F32 = 3 };

struct GemmArgs {
  int num_groups;
  const int* group_off;          // [G+1], 128-aligned, device
  int M;                         // ragged-K: rows of C per group (multiple of 128; a partial
                                 //   last 256-row tile is clipped by the 3-D C map)
  int N;                         // multiple of 128 (2-SM path; a partial last 256-column tile
                                 //   reads zero-filled / discarded B rows, its stores are clipped)
  int K;                         // ragged-M: reduction length (multiple of 64)
  int b_group_rows;              // ragged-M: rows of the B tensor owned by one weight matrix
  int b_groups;                  // ragged-M: group g multiplies weight matrix (g / b_div) % b_groups
  int b_div;                     // ragged-M: consecutive groups sharing a weight matrix (>= 1)
  const int* group_end;          // ragged-M, optional: group g = rows [group_off[g], group_end[g])
                                 //   (group_off then holds G starts); null: contiguous groups
  void* C;
  long long ldc;
  long long c_group_stride;      // ragged-K: elements between groups' C blocks
  __nv_bfloat16* aux;            // SwiGLU fwd: h13 out; SwiGLU bwd: dh13 out
  long long ld_aux;
  const __nv_bfloat16* aux_in;   // SwiGLU bwd: h13 in
  long long ld_aux_in;
  float beta;                    // EPI_F32: C = acc + beta * C
  // ragged-K: group g's K rows are the union over segments i < nseg of
  // [i*seg_stride_rows + seg_off[i*(G+1)+g], i*seg_stride_rows + seg_off[i*(G+1)+g+1])
  const int* seg_off;
  int nseg;
  int seg_stride_rows;
  // diagnostic only (env DM_GEMM_DIAG=1, results invalid): load the A tile of the
  // first k-block of every tile only, so the mainloop streams half the bytes. Used to
  // tell operand-supply-bound from MMA-bound mainloops; never set on the product path.
  int diag_skip_a;
  // 1: warp 0 streams A and warp 3 streams B (two issuers); 0: warp 0 issues both
  int dual_producer;
  // optional instrumentation (dm_debug_gemm_profile): u64 cycle counters
  // [0] producer waits on empty, [1] MMA waits on tempty, [2] MMA waits on full,
  // [3] epilogue waits on tfull (lane 0 of each epilogue warp), [4] CTA lifetime
  unsigned long long* prof;
};

#define DM_PROF_WAIT(slot, call)                                                  \
  do {                                                                            \
    if (args.prof) {                                                              \
      const long long _t = clock64();                                             \
      call;                                                                       \
      if ((threadIdx.x & 31) == 0) atomicAdd(args.prof + (slot), (unsigned long long)(clock64() - _t)); \
    } else {                                                                      \
      call;                                                                       \
    }                                                                             \
  } while (0)

struct TileInfo {
  int g, m0, n0, kb_count, row_base;
  int half;   // 2-SM ragged-M tail tile with 128 valid rows: M = 128 MMA, 64 rows per CTA
};

template <int RAGGED_K>
__device__ __forceinline__ TileInfo decode_tile(int t, const int* tile_start, const int* off,
                                                int G, const GemmArgs& a) {
  int lo = 0, hi = G - 1;
  while (lo < hi) {
    int mid = (lo + hi + 1) >> 1;
    if (tile_start[mid] <= t) lo = mid; else hi = mid - 1;
  }
  TileInfo ti;
  ti.g = lo;
  ti.half = 0;
  const int local = t - tile_start[lo];
  const int row_off = RAGGED_K ? 0 : off[lo];
  const int rows = RAGGED_K ? 0 : off[lo + 1] - row_off;
  ti.row_base = row_off;
  if (!RAGGED_K) {
    const int mt = rows / GBM;
    ti.m0 = row_off + (local % mt) * GBM;
    ti.n0 = (local / mt) * GBN;
    ti.kb_count = a.K / GBK;
  } else {
    const int mt = a.M / GBM;
    ti.m0 = (local % mt) * GBM;
    ti.n0 = (local / mt) * GBN;
    int kb = 0;
    for (int i = 0; i < a.nseg; ++i)
      kb += (a.seg_off[i * (G + 1) + lo + 1] - a.seg_off[i * (G + 1) + lo]) / GBK;
    ti.kb_count = kb;
  }
  return ti;
}

__device__ __forceinline__ float silu_f(float g) { return g / (1.0f + __expf(-g)); }

// One thread owns one accumulator row (TMEM lane) of the 128x256 tile.
template <int EPI>
__device__ __forceinline__ void epilogue_row(const TileInfo& ti, uint32_t trow, int r,
                                             const GemmArgs& a) {
  if constexpr (EPI == EPI_BF16) {
    const long long row = ti.m0 + r;
    __nv_bfloat16* out = reinterpret_cast<__nv_bfloat16*>(a.C) + row * a.ldc + ti.n0;
#pragma unroll 1
    for (int c = 0; c < GBN; c += 32) {
      uint32_t v0[16], v1[16];
      tmem_ld16(trow + c, v0);
      tmem_ld16(trow + c + 16, v1);
      tmem_wait_ld();
      int4 o[4];
      uint32_t* op = reinterpret_cast<uint32_t*>(o);
#pragma unroll
      for (int i = 0; i < 8; ++i) op[i] = pack_bf16(__uint_as_float(v0[2 * i]), __uint_as_float(v0[2 * i + 1]));
#pragma unroll
      for (int i = 0; i < 8; ++i) op[8 + i] = pack_bf16(__uint_as_float(v1[2 * i]), __uint_as_float(v1[2 * i + 1]));
#pragma unroll
      for (int i = 0; i < 4; ++i) st_v4(out + c + 8 * i, o[i]);
    }
  } else if constexpr (EPI == EPI_SWIGLU_FWD) {
    // Tile columns alternate DM_GLU_BLOCK gate rows of W13 and the matching up rows.
    const long long row = ti.m0 + r;
    __nv_bfloat16* hout = a.aux + row * a.ld_aux + ti.n0;
    __nv_bfloat16* aout = reinterpret_cast<__nv_bfloat16*>(a.C) + row * a.ldc + (ti.n0 >> 1);
#pragma unroll 1
    for (int c = 0; c < GBN / 2; c += 16) {   // c: act column within the tile
      const int gc = (c / DM_GLU_BLOCK) * 2 * DM_GLU_BLOCK + c % DM_GLU_BLOCK;
      uint32_t g[16], u[16];
      tmem_ld16(trow + gc, g);
      tmem_ld16(trow + gc + DM_GLU_BLOCK, u);
      tmem_wait_ld();
      int4 hg[2], hu[2], ao[2];
      uint32_t* hgp = reinterpret_cast<uint32_t*>(hg);
      uint32_t* hup = reinterpret_cast<uint32_t*>(hu);
      uint32_t* aop = reinterpret_cast<uint32_t*>(ao);
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const float g0 = __uint_as_float(g[2 * i]), g1 = __uint_as_float(g[2 * i + 1]);
        const float u0 = __uint_as_float(u[2 * i]), u1 = __uint_as_float(u[2 * i + 1]);
        hgp[i] = pack_bf16(g0, g1);
        hup[i] = pack_bf16(u0, u1);
        aop[i] = pack_bf16(silu_f(g0) * u0, silu_f(g1) * u1);
      }
      st_v4(hout + gc, hg[0]);                st_v4(hout + gc + 8, hg[1]);
      st_v4(hout + gc + DM_GLU_BLOCK, hu[0]); st_v4(hout + gc + DM_GLU_BLOCK + 8, hu[1]);
      st_v4(aout + c, ao[0]);                 st_v4(aout + c + 8, ao[1]);
    }
  } else if constexpr (EPI == EPI_SWIGLU_BWD) {
    // Accumulator = d_act for D_e columns [n0, n0+256); gate/up live in the
    // DM_GLU_BLOCK-interleaved h13 layout: d -> (d/B)*2B + d%B (+B for up).
    const long long row = ti.m0 + r;
    const __nv_bfloat16* hin = a.aux_in + row * a.ld_aux_in;
    __nv_bfloat16* dhout = a.aux + row * a.ld_aux;
#pragma unroll 1
    for (int c = 0; c < GBN; c += 16) {
      uint32_t d[16];
      tmem_ld16(trow + c, d);
      const int dcol = ti.n0 + c;
      const long long gcol = (long long)(dcol / DM_GLU_BLOCK) * 2 * DM_GLU_BLOCK + dcol % DM_GLU_BLOCK;
      int4 gv[2], uv[2];
      gv[0] = ld_v4(hin + gcol);                uv[0] = ld_v4(hin + gcol + DM_GLU_BLOCK);
      gv[1] = ld_v4(hin + gcol + 8);            uv[1] = ld_v4(hin + gcol + DM_GLU_BLOCK + 8);
      tmem_wait_ld();
      const uint32_t* gp = reinterpret_cast<const uint32_t*>(gv);
      const uint32_t* up = reinterpret_cast<const uint32_t*>(uv);
      int4 dg[2], du[2];
      uint32_t* dgp = reinterpret_cast<uint32_t*>(dg);
      uint32_t* dup = reinterpret_cast<uint32_t*>(du);
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        float gg[2] = {bf16lo(gp[i]), bf16hi(gp[i])};
        float uu[2] = {bf16lo(up[i]), bf16hi(up[i])};
        float da[2] = {__uint_as_float(d[2 * i]), __uint_as_float(d[2 * i + 1])};
        float rg[2], ru[2];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const float sg = 1.0f / (1.0f + __expf(-gg[h]));
          const float sl = gg[h] * sg;
          ru[h] = da[h] * sl;
          rg[h] = da[h] * uu[h] * sg * (1.0f + gg[h] * (1.0f - sg));
        }
        dgp[i] = pack_bf16(rg[0], rg[1]);
        dup[i] = pack_bf16(ru[0], ru[1]);
      }
      st_v4(dhout + gcol, dg[0]);                st_v4(dhout + gcol + 8, dg[1]);
      st_v4(dhout + gcol + DM_GLU_BLOCK, du[0]); st_v4(dhout + gcol + DM_GLU_BLOCK + 8, du[1]);
    }
  } else {  // EPI_F32 (wgrad): C_g[m, n] = acc + beta * C_g[m, n]
    float* out = reinterpret_cast<float*>(a.C) + (long long)ti.g * a.c_group_stride +
                 (long long)(ti.m0 + r) * a.ldc + ti.n0;
    const bool empty = ti.kb_count == 0;
#pragma unroll 1
    for (int c = 0; c < GBN; c += 16) {
      uint32_t v[16];
      if (!empty) {
        tmem_ld16(trow + c, v);
        tmem_wait_ld();
      } else {
#pragma unroll
        for (int i = 0; i < 16; ++i) v[i] = 0u;
      }
      float4* o4 = reinterpret_cast<float4*>(out + c);
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        float4 f = make_float4(__uint_as_float(v[4 * i]), __uint_as_float(v[4 * i + 1]),
                               __uint_as_float(v[4 * i + 2]), __uint_as_float(v[4 * i + 3]));
        if (a.beta != 0.0f) {
          const float4 old = o4[i];
          f.x += a.beta * old.x; f.y += a.beta * old.y; f.z += a.beta * old.z; f.w += a.beta * old.w;
        }
        o4[i] = f;
      }
    }
  }
}

template <int A_MN, int B_MN, int RAGGED_K, int EPI>
__global__ void __launch_bounds__(GEMM_THREADS, 1)
grouped_gemm_kernel(const __grid_constant__ CUtensorMap tmA,
                    const __grid_constant__ CUtensorMap tmB, const GemmArgs args) {
  extern __shared__ uint8_t smem_raw[];
  const uint32_t pad = (1024u - (smem_u32(smem_raw) & 1023u)) & 1023u;
  uint8_t* smem = smem_raw + pad;
  uint8_t* sA = smem;
  uint8_t* sB = smem + GSTAGES * GA_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(sB + GSTAGES * GB_BYTES);
  uint64_t* empty = full + GSTAGES;
  uint64_t* tfull = empty + GSTAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  int* s_tile = reinterpret_cast<int*>(smem + GSTAGES * (GA_BYTES + GB_BYTES) + 256);
  int* s_off = s_tile + (GEMM_MAX_GROUPS + 1);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int G = args.num_groups;

  if (!RAGGED_K)
    for (int i = threadIdx.x; i <= G; i += GEMM_THREADS) s_off[i] = args.group_off[i];
  if (threadIdx.x == 0) {
#pragma unroll
    for (int s = 0; s < GSTAGES; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
#pragma unroll
    for (int s = 0; s < 2; ++s) { mbar_init(&tfull[s], 1); mbar_init(&tempty[s], 128); }
    fence_mbar_init();
  }
  if (warp == 0 && lane == 0) { tma_prefetch_desc(&tmA); tma_prefetch_desc(&tmB); }
  if (warp == 2) tmem_alloc(tmem_slot, 512);
  __syncthreads();
  if (threadIdx.x == 32 * 3) {
    int acc = 0;
    for (int g = 0; g < G; ++g) {
      s_tile[g] = acc;
      const int rows = RAGGED_K ? 0 : s_off[g + 1] - s_off[g];
      acc += RAGGED_K ? (args.M / GBM) * (args.N / GBN) : (rows / GBM) * (args.N / GBN);
    }
    s_tile[G] = acc;
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  const int total_tiles = s_tile[G];

  if (warp == 0) {
    // ---------------------------------------------------------- TMA producer
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int t = blockIdx.x; t < total_tiles; t += gridDim.x) {
        const TileInfo ti = decode_tile<RAGGED_K>(t, s_tile, s_off, G, args);
        const int b_gofs = RAGGED_K ? 0 : (ti.g % args.b_groups) * args.b_group_rows;
        int seg = 0, seg_kb = 0, seg_nkb = 0, seg_row0 = 0;
        for (int kb = 0; kb < ti.kb_count; ++kb) {
          int kcoord;
          if (RAGGED_K) {
            while (seg_kb == seg_nkb) {  // advance to the next non-empty segment
              const int* so = args.seg_off + seg * (G + 1) + ti.g;
              seg_row0 = seg * args.seg_stride_rows + so[0];
              seg_nkb = (so[1] - so[0]) / GBK;
              seg_kb = 0;
              ++seg;
            }
            kcoord = seg_row0 + seg_kb * GBK;
            ++seg_kb;
          } else {
            kcoord = kb * GBK;
          }
          mbar_wait(&empty[stage], phase ^ 1);
          mbar_expect_tx(&full[stage], GA_BYTES + GB_BYTES);
          uint8_t* a_dst = sA + stage * GA_BYTES;
          uint8_t* b_dst = sB + stage * GB_BYTES;
          if (!A_MN) {
            tma_load_2d(a_dst, &tmA, &full[stage], kcoord, ti.m0);
          } else {
#pragma unroll
            for (int j = 0; j < GBM / 64; ++j)
              tma_load_2d(a_dst + j * 8192, &tmA, &full[stage], ti.m0 + 64 * j, kcoord);
          }
          if (!B_MN) {
            tma_load_2d(b_dst, &tmB, &full[stage], kcoord, b_gofs + ti.n0);
          } else {
#pragma unroll
            for (int j = 0; j < GBN / 64; ++j)
              tma_load_2d(b_dst + j * 8192, &tmB, &full[stage], ti.n0 + 64 * j, b_gofs + kcoord);
          }
          if (++stage == GSTAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    if (lane == 0) {
      constexpr uint32_t idesc = make_idesc_bf16(GBM, GBN, A_MN, B_MN);
      int stage = 0;
      uint32_t phase = 0;
      int it = 0;
      for (int t = blockIdx.x; t < total_tiles; t += gridDim.x, ++it) {
        const TileInfo ti = decode_tile<RAGGED_K>(t, s_tile, s_off, G, args);
        const int as = it & 1;
        const uint32_t aphase = (it >> 1) & 1;
        mbar_wait(&tempty[as], aphase ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + as * GBN;
        for (int kb = 0; kb < ti.kb_count; ++kb) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint32_t a_addr = smem_u32(sA + stage * GA_BYTES);
          const uint32_t b_addr = smem_u32(sB + stage * GB_BYTES);
#pragma unroll
          for (int k = 0; k < GBK / 16; ++k) {
            const uint64_t ad = A_MN ? make_sdesc_sw128(a_addr + k * 2048, 8192, 1024)
                                     : make_sdesc_sw128(a_addr + k * 32, 16, 1024);
            const uint64_t bd = B_MN ? make_sdesc_sw128(b_addr + k * 2048, 8192, 1024)
                                     : make_sdesc_sw128(b_addr + k * 32, 16, 1024);
            umma_bf16_ss(d_tmem, ad, bd, idesc, (kb | k) != 0 ? 1u : 0u);
          }
          umma_commit(&empty[stage]);
          if (++stage == GSTAGES) { stage = 0; phase ^= 1; }
        }
        umma_commit(&tfull[as]);
      }
    }
    __syncwarp();
  } else if (warp >= 4) {
    // --------------------------------------------------------- epilogue warps
    const int q = warp & 3;  // TMEM lane quarter this warp may access
    int it = 0;
    for (int t = blockIdx.x; t < total_tiles; t += gridDim.x, ++it) {
      const TileInfo ti = decode_tile<RAGGED_K>(t, s_tile, s_off, G, args);
      const int as = it & 1;
      const uint32_t aphase = (it >> 1) & 1;
      mbar_wait(&tfull[as], aphase);
      tc_fence_after();
      const uint32_t trow = tmem_base + (static_cast<uint32_t>(q * 32) << 16) + as * GBN;
      epilogue_row<EPI>(ti, trow, q * 32 + lane, args);
      tc_fence_before();
      mbar_arrive(&tempty[as]);
    }
  }

  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 2) tmem_dealloc(tmem_base, 512);
}

// ==================================================================== 2-SM path
// CTA pair (cluster of 2) computing 256x256 output tiles with
// tcgen05.mma.cta_group::2 (UMMA M=256): each CTA stages its 128 rows of A and
// its 128 rows (N half) of B per k-block, so per-SM smem operand traffic is
// 32 KiB per 256x256x64 step instead of 48 KiB per 128x256x64 step of the
// 1-SM kernel. The leader (rank 0) issues all MMAs; both CTAs' TMEM hold their
// 128 accumulator rows; each CTA's epilogue drains its own half through
// SWIZZLE_128B smem boxes and TMA bulk stores (fp32 accumulation into dW uses
// the TMA reduce-add, so no read-modify-write passes through the SMs).
constexpr uint32_t G2_A_BYTES = 128 * GBK * 2;   // 16 KiB (this CTA's M half)
constexpr uint32_t G2_B_BYTES = 128 * GBK * 2;   // 16 KiB (this CTA's N half)
constexpr uint32_t BOX_BYTES = 4096;             // one 32-row x 128-byte staging box

// Ring depth. The MMA issuer waits on TMA data 12-20% of the time
// (scripts/gemm_waits.py); a 6-stage ring did not reduce that (supply-rate, not
// latency, bound) and was slower, so 5 stages (4 next to the SwiGLU-bwd staging).
template <int EPI> constexpr int g2_stages() { return EPI == EPI_SWIGLU_BWD ? 4 : 5; }
// per-epilogue-warp staging: BF16/F32 2 boxes (double buffer); SwiGLU fwd gate/up/act;
// SwiGLU bwd dg/du out + g/u in
template <int EPI> constexpr uint32_t g2_stg_bytes() {
  return EPI == EPI_SWIGLU_FWD ? 3 * BOX_BYTES : EPI == EPI_SWIGLU_BWD ? 4 * BOX_BYTES : 2 * BOX_BYTES;
}
// fixed part; the three [G+1]-int tables (tile starts, group starts / ends) are appended at launch
template <int EPI> constexpr size_t g2_smem_bytes() {
  return 1024 + g2_stages<EPI>() * (G2_A_BYTES + G2_B_BYTES) + 4 * g2_stg_bytes<EPI>() + 256;
}

template <int RAGGED_K>
__device__ __forceinline__ TileInfo decode_tile_2sm(int t, const int* tile_start, const int* off, const int* end,
                                                    int G, const GemmArgs& a, uint32_t rank, bool& active) {
  // merged mode (group ranges with b_div > 1): the tile table runs over the G / b_div weight
  // groups, each the union of its b_div member ranges cut into 128-row chunks
  const bool merged = !RAGGED_K && a.group_end && a.b_div > 1;
  const int NG = merged ? G / a.b_div : G;
  int lo = 0, hi = NG - 1;
  while (lo < hi) {
    int mid = (lo + hi + 1) >> 1;
    if (tile_start[mid] <= t) lo = mid; else hi = mid - 1;
  }
  TileInfo ti;
  ti.g = lo;
  const int local = t - tile_start[lo];
  ti.half = 0;
  if (merged) {
    // a pair tile = two 128-row chunks of the weight group in (member, row) order — rank 0
    // takes the first, rank 1 the second, wherever their rows lie; an odd last chunk runs
    // as an M = 128 pair MMA (64 rows per CTA)
    const int g0 = lo * a.b_div;
    int chunks = 0;
    for (int i = 0; i < a.b_div; ++i) chunks += (end[g0 + i] - off[g0 + i]) >> 7;
    const int mt = (chunks + 1) >> 1;
    const int c0 = 2 * (local % mt);
    ti.half = c0 + 1 >= chunks;
    int c = ti.half ? c0 : c0 + (int)rank, row = 0;
    for (int i = 0; i < a.b_div; ++i) {
      const int cnt = (end[g0 + i] - off[g0 + i]) >> 7;
      if (c < cnt) { row = off[g0 + i] + (c << 7); break; }
      c -= cnt;
    }
    ti.g = g0;                                          // weight (g0 / b_div) % b_groups
    ti.m0 = row + (ti.half ? 64 * (int)rank : 0);
    ti.n0 = (local / mt) * GBN;
    ti.kb_count = a.K / GBK;
    ti.row_base = 0;
    active = true;
  } else if (!RAGGED_K) {
    const int row_off = off[lo];
    const int rows = end[lo] - row_off;
    const int mt = (rows + 255) / 256;
    const int tm0 = row_off + (local % mt) * 256;
    // Groups are 128-row aligned, so a tile has 256 or (the group's tail) 128 valid
    // rows. A tail tile runs as an M = 128 pair MMA (64 rows per CTA) instead of an
    // M = 256 MMA with an idle half: the padding-to-256 MMA work disappears.
    ti.half = (row_off + rows - tm0) <= 128;
    ti.m0 = tm0 + (ti.half ? 64 : 128) * (int)rank;   // this CTA's first row
    ti.n0 = (local / mt) * GBN;
    ti.kb_count = a.K / GBK;
    ti.row_base = row_off;
    active = true;
  } else {
    // Rasterise along the smaller output dimension so concurrent tiles share the
    // larger operand's tile (streamed once) while the smaller operand stays in L2:
    // dW13 (M = 2*D_e >> N = H) goes n-fastest, dW2 (M = H < N = D_e) m-fastest.
    const int mt = (a.M + 255) / 256, nt = (a.N + GBN - 1) / GBN;
    if (a.M >= a.N) {
      ti.m0 = (local / nt) * 256 + 128 * rank;
      ti.n0 = (local % nt) * GBN;
    } else {
      ti.m0 = (local % mt) * 256 + 128 * rank;
      ti.n0 = (local / mt) * GBN;
    }
    int kb = 0;
    for (int i = 0; i < a.nseg; ++i)
      kb += (a.seg_off[i * (G + 1) + lo + 1] - a.seg_off[i * (G + 1) + lo]) / GBK;
    ti.kb_count = kb;
    ti.row_base = 0;
    active = true;
  }
  return ti;
}

__device__ __forceinline__ void tmem_ld64(uint32_t taddr, uint32_t* r) {
  tmem_ld16(taddr, *reinterpret_cast<uint32_t(*)[16]>(r));
  tmem_ld16(taddr + 16, *reinterpret_cast<uint32_t(*)[16]>(r + 16));
  tmem_ld16(taddr + 32, *reinterpret_cast<uint32_t(*)[16]>(r + 32));
  tmem_ld16(taddr + 48, *reinterpret_cast<uint32_t(*)[16]>(r + 48));
}

// Write one thread's 64 fp32 accumulators (as bf16) into its 128-byte row of a box.
__device__ __forceinline__ void box_row_bf16(uint32_t box, int lane, const uint32_t* v) {
#pragma unroll
  for (int j = 0; j < 8; ++j)
    st_shared_v4(box + sw128(lane, j),
                 pack_bf16(__uint_as_float(v[8 * j + 0]), __uint_as_float(v[8 * j + 1])),
                 pack_bf16(__uint_as_float(v[8 * j + 2]), __uint_as_float(v[8 * j + 3])),
                 pack_bf16(__uint_as_float(v[8 * j + 4]), __uint_as_float(v[8 * j + 5])),
                 pack_bf16(__uint_as_float(v[8 * j + 6]), __uint_as_float(v[8 * j + 7])));
}

// Epilogue of one epilogue warp (TMEM lane quarter q = rows q*32 .. q*32+31 of
// this CTA's 128-row half). `stg` is the warp's private staging area; only lane 0
// issues TMA and owns the bulk groups.
//
// TMEM geometry of the warp's accumulator slice. Full tiles (M = 256 pair MMA): lane =
// row, all 256 columns. Half tiles (M = 128 pair MMA, 64 rows per CTA): the "2x2"
// data-path layout, lanes 0-63 hold rows 0-63 x tile columns [0,128) and lanes 64-127
// the same rows x columns [128,256), both at TMEM columns [0,128); so warp q drains
// rows (q&1)*32.. of the 128-column half (q>>1) — each warp still owns whole SwiGLU
// pairs because gate/up blocks are DM_GLU_BLOCK = 64 wide.
template <int EPI>
__device__ __forceinline__ void epilogue_tma(const TileInfo& ti, uint32_t tacc, int q, int lane,
                                             const GemmArgs& a, const CUtensorMap* tmC,
                                             const CUtensorMap* tmAux, const CUtensorMap* tmIn,
                                             uint8_t* stg, uint64_t* ibar, uint32_t& iphase) {
  const uint32_t s0 = smem_u32(stg);
  const int row0 = ti.m0 + (ti.half ? (q & 1) : q) * 32;   // first row of this warp
  const int col0 = ti.n0 + (ti.half ? (q >> 1) * 128 : 0);  // first tile column it holds
  const int ncols = ti.half ? 128 : GBN;
  if constexpr (EPI == EPI_BF16) {
#pragma unroll 1
    for (int c = 0; c < ncols / 64; ++c) {
      uint32_t v[64];
      tmem_ld64(tacc + c * 64, v);
      tmem_wait_ld();
      if (c >= 2) {
        if (lane == 0) bulk_wait_read<1>();
        __syncwarp();
      }
      box_row_bf16(s0 + (c & 1) * BOX_BYTES, lane, v);
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) {
        tma_store_2d(tmC, stg + (c & 1) * BOX_BYTES, col0 + c * 64, row0);
        bulk_commit();
      }
    }
  } else if constexpr (EPI == EPI_SWIGLU_FWD) {
    // accumulator columns alternate DM_GLU_BLOCK gate rows of W13 and the matching
    // up rows; c walks the warp's act columns (ncols / 2) in 64-column boxes
#pragma unroll 1
    for (int c = 0; c < ncols / 2; c += 64) {
      const int gc = (c / DM_GLU_BLOCK) * 2 * DM_GLU_BLOCK + c % DM_GLU_BLOCK;
      uint32_t g[64], u[64];
      tmem_ld64(tacc + gc, g);
      tmem_ld64(tacc + gc + DM_GLU_BLOCK, u);
      tmem_wait_ld();
      if (c > 0) {
        if (lane == 0) bulk_wait_read<0>();
        __syncwarp();
      }
      box_row_bf16(s0, lane, g);
      box_row_bf16(s0 + BOX_BYTES, lane, u);
#pragma unroll
      for (int i = 0; i < 64; ++i) {
        const float gf = __uint_as_float(g[i]), uf = __uint_as_float(u[i]);
        g[i] = __float_as_uint(silu_f(gf) * uf);
      }
      box_row_bf16(s0 + 2 * BOX_BYTES, lane, g);
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) {
        tma_store_2d(tmAux, stg, col0 + gc, row0);
        tma_store_2d(tmAux, stg + BOX_BYTES, col0 + gc + DM_GLU_BLOCK, row0);
        tma_store_2d(tmC, stg + 2 * BOX_BYTES, (col0 >> 1) + c, row0);
        bulk_commit();
      }
    }
  } else if constexpr (EPI == EPI_SWIGLU_BWD) {
    // accumulator = d_act for this warp's D_e columns [col0, col0 + ncols); g/u come
    // from the DM_GLU_BLOCK-interleaved h13 (d -> (d/B)*2B + d%B, +B for up)
    const int nch = ncols / 64;
    const uint32_t in_g = s0 + 2 * BOX_BYTES, in_u = s0 + 3 * BOX_BYTES;
    auto gcol_of = [&](int c) {
      const int dcol = col0 + c * 64;
      return (dcol / DM_GLU_BLOCK) * 2 * DM_GLU_BLOCK + dcol % DM_GLU_BLOCK;
    };
    if (lane == 0) {
      mbar_expect_tx(ibar, 2 * BOX_BYTES);
      tma_load_2d(stg + 2 * BOX_BYTES, tmIn, ibar, gcol_of(0), row0);
      tma_load_2d(stg + 3 * BOX_BYTES, tmIn, ibar, gcol_of(0) + DM_GLU_BLOCK, row0);
    }
#pragma unroll 1
    for (int c = 0; c < nch; ++c) {
      const int gcol = gcol_of(c);
      uint32_t d[64];
      tmem_ld64(tacc + c * 64, d);
      mbar_wait(ibar, iphase);
      iphase ^= 1;
      uint32_t gu[32], uu[32];
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int4 gv = ld_shared_v4(in_g + sw128(lane, j));
        const int4 uv = ld_shared_v4(in_u + sw128(lane, j));
        gu[4 * j] = gv.x; gu[4 * j + 1] = gv.y; gu[4 * j + 2] = gv.z; gu[4 * j + 3] = gv.w;
        uu[4 * j] = uv.x; uu[4 * j + 1] = uv.y; uu[4 * j + 2] = uv.z; uu[4 * j + 3] = uv.w;
      }
      tmem_wait_ld();
      __syncwarp();
      if (c + 1 < nch && lane == 0) {  // inputs consumed: prefetch the next chunk's g/u
        fence_proxy_async_smem();
        mbar_expect_tx(ibar, 2 * BOX_BYTES);
        tma_load_2d(stg + 2 * BOX_BYTES, tmIn, ibar, gcol_of(c + 1), row0);
        tma_load_2d(stg + 3 * BOX_BYTES, tmIn, ibar, gcol_of(c + 1) + DM_GLU_BLOCK, row0);
      }
      // d[i] <- dg (bf16-pair packed later), reuse gu/uu for du
#pragma unroll
      for (int i = 0; i < 32; ++i) {
        float gg[2] = {bf16lo(gu[i]), bf16hi(gu[i])};
        float uv2[2] = {bf16lo(uu[i]), bf16hi(uu[i])};
        float rg[2], ru[2];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const float da = __uint_as_float(d[2 * i + h]);
          const float sg = 1.0f / (1.0f + __expf(-gg[h]));
          ru[h] = da * gg[h] * sg;
          rg[h] = da * uv2[h] * sg * (1.0f + gg[h] * (1.0f - sg));
        }
        gu[i] = pack_bf16(rg[0], rg[1]);
        uu[i] = pack_bf16(ru[0], ru[1]);
      }
      if (c > 0) {
        if (lane == 0) bulk_wait_read<0>();
        __syncwarp();
      }
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        st_shared_v4(s0 + sw128(lane, j), gu[4 * j], gu[4 * j + 1], gu[4 * j + 2], gu[4 * j + 3]);
        st_shared_v4(s0 + BOX_BYTES + sw128(lane, j), uu[4 * j], uu[4 * j + 1], uu[4 * j + 2], uu[4 * j + 3]);
      }
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) {
        tma_store_2d(tmAux, stg, gcol, row0);
        tma_store_2d(tmAux, stg + BOX_BYTES, gcol + DM_GLU_BLOCK, row0);
        bulk_commit();
      }
    }
  } else {  // EPI_F32: dW_g rows (g*M + m) of a [G*M, N] fp32 matrix (ragged K, a.M > 0) or
            // C rows m (ragged M, a.M = 0); beta in {0, 1}
    // ragged K (a.M > 0): the 3-D map [G][M][N] clips this group's rows/cols; ragged M:
    // 2-D [rows, N] map
    const bool empty = ti.kb_count == 0;
    if (empty && a.beta != 0.0f) return;  // adding zeros
#pragma unroll 1
    for (int c = 0; c < ncols / 32; ++c) {
      uint32_t v[32];
      if (!empty) {
        tmem_ld16(tacc + c * 32, *reinterpret_cast<uint32_t(*)[16]>(v));
        tmem_ld16(tacc + c * 32 + 16, *reinterpret_cast<uint32_t(*)[16]>(v + 16));
        tmem_wait_ld();
      } else {
#pragma unroll
        for (int i = 0; i < 32; ++i) v[i] = 0u;
      }
      if (c >= 2) {
        if (lane == 0) bulk_wait_read<1>();
        __syncwarp();
      }
      const uint32_t box = s0 + (c & 1) * BOX_BYTES;
#pragma unroll
      for (int j = 0; j < 8; ++j) st_shared_v4(box + sw128(lane, j), v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) {
        uint8_t* box = stg + (c & 1) * BOX_BYTES;
        if (a.M > 0) {
          if (a.beta != 0.0f) tma_reduce_add_3d(tmC, box, col0 + c * 32, row0, ti.g);
          else tma_store_3d(tmC, box, col0 + c * 32, row0, ti.g);
        } else {
          if (a.beta != 0.0f) tma_reduce_add_2d(tmC, box, col0 + c * 32, row0);
          else tma_store_2d(tmC, box, col0 + c * 32, row0);
        }
        bulk_commit();
      }
    }
  }
}

template <int A_MN, int B_MN, int RAGGED_K, int EPI>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(GEMM_THREADS, 1)
grouped_gemm_2sm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                        const __grid_constant__ CUtensorMap tmC, const __grid_constant__ CUtensorMap tmAux,
                        const __grid_constant__ CUtensorMap tmIn, const GemmArgs args) {
  constexpr int STAGES = g2_stages<EPI>();
  constexpr uint32_t STG = g2_stg_bytes<EPI>();
  const long long prof_t0 = clock64();
  extern __shared__ uint8_t smem_raw[];
  const uint32_t pad = (1024u - (smem_u32(smem_raw) & 1023u)) & 1023u;
  uint8_t* smem = smem_raw + pad;
  uint8_t* sA = smem;
  uint8_t* sB = smem + STAGES * G2_A_BYTES;
  uint8_t* sStg = sB + STAGES * G2_B_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(sStg + 4 * STG);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 2;
  uint64_t* ibar = tempty + 2;   // [4] per-epilogue-warp input barriers
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(ibar + 4);
  int* s_tile = reinterpret_cast<int*>(sStg + 4 * STG + 256);
  int* s_off = s_tile + (args.num_groups + 1);     // group starts
  int* s_end = s_off + (args.num_groups + 1);      // group ends

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int G = args.num_groups;
  const uint32_t rank = cluster_ctarank();
  const bool leader = rank == 0;
  const int cluster_id = blockIdx.x >> 1;
  const int num_clusters = gridDim.x >> 1;

  if (!RAGGED_K) {
    for (int i = threadIdx.x; i < G; i += GEMM_THREADS) {
      s_off[i] = args.group_off[i];
      s_end[i] = args.group_end ? args.group_end[i] : args.group_off[i + 1];
    }
  }
  if (threadIdx.x == 0) {
#pragma unroll
    for (int s = 0; s < STAGES; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
#pragma unroll
    // tempty: one arrival per epilogue warp of both CTAs (lane 0 after a __syncwarp)
    for (int s = 0; s < 2; ++s) { mbar_init(&tfull[s], 1); mbar_init(&tempty[s], 2 * 4); }
#pragma unroll
    for (int s = 0; s < 4; ++s) mbar_init(&ibar[s], 1);
    fence_mbar_init();
  }
  if (warp == 0 && lane == 0) { tma_prefetch_desc(&tmA); tma_prefetch_desc(&tmB); }
  if (warp == 3 && lane == 0) { tma_prefetch_desc(&tmC); tma_prefetch_desc(&tmAux); }
  if (warp == 2) tmem_alloc_2sm(tmem_slot, 512);
  __syncthreads();
  if (threadIdx.x == 32 * 3) {
    int acc = 0;
    const int nt = (args.N + GBN - 1) / GBN;   // last column tile may be partial (N % 256 == 128)
    if (!RAGGED_K && args.group_end && args.b_div > 1) {   // merged: per weight group
      const int NG = G / args.b_div;
      for (int w = 0; w < NG; ++w) {
        s_tile[w] = acc;
        int chunks = 0;
        for (int i = 0; i < args.b_div; ++i) chunks += (s_end[w * args.b_div + i] - s_off[w * args.b_div + i]) >> 7;
        acc += ((chunks + 1) >> 1) * nt;
      }
      s_tile[NG] = acc;
    } else {
      for (int g = 0; g < G; ++g) {
        s_tile[g] = acc;
        const int rows = RAGGED_K ? 0 : s_end[g] - s_off[g];
        acc += RAGGED_K ? ((args.M + 255) / 256) * nt : ((rows + 255) / 256) * nt;
      }
      s_tile[G] = acc;
    }
  }
  tc_fence_before();
  cluster_sync_all();   // barriers initialised and TMEM allocated in both CTAs
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  const int total_tiles = s_tile[(!RAGGED_K && args.group_end && args.b_div > 1) ? G / args.b_div : G];

  if (warp == 0 || (warp == 3 && args.dual_producer)) {
    // ------------------------------------------- TMA producers (both CTAs)
    // warp 0 streams the A operand, warp 3 the B operand: two independent issuing
    // threads per CTA (the MN-major wgrad operands need two 64-column boxes each and a
    // single issuer starved the MMA). Both walk the same tile/k schedule and ring; the
    // A producer posts the stage's expected bytes (complete_tx may land first).
    if (lane == 0) {
      // L2 policy: evict-last/evict-first hints on the re-read/streamed operand
      // were measured slower than the default policy on every variant.
      const uint64_t pol = L2_EVICT_NORMAL;
      const bool is_a = warp == 0;
      const bool do_a = is_a, do_b = !is_a || !args.dual_producer;
      int stage = 0;
      uint32_t phase = 0;
      for (int t = cluster_id; t < total_tiles; t += num_clusters) {
        bool active;
        const TileInfo ti = decode_tile_2sm<RAGGED_K>(t, s_tile, s_off, s_end, G, args, rank, active);
        const int b_gofs = RAGGED_K ? 0 : ((ti.g / args.b_div) % args.b_groups) * args.b_group_rows;
        const int nb0 = ti.n0 + 128 * (int)rank;   // this CTA's half of the N tile
        int seg = 0, seg_kb = 0, seg_nkb = 0, seg_row0 = 0;
        for (int kb = 0; kb < ti.kb_count; ++kb) {
          int kcoord;
          if (RAGGED_K) {
            while (seg_kb == seg_nkb) {
              const int* so = args.seg_off + seg * (G + 1) + ti.g;
              seg_row0 = seg * args.seg_stride_rows + so[0];
              seg_nkb = (so[1] - so[0]) / GBK;
              seg_kb = 0;
              ++seg;
            }
            kcoord = seg_row0 + seg_kb * GBK;
            ++seg_kb;
          } else {
            kcoord = kb * GBK;
          }
          if (is_a) DM_PROF_WAIT(0, mbar_wait(&empty[stage], phase ^ 1));
          else mbar_wait(&empty[stage], phase ^ 1);
          const bool load_a = !args.diag_skip_a || kb < STAGES;
          if (do_a) {
            if (leader) mbar_expect_tx(&full[stage], 2 * ((load_a ? G2_A_BYTES : 0) + G2_B_BYTES));
            uint8_t* a_dst = sA + stage * G2_A_BYTES;
            if (!load_a) {
            } else if (!A_MN) {
              tma_load_2d_2sm(a_dst, &tmA, &full[stage], kcoord, ti.m0, pol);
            } else {
              tma_load_2d_2sm(a_dst, &tmA, &full[stage], ti.m0, kcoord, pol);
              tma_load_2d_2sm(a_dst + 8192, &tmA, &full[stage], ti.m0 + 64, kcoord, pol);
            }
          }
          if (do_b) {
            uint8_t* b_dst = sB + stage * G2_B_BYTES;
            if (!B_MN) {
              tma_load_2d_2sm(b_dst, &tmB, &full[stage], kcoord, b_gofs + nb0, pol);
            } else {
              tma_load_2d_2sm(b_dst, &tmB, &full[stage], nb0, b_gofs + kcoord, pol);
              tma_load_2d_2sm(b_dst + 8192, &tmB, &full[stage], nb0 + 64, b_gofs + kcoord, pol);
            }
          }
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    // ------------------------------------------------ MMA issuer (leader)
    if (leader && lane == 0) {
      constexpr uint32_t idesc_full = make_idesc_bf16(256, GBN, A_MN, B_MN);
      constexpr uint32_t idesc_half = make_idesc_bf16(128, GBN, A_MN, B_MN);
      int stage = 0;
      uint32_t phase = 0;
      int it = 0;
      for (int t = cluster_id; t < total_tiles; t += num_clusters, ++it) {
        bool active;
        const TileInfo ti = decode_tile_2sm<RAGGED_K>(t, s_tile, s_off, s_end, G, args, rank, active);
        const int as = it & 1;
        const uint32_t aphase = (it >> 1) & 1;
        DM_PROF_WAIT(1, mbar_wait(&tempty[as], aphase ^ 1));
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + as * GBN;
        const uint32_t idesc = ti.half ? idesc_half : idesc_full;
        for (int kb = 0; kb < ti.kb_count; ++kb) {
          DM_PROF_WAIT(2, mbar_wait(&full[stage], phase));
          tc_fence_after();
          const uint32_t a_addr = smem_u32(sA + stage * G2_A_BYTES);
          const uint32_t b_addr = smem_u32(sB + stage * G2_B_BYTES);
#pragma unroll
          for (int k = 0; k < GBK / 16; ++k) {
            const uint64_t ad = A_MN ? make_sdesc_sw128(a_addr + k * 2048, 8192, 1024)
                                     : make_sdesc_sw128(a_addr + k * 32, 16, 1024);
            const uint64_t bd = B_MN ? make_sdesc_sw128(b_addr + k * 2048, 8192, 1024)
                                     : make_sdesc_sw128(b_addr + k * 32, 16, 1024);
            umma_bf16_ss_2sm(d_tmem, ad, bd, idesc, (kb | k) != 0 ? 1u : 0u);
          }
          umma_commit_2sm_mc(&empty[stage]);
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
        umma_commit_2sm_mc(&tfull[as]);
      }
    }
    __syncwarp();
  } else if (warp >= 4) {
    // ------------------------------------------- epilogue warps (both CTAs)
    const int q = warp & 3;
    uint8_t* stg = sStg + q * STG;
    uint32_t iphase = 0;
    int it = 0;
    for (int t = cluster_id; t < total_tiles; t += num_clusters, ++it) {
      bool active;
      const TileInfo ti = decode_tile_2sm<RAGGED_K>(t, s_tile, s_off, s_end, G, args, rank, active);
      const int as = it & 1;
      const uint32_t aphase = (it >> 1) & 1;
      DM_PROF_WAIT(3, mbar_wait(&tfull[as], aphase));
      tc_fence_after();
      if (active) {
        const uint32_t tacc = tmem_base + (static_cast<uint32_t>(q * 32) << 16) + as * GBN;
        epilogue_tma<EPI>(ti, tacc, q, lane, args, &tmC, &tmAux, &tmIn, stg, &ibar[q], iphase);
      }
      // TMEM buffer drained: one (remote) arrival per warp instead of per thread — the
      // per-thread cluster arrives cost ~10% of the epilogue on short-K (wgrad) tiles
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        if (leader) mbar_arrive(&tempty[as]);
        else mbar_arrive_cluster(&tempty[as], 0);
      }
    }
    if (lane == 0) bulk_wait_all();
    __syncwarp();
  }

  tc_fence_before();
  cluster_sync_all();
  tc_fence_after();
  if (warp == 2) tmem_dealloc_2sm(tmem_base, 512);
  if (args.prof && threadIdx.x == 0) atomicAdd(args.prof + 4, (unsigned long long)(clock64() - prof_t0));
}

// ------------------------------------------------------------------- host side

static unsigned long long* g_gemm_prof = nullptr;

// Environment switches, read once (thread-safe static initialisation).
static int env_flag(const char* name, char on, int if_on, int otherwise) {
  const char* e = getenv(name);
  return (e && e[0] == on) ? if_on : otherwise;
}

static bool use_2sm() {
  static const bool v = env_flag("DM_GEMM_1SM", '1', 0, 1) == 1;
  return v;
}

// TMA L2 promotion. K-major operand boxes and epilogue boxes keep 256 B (the next k-block
// / column box follows); MN-major operand boxes (64 x 64, 128-byte rows) use none: at the
// Mixtral w13 dgrad (MN-major W13, K = 28672) 256 B promotion read 4.38 GB of DRAM per
// launch vs 3.76 GB without (algorithmic 2.35 GB), and ran 2.3% slower
// (scripts/gemm_traffic_probe.sh). DM_GEMM_PROMO = 0 / 64 / 128 / 256 forces one setting.
static CUtensorMapL2promotion l2_promotion(bool mn_major_operand) {
  static const int forced = [] {
    const char* e = getenv("DM_GEMM_PROMO");
    return e ? atoi(e) : -1;
  }();
  const int v = forced >= 0 ? forced : (mn_major_operand ? 0 : 256);
  return v == 0 ? CU_TENSOR_MAP_L2_PROMOTION_NONE : v == 64 ? CU_TENSOR_MAP_L2_PROMOTION_L2_64B
       : v == 128 ? CU_TENSOR_MAP_L2_PROMOTION_L2_128B : CU_TENSOR_MAP_L2_PROMOTION_L2_256B;
}

// groups > 0: a rank-3 map [groups][outer][inner] of back-to-back [outer, inner] blocks
// (box depth 1), so every group's edges clip independently.
static int make_tmap_2d(CUtensorMap* tm, const void* base, bool fp32, uint64_t inner, uint64_t outer,
                       uint64_t row_stride_elems, uint32_t box_inner, uint32_t box_outer, uint64_t groups = 0,
                       bool mn_major_operand = false) {
  PFN_cuTensorMapEncodeTiled_v12000 enc = tensor_map_encoder();
  if (!enc) return set_error(DM_ERR_DRIVER, "cuTensorMapEncodeTiled entry point unavailable");
  const uint64_t esz = fp32 ? 4 : 2;
  if ((reinterpret_cast<uintptr_t>(base) & 15) || ((row_stride_elems * esz) & 15))
    return set_error(DM_ERR_ALIGN, "TMA operand base/stride not 16-byte aligned");
  cuuint64_t dims[3] = {inner, outer, groups};
  cuuint64_t strides[2] = {row_stride_elems * esz, row_stride_elems * esz * outer};
  cuuint32_t box[3] = {box_inner, box_outer, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = enc(tm, fp32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, groups ? 3 : 2,
                   const_cast<void*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_128B, l2_promotion(mn_major_operand),
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return set_error(DM_ERR_DRIVER, "cuTensorMapEncodeTiled failed (%d)", (int)r);
  return DM_OK;
}

static int make_tmap_bf16_2d(CUtensorMap* tm, const void* base, uint64_t inner, uint64_t outer,
                             uint64_t row_stride_elems, uint32_t box_inner, uint32_t box_outer) {
  return make_tmap_2d(tm, base, false, inner, outer, row_stride_elems, box_inner, box_outer);
}

// Builds both operand maps for the chosen path: the 2-SM kernel stages a
// 128-row half of the N tile per CTA, the 1-SM kernel the full 256 rows.
struct GemmOperand {
  const void* base;
  uint64_t inner, outer, ld;
  bool mn_major;
  bool is_b;
};

// A row-major epilogue tensor written (or, for `in`, read) by TMA in 32-row x
// 128-byte boxes: 64 bf16 or 32 fp32 columns.
struct EpiTensor {
  const void* base = nullptr;
  bool fp32 = false;
  uint64_t cols = 0, rows = 0, ld = 0;
  uint64_t groups = 0;   // > 0: rank-3 map, `groups` blocks of [rows, cols]
};

struct EpiTensors {
  EpiTensor c, aux, in;
};

static int make_operand_map(CUtensorMap* tm, const GemmOperand& o, bool two_sm) {
  if (o.mn_major) return make_tmap_2d(tm, o.base, false, o.inner, o.outer, o.ld, 64, 64, 0, true);
  const uint32_t rows = (o.is_b && !two_sm) ? 256 : 128;
  return make_tmap_bf16_2d(tm, o.base, o.inner, o.outer, o.ld, 64, rows);
}

static int make_epi_map(CUtensorMap* tm, const EpiTensor& t, const CUtensorMap& dummy) {
  if (!t.base) {
    *tm = dummy;
    return DM_OK;
  }
  return make_tmap_2d(tm, t.base, t.fp32, t.cols, t.rows, t.ld, t.fp32 ? 32 : 64, 32, t.groups);
}

template <int A_MN, int B_MN, int RAGGED_K, int EPI>
static int launch_gemm(const GemmOperand& oa, const GemmOperand& ob, const EpiTensors& et,
                       const GemmArgs& args, cudaStream_t stream) {
  const bool two = use_2sm();
  CUtensorMap ta, tb;
  int rc;
  if ((rc = make_operand_map(&ta, oa, two))) return rc;
  if ((rc = make_operand_map(&tb, ob, two))) return rc;
  int grid = num_sms_current();
  if (two) {
    if (EPI == EPI_F32 && args.beta != 0.0f && args.beta != 1.0f)
      return set_error(DM_ERR_ARG, "wgrad beta must be 0 (overwrite) or 1 (TMA reduce-add)");
    CUtensorMap tc, tx, ti;
    if ((rc = make_epi_map(&tc, et.c, ta))) return rc;
    if ((rc = make_epi_map(&tx, et.aux, ta))) return rc;
    if ((rc = make_epi_map(&ti, et.in, ta))) return rc;
    auto kern = grouped_gemm_2sm_kernel<A_MN, B_MN, RAGGED_K, EPI>;
    const size_t smem = g2_smem_bytes<EPI>() + 3 * ((size_t)args.num_groups + 1) * sizeof(int);
    if (smem > 232448) return set_error(DM_ERR_SHAPE, "too many groups (%d) for the GEMM smem budget", args.num_groups);
    if ((rc = ensure_smem_attr((const void*)kern, 232448, "cudaFuncSetAttribute(gemm2 smem)"))) return rc;
    grid &= ~1;
    GemmArgs a2 = args;
    if (a2.b_div < 1) a2.b_div = 1;
    a2.prof = g_gemm_prof;
    static const int diag = env_flag("DM_GEMM_DIAG", '1', 1, 0);
    static const int dual = env_flag("DM_GEMM_DUAL", '0', 0, 1);
    a2.diag_skip_a = diag;
    a2.dual_producer = dual;
    kern<<<grid, GEMM_THREADS, smem, stream>>>(ta, tb, tc, tx, ti, a2);
  } else {
    if (args.group_end || args.b_div > 1)
      return set_error(DM_ERR_ARG, "group row ranges need the 2-SM GEMM path (unset DM_GEMM_1SM)");
    if (args.N % GBN || (RAGGED_K && args.M % 256))
      return set_error(DM_ERR_SHAPE, "the 1-SM debug GEMM path needs full 256-wide tiles (N=%d, M=%d)", args.N, args.M);
    auto kern = grouped_gemm_kernel<A_MN, B_MN, RAGGED_K, EPI>;
    if ((rc = ensure_smem_attr((const void*)kern, (int)GEMM_SMEM_BYTES, "cudaFuncSetAttribute(gemm smem)"))) return rc;
    kern<<<grid, GEMM_THREADS, GEMM_SMEM_BYTES, stream>>>(ta, tb, args);
  }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return set_cuda_error(e, "grouped_gemm launch");
  note_launch();
  return DM_OK;
}

static int check_groups(int G, int E, int cap_rows) {
  if (G < 1 || G > GEMM_MAX_GROUPS) return set_error(DM_ERR_SHAPE, "group count %d outside [1, %d]", G, GEMM_MAX_GROUPS);
  if (E < 1 || E > G) return set_error(DM_ERR_SHAPE, "weight count %d outside [1, G=%d]", E, G);
  if (cap_rows < 0 || (cap_rows % GBM)) return set_error(DM_ERR_SHAPE, "cap_rows %d must be a multiple of %d", cap_rows, GBM);
  return DM_OK;
}

}  // namespace dm

using namespace dm;

extern "C" {

static int dm_grouped_w13_swiglu_fwd_impl(const void* x_perm, const void* w13, const int32_t* group_off, const int32_t* group_end, int b_div, int G,
                              int E, int cap_rows, int H, int De, void* h13, void* act, void* stream) {
  int rc = check_groups(G, E, cap_rows);
  if (rc) return rc;
  if (H % GBK || H < GBK || De % 128 || De < 128)
    return set_error(DM_ERR_SHAPE, "w13 fwd needs H %% 64 == 0 and D_e %% 128 == 0 (H=%d, D_e=%d)", H, De);
  const GemmOperand A{x_perm, (uint64_t)H, (uint64_t)cap_rows, (uint64_t)H, false, false};
  const GemmOperand B{w13, (uint64_t)H, (uint64_t)E * 2 * De, (uint64_t)H, false, true};
  GemmArgs a{};
  a.group_end = group_end; a.b_div = b_div;
  a.num_groups = G; a.b_groups = E; a.group_off = group_off; a.N = 2 * De; a.K = H; a.b_group_rows = 2 * De;
  a.C = act; a.ldc = De; a.aux = reinterpret_cast<__nv_bfloat16*>(h13); a.ld_aux = 2 * De;
  EpiTensors et;
  et.c = {act, false, (uint64_t)De, (uint64_t)cap_rows, (uint64_t)De};
  et.aux = {h13, false, (uint64_t)2 * De, (uint64_t)cap_rows, (uint64_t)2 * De};
  return launch_gemm<0, 0, 0, EPI_SWIGLU_FWD>(A, B, et, a, (cudaStream_t)stream);
}

static int dm_grouped_w2_fwd_impl(const void* act, const void* w2, const int32_t* group_off, const int32_t* group_end, int b_div, int G, int E,
                      int cap_rows, int H, int De, void* y_perm, void* stream) {
  int rc = check_groups(G, E, cap_rows);
  if (rc) return rc;
  if (H % 128 || H < 128 || De % GBK || De < GBK)
    return set_error(DM_ERR_SHAPE, "w2 fwd needs H %% 128 == 0 and D_e %% 64 == 0 (H=%d, D_e=%d)", H, De);
  const GemmOperand A{act, (uint64_t)De, (uint64_t)cap_rows, (uint64_t)De, false, false};
  const GemmOperand B{w2, (uint64_t)De, (uint64_t)E * H, (uint64_t)De, false, true};
  GemmArgs a{};
  a.group_end = group_end; a.b_div = b_div;
  a.num_groups = G; a.b_groups = E; a.group_off = group_off; a.N = H; a.K = De; a.b_group_rows = H;
  a.C = y_perm; a.ldc = H;
  EpiTensors et;
  et.c = {y_perm, false, (uint64_t)H, (uint64_t)cap_rows, (uint64_t)H};
  return launch_gemm<0, 0, 0, EPI_BF16>(A, B, et, a, (cudaStream_t)stream);
}

static int dm_grouped_w2_dgrad_swiglu_bwd_impl(const void* dy_perm, const void* w2, const void* h13,
                                   const int32_t* group_off, const int32_t* group_end, int b_div, int G, int E, int cap_rows, int H, int De,
                                   void* dh13, void* stream) {
  int rc = check_groups(G, E, cap_rows);
  if (rc) return rc;
  if (H % GBK || H < GBK || De % 128 || De < 128)
    return set_error(DM_ERR_SHAPE, "w2 dgrad needs H %% 64 == 0 and D_e %% 128 == 0 (H=%d, D_e=%d)", H, De);
  const GemmOperand A{dy_perm, (uint64_t)H, (uint64_t)cap_rows, (uint64_t)H, false, false};
  const GemmOperand B{w2, (uint64_t)De, (uint64_t)E * H, (uint64_t)De, true, true};
  GemmArgs a{};
  a.group_end = group_end; a.b_div = b_div;
  a.num_groups = G; a.b_groups = E; a.group_off = group_off; a.N = De; a.K = H; a.b_group_rows = H;
  a.aux = reinterpret_cast<__nv_bfloat16*>(dh13); a.ld_aux = 2 * De;
  a.aux_in = reinterpret_cast<const __nv_bfloat16*>(h13); a.ld_aux_in = 2 * De;
  EpiTensors et;
  et.aux = {dh13, false, (uint64_t)2 * De, (uint64_t)cap_rows, (uint64_t)2 * De};
  et.in = {h13, false, (uint64_t)2 * De, (uint64_t)cap_rows, (uint64_t)2 * De};
  return launch_gemm<0, 1, 0, EPI_SWIGLU_BWD>(A, B, et, a, (cudaStream_t)stream);
}

static int dm_grouped_w13_dgrad_impl(const void* dh13, const void* w13, const int32_t* group_off, const int32_t* group_end, int b_div, int G, int E,
                         int cap_rows, int H, int De, void* dx_perm, void* stream) {
  int rc = check_groups(G, E, cap_rows);
  if (rc) return rc;
  if (H % 128 || H < 128 || De % 128 || De < 128)
    return set_error(DM_ERR_SHAPE, "w13 dgrad needs H %% 128 == 0 and D_e %% 128 == 0 (H=%d, D_e=%d)", H, De);
  const GemmOperand A{dh13, (uint64_t)2 * De, (uint64_t)cap_rows, (uint64_t)2 * De, false, false};
  const GemmOperand B{w13, (uint64_t)H, (uint64_t)E * 2 * De, (uint64_t)H, true, true};
  GemmArgs a{};
  a.group_end = group_end; a.b_div = b_div;
  a.num_groups = G; a.b_groups = E; a.group_off = group_off; a.N = H; a.K = 2 * De; a.b_group_rows = 2 * De;
  a.C = dx_perm; a.ldc = H;
  EpiTensors et;
  et.c = {dx_perm, false, (uint64_t)H, (uint64_t)cap_rows, (uint64_t)H};
  return launch_gemm<0, 1, 0, EPI_BF16>(A, B, et, a, (cudaStream_t)stream);
}

int dm_grouped_w13_swiglu_fwd(const void* x_perm, const void* w13, const int32_t* group_off, int G,
                              int E, int cap_rows, int H, int De, void* h13, void* act, void* stream) {
  return dm_grouped_w13_swiglu_fwd_impl(x_perm, w13, group_off, nullptr, 1, G, E, cap_rows, H, De, h13, act, stream);
}
int dm_grouped_w2_fwd(const void* act, const void* w2, const int32_t* group_off, int G, int E,
                      int cap_rows, int H, int De, void* y_perm, void* stream) {
  return dm_grouped_w2_fwd_impl(act, w2, group_off, nullptr, 1, G, E, cap_rows, H, De, y_perm, stream);
}
int dm_grouped_w2_dgrad_swiglu_bwd(const void* dy_perm, const void* w2, const void* h13,
                                   const int32_t* group_off, int G, int E, int cap_rows, int H, int De,
                                   void* dh13, void* stream) {
  return dm_grouped_w2_dgrad_swiglu_bwd_impl(dy_perm, w2, h13, group_off, nullptr, 1, G, E, cap_rows, H, De, dh13,
                                             stream);
}
int dm_grouped_w13_dgrad(const void* dh13, const void* w13, const int32_t* group_off, int G, int E,
                         int cap_rows, int H, int De, void* dx_perm, void* stream) {
  return dm_grouped_w13_dgrad_impl(dh13, w13, group_off, nullptr, 1, G, E, cap_rows, H, De, dx_perm, stream);
}

int dm_grouped_w13_swiglu_fwd_ranges(const void* x_perm, const void* w13, const int32_t* group_start,
                                     const int32_t* group_end, int G, int E, int b_div, int cap_rows, int H,
                                     int De, void* h13, void* act, void* stream) {
  if (b_div < 1 || G % b_div) return set_error(DM_ERR_ARG, "b_div %d must divide G = %d", b_div, G);
  return dm_grouped_w13_swiglu_fwd_impl(x_perm, w13, group_start, group_end, b_div, G, E, cap_rows, H, De, h13, act,
                                        stream);
}
int dm_grouped_w2_fwd_ranges(const void* act, const void* w2, const int32_t* group_start, const int32_t* group_end,
                             int G, int E, int b_div, int cap_rows, int H, int De, void* y_perm, void* stream) {
  if (b_div < 1 || G % b_div) return set_error(DM_ERR_ARG, "b_div %d must divide G = %d", b_div, G);
  return dm_grouped_w2_fwd_impl(act, w2, group_start, group_end, b_div, G, E, cap_rows, H, De, y_perm, stream);
}
int dm_grouped_w2_dgrad_swiglu_bwd_ranges(const void* dy_perm, const void* w2, const void* h13,
                                          const int32_t* group_start, const int32_t* group_end, int G, int E,
                                          int b_div, int cap_rows, int H, int De, void* dh13, void* stream) {
  if (b_div < 1 || G % b_div) return set_error(DM_ERR_ARG, "b_div %d must divide G = %d", b_div, G);
  return dm_grouped_w2_dgrad_swiglu_bwd_impl(dy_perm, w2, h13, group_start, group_end, b_div, G, E, cap_rows, H, De,
                                             dh13, stream);
}
int dm_grouped_w13_dgrad_ranges(const void* dh13, const void* w13, const int32_t* group_start,
                                const int32_t* group_end, int G, int E, int b_div, int cap_rows, int H, int De,
                                void* dx_perm, void* stream) {
  if (b_div < 1 || G % b_div) return set_error(DM_ERR_ARG, "b_div %d must divide G = %d", b_div, G);
  return dm_grouped_w13_dgrad_impl(dh13, w13, group_start, group_end, b_div, G, E, cap_rows, H, De, dx_perm, stream);
}

int dm_grouped_wgrad_strided(const void* a_tok, int M, int lda, const void* b_tok, int N, int ldb,
                             const int32_t* seg_off, int nseg, int E, int total_rows, int seg_stride_rows,
                             float* dW, float beta, void* stream) {
  int rc = check_groups(E, E, total_rows);
  if (rc) return rc;
  if (M % 128 || N % 128 || M <= 0 || N <= 0)
    return set_error(DM_ERR_SHAPE, "wgrad needs M %% 128 == 0 and N %% 128 == 0 (M=%d, N=%d)", M, N);
  if (lda < M || ldb < N || lda % 8 || ldb % 8)
    return set_error(DM_ERR_SHAPE, "wgrad row strides (lda=%d, ldb=%d) must be >= M/N and multiples of 8", lda, ldb);
  if (nseg < 1 || nseg > 64) return set_error(DM_ERR_SHAPE, "wgrad segments %d outside [1, 64]", nseg);
  if (seg_stride_rows < 0 || (long long)(nseg - 1) * seg_stride_rows > total_rows)
    return set_error(DM_ERR_SHAPE, "wgrad segment stride %d inconsistent with %d rows", seg_stride_rows, total_rows);
  if (reinterpret_cast<uintptr_t>(dW) & 15) return set_error(DM_ERR_ALIGN, "dW not 16-byte aligned");
  const GemmOperand A{a_tok, (uint64_t)M, (uint64_t)total_rows, (uint64_t)lda, true, false};
  const GemmOperand B{b_tok, (uint64_t)N, (uint64_t)total_rows, (uint64_t)ldb, true, true};
  GemmArgs a{};
  a.num_groups = E; a.group_off = seg_off; a.M = M; a.N = N;
  a.C = dW; a.ldc = N; a.c_group_stride = (long long)M * N; a.beta = beta;
  a.seg_off = seg_off; a.nseg = nseg; a.seg_stride_rows = seg_stride_rows;
  EpiTensors et;
  et.c = {dW, true, (uint64_t)N, (uint64_t)M, (uint64_t)N};
  et.c.groups = (uint64_t)E;
  return launch_gemm<1, 1, 1, EPI_F32>(A, B, et, a, (cudaStream_t)stream);
}

int dm_grouped_wgrad(const void* a_tok, int M, const void* b_tok, int N, const int32_t* seg_off,
                     int nseg, int E, int total_rows, int seg_stride_rows, float* dW, float beta,
                     void* stream) {
  return dm_grouped_wgrad_strided(a_tok, M, M, b_tok, N, N, seg_off, nseg, E, total_rows, seg_stride_rows, dW,
                                  beta, stream);
}

int dm_grouped_gemm_f32(const void* a3, const void* b3, int b_mn_major, const int32_t* group_off, int G, int E,
                        int cap_rows, int N, int K3, float* c, void* stream) {
  int rc = check_groups(G, E, cap_rows);
  if (rc) return rc;
  if (K3 % GBK || K3 < GBK || N % 128 || N < 128)
    return set_error(DM_ERR_SHAPE, "gemm_f32 needs K3 %% 64 == 0 and N %% 128 == 0 (K3=%d, N=%d)", K3, N);
  if (reinterpret_cast<uintptr_t>(c) & 15) return set_error(DM_ERR_ALIGN, "C not 16-byte aligned");
  const GemmOperand A{a3, (uint64_t)K3, (uint64_t)cap_rows, (uint64_t)K3, false, false};
  GemmArgs a{};
  a.num_groups = G; a.b_groups = E; a.group_off = group_off; a.N = N; a.K = K3; a.M = 0;
  a.C = c; a.ldc = N; a.beta = 0.0f;
  EpiTensors et;
  et.c = {c, true, (uint64_t)N, (uint64_t)cap_rows, (uint64_t)N};
  if (b_mn_major) {
    const GemmOperand B{b3, (uint64_t)N, (uint64_t)E * K3, (uint64_t)N, true, true};
    a.b_group_rows = K3;
    return launch_gemm<0, 1, 0, EPI_F32>(A, B, et, a, (cudaStream_t)stream);
  }
  const GemmOperand B{b3, (uint64_t)K3, (uint64_t)E * N, (uint64_t)K3, false, true};
  a.b_group_rows = N;
  return launch_gemm<0, 0, 0, EPI_F32>(A, B, et, a, (cudaStream_t)stream);
}

/* Debug/profiling hook: when `buf` (device, >= 5 u64, zeroed by the caller) is
 * non-NULL every subsequent 2-SM GEMM launch accumulates per-role wait cycles. */
int dm_debug_gemm_profile(void* buf) {
  g_gemm_prof = reinterpret_cast<unsigned long long*>(buf);
  return DM_OK;
}

}  // extern "C"
