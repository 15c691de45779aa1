/*
 * dm_moe.h — C ABI of the B200 (sm_100a) DisagMoE MoE hot path.
 *
 * The reference (arxiv/paper_2605_11005, package `afpipe`) ships no kernel and
 * no FFI: the hot path exists there only as durations and byte counts. Each
 * entry point below replaces the reference quantity that *models* that stage
 * (citations relative to /root/reference):
 *
 *   router / dispatch  (dm_router_*, dm_expert_scan, dm_permute,
 *                       dm_route_and_dispatch)
 *       replaces: m2n_comm_bytes V = e*b*s*k*H   pkg/src/afpipe/costs.py:95-103
 *                 A->F M2NSend/M2NRecv twins      pkg/src/afpipe/taskgraph.py:331-332
 *                 gating semantics
 *   expert FFN fwd     (dm_grouped_w13_swiglu_fwd, dm_grouped_w2_fwd)
 *       replaces: ffn_flops C_f = 4*b*k*s*H*D_e   pkg/src/afpipe/costs.py:90-92
 *                 F FwdCompute task duration       pkg/src/afpipe/taskgraph.py:333-334, :152
 *   expert FFN bwd     (dm_grouped_w2_dgrad_swiglu_bwd, dm_grouped_w13_dgrad,
 *                       dm_grouped_wgrad)
 *       replaces: backward_scale (2x fwd)          pkg/src/afpipe/costs.py:146-150
 *                 F BwdCompute task               pkg/src/afpipe/taskgraph.py:346-347
 *   combine fwd/bwd    (dm_combine_fwd, dm_combine_bwd, dm_permute_bwd,
 *                       dm_router_wgrad)
 *       replaces: F->A transfer + weighted sum     pkg/src/afpipe/taskgraph.py:335-339
 *                 backward chain                   pkg/src/afpipe/taskgraph.py:343-356
 *
 * Conventions (no exceptions cross this boundary):
 *   - The caller owns all memory; pointers are device pointers; nothing here
 *     allocates, frees or synchronises. `stream` is a cudaStream_t (NULL = legacy).
 *   - Return 0 on success, >0 = cudaError_t of a failing launch, <0 = DM_ERR_*.
 *     dm_last_error_string() gives the thread-local message.
 *   - bf16 row-major tensors; H (hidden) rows must be 16-byte aligned.
 *   - Permuted buffers are expert-contiguous with every expert block padded to
 *     DM_ROW_ALIGN rows (zero-filled); pad_off[E+1] holds the block offsets and
 *     dm_capacity_rows() bounds their total, so no host sync is ever needed.
 *   - W13 is [E, 2*D_e, H] with gate/up rows interleaved in blocks of DM_GLU_BLOCK
 *     = 64 (rows 128b..128b+63 = gate rows 64b.., next 64 = up rows 64b..), so each
 *     64-column half of a 128-column accumulator slice holds a gate block and its
 *     up block; h13 / dh13 columns follow the same interleave;
 *     W2 is [E, H, D_e]; router weight W_g is fp32 [E, H].
 */
#ifndef DM_MOE_H_
#define DM_MOE_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#if defined(__GNUC__)
#define DM_API __attribute__((visibility("default")))
#else
#define DM_API
#endif

#define DM_OK 0
#define DM_ERR_SHAPE (-1)
#define DM_ERR_DTYPE (-2)
#define DM_ERR_ALIGN (-3)
#define DM_ERR_ARG (-4)
#define DM_ERR_DRIVER (-5)

#define DM_ABI_VERSION 1
#define DM_CHUNK_TOKENS 32      /* tokens per histogram chunk (stable sort unit) */
#define DM_ROW_ALIGN 128        /* expert block alignment in permuted buffers   */
#define DM_GLU_BLOCK 64         /* gate/up interleave block of W13 / h13 / dh13 */
#define DM_MAX_TOPK 16
#define DM_MAX_EXPERTS 1024

static inline int dm_num_chunks(int T) { return (T + DM_CHUNK_TOKENS - 1) / DM_CHUNK_TOKENS; }

/* dm_route_and_dispatch's streaming router (E <= 16) sorts in units of
 * DM_ROUTE_UNIT_TOKENS tokens (one warp's tokens); its workspace holds one histogram
 * row per unit, which also covers the DM_CHUNK_TOKENS chunks of the two-pass path. */
#define DM_ROUTE_UNIT_TOKENS 4
static inline int dm_num_route_units(int T) { return (T + DM_ROUTE_UNIT_TOKENS - 1) / DM_ROUTE_UNIT_TOKENS; }

/* Upper bound on sum_e roundup(count_e, DM_ROW_ALIGN) for T tokens, top-k. */
static inline int dm_capacity_rows(int T, int E, int k) {
  long long r = (long long)T * k + (long long)E * (DM_ROW_ALIGN - 1);
  return (int)((r + DM_ROW_ALIGN - 1) / DM_ROW_ALIGN * DM_ROW_ALIGN);
}

typedef struct dm_route_ws {
  float* logits;        /* [T, E] fp32 */
  int32_t* chunk_hist;  /* [nunit, E] (two-pass path: [nchunk, E]) */
  int32_t* chunk_base;  /* [nunit, E] (two-pass path: [nchunk, E]) */
  int32_t* rank;        /* [T, k] stable rank of (t, j) among its chunk's slots of the same expert */
  uint32_t* done;       /* CTA completion counters of the streaming router (4 KB): zero when
                           the workspace is first used (allocate it zeroed); left zero */
} dm_route_ws;

static inline size_t dm_align256(size_t v) { return (v + 255) & ~(size_t)255; }

static inline size_t dm_route_workspace_size(int T, int H, int E, int k) {
  (void)H;
  size_t nunit = (size_t)dm_num_route_units(T);
  return dm_align256((size_t)T * E * 4) + 2 * dm_align256(nunit * E * 4) + dm_align256((size_t)T * k * 4) + 4096;
}

static inline void dm_route_workspace_layout(int T, int H, int E, int k, void* ws, dm_route_ws* out) {
  (void)H;
  char* p = (char*)ws;
  size_t nunit = (size_t)dm_num_route_units(T);
  out->logits = (float*)p;
  p += dm_align256((size_t)T * E * 4);
  out->chunk_hist = (int32_t*)p;
  p += dm_align256(nunit * E * 4);
  out->chunk_base = (int32_t*)p;
  p += dm_align256(nunit * E * 4);
  out->rank = (int32_t*)p;
  p += dm_align256((size_t)T * k * 4);
  out->done = (uint32_t*)p;
}

/* Tokens per router-wgrad partial block: small blocks (more parallelism) when the
 * per-block partials are small, i.e. for few experts. */
static inline int dm_router_wgrad_token_block(int E) { return E <= 16 ? 128 : 512; }

/* Partial blocks [ntb][E][H] fp32, then the completion counters of dm_router_wgrad_sorted
 * (one int per (1024-column chunk, expert)) and of dm_router_wgrad (one per 256-column
 * chunk): zero when the workspace is first used (allocate it zeroed), left zero. */
static inline size_t dm_router_wgrad_workspace_size(int T, int H, int E) {
  int tb = dm_router_wgrad_token_block(E);
  size_t ntb = (size_t)((T + tb - 1) / tb);
  size_t ctr = ((size_t)((H + 1023) / 1024) * (size_t)E + (size_t)((H + 255) / 256)) * 4;
  return ntb * (size_t)E * (size_t)H * 4 + ((ctr + 255) & ~(size_t)255);
}

/* ---- library ---------------------------------------------------------- */
DM_API int dm_version(void);
DM_API const char* dm_last_error_string(void);
DM_API int dm_num_sms(int device);
/* Kernel launches issued through this ABI since load (evidence for benches). */
DM_API long long dm_launch_count(void);
/* Exported copies of the inline sizing helpers (for FFI users without a C compiler). */
DM_API int dm_capacity_rows_fn(int T, int E, int k);
DM_API size_t dm_route_workspace_size_fn(int T, int H, int E, int k);
DM_API size_t dm_router_wgrad_workspace_size_fn(int T, int H, int E);

/* ---- dispatch (A side) ------------------------------------------------ */
/* logits[T,E] = x[T,H] (bf16) . W_g[E,H]^T (fp32) in the canonical fixed order. */
DM_API int dm_router_logits(const void* x, const float* wg, float* logits, int T, int H, int E, void* stream);
/* top-k by logit (ties -> lower expert id); w = softmax over the selected logits;
 * rank[T, k] = stable rank of slot (t, j) among the slots of its DM_CHUNK_TOKENS-token
 * chunk that chose the same expert; chunk_hist[nchunk, E] per-chunk expert counts. */
DM_API int dm_router_topk(const float* logits, int T, int E, int k, int32_t* idx, float* w, int32_t* rank,
                          int32_t* chunk_hist, void* stream);
/* counts[E], pad_off[E+1] (DM_ROW_ALIGN-padded block offsets), chunk_base[nchunk, E]. */
DM_API int dm_expert_scan(const int32_t* chunk_hist, int T, int E, int32_t* counts, int32_t* pad_off,
                   int32_t* chunk_base, void* stream);
/* Stable counting sort: row_map[t*k+j] = chunk_base[chunk(t), e] + rank[t*k+j];
 * src_token[pos] = t (-1 for padding); x_perm[pos] = x[t]; padding rows zeroed. */
DM_API int dm_permute(const void* x, const int32_t* idx, const int32_t* rank, const int32_t* chunk_base,
                      const int32_t* counts, const int32_t* pad_off, int T, int H, int E, int k,
                      int32_t* row_map, int32_t* src_token, void* x_perm, void* stream);
/* logits -> topk -> scan -> permute; workspace of dm_route_workspace_size bytes. */
DM_API int dm_route_and_dispatch(const void* x, const float* wg, int T, int H, int E, int k, void* workspace,
                          int32_t* idx, float* w, int32_t* counts, int32_t* pad_off,
                          int32_t* row_map, int32_t* src_token, void* x_perm, void* stream);

/* ---- expert FFN (F side), grouped by 128-aligned row offsets ------------
 * group_off[G+1] partitions the permuted rows into G groups (each a multiple
 * of 128 rows); group g multiplies weight matrix g % E. On the fused path
 * G = E (one group per expert, group_off = pad_off); an F rank of the AF-Pipe
 * runtime passes G = n_attention_ranks * E_local groups ordered (A rank, expert). */
/* h13[r, :] = x_perm[r, :] . W13_e^T ; act = silu(gate) * up.  h13 [cap, 2*D_e], act [cap, D_e]. */
DM_API int dm_grouped_w13_swiglu_fwd(const void* x_perm, const void* w13, const int32_t* group_off, int G,
                                     int E, int cap_rows, int H, int De, void* h13, void* act, void* stream);
/* y_perm[r, :] = act[r, :] . W2_e^T */
DM_API int dm_grouped_w2_fwd(const void* act, const void* w2, const int32_t* group_off, int G, int E,
                             int cap_rows, int H, int De, void* y_perm, void* stream);
/* d_act = dy_perm . W2_e ; dh13 = SwiGLU'(h13) (.) d_act  (same interleaved layout as h13). */
DM_API int dm_grouped_w2_dgrad_swiglu_bwd(const void* dy_perm, const void* w2, const void* h13,
                                          const int32_t* group_off, int G, int E, int cap_rows, int H,
                                          int De, void* dh13, void* stream);
/* dx_perm = dh13 . W13_e */
DM_API int dm_grouped_w13_dgrad(const void* dh13, const void* w13, const int32_t* group_off, int G, int E,
                                int cap_rows, int H, int De, void* dx_perm, void* stream);
/* dW[e] (fp32 [M, N]) = sum over segments i < nseg of
 *   a_tok[rows_{i,e}, :M]^T . b_tok[rows_{i,e}, :N]   (+ beta * dW[e]),
 * rows_{i,e} = i*seg_stride_rows + [seg_off[i*(E+1)+e], seg_off[i*(E+1)+e+1]),
 * a_tok / b_tok having total_rows rows. With seg_stride_rows = cap and one
 * segment per micro-batch, one launch reduces an expert's gradient over every
 * micro-batch of an iteration (deferred weight-gradient pass); seg_stride_rows = 0
 * takes absolute offsets (F ranks: one segment per (micro-batch, A rank)).
 * dW2 = wgrad(dy_perm, M=H, act, N=D_e); dW13 = wgrad(dh13, M=2*D_e, x_perm, N=H). */
DM_API int dm_grouped_wgrad(const void* a_tok, int M, const void* b_tok, int N, const int32_t* seg_off,
                            int nseg, int E, int total_rows, int seg_stride_rows, float* dW, float beta,
                            void* stream);

/* The same four GEMMs over explicit group row ranges: group g = rows [group_start[g], group_end[g])
 * (device arrays, each start a multiple of 128, each range 128-row padded), multiplying weight
 * matrix (g / b_div) % E. With dm_batch_group_ranges this runs n micro-batches stacked cap rows
 * apart as ONE launch, groups ordered expert-major (b_div = n), so each expert's weights stream
 * once for all micro-batches (fused single-device iteration). 2-SM path only. */
DM_API int dm_grouped_w13_swiglu_fwd_ranges(const void* x_perm, const void* w13, const int32_t* group_start,
                                            const int32_t* group_end, int G, int E, int b_div, int cap_rows, int H,
                                            int De, void* h13, void* act, void* stream);
DM_API int dm_grouped_w2_fwd_ranges(const void* act, const void* w2, const int32_t* group_start,
                                    const int32_t* group_end, int G, int E, int b_div, int cap_rows, int H, int De,
                                    void* y_perm, void* stream);
DM_API int dm_grouped_w2_dgrad_swiglu_bwd_ranges(const void* dy_perm, const void* w2, const void* h13,
                                                 const int32_t* group_start, const int32_t* group_end, int G, int E,
                                                 int b_div, int cap_rows, int H, int De, void* dh13, void* stream);
DM_API int dm_grouped_w13_dgrad_ranges(const void* dh13, const void* w13, const int32_t* group_start,
                                       const int32_t* group_end, int G, int E, int b_div, int cap_rows, int H, int De,
                                       void* dx_perm, void* stream);
/* group_start / group_end [E * n] from the [n, E+1] padded offsets of n micro-batches stacked cap
 * rows apart: expert_major != 0 orders them g = e * n + i (pass b_div = n to the GEMMs: one weight
 * pass serves every micro-batch, 128-row chunks of different micro-batches share a pair tile),
 * else g = i * E + e (b_div = 1: the per-micro-batch tile order, one launch). */
DM_API int dm_batch_group_ranges(const int32_t* pad_off, int n, int E, int cap, int expert_major,
                                 int32_t* group_start, int32_t* group_end, void* stream);

/* Debug: route 2-SM GEMM wait-cycle counters into a device u64[5] buffer (NULL = off). */
DM_API int dm_debug_gemm_profile(void* buf);
/* Debug: per-CTA globaltimer timeline of the streaming router (>= 64 u64 per CTA, zeroed;
 * NULL turns it off). */
DM_API int dm_debug_route_profile(void* buf);

/* ---- combine (A side) ------------------------------------------------- */
/* y[t] = resid[t] + sum_j w[t,j] * y_perm[row_map[t,j]]  (fp32 accumulation; resid may be
 * NULL, else the residual stream of a layer stack; it must not alias y). */
DM_API int dm_combine_fwd(const void* y_perm, const int32_t* row_map, const float* w, int T, int H, int k,
                          const void* resid, void* y, void* stream);
/* dy_perm = w * dy scattered (padding zeroed); dw = <dy, y_perm>;
 * dlogit[t,j] = w_j (dw_j - sum_i w_i dw_i); optional dl_perm[row_map[t,j]] = dlogit[t,j]. */
DM_API int dm_combine_bwd(const void* dy, const void* y_perm, const int32_t* row_map, const float* w,
                          const int32_t* counts, const int32_t* pad_off, int T, int H, int E, int k,
                          void* dy_perm, float* dw, float* dlogit, float* dl_perm, void* stream);
/* dx = resid + sum_j dx_perm[row_map] + sum_j dlogit * W_g[idx]  (dlogit and resid may be
 * NULL; resid is the residual-path gradient of a layer stack and must not alias dx). */
DM_API int dm_permute_bwd(const void* dx_perm, const int32_t* row_map, const int32_t* idx,
                          const float* dlogit, const float* wg, int T, int H, int E, int k,
                          const void* resid, void* dx, void* stream);
/* dW_g[E,H] = sum_{t,j} dlogit[t,j] x[t] at row idx[t,j] (+ beta * dW_g);
 * partial_ws of dm_router_wgrad_workspace_size bytes. */
DM_API int dm_router_wgrad(const void* x, const int32_t* idx, const float* dlogit, int T, int H, int E,
                    int k, float* partial_ws, float* dwg, float beta, void* stream);

/* dW_g[e,:] = sum over expert e's permuted rows r of dl_perm[r] * x[src_token[r], :]
 * (+ beta * dW_g), deterministic. partial_ws (dm_router_wgrad_workspace_size bytes, zeroed
 * before first use, may be NULL) lets few-expert layers split each expert's rows into
 * segments; the last segment CTA of each (column chunk, expert) sums them in order. */
DM_API int dm_router_wgrad_sorted(const void* x, const int32_t* src_token, const float* dl_perm,
                                  const int32_t* counts, const int32_t* pad_off, int T, int H, int E,
                                  float* partial_ws, float* dwg, float beta, void* stream);

/* ---- fp32 mode (experiment bytes_per_element = 4; 1e-4 parity) ---------------
 * fp32 activations / gradients / master weights. GEMM operands are bf16 "split-3":
 * v = hi + lo with hi = bf16(v), lo = bf16(v - hi); activations are stored as rows
 * [hi | hi | lo] along K (3K columns), weights as [hi | lo | hi] (K-major) or with
 * per-matrix stacked rows [hi; lo; hi] (MN-major), so one tcgen05 bf16 GEMM over
 * K3 = 3K sums a_hi.b_hi + a_hi.b_lo + a_lo.b_hi into fp32 (error ~2^-16).
 *   replaces (reference): the fp32 path selected by ModelConfig.bytes_per_element
 *                          pkg/src/afpipe/config.py:45-60 (costs only, costs.py:95-103) */
/* Router (fp32 x, canonical order) + top-k + scan + permute into x3 [cap, 3H]. */
DM_API int dm_route_and_dispatch_f32(const float* x, const float* wg, int T, int H, int E, int k, void* workspace,
                                     int32_t* idx, float* w, int32_t* counts, int32_t* pad_off, int32_t* row_map,
                                     int32_t* src_token, void* x3, void* stream);
/* C[cap, N] fp32 = A3[cap, K3] . B3_g (group g uses matrix g % E): B3 K-major [E*N, K3]
 * (b_mn_major 0) or MN-major [E*K3, N] (1). Groups as in the bf16 GEMMs. */
DM_API int dm_grouped_gemm_f32(const void* a3, const void* b3, int b_mn_major, const int32_t* group_off, int G,
                               int E, int cap_rows, int N, int K3, float* c, void* stream);
DM_API int dm_combine_fwd_f32(const float* y_perm, const int32_t* row_map, const float* w, int T, int H, int k,
                              const float* resid, float* y, void* stream);
/* dy3 [cap, 3H] = split-3 of w * dy at the permuted rows (padding zeroed). */
DM_API int dm_combine_bwd_f32(const float* dy, const float* y_perm, const int32_t* row_map, const float* w,
                              const int32_t* counts, const int32_t* pad_off, int T, int H, int E, int k,
                              void* dy3, float* dw, float* dlogit, float* dl_perm, void* stream);
DM_API int dm_permute_bwd_f32(const float* dx_perm, const int32_t* row_map, const int32_t* idx,
                              const float* dlogit, const float* wg, int T, int H, int E, int k, const float* resid,
                              float* dx, void* stream);
DM_API int dm_router_wgrad_sorted_f32(const float* x, const int32_t* src_token, const float* dl_perm,
                                      const int32_t* counts, const int32_t* pad_off, int T, int H, int E,
                                      float* partial_ws, float* dwg, float beta, void* stream);
/* act3 [rows, 3De] = split-3(silu(gate) * up) of fp32 h13 [rows, 2De] (DM_GLU_BLOCK interleave). */
DM_API int dm_swiglu_fwd_split(const float* h13, int rows, int De, void* act3, void* stream);
/* dh13_3 [rows, 6De] = split-3 of the SwiGLU backward of fp32 d_act [rows, De]. */
DM_API int dm_swiglu_bwd_split(const float* d_act, const float* h13, int rows, int De, void* dh13_3,
                               void* stream);
/* dm_grouped_wgrad with explicit row strides (elements) of the token-major operands,
 * e.g. the hi / lo column blocks of split-3 activations. */
DM_API int dm_grouped_wgrad_strided(const void* a_tok, int M, int lda, const void* b_tok, int N, int ldb,
                                    const int32_t* seg_off, int nseg, int E, int total_rows, int seg_stride_rows,
                                    float* dW, float beta, void* stream);
/* fp32 [groups*rows, cols] -> bf16 split-3; layout 0: [hi|hi|lo] rows, 1: [hi|lo|hi]
 * rows, 2: per group of `rows` rows, stacked [hi; lo; hi] (dst [groups*3*rows, cols]). */
DM_API int dm_split3(const float* src, int groups, int rows, int cols, int layout, void* dst, void* stream);

/* ---- A-side attention (reference cost C_a, costs.py:84-87) ----
 * Causal GQA flash-attention forward, head_dim 128, tcgen05/TMEM/TMA. qkv is the bf16
 * projection [T, (nh + 2*nkv) * 128] (q heads, then k heads, then v heads; T = batch *
 * seq_len, sequences contiguous); out [T, nh * 128] bf16; lse [batch, nh, seq_len] fp32
 * natural-log softmax normaliser of the scaled logits (scale 1/sqrt(128)).
 * seq_len must be a multiple of 128 (of 256 when nh / nkv is odd). */
DM_API int dm_attention_fwd(const void* qkv, int T, int seq_len, int nh, int nkv, int head_dim, void* out,
                            float* lse, void* stream);
/* Its backward: dqkv [T, (nh + 2*nkv) * 128] bf16 (dQ, dK, dV in the qkv layout) from qkv, the
 * forward's out and lse, and dout [T, nh * 128]; dl_ws is a [2, batch, nh, seq_len] fp32
 * workspace (rowsum(dout * out), then the log2-domain lse). seq_len must be a multiple of 128.
 * Deterministic (no atomics). */
DM_API int dm_attention_bwd(const void* qkv, const void* out, const void* dout, const float* lse, int T,
                            int seq_len, int nh, int nkv, int head_dim, float* dl_ws, void* dqkv, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* DM_MOE_H_ */
