/*
 * moe_oracle.c — CPU ORACLE for the DisagMoE MoE hot path. TEST INFRASTRUCTURE
 * ONLY: imported by tests/, __graft_entry__.smoke() and bench.py's cpu_baseline
 * leg as the checker; never linked into or called by the product path.
 *
 * PARITY UNPINNED (by the reference): arxiv/paper_2605_11005 ships no MoE
 * arithmetic (SPEC.md:14 puts "real tensor computation/autograd" out of scope;
 * the package is a cost model + simulator, pkg/pyproject.toml:8). This file
 * restates the paper's gating semantics — "trainable gate network to select
 * the top-k experts ... outputs ... reduced by a weighted sum"
 * — under the conventions written in DESIGN.md §3:
 *   1. logits = x . W_g^T in fp32, canonical order:
 *        partial[p][s] (lane p in [0,32), parity s in {0,1}) = fmaf chain over
 *        the 8-element chunks c with c % 32 == p (c ascending) and, inside each
 *        chunk, the elements j with j % 2 == s (j ascending), starting at +0.0f;
 *        v[p] = partial[p][0] + partial[p][1]; then an xor butterfly with
 *        offsets 16,8,4,2,1 of round-to-nearest adds over v.
 *        (Two chains per lane let the GPU use packed fp32x2 FMAs, FFMA2.)
 *   2. top-k by descending logit, ties -> lower expert id.
 *   3. weights = softmax over the k selected logits (== softmax, then
 *      renormalise over the top-k).
 *   4. permutation = stable counting sort by expert over token-major (t, j);
 *      each expert block padded to `align` rows; row_map[t*k+j] = position.
 * Compile with -ffp-contract=off (oracle/Makefile) so every fp32 op is a single
 * IEEE op; fmaf() is the correctly rounded fused multiply-add, bit-identical to
 * the GPU's __fmaf_rn.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

static inline float bf16_to_f32(uint16_t v) {
  uint32_t u = ((uint32_t)v) << 16;
  float f;
  memcpy(&f, &u, 4);
  return f;
}

/* logits[T*E] in the canonical order (convention 1). The loops run over experts
 * innermost so the (exact) fmaf chains vectorise; each (t, e, p) chain still
 * visits its elements in ascending order, which is all the convention fixes.
 * target_clones picks a hardware-FMA build at load time when the CPU has one. */
__attribute__((target_clones("fma", "default")))
static void router_logits_core(const uint16_t* xb, const float* xf, const float* wg, int T, int H, int E,
                               float* logits) {
  const int nch = H / 8;
  float* part = (float*)malloc(sizeof(float) * 64 * (size_t)E);   /* [p][s][e] */
  float* xr = (float*)malloc(sizeof(float) * (size_t)H);
  for (int t = 0; t < T; ++t) {
    for (int h = 0; h < H; ++h) xr[h] = xb ? bf16_to_f32(xb[(size_t)t * H + h]) : xf[(size_t)t * H + h];
    for (int i = 0; i < 64 * E; ++i) part[i] = 0.0f;
    for (int c = 0; c < nch; ++c) {
      for (int j = 0; j < 8; ++j) {
        float* pp = part + ((size_t)(c % 32) * 2 + (j & 1)) * E;
        const int h = c * 8 + j;
        const float xv = xr[h];
        for (int e = 0; e < E; ++e) pp[e] = fmaf(xv, wg[(size_t)e * H + h], pp[e]);
      }
    }
    for (int e = 0; e < E; ++e) {
      float v[32];
      for (int p = 0; p < 32; ++p) v[p] = part[((size_t)p * 2) * E + e] + part[((size_t)p * 2 + 1) * E + e];
      for (int off = 16; off > 0; off >>= 1) {
        float nxt[32];
        for (int l = 0; l < 32; ++l) nxt[l] = v[l] + v[l ^ off];
        memcpy(v, nxt, sizeof(v));
      }
      logits[(size_t)t * E + e] = v[0];
    }
  }
  free(xr);
  free(part);
}

void dm_oracle_router_logits(const uint16_t* x, const float* wg, int T, int H, int E, float* logits) {
  router_logits_core(x, NULL, wg, T, H, E, logits);
}

/* fp32 mode (bytes_per_element 4): the same canonical order on fp32 activations. */
void dm_oracle_router_logits_f32(const float* x, const float* wg, int T, int H, int E, float* logits) {
  router_logits_core(NULL, x, wg, T, H, E, logits);
}

/* idx[T*k], w[T*k] from logits (conventions 2-3). */
void dm_oracle_topk(const float* logits, int T, int E, int k, int32_t* idx, float* w) {
  for (int t = 0; t < T; ++t) {
    const float* row = logits + (size_t)t * E;
    int sel[64];
    float val[64];
    for (int j = 0; j < k; ++j) {
      int be = -1;
      float bv = -INFINITY;
      for (int e = 0; e < E; ++e) {
        int taken = 0;
        for (int q = 0; q < j; ++q) taken |= (sel[q] == e);
        if (taken) continue;
        if (be < 0 || row[e] > bv) { bv = row[e]; be = e; }  /* strict > keeps the lower id on ties */
      }
      sel[j] = be;
      val[j] = bv;
    }
    float s = 0.0f;
    for (int j = 0; j < k; ++j) s += expf(val[j] - val[0]);
    for (int j = 0; j < k; ++j) {
      idx[(size_t)t * k + j] = sel[j];
      w[(size_t)t * k + j] = expf(val[j] - val[0]) / s;
    }
  }
}

void dm_oracle_router(const uint16_t* x, const float* wg, int T, int H, int E, int k, float* logits,
                      int32_t* idx, float* w) {
  dm_oracle_router_logits(x, wg, T, H, E, logits);
  dm_oracle_topk(logits, T, E, k, idx, w);
}

/* Convention 4. src_token has `cap` entries (-1 = padding / unused). */
int dm_oracle_dispatch(const int32_t* idx, int T, int k, int E, int align, int cap, int32_t* counts,
                       int32_t* pad_off, int32_t* row_map, int32_t* src_token) {
  memset(counts, 0, sizeof(int32_t) * (size_t)E);
  for (size_t s = 0; s < (size_t)T * k; ++s) {
    if (idx[s] < 0 || idx[s] >= E) return -1;
    counts[idx[s]]++;
  }
  int acc = 0;
  for (int e = 0; e < E; ++e) {
    pad_off[e] = acc;
    acc += (counts[e] + align - 1) / align * align;
  }
  pad_off[E] = acc;
  if (acc > cap) return -2;
  for (int i = 0; i < cap; ++i) src_token[i] = -1;
  int32_t* next = (int32_t*)malloc(sizeof(int32_t) * (size_t)E);
  for (int e = 0; e < E; ++e) next[e] = pad_off[e];
  for (int t = 0; t < T; ++t)
    for (int j = 0; j < k; ++j) {
      const int e = idx[(size_t)t * k + j];
      const int pos = next[e]++;
      row_map[(size_t)t * k + j] = pos;
      src_token[pos] = t;
    }
  free(next);
  return 0;
}
