/*
 * TEST INFRASTRUCTURE ONLY -- CPU oracle for the router / traffic-matrix /
 * pack stage (kernels K1 + K3). The reference has no router: it models the
 * gate only as LayerProfile.gate_work (reference pkg/src/moeplan/core.py:194-221)
 * and the traffic matrix as TrafficMatrix (core.py:75-117), built per source
 * shard as in workload.py:55-87. This file pins the arithmetic the device
 * router is DEFINED by:
 *
 *   raw(t,e) = tree32( p_0..p_31 ),
 *     p_l    = fold over i = 0..H/256-1, jj = 0..7 of
 *              acc = fmaf(x[t][256 i + 8 l + jj], w[e][256 i + 8 l + jj], acc), acc0 = 0
 *     tree32 = pairwise lane sums with xor offsets 16, 8, 4, 2, 1
 *   logit(t,e) = raw(t,e) + bias[e]                      (fp32)
 *   top-k: repeatedly take the largest logit, lowest expert index on ties
 *   weights: softmax over the k selected logits (Mixtral convention)
 *
 * bf16 x bf16 products are exact in fp32, so fmaf == mul+add here and only
 * the summation order matters; the tree and the lane striding are fixed, so
 * the logits (hence expert choice, traffic matrix and token permutation) are
 * bit-exact between this file and the kernel.
 */
#include <math.h>
#include <stdint.h>
#include <string.h>

static float bf16_to_f32(uint16_t b) {
  uint32_t u = (uint32_t)b << 16;
  float f;
  memcpy(&f, &u, 4);
  return f;
}

/* logits[T][E] (bias included) */
void oracle_router_logits(const uint16_t *x, const uint16_t *w, const float *bias,
                          int T, int H, int E, float *logits) {
  int iters = H / 256;
  for (int t = 0; t < T; t++) {
    const uint16_t *xr = x + (size_t)t * H;
    for (int e = 0; e < E; e++) {
      const uint16_t *wr = w + (size_t)e * H;
      float p[32];
      for (int l = 0; l < 32; l++) {
        float acc = 0.0f;
        for (int i = 0; i < iters; i++)
          for (int jj = 0; jj < 8; jj++) {
            int h = 256 * i + 8 * l + jj;
            acc = fmaf(bf16_to_f32(xr[h]), bf16_to_f32(wr[h]), acc);
          }
        p[l] = acc;
      }
      for (int o = 16; o >= 1; o >>= 1)
        for (int l = 0; l < o; l++) p[l] = p[l] + p[l + o];
      logits[(size_t)t * E + e] = p[0] + bias[e];
    }
  }
}

/* top-k with lowest-index tie-break + softmax over the selected logits. */
void oracle_router_topk(const float *logits, int T, int E, int k,
                        int32_t *topk_idx, float *topk_w) {
  for (int t = 0; t < T; t++) {
    const float *l = logits + (size_t)t * E;
    uint64_t taken[2] = {0, 0};
    float sel[16];
    for (int s = 0; s < k; s++) {
      int best = -1;
      float bv = 0.0f;
      for (int e = 0; e < E; e++) {
        if (taken[e >> 6] >> (e & 63) & 1) continue;
        if (best < 0 || l[e] > bv) { best = e; bv = l[e]; }
      }
      taken[best >> 6] |= 1ull << (best & 63);
      topk_idx[(size_t)t * k + s] = best;
      sel[s] = bv;
    }
    float m = sel[0], z = 0.0f, ex[16];
    for (int s = 0; s < k; s++) { ex[s] = expf(sel[s] - m); z += ex[s]; }
    for (int s = 0; s < k; s++) topk_w[(size_t)t * k + s] = ex[s] / z;
  }
}
