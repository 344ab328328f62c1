// K1 router (top-k gating + GPU x GPU traffic histogram) and K3 pack (token
// permutation into per-destination send lists).
//
// The reference has no router: it models the gate as LayerProfile.gate_work
// (pkg/src/moeplan/core.py:194-221) and consumes its output as a
// TrafficMatrix (core.py:75-117) of one batch shard per GPU (workload.py:55-87).
// The arithmetic below DEFINES the router (oracle/router_oracle.c restates
// it bit-for-bit):
//   raw(t,e) = xor-tree over 32 lanes (offsets 16,8,4,2,1) of
//              p_l = sequential fmaf over h = 256 i + 8 l + jj  (i asc, jj asc)
//   logit    = raw + bias[e];  top-k with lowest index on ties;
//   weights  = softmax over the k selected logits.
// The tree is evaluated as a reduce-scatter (lane q ends with pair q), which
// has the same tree shape, hence the same bits, as the butterfly.
//
// HBM-bound: x is streamed once with 16-byte non-allocating loads; w_gate
// (E*H*2 bytes) stays L1/L2-resident.
#include "common.cuh"

namespace {

constexpr int TILE = 64;      // tokens per CTA (blk_cnt granularity)
constexpr int WARPS = 8;      // 256 threads
constexpr int MAXK = 8;
constexpr int MAXE = 64;

__device__ __forceinline__ void bf16x8_to_f32(const int4& v, float* f) {
  const uint32_t w[4] = {(uint32_t)v.x, (uint32_t)v.y, (uint32_t)v.z, (uint32_t)v.w};
#pragma unroll
  for (int q = 0; q < 4; q++) {
    f[2 * q] = __uint_as_float(w[q] << 16);
    f[2 * q + 1] = __uint_as_float(w[q] & 0xffff0000u);
  }
}

// One warp computes the logits of TG tokens x EP experts (TG*EP == 32) and
// leaves pair q = lane (token q / EP, expert q % EP) in its return value.
template <int TG, int EP>
__device__ __forceinline__ float warp_logits(const int4* __restrict__ xrow[TG],
                                             const int4* __restrict__ wrow, int h_chunks, int lane,
                                             int hv, int e_valid) {
  static_assert(TG * EP == 32, "tile");
  float acc[TG][EP];
#pragma unroll
  for (int t = 0; t < TG; t++)
#pragma unroll
    for (int e = 0; e < EP; e++) acc[t][e] = 0.0f;
  for (int i = 0; i < h_chunks; i++) {
    const int c = 32 * i + lane;  // 16-byte chunk index within the row
    float xf[TG][8];
#pragma unroll
    for (int t = 0; t < TG; t++) {
      int4 v = ld_nc_v4(xrow[t] + c);
      bf16x8_to_f32(v, xf[t]);
    }
#pragma unroll
    for (int e = 0; e < EP; e++) {
      // experts past the last one of this pass re-read a valid row; their sums are dropped
      int4 wv = __ldg(wrow + (size_t)min(e, e_valid - 1) * hv + c);
      float wf[8];
      bf16x8_to_f32(wv, wf);
#pragma unroll
      for (int t = 0; t < TG; t++)
#pragma unroll
        for (int jj = 0; jj < 8; jj++) acc[t][e] = fmaf(xf[t][jj], wf[jj], acc[t][e]);
    }
  }
  // reduce-scatter: 32 values per lane -> 1, keeping the upper half when (lane & o)
  float v[32];
#pragma unroll
  for (int q = 0; q < 32; q++) v[q] = acc[q / EP][q % EP];
#pragma unroll
  for (int o = 16, s = 32; o >= 1; o >>= 1, s >>= 1) {
    const bool upper = lane & o;
#pragma unroll
    for (int q = 0; q < s / 2; q++) {
      float mine = upper ? v[q + s / 2] : v[q];
      float send = upper ? v[q] : v[q + s / 2];
      float got = __shfl_xor_sync(0xffffffffu, send, o);
      v[q] = mine + got;
    }
  }
  return v[0];
}

// top-k + softmax + destinations (thread per token, first 64 threads) and the
// tile's destination histogram (warp-aggregated), shared by both router kernels
__device__ __forceinline__ void route_tail(const float (*logit_s)[MAXE + 1], int* hist_s, int t0, int T, int E,
                                           int k, const int32_t* __restrict__ gpu_of_expert, int n,
                                           int rank_base, int tokens_per_rank, int32_t* __restrict__ topk_idx,
                                           float* __restrict__ topk_w, int32_t* __restrict__ slot_dst,
                                           int32_t* __restrict__ blk_cnt, int32_t* __restrict__ counts) {
  const int lane = threadIdx.x & 31;
  if (threadIdx.x < TILE) {
    const int tl = threadIdx.x, t = t0 + tl;
    const bool valid = t < T;
    int dst[MAXK];
    if (valid) {
      uint64_t taken = 0;
      int sel[MAXK];
      float sv[MAXK];
      for (int s = 0; s < k; s++) {
        int best = -1;
        float bv = 0.0f;
        for (int e = 0; e < E; e++) {
          if ((taken >> e) & 1) continue;
          float l = logit_s[tl][e];
          if (best < 0 || l > bv) { best = e; bv = l; }
        }
        taken |= 1ull << best;
        sel[s] = best;
        sv[s] = bv;
      }
      float z = 0.0f, ex[MAXK];
      for (int s = 0; s < k; s++) { ex[s] = expf(sv[s] - sv[0]); z += ex[s]; }
      for (int s = 0; s < k; s++) {
        topk_idx[(size_t)t * k + s] = sel[s];
        topk_w[(size_t)t * k + s] = ex[s] / z;
        int g = gpu_of_expert[sel[s]];
        bool dup = false;
        for (int q = 0; q < s; q++) dup |= (gpu_of_expert[sel[q]] == g);
        dst[s] = dup ? -1 : g;
        slot_dst[(size_t)t * k + s] = dup ? -(g + 1) : g;  // duplicates encoded as -(rank+1)
      }
    }
    // warp-aggregated histogram: one shared atomic per distinct destination per warp
    const unsigned active = __ballot_sync(0xffffffffu, valid);
    for (int s = 0; s < k; s++) {
      int dd = valid ? dst[s] : -1;
      unsigned peers = __match_any_sync(0xffffffffu, dd);
      if (valid && dd >= 0 && (__ffs(peers & active) - 1) == lane) atomicAdd(&hist_s[dd], __popc(peers));
    }
  }
  __syncthreads();
  if (threadIdx.x < n) {
    const int c = hist_s[threadIdx.x];
    blk_cnt[(size_t)blockIdx.x * n + threadIdx.x] = c;
    const int src = rank_base + t0 / tokens_per_rank;
    if (c) atomicAdd(&counts[src * n + threadIdx.x], c);
  }
}

template <int TG, int EP>
__global__ void __launch_bounds__(WARPS * 32) route_kernel(
    const __nv_bfloat16* __restrict__ x, const __nv_bfloat16* __restrict__ wg,
    const float* __restrict__ bias, int T, int H, int E, int k,
    const int32_t* __restrict__ gpu_of_expert, int n, int rank_base, int tokens_per_rank,
    int32_t* __restrict__ topk_idx, float* __restrict__ topk_w, int32_t* __restrict__ slot_dst,
    int32_t* __restrict__ blk_cnt, int32_t* __restrict__ counts) {
  __shared__ float logit_s[TILE][MAXE + 1];
  __shared__ int hist_s[AUR_MAXN];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int t0 = blockIdx.x * TILE;
  const int hv = H / 8;         // int4 per row
  const int h_chunks = H / 256;
  if (threadIdx.x < AUR_MAXN) hist_s[threadIdx.x] = 0;

  // ---- logits: warp w owns tokens [t0 + 8w, t0 + 8w + 8)
  for (int tg = 0; tg < 8; tg += TG) {
    const int tb = t0 + warp * 8 + tg;
    const int4* xrow[TG];
#pragma unroll
    for (int t = 0; t < TG; t++) {
      int tt = min(tb + t, T - 1);
      xrow[t] = reinterpret_cast<const int4*>(x + (size_t)tt * H);
    }
    for (int e0 = 0; e0 < E; e0 += EP) {
      const int4* wrow = reinterpret_cast<const int4*>(wg + (size_t)e0 * H);
      float r = warp_logits<TG, EP>(xrow, wrow, h_chunks, lane, hv, min(EP, E - e0));
      const int tq = lane / EP, eq = e0 + lane % EP;
      if (eq < E) logit_s[warp * 8 + tg + tq][eq] = r + bias[eq];
    }
  }
  __syncthreads();

  route_tail(logit_s, hist_s, t0, T, E, k, gpu_of_expert, n, rank_base, tokens_per_rank, topk_idx, topk_w,
             slot_dst, blk_cnt, counts);
}

// Many experts (E > 8): the gate no longer fits L1, and streaming it from L2
// for every 4-token group makes the router L2-bound. Here each CTA stages, per
// pass of 8 experts and per 256-wide h chunk, that gate slice once in shared
// memory as fp32 (double-buffered; every warp of the CTA reuses it for its 8
// tokens). The arithmetic is the defined one: lane l of the token's warp
// accumulates h = 256 i + 8 l + jj (i asc, jj asc) with fmaf, then the xor tree.
constexpr int SEP = 8;  // experts per pass
__global__ void __launch_bounds__(WARPS * 32, 1) route_staged_kernel(
    const __nv_bfloat16* __restrict__ x, const __nv_bfloat16* __restrict__ wg,
    const float* __restrict__ bias, int T, int H, int E, int k,
    const int32_t* __restrict__ gpu_of_expert, int n, int rank_base, int tokens_per_rank,
    int32_t* __restrict__ topk_idx, float* __restrict__ topk_w, int32_t* __restrict__ slot_dst,
    int32_t* __restrict__ blk_cnt, int32_t* __restrict__ counts) {
  __shared__ float logit_s[TILE][MAXE + 1];
  __shared__ int hist_s[AUR_MAXN];
  // [buffer][expert][plane][lane * 4 + q]: lane l's h = 8 l + 4 plane + q (conflict-free LDS.128)
  __shared__ __align__(16) float w_s[2][SEP][2][128];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int t0 = blockIdx.x * TILE;
  const int h_chunks = H / 256;
  if (tid < AUR_MAXN) hist_s[tid] = 0;
  const int4* xrow[8];
#pragma unroll
  for (int t = 0; t < 8; t++) xrow[t] = reinterpret_cast<const int4*>(x + (size_t)min(t0 + warp * 8 + t, T - 1) * H);
  const int se = tid >> 5, sl = tid & 31;  // staging: expert se of the pass, lane slot sl (8 h values)

  for (int e0 = 0; e0 < E; e0 += SEP) {
    const int ev = min(SEP, E - e0);
    const int4* wsrc = reinterpret_cast<const int4*>(wg + (size_t)(e0 + min(se, ev - 1)) * H) + sl;
    auto stage = [&](int buf, int4 v) {
      float f[8];
      bf16x8_to_f32(v, f);
      *reinterpret_cast<float4*>(&w_s[buf][se][0][sl * 4]) = make_float4(f[0], f[1], f[2], f[3]);
      *reinterpret_cast<float4*>(&w_s[buf][se][1][sl * 4]) = make_float4(f[4], f[5], f[6], f[7]);
    };
    stage(0, __ldg(wsrc));
    __syncthreads();
    float acc[8][SEP];
#pragma unroll
    for (int t = 0; t < 8; t++)
#pragma unroll
      for (int e = 0; e < SEP; e++) acc[t][e] = 0.0f;
    for (int i = 0; i < h_chunks; i++) {
      const int buf = i & 1;
      int4 wn = make_int4(0, 0, 0, 0);
      if (i + 1 < h_chunks) wn = __ldg(wsrc + 32 * (i + 1));  // next slice, in flight during the FMAs
      float wf[SEP][8];
#pragma unroll
      for (int e = 0; e < SEP; e++) {
        const float4 a = *reinterpret_cast<const float4*>(&w_s[buf][e][0][lane * 4]);
        const float4 b = *reinterpret_cast<const float4*>(&w_s[buf][e][1][lane * 4]);
        wf[e][0] = a.x; wf[e][1] = a.y; wf[e][2] = a.z; wf[e][3] = a.w;
        wf[e][4] = b.x; wf[e][5] = b.y; wf[e][6] = b.z; wf[e][7] = b.w;
      }
#pragma unroll
      for (int t = 0; t < 8; t++) {
        float xf[8];
        bf16x8_to_f32(ld_nc_v4(xrow[t] + 32 * i + lane), xf);
#pragma unroll
        for (int e = 0; e < SEP; e++)
#pragma unroll
          for (int jj = 0; jj < 8; jj++) acc[t][e] = fmaf(xf[jj], wf[e][jj], acc[t][e]);
      }
      if (i + 1 < h_chunks) stage(buf ^ 1, wn);
      __syncthreads();
    }
    // xor tree over the lanes: reduce-scatter per group of 32 pairs (pair p = t * SEP + e)
#pragma unroll
    for (int g = 0; g < 2; g++) {
      float v[32];
#pragma unroll
      for (int q = 0; q < 32; q++) v[q] = acc[(g * 32 + q) / SEP][(g * 32 + q) % SEP];
#pragma unroll
      for (int o = 16, sz = 32; o >= 1; o >>= 1, sz >>= 1) {
        const bool upper = lane & o;
#pragma unroll
        for (int q = 0; q < sz / 2; q++) {
          float mine = upper ? v[q + sz / 2] : v[q];
          float send = upper ? v[q] : v[q + sz / 2];
          float got = __shfl_xor_sync(0xffffffffu, send, o);
          v[q] = mine + got;
        }
      }
      const int pr = g * 32 + lane, tq = pr / SEP, eq = e0 + pr % SEP;
      if (eq < E) logit_s[warp * 8 + tq][eq] = v[0] + bias[eq];
    }
  }
  __syncthreads();
  route_tail(logit_s, hist_s, t0, T, E, k, gpu_of_expert, n, rank_base, tokens_per_rank, topk_idx, topk_w,
             slot_dst, blk_cnt, counts);
}

// K3: token permutation. CTA = 64 threads = the 64 tokens of one route tile.
// list(i, j) = rank i's tokens bound for j in ascending order; the entry for
// token t lands at soff[i][j] + (entries of earlier tiles of rank i, from
// blk_cnt) + (entries of earlier tokens in this tile, from warp ballots).
__global__ void __launch_bounds__(TILE) pack_kernel(
    const int32_t* __restrict__ slot_dst, const int32_t* __restrict__ blk_cnt,
    const int32_t* __restrict__ counts, int T, int k, int n, int rank_base, int tokens_per_rank,
    int32_t* __restrict__ send_list, int32_t* __restrict__ pos, int32_t* __restrict__ soff,
    int32_t* __restrict__ roff, int32_t* __restrict__ rtot, int32_t* __restrict__ rloc,
    int32_t* __restrict__ rrem, const int32_t* __restrict__ topk_idx,
    const float* __restrict__ topk_w, const int32_t* __restrict__ local_of_expert,
    uint8_t* __restrict__ meta, int meta_bytes) {
  __shared__ int base_s[AUR_MAXN];   // entries of earlier tiles of rank i, per destination
  __shared__ int soff_s[AUR_MAXN];   // start of list(i, j) in rank i's send list
  __shared__ int warp0_s[AUR_MAXN];  // entries of warp 0 per destination
  const int tl = threadIdx.x, warp = tl >> 5, lane = tl & 31;
  const int t0 = blockIdx.x * TILE, t = t0 + tl;
  if (blockIdx.x == 0 && tl < n) {  // buffer layout of every rank (thread tl: sender row / receiver column tl)
    int acc = 0;
    for (int j = 0; j < n; j++) {
      soff[tl * n + j] = acc;
      acc += counts[tl * n + j];
    }
    const int loc = counts[tl * n + tl];
    roff[tl * n + tl] = 0;  // local rows first
    acc = loc;
    for (int i = 0; i < n; i++) {
      if (i == tl) continue;
      roff[i * n + tl] = acc;
      acc += counts[i * n + tl];
    }
    rtot[tl] = acc;
    rloc[tl] = loc;
    rrem[tl] = acc - loc;
  }
  const int i_local = t0 / tokens_per_rank, i = rank_base + i_local;
  const int b_first = i_local * (tokens_per_rank / TILE);
  if (tl < n) {
    int so = 0, acc = 0;
    for (int jj = 0; jj < tl; jj++) so += counts[i * n + jj];
    for (int b = b_first; b < (int)blockIdx.x; b++) acc += blk_cnt[(size_t)b * n + tl];
    base_s[tl] = acc;
    soff_s[tl] = so;
  }
  const bool valid = t < T;
  int full[MAXK];  // destination rank of every slot (duplicates decoded)
  uint32_t mine = 0;
  for (int s = 0; s < k; s++) {
    int v = valid ? slot_dst[(size_t)t * k + s] : 0;
    full[s] = v >= 0 ? v : -(v + 1);
    if (valid) mine |= 1u << full[s];
  }
  int* list = send_list + (size_t)i_local * ((size_t)tokens_per_rank * k);
  const unsigned lt = (1u << lane) - 1;
  unsigned bal[AUR_MAXN];
  for (int j = 0; j < n; j++) {
    bal[j] = __ballot_sync(0xffffffffu, (mine >> j) & 1);
    if (warp == 0 && lane == 0) warp0_s[j] = __popc(bal[j]);
  }
  __syncthreads();
  if (valid) {
    for (int s = 0; s < k; s++) {
      const int j = full[s];
      const int p = base_s[j] + (warp ? warp0_s[j] : 0) + __popc(bal[j] & lt);
      pos[(size_t)t * k + s] = p;
      if (slot_dst[(size_t)t * k + s] >= 0) {
        list[soff_s[j] + p] = t - i_local * tokens_per_rank;
        if (meta) {  // the row's expert slots on rank j: {local expert, gate weight} or {-1, 0}
          int2* m = reinterpret_cast<int2*>(meta + ((size_t)i_local * tokens_per_rank * k +
                                                    soff_s[j] + p) * meta_bytes);
          for (int q = 0; q < k; q++) {
            const bool here = full[q] == j;
            const int e = here ? local_of_expert[topk_idx[(size_t)t * k + q]] : -1;
            m[q] = make_int2(e, here ? __float_as_int(topk_w[(size_t)t * k + q]) : 0);
          }
        }
      }
    }
  }
}

}  // namespace

extern "C" int aurora_route(const void* x, const void* w_gate, const float* bias, int T, int H,
                            int E, int k, const int32_t* gpu_of_expert, int n, int rank_base,
                            int tokens_per_rank, int32_t* topk_idx, float* topk_w,
                            int32_t* slot_dst, int32_t* blk_cnt, int32_t* counts, void* stream) {
  if (T <= 0 || H % 256 || k < 1 || k > MAXK || k > E || n < 1 || n > AUR_MAXN ||
      tokens_per_rank % TILE || T % tokens_per_rank)
    return AURORA_EINVAL;
  const int blocks = (T + TILE - 1) / TILE;
  cudaStream_t s = (cudaStream_t)stream;
  const __nv_bfloat16* xb = (const __nv_bfloat16*)x;
  const __nv_bfloat16* wb = (const __nv_bfloat16*)w_gate;
#define LAUNCH(TG, EP)                                                                          \
  route_kernel<TG, EP><<<blocks, WARPS * 32, 0, s>>>(xb, wb, bias, T, H, E, k, gpu_of_expert, n, \
                                                    rank_base, tokens_per_rank, topk_idx,        \
                                                    topk_w, slot_dst, blk_cnt, counts)
  // 4 tokens x 8 experts per warp pass: the gate matrix is streamed once per
  // 4 tokens (ceil(E/8) passes), x re-read from L1 between passes; E <= 4 in one pass
  if (E < 1 || E > MAXE) return AURORA_EUNSUPPORTED;
  if (E <= 4)
    LAUNCH(8, 4);
  else if (E <= 8)
    LAUNCH(4, 8);
  else
    route_staged_kernel<<<blocks, WARPS * 32, 0, s>>>(xb, wb, bias, T, H, E, k, gpu_of_expert, n, rank_base,
                                                     tokens_per_rank, topk_idx, topk_w, slot_dst, blk_cnt, counts);
#undef LAUNCH
  AUR_CHECK_LAUNCH();
  return AURORA_OK;
}

extern "C" int aurora_pack(const int32_t* slot_dst, const int32_t* blk_cnt, const int32_t* counts,
                           int T, int k, int n, int rank_base, int tokens_per_rank,
                           int32_t* send_list, int32_t* pos, int32_t* soff, int32_t* roff,
                           int32_t* rtot, int32_t* rloc, int32_t* rrem,
                           const int32_t* topk_idx, const float* topk_w,
                           const int32_t* local_of_expert, void* meta, void* stream) {
  if (T <= 0 || k < 1 || k > MAXK || n < 1 || n > AUR_MAXN || tokens_per_rank % TILE ||
      T % tokens_per_rank || !soff || !roff || !rtot || !rloc || !rrem)
    return AURORA_EINVAL;
  pack_kernel<<<T / TILE, TILE, 0, (cudaStream_t)stream>>>(
      slot_dst, blk_cnt, counts, T, k, n, rank_base, tokens_per_rank, send_list, pos, soff, roff,
      rtot, rloc, rrem, topk_idx, topk_w, local_of_expert, (uint8_t*)meta, ((k * 8 + 15) / 16) * 16);
  AUR_CHECK_LAUNCH();
  return AURORA_OK;
}
