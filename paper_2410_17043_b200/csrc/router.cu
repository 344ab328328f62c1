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
// x is streamed by TMA (2-D tiles of 64 tokens x 256 h into a 4-stage
// shared-memory ring) beside the matching block of the gate, prepared once
// per layer as fp32 in a lane-major expert-pair layout; the FMAs run as
// fp32x2 (FFMA2) over expert pairs -- two independent RN fmas, same bits.
#include <cuda.h>

#include "common.cuh"
#include "tc_helpers.cuh"

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

// 16-byte shared-memory load by 32-bit shared address (a generic load of the
// realigned dynamic smem pointer would go through the long-scoreboard path)
__device__ __forceinline__ int4 lds128(uint32_t addr) {
  int4 v;
  asm volatile("ld.shared.v4.b32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(addr));
  return v;
}

// top-k + softmax + destinations (thread per token, first 64 threads) and the
// tile's destination histogram (warp-aggregated), shared by both router kernels
// presel (sel_s / sv_s non-null): the selection was made by warp_topk, read it from shared memory
template <bool PRESEL = false>
__device__ __forceinline__ void route_tail(const float (*logit_s)[MAXE + 1], int* hist_s, int t0, int T, int E,
                                           int k, const int32_t* __restrict__ gpu_of_expert, int n,
                                           int rank_base, int tokens_per_rank, int32_t* __restrict__ topk_idx,
                                           float* __restrict__ topk_w, int32_t* __restrict__ slot_dst,
                                           int32_t* __restrict__ blk_cnt, int32_t* __restrict__ counts,
                                           const int (*sel_s)[MAXK] = nullptr, const float (*sv_s)[MAXK] = nullptr) {
  const int lane = threadIdx.x & 31;
  if (threadIdx.x < TILE) {
    const int tl = threadIdx.x, t = t0 + tl;
    const bool valid = t < T;
    int dst[MAXK];
    if (valid) {
      int sel[MAXK];
      float sv[MAXK];
      if (PRESEL) {
        for (int s = 0; s < k; s++) {
          sel[s] = sel_s[tl][s];
          sv[s] = sv_s[tl][s];
        }
      } else {
        uint64_t taken = 0;
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

__device__ __forceinline__ void mbar_arrive_cta(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(tc::smem_u32(bar)) : "memory");
}

constexpr int XS = 4;                      // stages
constexpr int REP = 8;                     // experts per pass
constexpr int XBYTES = TILE * 256 * 2;     // x part of a stage: 64 tokens x 256 h (bf16)
constexpr int WBYTES = REP * 256 * 4;      // gate part: the pass's 8 experts x 256 h (fp32, lane-major pairs)
constexpr int XCHUNK = XBYTES + WBYTES;    // bytes per stage

__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];"
      ::"r"(tc::smem_u32(dst)), "l"(reinterpret_cast<uint64_t>(map)), "r"(tc::smem_u32(bar)), "r"(c0), "r"(c1)
      : "memory");
}
__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   tc::smem_u32(dst)), "l"(src), "r"(bytes), "r"(tc::smem_u32(bar))
               : "memory");
}

// The gate, prepared once per layer (aurora_route_prepare_gate): widened to
// fp32 (exact) and laid out per (8-expert pass, 256-h chunk) block of 2048
// floats so that one 16-byte shared load per lane yields two expert pairs:
//   float index ((p * 4 + jp) * 32 + l) * 4 + q,  q = 2 * (jj & 1) + (e & 1)
//   for expert e = 8 pass + 2 p + (q & 1), h = 256 chunk + 8 l + 2 jp + (q >> 1)
// (experts past E are zero). Lane l's accumulation order is unchanged.
__global__ void prepare_gate_kernel(const __nv_bfloat16* __restrict__ w, int E, int H, float* __restrict__ wp) {
  const int h_chunks = H / 256, passes = (E + REP - 1) / REP;
  const long long total = (long long)passes * h_chunks * 2048;
  for (long long o = (long long)blockIdx.x * blockDim.x + threadIdx.x; o < total; o += (long long)gridDim.x * blockDim.x) {
    const int blk = (int)(o >> 11), f = (int)(o & 2047);
    const int pass = blk / h_chunks, c = blk - pass * h_chunks;
    const int q = f & 3, l = (f >> 2) & 31, jp = (f >> 7) & 3, p = f >> 9;
    const int e = pass * REP + 2 * p + (q & 1), h = c * 256 + 8 * l + 2 * jp + (q >> 1);
    wp[o] = e < E ? __bfloat162float(w[(size_t)e * H + h]) : 0.0f;
  }
}

// one 256-h chunk of the warp's 8 tokens x 8 experts: fp32x2 FMAs (FFMA2) over
// expert pairs, x broadcast into both halves; per (token, expert) the same
// sequential fmaf chain over h = 256 i + 8 l + jj as the scalar definition
template <int XB = XBYTES>
__device__ __forceinline__ void gate_chunk(float2 (&acc)[8][REP / 2], uint32_t stage_u, int warp, int lane) {
  float2 wp[REP / 2][8];
#pragma unroll
  for (int p = 0; p < REP / 2; p++)
#pragma unroll
    for (int jp = 0; jp < 4; jp++) {
      const int4 v = lds128(stage_u + XB + ((p * 4 + jp) * 32 + lane) * 16);
      wp[p][2 * jp] = make_float2(__int_as_float(v.x), __int_as_float(v.y));
      wp[p][2 * jp + 1] = make_float2(__int_as_float(v.z), __int_as_float(v.w));
    }
  const uint32_t xb = stage_u + (warp * 8) * 512 + 16 * lane;
  // tokens in groups of TG, jj outer: TG * 4 independent accumulator chains per step
  constexpr int TG = 4;
#pragma unroll
  for (int t0 = 0; t0 < 8; t0 += TG) {
    float xf[TG][8];
#pragma unroll
    for (int t = 0; t < TG; t++) bf16x8_to_f32(lds128(xb + (t0 + t) * 512), xf[t]);
#pragma unroll
    for (int jj = 0; jj < 8; jj++)
#pragma unroll
      for (int t = 0; t < TG; t++) {
        const float2 xx = make_float2(xf[t][jj], xf[t][jj]);
#pragma unroll
        for (int p = 0; p < REP / 2; p++) acc[t0 + t][p] = __ffma2_rn(xx, wp[p][jj], acc[t0 + t][p]);
      }
  }
}

// xor tree over the lanes: reduce-scatter per group of 32 (token, expert) pairs;
// lane q ends with pair g * 32 + q (t = pair / 8, e = pair % 8)
__device__ __forceinline__ float gate_reduce(const float2 (&acc)[8][REP / 2], int g, int lane) {
  float v[32];
#pragma unroll
  for (int qq = 0; qq < 32; qq++) {
    const int pr = g * 32 + qq, t = pr / REP, e = pr % REP;
    v[qq] = (e & 1) ? acc[t][e >> 1].y : acc[t][e >> 1].x;
  }
#pragma unroll
  for (int o = 16, sz = 32; o >= 1; o >>= 1, sz >>= 1) {
    const bool upper = lane & o;
#pragma unroll
    for (int qq = 0; qq < sz / 2; qq++) {
      float mine = upper ? v[qq + sz / 2] : v[qq];
      float send = upper ? v[qq] : v[qq + sz / 2];
      float got = __shfl_xor_sync(0xffffffffu, send, o);
      v[qq] = mine + got;
    }
  }
  return v[0];
}

template <int NS = XS, int NW = WARPS>
__device__ __forceinline__ void init_ring(uint64_t* full, uint64_t* empty) {
  if (threadIdx.x == 0) {
    for (int q = 0; q < NS; q++) {
      tc::mbar_init(&full[q], 1);
      tc::mbar_init(&empty[q], NW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
}

// E <= 8 (one pass) or no logits workspace: one CTA per 64-token tile, every pass, then the tail
__global__ void __launch_bounds__(WARPS * 32, 1) route_tma_kernel(
    const __grid_constant__ CUtensorMap xmap, const float* __restrict__ wperm,
    const float* __restrict__ bias, int T, int H, int E, int k,
    const int32_t* __restrict__ gpu_of_expert, int n, int rank_base, int tokens_per_rank,
    int32_t* __restrict__ topk_idx, float* __restrict__ topk_w, int32_t* __restrict__ slot_dst,
    int32_t* __restrict__ blk_cnt, int32_t* __restrict__ counts) {
  extern __shared__ __align__(1024) uint8_t xs_raw[];
  uint8_t* xs = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(xs_raw) + 1023) & ~uintptr_t(1023));
  __shared__ float logit_s[TILE][MAXE + 1];
  __shared__ int hist_s[AUR_MAXN];
  __shared__ __align__(8) uint64_t full[XS], empty[XS];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint32_t xs_u = tc::smem_u32(xs);
  const int t0 = blockIdx.x * TILE;
  const int h_chunks = H / 256, passes = (E + REP - 1) / REP, total = passes * h_chunks;
  if (tid < AUR_MAXN) hist_s[tid] = 0;
  init_ring(full, empty);
  __syncthreads();
  // stage q: x chunk (q % h_chunks) of the CTA's tokens + gate block q (pass q / h_chunks)
  auto fill = [&](int q, int st) {
    tc::mbar_expect_tx(&full[st], XCHUNK);
    tma_load_2d(xs + st * XCHUNK, &xmap, &full[st], 256 * (q % h_chunks), t0);
    bulk_load(xs + st * XCHUNK + XBYTES, wperm + (size_t)q * 2048, WBYTES, &full[st]);
  };
  if (tid == 0)
    for (int q = 0; q < XS && q < total; q++) fill(q, q);

  for (int pass = 0; pass < passes; pass++) {
    const int e0 = pass * REP;
    float2 acc[8][REP / 2];
#pragma unroll
    for (int t = 0; t < 8; t++)
#pragma unroll
      for (int p = 0; p < REP / 2; p++) acc[t][p] = make_float2(0.0f, 0.0f);
    for (int i = 0; i < h_chunks; i++) {
      const int q = pass * h_chunks + i, s = q % XS;
      const uint32_t ph = (uint32_t)(q / XS) & 1u;
      tc::mbar_wait(&full[s], ph);
      gate_chunk(acc, xs_u + s * XCHUNK, warp, lane);
      __syncwarp();
      if (lane == 0) mbar_arrive_cta(&empty[s]);
      if (tid == 0 && q + XS < total) {  // refill this stage once every warp is done with it
        tc::mbar_wait(&empty[s], ph);
        fill(q + XS, s);
      }
    }
#pragma unroll
    for (int g = 0; g < 2; g++) {
      const float v = gate_reduce(acc, g, lane);
      const int pr = g * 32 + lane, tq = pr / REP, eq = e0 + pr % REP;
      if (eq < E) logit_s[warp * 8 + tq][eq] = v + bias[eq];
    }
  }
  __syncthreads();
  route_tail(logit_s, hist_s, t0, T, E, k, gpu_of_expert, n, rank_base, tokens_per_rank, topk_idx, topk_w,
             slot_dst, blk_cnt, counts);
}

// E > 8: the (64-token tile, 8-expert pass) units of the gate are spread over a
// persistent grid (C5: 256 tiles x 8 passes = 2048 units over 148 CTAs, so the
// FMA-bound work balances across the SMs instead of running 256 whole tiles in
// 1.7 waves). The x / gate stages stream through one TMA ring across units;
// each unit stores its 64 x 8 logits (+ bias) and route_tail_kernel finishes
// every tile. Same per-lane order and xor tree as route_tma_kernel: same bits.
// NW warps x 8 tokens per unit, NS stages. 16 warps (four per scheduler: the FFMA2
// chains need more than two warps to keep the FMA pipe busy) with two stages beat
// 12 x 3 and 8 x 4 (C5: 247 / 258 / 277 us)
template <int NW, int NS>
__global__ void __launch_bounds__(NW * 32, 1) route_units_kernel(
    const __grid_constant__ CUtensorMap xmap, const float* __restrict__ wperm,
    const float* __restrict__ bias, int T, int H, int E, float* __restrict__ logits) {
  extern __shared__ __align__(1024) uint8_t xs_raw[];
  uint8_t* xs = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(xs_raw) + 1023) & ~uintptr_t(1023));
  constexpr int UT = NW * 8, UXB = UT * 512, UCH = UXB + WBYTES;  // unit tokens, x bytes, stage bytes
  __shared__ __align__(8) uint64_t full[NS], empty[NS];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint32_t xs_u = tc::smem_u32(xs);
  const int h_chunks = H / 256, passes = (E + REP - 1) / REP, tiles = (T + UT - 1) / UT;
  const int units = tiles * passes;
  const int my_units = units > (int)blockIdx.x ? (units - 1 - (int)blockIdx.x) / (int)gridDim.x + 1 : 0;
  const int total = my_units * h_chunks;
  init_ring<NS, NW>(full, empty);
  __syncthreads();
  // stage q: chunk q % h_chunks of this CTA's unit q / h_chunks (unit u = tile * passes + pass)
  auto fill = [&](int q, int st) {
    const int u = (int)blockIdx.x + (q / h_chunks) * (int)gridDim.x, c = q % h_chunks;
    tc::mbar_expect_tx(&full[st], UCH);
    tma_load_2d(xs + st * UCH, &xmap, &full[st], 256 * c, (u / passes) * UT);
    bulk_load(xs + st * UCH + UXB, wperm + ((size_t)(u % passes) * h_chunks + c) * 2048, WBYTES, &full[st]);
  };
  if (tid == 0)
    for (int q = 0; q < NS && q < total; q++) fill(q, q);
  for (int ui = 0; ui < my_units; ui++) {
    const int u = (int)blockIdx.x + ui * (int)gridDim.x;
    const int t0 = (u / passes) * UT, e0 = (u % passes) * REP;
    float2 acc[8][REP / 2];
#pragma unroll
    for (int t = 0; t < 8; t++)
#pragma unroll
      for (int p = 0; p < REP / 2; p++) acc[t][p] = make_float2(0.0f, 0.0f);
    for (int i = 0; i < h_chunks; i++) {
      const int q = ui * h_chunks + i, s = q % NS;
      const uint32_t ph = (uint32_t)(q / NS) & 1u;
      tc::mbar_wait(&full[s], ph);
      gate_chunk<UXB>(acc, xs_u + s * UCH, warp, lane);
      __syncwarp();
      if (lane == 0) mbar_arrive_cta(&empty[s]);
      if (tid == 0 && q + NS < total) {
        tc::mbar_wait(&empty[s], ph);
        fill(q + NS, s);
      }
    }
#pragma unroll
    for (int g = 0; g < 2; g++) {
      const float v = gate_reduce(acc, g, lane);
      const int pr = g * 32 + lane, t = t0 + warp * 8 + pr / REP, eq = e0 + pr % REP;
      if (eq < E && t < T) logits[(size_t)t * E + eq] = v + bias[eq];
    }
  }
}

// the tail of the split router: one CTA per 64-token tile (blk_cnt row = blockIdx.x)
__global__ void __launch_bounds__(WARPS * 32) route_tail_kernel(
    const float* __restrict__ logits, int T, int E, int k, const int32_t* __restrict__ gpu_of_expert, int n,
    int rank_base, int tokens_per_rank, int32_t* __restrict__ topk_idx, float* __restrict__ topk_w,
    int32_t* __restrict__ slot_dst, int32_t* __restrict__ blk_cnt, int32_t* __restrict__ counts) {
  __shared__ int hist_s[AUR_MAXN];
  __shared__ int sel_s[TILE][MAXK];
  __shared__ float sv_s[TILE][MAXK];
  const int t0 = blockIdx.x * TILE;
  if (threadIdx.x < AUR_MAXN) hist_s[threadIdx.x] = 0;
  // 4 threads per token (all 256 threads: the tile's 64 tokens at once); thread
  // sub holds experts e = sub + 4 j. Each of the k rounds takes the larger logit,
  // the lower index on ties -- the sequential scan's choice.
  {
    const int tl = threadIdx.x >> 2, sub = threadIdx.x & 3, t = t0 + tl;
    float v[16];
    uint32_t live = 0;
#pragma unroll
    for (int j = 0; j < 16; j++) {
      const int e = sub + 4 * j;
      v[j] = 0.0f;
      if (t < T && e < E) {
        v[j] = logits[(size_t)t * E + e];
        live |= 1u << j;
      }
    }
    for (int s = 0; s < k; s++) {
      float bv = 0.0f;
      int bi = 1 << 30;
#pragma unroll
      for (int j = 0; j < 16; j++)
        if (((live >> j) & 1) && (bi == (1 << 30) || v[j] > bv)) { bv = v[j]; bi = sub + 4 * j; }
#pragma unroll
      for (int o = 1; o <= 2; o <<= 1) {
        const float ov = __shfl_xor_sync(0xffffffffu, bv, o);
        const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
        if (oi != (1 << 30) && (bi == (1 << 30) || ov > bv || (ov == bv && oi < bi))) { bv = ov; bi = oi; }
      }
      if (sub == 0 && t < T) {
        sel_s[tl][s] = bi;
        sv_s[tl][s] = bv;
      }
      if (bi != (1 << 30) && (bi & 3) == sub) live &= ~(1u << (bi >> 2));
    }
  }
  __syncthreads();
  route_tail<true>(nullptr, hist_s, t0, T, E, k, gpu_of_expert, n, rank_base, tokens_per_rank, topk_idx, topk_w,
                   slot_dst, blk_cnt, counts, sel_s, sv_s);
}

typedef CUresult (*EncodeTiledFnR)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                   const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

bool make_x_map(CUtensorMap* m, const void* x, uint64_t T, uint64_t H, uint32_t box_rows = TILE) {
  static EncodeTiledFnR fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      return false;
    fn = reinterpret_cast<EncodeTiledFnR>(p);
  }
  cuuint64_t dims[2] = {H, T};
  cuuint64_t strides[1] = {H * 2};
  cuuint32_t box[2] = {256, box_rows};
  cuuint32_t estr[2] = {1, 1};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(x), dims, strides, box, estr,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// K3: token permutation. CTA = 64 threads = the 64 tokens of one route tile.
// list(i, j) = rank i's tokens bound for j in ascending order; the entry for
// token t lands at soff[i][j] + (entries of earlier tiles of rank i, from
// blk_cnt) + (entries of earlier tokens in this tile, from warp ballots).
// Grouped placement (several experts per rank, GROUPED): the receiver keeps its
// rows grouped by local expert -- group (r_local, local expert) of a process,
// rows ordered by (sender, token) -- and each dispatched row lands straight at
// its position in every group it belongs to (the engine reads the positions from
// the row's meta record), so no receiver-side sort or gather is needed.
struct GroupedArgs {
  const int32_t* blk_cnt_e;       // [T/64][E] tokens of each tile choosing each expert
  const int32_t* cnt_e;           // [n][E] tokens of each sender rank choosing each expert (all senders)
  const int32_t* gpu_of_expert;   // [E]
  int E, G, n_local;              // experts, experts per rank, ranks per process (uniform)
  int32_t* g_off;                 // [n_local * G + 1] this process's packed group offsets
  int32_t* g_rows;                // [n_local * G]
  int4* const* ginfo;             // [n] per rank: its process's {recv row, weight, single, 0} per packed row (nullable)
};

template <bool GROUPED>
__global__ void __launch_bounds__(TILE) pack_kernel(
    const int32_t* __restrict__ slot_dst, const int32_t* __restrict__ blk_cnt,
    const int32_t* __restrict__ counts, int T, int k, int n, int rank_base, int tokens_per_rank,
    int32_t* __restrict__ send_list, int32_t* __restrict__ pos, int32_t* __restrict__ soff,
    int32_t* __restrict__ roff, int32_t* __restrict__ rtot, int32_t* __restrict__ rloc,
    int32_t* __restrict__ rrem, const int32_t* __restrict__ topk_idx,
    const float* __restrict__ topk_w, const int32_t* __restrict__ local_of_expert,
    uint8_t* __restrict__ meta, int meta_bytes, const GroupedArgs ga) {
  __shared__ int base_s[AUR_MAXN];   // entries of earlier tiles of rank i, per destination
  __shared__ int soff_s[AUR_MAXN];   // start of list(i, j) in rank i's send list
  __shared__ int warp0_s[AUR_MAXN];  // entries of warp 0 per destination
  __shared__ int gbase_s[GROUPED ? MAXE : 1];                 // grouped position of this tile's first row per expert
  __shared__ unsigned long long tmask_s[GROUPED ? MAXE : 1];  // tokens of the tile choosing each expert
  __shared__ int roffi_s[GROUPED ? AUR_MAXN : 1];               // roff[i][j] of this tile's sender i
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
  if (GROUPED) {
    const int E = ga.E;
    if (tl < n) {  // receiver j = tl: local rows first, then the other senders in index order
      const int j = tl;
      int ro = 0;
      if (i != j) {
        ro = counts[j * n + j];
        for (int i2 = 0; i2 < i; i2++)
          if (i2 != j) ro += counts[i2 * n + j];
      }
      roffi_s[j] = ro;
    }
    __shared__ int rows_s[MAXE], key_s[MAXE];
    int rows_e = 0, earlier_senders = 0, key = 0, proc = 0;
    if (tl < E) {  // expert tl: rows of its group (all senders), rows from senders before i
      const int e = tl, j = ga.gpu_of_expert[e];
      proc = j / ga.n_local;
      key = j * ga.G + local_of_expert[e];  // group order: (rank, local expert)
      for (int i2 = 0; i2 < n; i2++) {
        const int c = ga.cnt_e[i2 * E + e];
        rows_e += c;
        if (i2 < i) earlier_senders += c;
      }
      rows_s[e] = rows_e;
      key_s[e] = key;
    }
    __syncthreads();
    if (tl < E) {  // the group's offset in its process's packed buffer, this tile's base
      const int e = tl;
      int before = 0;
      for (int e2 = 0; e2 < E; e2++)
        if (key_s[e2] < key && key_s[e2] / (ga.n_local * ga.G) == proc) before += rows_s[e2];
      key = key - proc * ga.n_local * ga.G;  // the group's index inside its process
      int acc = 0;
      for (int b = b_first; b < (int)blockIdx.x; b++) acc += ga.blk_cnt_e[(size_t)b * E + e];
      gbase_s[e] = before + earlier_senders + acc;
      tmask_s[e] = 0ull;
      if (blockIdx.x == 0 && proc * ga.n_local == rank_base) {  // this process's packed groups
        const int g = key;
        ga.g_rows[g] = rows_e;
        ga.g_off[g] = before;
      }
    }
    if (blockIdx.x == 0 && tl == 0) {  // total rows of this process
      int tot = 0;
      for (int e2 = 0; e2 < E; e2++)
        if (key_s[e2] / (ga.n_local * ga.G) == rank_base / ga.n_local) tot += rows_s[e2];
      ga.g_off[ga.n_local * ga.G] = tot;
    }
    __syncthreads();
    if (t < T)
      for (int s2 = 0; s2 < k; s2++) atomicOr(&tmask_s[topk_idx[(size_t)t * k + s2]], 1ull << tl);
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
        if (meta) {  // the row's expert slots on rank j: {local expert (grouped: the
                     // row's position in that expert's group), gate weight} or {-1, 0}
          int2* m = reinterpret_cast<int2*>(meta + ((size_t)i_local * tokens_per_rank * k +
                                                    soff_s[j] + p) * meta_bytes);
          int nhere = 0;
          for (int q = 0; q < k; q++) nhere += full[q] == j;
          for (int q = 0; q < k; q++) {
            const bool here = full[q] == j;
            const int eg = topk_idx[(size_t)t * k + q];
            int e = -1;
            if (here) {
              if (GROUPED)
                e = gbase_s[eg] + __popcll(tmask_s[eg] & ((1ull << tl) - 1ull));
              else
                e = local_of_expert[eg];
            }
            const int wb = here ? __float_as_int(topk_w[(size_t)t * k + q]) : 0;
            m[q] = make_int2(e, wb);
            // grouped: the receiver's per-position record for GEMM2's single-row epilogue
            if (GROUPED && here && ga.ginfo) ga.ginfo[j][e] = make_int4(roffi_s[j] + p, wb, nhere == 1 ? 1 : 0, 0);
          }
          if (GROUPED)  // padding records: no position (the engine reads meta_bytes / 8 records)
            for (int q = k; q < meta_bytes / 8; q++) m[q] = make_int2(-1, 0);
        }
      }
    }
  }
}

}  // namespace

extern "C" int aurora_route_gate_floats(int E, int H) {
  if (E < 1 || E > MAXE || H <= 0 || H % 256) return -AURORA_EINVAL;
  return ((E + REP - 1) / REP) * H * REP;
}

extern "C" int aurora_route_prepare_gate(const void* w_gate, int E, int H, float* gate_prep, void* stream) {
  if (!w_gate || !gate_prep || E < 1 || E > MAXE || H <= 0 || H % 256) return AURORA_EINVAL;
  prepare_gate_kernel<<<256, 256, 0, (cudaStream_t)stream>>>((const __nv_bfloat16*)w_gate, E, H, gate_prep);
  AUR_CHECK_LAUNCH();
  return AURORA_OK;
}

extern "C" int aurora_route(const void* x, const float* gate_prep, const float* bias, int T, int H,
                            int E, int k, const int32_t* gpu_of_expert, int n, int rank_base,
                            int tokens_per_rank, int32_t* topk_idx, float* topk_w,
                            int32_t* slot_dst, int32_t* blk_cnt, int32_t* counts, float* logits,
                            void* stream) {
  if (T <= 0 || H % 256 || k < 1 || k > MAXK || k > E || n < 1 || n > AUR_MAXN ||
      tokens_per_rank % TILE || T % tokens_per_rank || !x || !gate_prep || !bias)
    return AURORA_EINVAL;
  const int blocks = (T + TILE - 1) / TILE;
  cudaStream_t s = (cudaStream_t)stream;
  if (E < 1 || E > MAXE) return AURORA_EUNSUPPORTED;
  CUtensorMap xmap;
  if (!make_x_map(&xmap, x, (uint64_t)T, (uint64_t)H)) return AURORA_ECUDA;
  constexpr int dyn = XS * XCHUNK + 1024;
  constexpr int UNW = 16, UNS = 2;  // balanced units: 16 warps x 8 tokens, 2 stages
  constexpr int udyn = UNS * (UNW * 8 * 512 + WBYTES) + 1024;
  static bool attr = false;
  if (!attr) {
    if (cudaFuncSetAttribute(route_tma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, dyn) != cudaSuccess ||
        cudaFuncSetAttribute(route_units_kernel<UNW, UNS>, cudaFuncAttributeMaxDynamicSharedMemorySize, udyn) !=
            cudaSuccess)
      return AURORA_ECUDA;
    attr = true;
  }
  if (logits && E > REP) {  // several 8-expert passes: balance (tile, pass) units over a persistent grid
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    CUtensorMap umap;
    if (!make_x_map(&umap, x, (uint64_t)T, (uint64_t)H, UNW * 8)) return AURORA_ECUDA;
    const int units = ((T + UNW * 8 - 1) / (UNW * 8)) * ((E + REP - 1) / REP);
    route_units_kernel<UNW, UNS><<<units < sms ? units : sms, UNW * 32, udyn, s>>>(umap, gate_prep, bias, T, H, E,
                                                                                   logits);
    route_tail_kernel<<<blocks, WARPS * 32, 0, s>>>(logits, T, E, k, gpu_of_expert, n, rank_base, tokens_per_rank,
                                                     topk_idx, topk_w, slot_dst, blk_cnt, counts);
    AUR_CHECK_LAUNCH();
    return AURORA_OK;
  }
  route_tma_kernel<<<blocks, WARPS * 32, dyn, s>>>(xmap, gate_prep, bias, T, H, E, k, gpu_of_expert, n, rank_base,
                                                   tokens_per_rank, topk_idx, topk_w, slot_dst, blk_cnt, counts);
  AUR_CHECK_LAUNCH();
  return AURORA_OK;
}

// per 64-token tile and expert: tokens choosing the expert (+ per sender rank totals)
__global__ void __launch_bounds__(TILE) expert_hist_kernel(const int32_t* __restrict__ topk_idx, int T, int k, int E,
                                                         int rank_base, int tokens_per_rank,
                                                         int32_t* __restrict__ blk_cnt_e, int32_t* __restrict__ cnt_e) {
  __shared__ int h[MAXE];
  const int tl = threadIdx.x, t = blockIdx.x * TILE + tl;
  if (tl < E) h[tl] = 0;
  __syncthreads();
  if (t < T)
    for (int s = 0; s < k; s++) atomicAdd(&h[topk_idx[(size_t)t * k + s]], 1);
  __syncthreads();
  if (tl < E) {
    blk_cnt_e[(size_t)blockIdx.x * E + tl] = h[tl];
    const int src = rank_base + (blockIdx.x * TILE) / tokens_per_rank;
    if (h[tl]) atomicAdd(&cnt_e[src * E + tl], h[tl]);
  }
}

extern "C" int aurora_expert_hist(const int32_t* topk_idx, int T, int k, int E, int rank_base, int tokens_per_rank,
                                  int32_t* blk_cnt_e, int32_t* cnt_e, void* stream) {
  if (!topk_idx || !blk_cnt_e || !cnt_e || T <= 0 || k < 1 || k > MAXK || E < 1 || E > MAXE ||
      tokens_per_rank % TILE || T % tokens_per_rank)
    return AURORA_EINVAL;
  expert_hist_kernel<<<T / TILE, TILE, 0, (cudaStream_t)stream>>>(topk_idx, T, k, E, rank_base, tokens_per_rank,
                                                                   blk_cnt_e, cnt_e);
  AUR_CHECK_LAUNCH();
  return AURORA_OK;
}

extern "C" int aurora_pack_grouped(const int32_t* slot_dst, const int32_t* blk_cnt, const int32_t* counts,
                                   int T, int k, int n, int rank_base, int tokens_per_rank,
                                   int32_t* send_list, int32_t* pos, int32_t* soff, int32_t* roff,
                                   int32_t* rtot, int32_t* rloc, int32_t* rrem,
                                   const int32_t* topk_idx, const float* topk_w,
                                   const int32_t* local_of_expert, void* meta,
                                   const int32_t* blk_cnt_e, const int32_t* cnt_e, const int32_t* gpu_of_expert,
                                   int E, int G, int n_local, int32_t* g_off, int32_t* g_rows,
                                   void* const* ginfo_bufs, void* stream) {
  if (T <= 0 || k < 1 || k > MAXK || n < 1 || n > AUR_MAXN || tokens_per_rank % TILE ||
      T % tokens_per_rank || !soff || !roff || !rtot || !rloc || !rrem || !meta || !blk_cnt_e || !cnt_e ||
      !gpu_of_expert || !local_of_expert || !g_off || !g_rows || E < 1 || E > MAXE || G < 1 || n_local < 1 ||
      n % n_local || rank_base % n_local || E != n * G)
    return AURORA_EINVAL;
  const GroupedArgs ga{blk_cnt_e, cnt_e, gpu_of_expert, E, G, n_local, g_off, g_rows,
                       reinterpret_cast<int4* const*>(ginfo_bufs)};
  pack_kernel<true><<<T / TILE, TILE, 0, (cudaStream_t)stream>>>(
      slot_dst, blk_cnt, counts, T, k, n, rank_base, tokens_per_rank, send_list, pos, soff, roff,
      rtot, rloc, rrem, topk_idx, topk_w, local_of_expert, (uint8_t*)meta, ((k * 8 + 15) / 16) * 16, ga);
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
  pack_kernel<false><<<T / TILE, TILE, 0, (cudaStream_t)stream>>>(
      slot_dst, blk_cnt, counts, T, k, n, rank_base, tokens_per_rank, send_list, pos, soff, roff,
      rtot, rloc, rrem, topk_idx, topk_w, local_of_expert, (uint8_t*)meta, ((k * 8 + 15) / 16) * 16,
      GroupedArgs{});
  AUR_CHECK_LAUNCH();
  return AURORA_OK;
}
