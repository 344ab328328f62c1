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

// fp32 += bf16 x bf16 with one rounding (fma.rn.f32.bf16 -> FHFMA.BF16, reading either half of a
// packed register directly): the product of two bf16 is exact in fp32, so this is fmaf on the
// widened values -- the same bits, without the widening instructions
__device__ __forceinline__ float fma_bf16_lo(uint32_t a, uint32_t b, float c) {
  unsigned short al, ah, bl, bh;
  asm("mov.b32 {%0, %1}, %2;" : "=h"(al), "=h"(ah) : "r"(a));
  asm("mov.b32 {%0, %1}, %2;" : "=h"(bl), "=h"(bh) : "r"(b));
  asm("fma.rn.f32.bf16 %0, %1, %2, %0;" : "+f"(c) : "h"(al), "h"(bl));
  return c;
}
__device__ __forceinline__ float fma_bf16_hi(uint32_t a, uint32_t b, float c) {
  unsigned short al, ah, bl, bh;
  asm("mov.b32 {%0, %1}, %2;" : "=h"(al), "=h"(ah) : "r"(a));
  asm("mov.b32 {%0, %1}, %2;" : "=h"(bl), "=h"(bh) : "r"(b));
  asm("fma.rn.f32.bf16 %0, %1, %2, %0;" : "+f"(c) : "h"(ah), "h"(bh));
  return c;
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

// E <= 8: one CTA per 64-token tile, 16 warps x 4 tokens, the gate read as bf16 rows (a TMA box of
// 8 experts x 256 h per chunk, from the bf16 copy aurora_route_prepare_gate keeps after the fp32
// block) and every term one FHFMA.BF16 on the packed halves of x and the gate (= fmaf on the
// widened values): no widening instructions, half the gate's shared-memory bytes, and twice the
// warps of route_tma_kernel (whose fp32 gate fragments hold 64 registers per thread). Same per-lane
// chains and xor tree (a reduce-scatter: lane q ends with (token q / 8, expert q % 8)): same bits.
constexpr int BW = 16, BTPW = 4, BS = 5;
constexpr int BXB = TILE * 512, BWB = 8 * 512, BCH = BXB + BWB;
__global__ void __launch_bounds__(BW * 32, 1) route_bf16_kernel(
    const __grid_constant__ CUtensorMap xmap, const __grid_constant__ CUtensorMap wmap,
    const float* __restrict__ bias, int T, int H, int E, int k, const int32_t* __restrict__ gpu_of_expert, int n,
    int rank_base, int tokens_per_rank, int32_t* __restrict__ topk_idx, float* __restrict__ topk_w,
    int32_t* __restrict__ slot_dst, int32_t* __restrict__ blk_cnt, int32_t* __restrict__ counts) {
  extern __shared__ __align__(1024) uint8_t bs_raw[];
  uint8_t* xs = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(bs_raw) + 1023) & ~uintptr_t(1023));
  __shared__ float logit_s[TILE][MAXE + 1];
  __shared__ int hist_s[AUR_MAXN];
  __shared__ __align__(8) uint64_t full[BS], empty[BS];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint32_t xs_u = tc::smem_u32(xs);
  const int t0 = blockIdx.x * TILE, chunks = H / 256;
  if (tid < AUR_MAXN) hist_s[tid] = 0;
  init_ring<BS, BW>(full, empty);
  __syncthreads();
  auto fill = [&](int c, int st) {
    tc::mbar_expect_tx(&full[st], BCH);
    tma_load_2d(xs + st * BCH, &xmap, &full[st], 256 * c, t0);
    tma_load_2d(xs + st * BCH + BXB, &wmap, &full[st], 256 * c, 0);
  };
  if (tid == 0)
    for (int c = 0; c < BS && c < chunks; c++) fill(c, c);
  float acc[BTPW][8];
#pragma unroll
  for (int tt = 0; tt < BTPW; tt++)
#pragma unroll
    for (int e = 0; e < 8; e++) acc[tt][e] = 0.0f;
  for (int c = 0; c < chunks; c++) {
    const int s = c % BS;
    tc::mbar_wait(&full[s], (uint32_t)(c / BS) & 1u);
    const uint32_t st = xs_u + s * BCH;
    uint32_t w[8][4];
#pragma unroll
    for (int e = 0; e < 8; e++) {
      const int4 v = lds128(st + BXB + e * 512 + 16 * lane);
      w[e][0] = (uint32_t)v.x; w[e][1] = (uint32_t)v.y; w[e][2] = (uint32_t)v.z; w[e][3] = (uint32_t)v.w;
    }
#pragma unroll
    for (int tt = 0; tt < BTPW; tt++) {
      const int4 xv = lds128(st + (warp * BTPW + tt) * 512 + 16 * lane);
      const uint32_t xw[4] = {(uint32_t)xv.x, (uint32_t)xv.y, (uint32_t)xv.z, (uint32_t)xv.w};
#pragma unroll
      for (int e = 0; e < 8; e++) {
        float a = acc[tt][e];
#pragma unroll
        for (int q = 0; q < 4; q++) {
          a = fma_bf16_lo(xw[q], w[e][q], a);
          a = fma_bf16_hi(xw[q], w[e][q], a);
        }
        acc[tt][e] = a;
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive_cta(&empty[s]);
    if (tid == 0 && c + BS < chunks) {
      tc::mbar_wait(&empty[s], (uint32_t)(c / BS) & 1u);
      fill(c + BS, s);
    }
  }
  // reduce-scatter over the lanes: lane q ends with pair q = (token q / 8, expert q % 8)
  float v[32];
#pragma unroll
  for (int qq = 0; qq < 32; qq++) v[qq] = acc[qq >> 3][qq & 7];
#pragma unroll
  for (int o = 16, sz = 32; o >= 1; o >>= 1, sz >>= 1) {
    const bool upper = lane & o;
#pragma unroll
    for (int qq = 0; qq < sz / 2; qq++) {
      const float mine = upper ? v[qq + sz / 2] : v[qq];
      const float send = upper ? v[qq] : v[qq + sz / 2];
      v[qq] = mine + __shfl_xor_sync(0xffffffffu, send, o);
    }
  }
  {
    const int tq = lane >> 3, eq = lane & 7;
    if (eq < E) logit_s[warp * BTPW + tq][eq] = v[0] + bias[eq];
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

// ============================================================================
// Tensor-core router (E > 8): the gate's dense contraction on tcgen05, the
// logits that decide anything recomputed exactly.
//
// 1. La = x W_pad^T on the CTA-pair grouped GEMM (gemm2sm.cu; W_pad = the gate
//    padded to 256 rows, bf16 out): an approximation of every logit.
// 2. route_exact_kernel, per token: the m = min(k + 2, E) experts with the
//    largest approximate logits a_e = La_e + bias_e are the candidates; their
//    logits are recomputed in the DEFINED order (same per-lane fmaf chains and
//    xor tree as route_tma_kernel / oracle_router_logits: same bits). Every
//    other expert's logit is bounded above by
//        ub_e = a_e + 2^-8 |La_e| + 2^-20 (|a_e| + 1) + C * S_t,
//        S_t  = sum_h |x_th| max_e |w_eh|   (>= sum_h |x_th w_eh|),
//    covering the bf16 rounding of La, the tensor-core accumulation and the
//    defined order's own rounding: worst cases (K/16 + 32) 2^-23 S_t (one
//    ulp per accumulation step, truncating) and (K/32 + 5) 2^-24 S_t, together
//    < 2^-14.5 S_t at K = 5120; C = 2^-13, a 2.8x margin over the worst case
//    (measured errors are ~100x below it). When the k-th largest exact
//    candidate logit exceeds max ub over the non-candidates, the exact top-k
//    is among the candidates, so the top-k (the lowest index on ties), the
//    softmax weights, the traffic matrix and the permutation are those of the
//    exact logits; otherwise the token's logits are all recomputed exactly
//    (counted in n_fallback). logits[t][e] is then exact for every candidate
//    (and for every expert of a fallback token) and a_e for the others, which
//    lie strictly below the k-th selected value -- route_tail_kernel's top-k
//    over the row is the exact one.
// ============================================================================
constexpr int RX_W = 16, RX_TPW = 4, RX_TOK = RX_W * RX_TPW, RX_NS = 3;
constexpr int RX_XB = RX_TOK * 512;             // x chunk: 64 tokens x 256 h bf16
constexpr int RX_WB = MAXE * 512;               // gate chunk: E x 256 h bf16 (chunk-contiguous layout)
constexpr int RX_STAGE = RX_XB + RX_WB + 1024;  // + max_e |w_eh| for the chunk (256 fp32)

__device__ __forceinline__ uint32_t f2key(float f) {  // order-preserving float -> uint
  const uint32_t b = __float_as_uint(f);
  return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}
__device__ __forceinline__ float key2f(uint32_t k) {
  return __uint_as_float((k & 0x80000000u) ? (k & 0x7fffffffu) : ~k);
}
__device__ __forceinline__ float warp_sum_tree(float v) {  // xor tree 16, 8, 4, 2, 1: every lane ends with it
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// MC candidates per token (>= k + 2); slots past min(k + 2, E) repeat the last candidate and are
// ignored
template <int MC>
__global__ void __launch_bounds__(RX_W * 32, 1) route_exact_kernel(
    const __grid_constant__ CUtensorMap xmap, const __nv_bfloat16* __restrict__ x,
    const __nv_bfloat16* __restrict__ w_gate, const __nv_bfloat16* __restrict__ wchunk,
    const float* __restrict__ wmax, const __nv_bfloat16* __restrict__ la, const float* __restrict__ bias,
    int T, int H, int E, int k, float* __restrict__ logits, int32_t* __restrict__ n_fallback) {
  extern __shared__ __align__(1024) uint8_t rx_raw[];
  uint8_t* xs = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(rx_raw) + 1023) & ~uintptr_t(1023));
  __shared__ __align__(8) uint64_t full[RX_NS], empty[RX_NS];
  __shared__ int fb_s[RX_TOK];
  __shared__ int nfb_s;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint32_t xs_u = tc::smem_u32(xs);
  const int t0 = blockIdx.x * RX_TOK, chunks = H / 256;
  const int m = min(min(k + 2, E), MC);
  const uint32_t wbytes = (uint32_t)E * 512;
  if (tid == 0) nfb_s = 0;
  init_ring<RX_NS, RX_W>(full, empty);
  __syncthreads();
  auto fill = [&](int c, int st) {
    uint8_t* d = xs + st * RX_STAGE;
    tc::mbar_expect_tx(&full[st], RX_XB + wbytes + 1024);
    tma_load_2d(d, &xmap, &full[st], 256 * c, t0);
    bulk_load(d + RX_XB, wchunk + (size_t)c * E * 256, wbytes, &full[st]);
    bulk_load(d + RX_XB + RX_WB, wmax + 256 * c, 1024, &full[st]);
  };
  if (tid == 0)
    for (int c = 0; c < RX_NS && c < chunks; c++) fill(c, c);

  // ---- candidates: the m largest approximate logits (lane holds experts lane, lane + 32)
  uint32_t cpk[RX_TPW][(MC + 3) / 4];
  float thr[RX_TPW];
#pragma unroll
  for (int tt = 0; tt < RX_TPW; tt++) {
    const int t = t0 + warp * RX_TPW + tt;
    float a[2] = {-INFINITY, -INFINITY}, ub[2] = {-INFINITY, -INFINITY};
#pragma unroll
    for (int h = 0; h < 2; h++) {
      const int e = lane + 32 * h;
      if (t < T && e < E) {
        const float l = __bfloat162float(la[(size_t)t * 256 + e]);
        a[h] = l + bias[e];
        ub[h] = a[h] + ldexpf(fabsf(l), -8) + ldexpf(fabsf(a[h]) + 1.0f, -20);
      }
    }
    uint32_t taken = 0, elast = 0;
#pragma unroll
    for (int q = 0; q < (MC + 3) / 4; q++) cpk[tt][q] = 0;
#pragma unroll
    for (int j = 0; j < MC; j++) {
      if (j >= m) {  // padding slot: the last candidate again (its result is ignored)
        cpk[tt][j >> 2] |= elast << (8 * (j & 3));
        continue;
      }
      const bool ok0 = !(taken & 1u) && lane < E, ok1 = !(taken & 2u) && lane + 32 < E;
      const uint32_t k0 = ok0 ? f2key(a[0]) : 0u, k1 = ok1 ? f2key(a[1]) : 0u;
      const bool pick1 = k1 > k0;  // ties: the lower index (lane < lane + 32)
      const uint32_t kb = pick1 ? k1 : k0;
      const uint32_t kmax = __reduce_max_sync(0xffffffffu, kb);
      const uint32_t e = __reduce_min_sync(0xffffffffu, (kb == kmax && (ok0 || ok1)) ? (uint32_t)(lane + (pick1 ? 32 : 0)) : 255u);
      if ((int)e == lane) taken |= 1u;
      if ((int)e == lane + 32) taken |= 2u;
      cpk[tt][j >> 2] |= e << (8 * (j & 3));
      elast = e;
    }
    const uint32_t u0 = (!(taken & 1u) && lane < E) ? f2key(ub[0]) : 0u;
    const uint32_t u1 = (!(taken & 2u) && lane + 32 < E) ? f2key(ub[1]) : 0u;
    const uint32_t um = __reduce_max_sync(0xffffffffu, u0 > u1 ? u0 : u1);
    thr[tt] = um ? key2f(um) : -INFINITY;
  }

  // ---- exact candidate logits: per lane the defined chains over h = 256 c + 8 lane + jj,
  // jj = 2q (low half of word q), 2q + 1 (high half): one FHFMA.BF16 per term
  float acc[RX_TPW][MC], sab[RX_TPW];
#pragma unroll
  for (int tt = 0; tt < RX_TPW; tt++) {
    sab[tt] = 0.0f;
#pragma unroll
    for (int j = 0; j < MC; j++) acc[tt][j] = 0.0f;
  }
  for (int c = 0; c < chunks; c++) {
    const int s = c % RX_NS;
    tc::mbar_wait(&full[s], (uint32_t)(c / RX_NS) & 1u);
    const uint32_t st = xs_u + s * RX_STAGE;
    const uint32_t wst = st + RX_XB + 16 * lane;
    float mh[8];
    {
      const int4 m0 = lds128(st + RX_XB + RX_WB + 32 * lane), m1 = lds128(st + RX_XB + RX_WB + 32 * lane + 16);
      mh[0] = __int_as_float(m0.x); mh[1] = __int_as_float(m0.y); mh[2] = __int_as_float(m0.z); mh[3] = __int_as_float(m0.w);
      mh[4] = __int_as_float(m1.x); mh[5] = __int_as_float(m1.y); mh[6] = __int_as_float(m1.z); mh[7] = __int_as_float(m1.w);
    }
#pragma unroll
    for (int tt = 0; tt < RX_TPW; tt++) {
      const int4 xv = lds128(st + (warp * RX_TPW + tt) * 512 + 16 * lane);
      const uint32_t xw[4] = {(uint32_t)xv.x, (uint32_t)xv.y, (uint32_t)xv.z, (uint32_t)xv.w};
      {
        float xf[8];
        bf16x8_to_f32(xv, xf);
#pragma unroll
        for (int jj = 0; jj < 8; jj++) sab[tt] = fmaf(fabsf(xf[jj]), mh[jj], sab[tt]);
      }
#pragma unroll
      for (int j = 0; j < MC; j++) {
        const uint32_t e = (cpk[tt][j >> 2] >> (8 * (j & 3))) & 0xFFu;
        const int4 wv = lds128(wst + e * 512);
        const uint32_t ww[4] = {(uint32_t)wv.x, (uint32_t)wv.y, (uint32_t)wv.z, (uint32_t)wv.w};
        float a = acc[tt][j];
#pragma unroll
        for (int q = 0; q < 4; q++) {
          a = fma_bf16_lo(xw[q], ww[q], a);
          a = fma_bf16_hi(xw[q], ww[q], a);
        }
        acc[tt][j] = a;
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive_cta(&empty[s]);
    if (tid == 0 && c + RX_NS < chunks) {
      tc::mbar_wait(&empty[s], (uint32_t)(c / RX_NS) & 1u);
      fill(c + RX_NS, s);
    }
  }

  // ---- exact logits, the certificate, the row of logits
  constexpr float C_TC = 1.0f / 8192.0f;
#pragma unroll
  for (int tt = 0; tt < RX_TPW; tt++) {
    const int tl = warp * RX_TPW + tt, t = t0 + tl;
    const float S = warp_sum_tree(sab[tt]) * 1.001f;
    float ex[MC];
    uint32_t ce[MC];
#pragma unroll
    for (int j = 0; j < MC; j++) {
      ce[j] = (cpk[tt][j >> 2] >> (8 * (j & 3))) & 0xFFu;
      const float v = warp_sum_tree(acc[tt][j]);  // every lane: the tree's value
      ex[j] = j < m ? v + bias[ce[j]] : -INFINITY;
    }
    // k-th largest exact candidate logit
    uint32_t used = 0;
    float kth = INFINITY;
    for (int q = 0; q < k; q++) {
      int bj = -1;
      float bv = -INFINITY;
#pragma unroll
      for (int j = 0; j < MC; j++)
        if (j < m && !((used >> j) & 1u) && (bj < 0 || ex[j] > bv)) { bj = j; bv = ex[j]; }
      used |= 1u << bj;
      kth = bv;
    }
    const bool certified = m >= E || kth > thr[tt] + C_TC * S;
    if (t < T) {
      if (certified) {
#pragma unroll
        for (int h = 0; h < 2; h++) {
          const int e = lane + 32 * h;
          if (e < E) {
            float v = __bfloat162float(la[(size_t)t * 256 + e]) + bias[e];
#pragma unroll
            for (int j = 0; j < MC; j++)
              if (j < m && ce[j] == (uint32_t)e) v = ex[j];
            logits[(size_t)t * E + e] = v;
          }
        }
      } else if (lane == 0) {
        fb_s[atomicAdd(&nfb_s, 1)] = t;
      }
    }
  }
  __syncthreads();
  // ---- fallback (not certified): every logit of the token in the defined order, from global
  // memory; the CTA's 16 warps share the experts (warp w: e = w, w + 16, w + 32, w + 48)
  const int nfb = nfb_s;
  for (int q = 0; q < nfb; q++) {
    const int t = fb_s[q];
    float a[MAXE / RX_W];
#pragma unroll
    for (int r = 0; r < MAXE / RX_W; r++) a[r] = 0.0f;
#pragma unroll 4
    for (int c = 0; c < chunks; c++) {
      float xf[8];
      bf16x8_to_f32(__ldg(reinterpret_cast<const int4*>(x + (size_t)t * H + 256 * c + 8 * lane)), xf);
#pragma unroll
      for (int r = 0; r < MAXE / RX_W; r++) {
        const int e = warp + RX_W * r;
        if (e < E) {
          float wf[8];
          bf16x8_to_f32(__ldg(reinterpret_cast<const int4*>(w_gate + (size_t)e * H + 256 * c + 8 * lane)), wf);
#pragma unroll
          for (int jj = 0; jj < 8; jj++) a[r] = fmaf(xf[jj], wf[jj], a[r]);
        }
      }
    }
#pragma unroll
    for (int r = 0; r < MAXE / RX_W; r++) {
      const int e = warp + RX_W * r;
      const float v = warp_sum_tree(a[r]);
      if (e < E && lane == 0) logits[(size_t)t * E + e] = v + bias[e];
    }
  }
  if (tid == 0 && nfb && n_fallback) atomicAdd(n_fallback, nfb);
}

// gate in the exact kernel's layout: wchunk[c][e][256] = w[e][256 c ..], wmax[h] = max_e |w[e][h]|,
// wpad[256][H] = w rows (rows >= E zero)
__global__ void prepare_gate_tc_kernel(const __nv_bfloat16* __restrict__ w, int E, int H,
                                       __nv_bfloat16* __restrict__ wchunk, float* __restrict__ wmax,
                                       __nv_bfloat16* __restrict__ wpad) {
  const long long total = 256LL * H;
  for (long long o = (long long)blockIdx.x * blockDim.x + threadIdx.x; o < total; o += (long long)gridDim.x * blockDim.x) {
    const int e = (int)(o / H), h = (int)(o % H);
    const __nv_bfloat16 v = e < E ? w[(size_t)e * H + h] : __float2bfloat16(0.0f);
    wpad[o] = v;
    if (e < E) wchunk[((size_t)(h / 256) * E + e) * 256 + (h % 256)] = v;
    if (e == 0) {
      float mx = 0.0f;
      for (int q = 0; q < E; q++) mx = fmaxf(mx, fabsf(__bfloat162float(w[(size_t)q * H + h])));
      wmax[h] = mx;
    }
  }
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
  // E <= 8: + the bf16 rows [8][H] (zero past E) route_bf16_kernel reads, after the fp32 block
  return ((E + REP - 1) / REP) * H * REP + (E <= REP ? 4 * H : 0);
}

__global__ void prepare_gate_bf16_kernel(const __nv_bfloat16* __restrict__ w, int E, int H,
                                         __nv_bfloat16* __restrict__ wb) {
  for (int o = blockIdx.x * blockDim.x + threadIdx.x; o < 8 * H; o += gridDim.x * blockDim.x)
    wb[o] = o / H < E ? w[o] : __float2bfloat16(0.0f);
}

extern "C" int aurora_route_prepare_gate(const void* w_gate, int E, int H, float* gate_prep, void* stream) {
  if (!w_gate || !gate_prep || E < 1 || E > MAXE || H <= 0 || H % 256) return AURORA_EINVAL;
  prepare_gate_kernel<<<256, 256, 0, (cudaStream_t)stream>>>((const __nv_bfloat16*)w_gate, E, H, gate_prep);
  if (E <= REP)
    prepare_gate_bf16_kernel<<<256, 256, 0, (cudaStream_t)stream>>>(
        (const __nv_bfloat16*)w_gate, E, H, reinterpret_cast<__nv_bfloat16*>(gate_prep + (size_t)H * REP));
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
  if (E <= REP) {  // bf16 gate rows after the fp32 block (aurora_route_prepare_gate)
    constexpr int bdyn = BS * BCH + 1024;
    static bool battr = cudaFuncSetAttribute(route_bf16_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bdyn) ==
                        cudaSuccess;
    if (!battr) return AURORA_ECUDA;
    CUtensorMap wmap;
    if (!make_x_map(&wmap, gate_prep + (size_t)H * REP, 8, (uint64_t)H, 8)) return AURORA_ECUDA;
    route_bf16_kernel<<<blocks, BW * 32, bdyn, s>>>(xmap, wmap, bias, T, H, E, k, gpu_of_expert, n, rank_base,
                                                    tokens_per_rank, topk_idx, topk_w, slot_dst, blk_cnt, counts);
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

__global__ void set_rows_kernel(int32_t* rows, int T) { *rows = T; }

extern "C" int aurora_route_tc_bytes(int E, int H) {  // bytes of the tensor-core router's gate copies
  if (E < 9 || E > MAXE || H <= 0 || H % 256) return -AURORA_EINVAL;
  return 256 * H * 2 + E * H * 2 + H * 4;
}

extern "C" int aurora_route_prepare_gate_tc(const void* w_gate, int E, int H, void* gate_tc, void* stream) {
  if (!w_gate || !gate_tc || E < 9 || E > MAXE || H <= 0 || H % 256) return AURORA_EINVAL;
  uint8_t* b = (uint8_t*)gate_tc;
  __nv_bfloat16* wpad = (__nv_bfloat16*)b;
  __nv_bfloat16* wchunk = (__nv_bfloat16*)(b + (size_t)256 * H * 2);
  float* wmax = (float*)(b + (size_t)256 * H * 2 + (size_t)E * H * 2);
  prepare_gate_tc_kernel<<<256, 256, 0, (cudaStream_t)stream>>>((const __nv_bfloat16*)w_gate, E, H, wchunk, wmax, wpad);
  AUR_CHECK_LAUNCH();
  return AURORA_OK;
}

extern "C" int aurora_route_tc(const void* x, const void* w_gate, const void* gate_tc, const float* bias, int T,
                               int H, int E, int k, const int32_t* gpu_of_expert, int n, int rank_base,
                               int tokens_per_rank, int32_t* topk_idx, float* topk_w, int32_t* slot_dst,
                               int32_t* blk_cnt, int32_t* counts, float* logits, void* la_buf,
                               int32_t* t_rows, int32_t* tile_ctr, int32_t* n_fallback, void* stream) {
  if (T <= 0 || H % 256 || H > 8192 || k < 1 || k > MAXK || k > E || E < 9 || E > MAXE || n < 1 || n > AUR_MAXN ||
      tokens_per_rank % TILE || T % tokens_per_rank || !x || !w_gate || !gate_tc || !bias || !logits || !la_buf ||
      !t_rows)
    return AURORA_EINVAL;
  cudaStream_t s = (cudaStream_t)stream;
  const uint8_t* b = (const uint8_t*)gate_tc;
  const __nv_bfloat16* wpad = (const __nv_bfloat16*)b;
  const __nv_bfloat16* wchunk = (const __nv_bfloat16*)(b + (size_t)256 * H * 2);
  const float* wmax = (const float*)(b + (size_t)256 * H * 2 + (size_t)E * H * 2);
  // 1. approximate logits on the tensor cores: one group of T rows, N = 256 (the padded gate), K = H
  //    (the GEMM reads its row count on the device: written here, so a stale value cannot feed the
  //    certificate approximations of another batch)
  set_rows_kernel<<<1, 1, 0, s>>>(t_rows, T);
  int rc = aurora_grouped_gemm(x, wpad, la_buf, nullptr, t_rows, 1, (int64_t)T, 256, H, 0, tile_ctr, 0, stream);
  if (rc != AURORA_OK) return rc;
  // 2. exact candidates + certificate (fallback: the whole row)
  CUtensorMap xmap;
  if (!make_x_map(&xmap, x, (uint64_t)T, (uint64_t)H, RX_TOK)) return AURORA_ECUDA;
  constexpr int rdyn = RX_NS * RX_STAGE + 1024;
  static bool attr = cudaFuncSetAttribute(route_exact_kernel<8>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          rdyn) == cudaSuccess &&
                     cudaFuncSetAttribute(route_exact_kernel<10>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          rdyn) == cudaSuccess;
  if (!attr) return AURORA_ECUDA;
  auto kern = k + 2 <= 8 ? route_exact_kernel<8> : route_exact_kernel<10>;
  kern<<<(T + RX_TOK - 1) / RX_TOK, RX_W * 32, rdyn, s>>>(
      xmap, (const __nv_bfloat16*)x, (const __nv_bfloat16*)w_gate, wchunk, wmax, (const __nv_bfloat16*)la_buf, bias,
      T, H, E, k, logits, n_fallback);
  // 3. top-k, weights, destinations, histograms over the (certified) logits
  route_tail_kernel<<<(T + TILE - 1) / TILE, WARPS * 32, 0, s>>>(logits, T, E, k, gpu_of_expert, n, rank_base,
                                                                  tokens_per_rank, topk_idx, topk_w, slot_dst,
                                                                  blk_cnt, counts);
  AUR_CHECK_LAUNCH();
  return AURORA_OK;
}
