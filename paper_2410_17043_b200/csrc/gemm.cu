// K5: expert FFNs as grouped GEMMs on the 5th-gen tensor cores.
//
// C[g] = A[g] . B[g]^T for every local expert g (bf16 in, fp32 accumulate in
// TMEM, bf16 out) -- the one genuinely dense contraction of the MoE layer,
// which the reference only models as LayerProfile.ffn_work_per_token
// (pkg/src/moeplan/core.py:194-221; sim.py:71-89).
//
// Persistent, warp-specialised kernel, one CTA per SM:
//   warp 0  TMA producer: 128x64 A tile + 256x64 B tile per stage, SW128
//   warp 1  TMEM allocator + single-thread tcgen05.mma issuer (M=128, N=256, K=16)
//   warps 2-5 epilogue: tcgen05.ld 32x32b -> registers -> bf16 -> global
// 4-stage smem ring (full/empty mbarriers), 2 TMEM accumulators of 256
// columns (tmem_full/tmem_empty) so tile t's epilogue overlaps tile t+1's MMAs.
// Tiles are (group, n-tile, m-tile) with m fastest, so CTAs running at the
// same time share one B (weight) tile through L2 and A stays L2-resident.
// Group row counts are read on the device: no host synchronisation.
//
// Epilogue 1 (SwiGLU) expects B rows interleaved in 128-row blocks
// (gate block, up block): the 256-column tile holds matching gate / up
// columns and emits silu(gate) * up for 128 output columns.
#include <cuda.h>
#include <stdlib.h>

#include "common.cuh"

// the CTA-pair variant (gemm2sm.cu)
int aurora_launch_grouped_2sm(const void* a, const void* b, void* c, const int32_t* m_start,
                              const int32_t* m_rows, int G, int64_t cap, int64_t map_rows, int N,
                              int K, int epilogue, int32_t* tile_ctr, int num_sms, cudaStream_t stream,
                              const AuroraScatterArgs* scatter, const int32_t* cluster_part, int part_gp,
                              const AuroraArrivalArgs* arrival, int after_gemm);

namespace {

constexpr int BM = 128, BN = 256, BK = 64, STAGES = 4;
constexpr int UMMA_K = 16;
constexpr int THREADS = 192;
constexpr int A_BYTES = BM * BK * 2;  // 16 KB
constexpr int B_BYTES = BN * BK * 2;  // 32 KB
constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
constexpr int TMEM_COLS = 512;        // 2 accumulators x 256 fp32 columns
constexpr int MAX_GROUPS = 64;
constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + 1024 /*align*/ + 256 /*barriers*/;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@!P1 bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, uint64_t* bar,
                                            int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4}], [%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
      : "memory");
}

// K-major operand, 128-byte swizzle, 8-row core-matrix groups 1024 B apart
__device__ __forceinline__ uint64_t sw128_desc(const void* smem) {
  const uint64_t addr = smem_u32(smem);
  return ((addr & 0x3FFFFull) >> 4) | (1ull << 16) /*LBO (ignored for SW128 K-major)*/ |
         (64ull << 32) /*SBO = 1024 B*/ | (1ull << 46) /*sm100 version*/ | (2ull << 61) /*SW128*/;
}

// kind::f16 instruction descriptor: D f32, A/B bf16, both K-major, M x N
constexpr uint32_t IDESC = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(BN >> 3) << 17) |
                           ((uint32_t)(BM >> 4) << 24);

__device__ __forceinline__ void umma_bf16(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc,
                                          uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(IDESC), "r"(accumulate));
}
__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}

#define TMEM_LD32(taddr, r)                                                                       \
  asm volatile(                                                                                   \
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14," \
      "%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"              \
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),       \
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),   \
        "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]),             \
        "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]),             \
        "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])              \
      : "r"(taddr))

__device__ __forceinline__ void tmem_ld_wait() {
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

struct TileIter {
  int n_tiles_n;       // N / BN
  int total;           // total tiles
  int prefix[MAX_GROUPS + 1];
  int mt[MAX_GROUPS];  // m-tiles per group
  int ms[MAX_GROUPS];  // first row of the group's range (m_start)
};

// Tile t -> (group, m-tile, n-tile). Inside a group, tiles walk blocks of
// `gm` m-tiles: within a block the m-tile varies fastest (CTAs running
// together share one weight tile), and the block's A rows (gm x 128 x K)
// stay L2-resident while every n-tile passes over them.
__device__ __forceinline__ void tile_coords(const TileIter& it, int G, int gm, int t, int& g,
                                            int& mt, int& nt) {
  int lo = 0, hi = G - 1;  // the last g with prefix[g] <= t
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (it.prefix[mid] <= t) lo = mid;
    else hi = mid - 1;
  }
  g = lo;
  const int local = t - it.prefix[g];
  const int per_block = gm * it.n_tiles_n;
  const int sb = local / per_block, rem = local - sb * per_block;
  const int rows = min(gm, it.mt[g] - sb * gm);
  mt = sb * gm + rem % rows;
  nt = rem / rows;
}

__device__ __forceinline__ float silu_mul(float g, float u) { return g / (1.0f + __expf(-g)) * u; }

__global__ void __launch_bounds__(THREADS, 1)
    grouped_gemm_kernel(const __grid_constant__ CUtensorMap map_a,
                        const __grid_constant__ CUtensorMap map_b, __nv_bfloat16* __restrict__ c,
                        const int32_t* __restrict__ m_start, const int32_t* __restrict__ m_rows,
                        int G, long long cap, int N, int K,
                        int epilogue, int group_m) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_base_s = reinterpret_cast<uint32_t*>(tempty + 2);
  __shared__ TileIter it;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    it.n_tiles_n = N / BN;
    int acc = 0;
    for (int g = 0; g < G; g++) {
      const int m = m_rows[g];
      it.ms[g] = m_start ? m_start[g] : 0;
      it.mt[g] = (m + BM - 1) / BM;
      it.prefix[g] = acc;
      acc += it.mt[g] * it.n_tiles_n;
    }
    it.prefix[G] = acc;
    it.total = acc;
    for (int s = 0; s < STAGES; s++) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; a++) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 128);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_base_s)),
                 "r"(TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_base_s;
  const int k_blocks = K / BK;

  if (warp == 0) {
    if (lane == 0) {  // ---------------- TMA producer
      int s = 0;
      uint32_t ph = 0;
      for (int t = blockIdx.x; t < it.total; t += gridDim.x) {
        int g, mt, nt;
        tile_coords(it, G, group_m, t, g, mt, nt);
        const int a_row = (int)(g * cap) + it.ms[g] + mt * BM;
        const int b_row = g * N + nt * BN;
        for (int kb = 0; kb < k_blocks; kb++) {
          mbar_wait(&empty[s], ph ^ 1);
          uint8_t* sa = smem + s * STAGE_BYTES;
          mbar_expect_tx(&full[s], STAGE_BYTES);
          tma_load_2d(sa, &map_a, &full[s], kb * BK, a_row);
          tma_load_2d(sa + A_BYTES, &map_b, &full[s], kb * BK, b_row);
          if (++s == STAGES) { s = 0; ph ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // ---------------- MMA issuer
      int s = 0;
      uint32_t ph = 0;
      int local = 0;
      for (int t = blockIdx.x; t < it.total; t += gridDim.x, local++) {
        const int acc = local & 1;
        mbar_wait(&tempty[acc], ((local >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t d = tmem_base + acc * BN;
        for (int kb = 0; kb < k_blocks; kb++) {
          mbar_wait(&full[s], ph);
          tc_fence_after();
          uint8_t* sa = smem + s * STAGE_BYTES;
          const uint64_t ad = sw128_desc(sa), bd = sw128_desc(sa + A_BYTES);
#pragma unroll
          for (int k = 0; k < BK / UMMA_K; k++) {
            // advance 32 bytes (16 bf16) along K inside the swizzle atom: +2 in 16-byte units
            umma_bf16(d, ad + 2 * k, bd + 2 * k, (kb | k) != 0);
          }
          umma_commit(&empty[s]);  // frees the stage once these MMAs have read it
          if (++s == STAGES) { s = 0; ph ^= 1; }
        }
        umma_commit(&tfull[acc]);
      }
    }
  } else {  // ---------------- epilogue warps 2..5
    const int quarter = warp & 3;  // TMEM lanes [32*quarter, 32*quarter+32)
    int local = 0;
    for (int t = blockIdx.x; t < it.total; t += gridDim.x, local++) {
      int g, mt, nt;
      tile_coords(it, G, group_m, t, g, mt, nt);
      const int acc = local & 1;
      mbar_wait(&tfull[acc], (local >> 1) & 1);
      tc_fence_after();
      const int row_in_group = mt * BM + quarter * 32 + lane;
      const bool live = row_in_group < m_rows[g];
      const long long row = g * cap + it.ms[g] + row_in_group;
      const uint32_t tbase = tmem_base + ((uint32_t)(quarter * 32) << 16) + acc * BN;
      if (epilogue == 1) {
        __nv_bfloat16* out = c + row * (long long)(N / 2) + nt * (BN / 2);
        for (int c0 = 0; c0 < BN / 2; c0 += 32) {
          uint32_t gr[32], ur[32];
          TMEM_LD32(tbase + c0, gr);
          TMEM_LD32(tbase + BN / 2 + c0, ur);
          tmem_ld_wait();
          if (live) {
            uint32_t packed[16];
#pragma unroll
            for (int q = 0; q < 16; q++) {
              float a0 = silu_mul(__uint_as_float(gr[2 * q]), __uint_as_float(ur[2 * q]));
              float a1 = silu_mul(__uint_as_float(gr[2 * q + 1]), __uint_as_float(ur[2 * q + 1]));
              __nv_bfloat162 h2 = __floats2bfloat162_rn(a0, a1);
              packed[q] = *reinterpret_cast<uint32_t*>(&h2);
            }
            int4* o = reinterpret_cast<int4*>(out + c0);
#pragma unroll
            for (int q = 0; q < 4; q++)
              o[q] = make_int4(packed[4 * q], packed[4 * q + 1], packed[4 * q + 2], packed[4 * q + 3]);
          }
        }
      } else {
        __nv_bfloat16* out = c + row * (long long)N + nt * BN;
        for (int c0 = 0; c0 < BN; c0 += 32) {
          uint32_t r[32];
          TMEM_LD32(tbase + c0, r);
          tmem_ld_wait();
          if (live) {
            uint32_t packed[16];
#pragma unroll
            for (int q = 0; q < 16; q++) {
              __nv_bfloat162 h2 = __floats2bfloat162_rn(__uint_as_float(r[2 * q]), __uint_as_float(r[2 * q + 1]));
              packed[q] = *reinterpret_cast<uint32_t*>(&h2);
            }
            int4* o = reinterpret_cast<int4*>(out + c0);
#pragma unroll
            for (int q = 0; q < 4; q++)
              o[q] = make_int4(packed[4 * q], packed[4 * q + 1], packed[4 * q + 2], packed[4 * q + 3]);
          }
        }
      }
      tc_fence_before();
      mbar_arrive(&tempty[acc]);
    }
  }
  __syncthreads();
  if (warp == 1) {
    __syncwarp();
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                 "r"(TMEM_COLS));
  }
}

// ---------------------------------------------------------------- host side
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                  const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                  const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  }
  return fn;
}

// 2-D bf16 row-major [rows][cols] map with a (box_rows x 64) SW128 box
bool make_map(CUtensorMap* m, const void* base, uint64_t rows, uint64_t cols, uint32_t box_rows) {
  EncodeTiledFn fn = encode_fn();
  if (!fn) return false;
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {cols * 2};
  cuuint32_t box[2] = {BK, box_rows};
  cuuint32_t estr[2] = {1, 1};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box,
            estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// kernel choice: "2sm" = CTA-pair tcgen05 (gemm2sm.cu), "1sm" = this file's kernel
bool use_pair_kernel() {
  static int mode = -1;
  if (mode < 0) {
    const char* e = getenv("AURORA_GEMM");
    mode = (e && e[0] == '1') ? 0 : 1;
  }
  return mode == 1;
}

int launch_grouped(const void* a, const void* b, void* c, const int32_t* m_start,
                   const int32_t* m_rows, int G,
                   int64_t cap, int64_t map_rows, int N, int K, int epilogue, int32_t* tile_ctr, int num_sms,
                   cudaStream_t stream, const AuroraScatterArgs* scatter = nullptr,
                   const int32_t* cluster_part = nullptr, int part_gp = 1,
                   const AuroraArrivalArgs* arrival = nullptr, int after_gemm = 0) {
  // cap > 0: group g owns rows [g*cap, (g+1)*cap); cap == 0: groups packed,
  // m_start[g] absolute, map_rows = rows of the A buffer
  if (cap < 0 || (cap == 0 && (map_rows <= 0 || !m_start))) return AURORA_EINVAL;
  if (map_rows <= 0) map_rows = (int64_t)G * cap;
  if (use_pair_kernel())
    return aurora_launch_grouped_2sm(a, b, c, m_start, m_rows, G, cap, map_rows, N, K, epilogue, tile_ctr, num_sms,
                                     stream, scatter, cluster_part, part_gp, arrival, after_gemm);
  if (cluster_part || arrival) return AURORA_EINVAL;  // partitioned (emulated per-rank compute): pair kernel only
  if (scatter) return AURORA_EINVAL;  // the fused combine lives in the CTA-pair kernel
  if (G < 1 || G > MAX_GROUPS || N % BN || K % BK || N <= 0 || K <= 0 ||
      (epilogue != 0 && epilogue != 1) || !a || !b || !c || !m_rows)
    return AURORA_EINVAL;
  if ((reinterpret_cast<uintptr_t>(a) | reinterpret_cast<uintptr_t>(b)) & 15) return AURORA_EINVAL;
  CUtensorMap ma, mb;
  if (!make_map(&ma, a, (uint64_t)map_rows, K, BM) || !make_map(&mb, b, (uint64_t)G * N, K, BN))
    return AURORA_ECUDA;
  static bool attr_set = false;
  if (!attr_set) {
    if (cudaFuncSetAttribute(grouped_gemm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             SMEM_BYTES) != cudaSuccess)
      return AURORA_ECUDA;
    attr_set = true;
  }
  // m-tile block: ~32 MiB of A rows, re-read from L2 by every n-tile
  const int group_m = (int)max(1LL, min(64LL, (32LL << 20) / ((long long)BM * K * 2)));
  if (num_sms <= 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&num_sms, cudaDevAttrMultiProcessorCount, dev);
  }
  grouped_gemm_kernel<<<num_sms, THREADS, SMEM_BYTES, stream>>>(
      ma, mb, (__nv_bfloat16*)c, m_start, m_rows, G, (long long)cap, N, K, epilogue, group_m);
  AUR_CHECK_LAUNCH();
  return AURORA_OK;
}

}  // namespace

extern "C" int aurora_grouped_gemm(const void* a, const void* b, void* c, const int32_t* m_start,
                                   const int32_t* m_rows,
                                   int G, int64_t cap, int N, int K, int epilogue, int32_t* tile_ctr, int num_sms,
                                   void* stream) {
  return launch_grouped(a, b, c, m_start, m_rows, G, cap, 0, N, K, epilogue, tile_ctr, num_sms,
                        (cudaStream_t)stream);
}

extern "C" int aurora_expert_ffn(const void* a_buf, const void* w13, const void* w2, void* h_buf,
                                 void* y_buf, const int32_t* m_start, const int32_t* m_rows, int G,
                                 int64_t cap, int H,
                                 int F, const int32_t* cluster_part, int32_t* tile_ctr, int num_sms,
                                 void* stream) {
  // h = silu(x W1^T) * (x W3^T): N = 2F interleaved, K = H
  int rc = launch_grouped(a_buf, w13, h_buf, m_start, m_rows, G, cap, 0, 2 * F, H, 1, tile_ctr, num_sms,
                          (cudaStream_t)stream, nullptr, cluster_part);
  if (rc != AURORA_OK) return rc;
  // y = h W2^T: N = H, K = F
  return launch_grouped(h_buf, w2, y_buf, m_start, m_rows, G, cap, 0, H, F, 0, tile_ctr, num_sms,
                        (cudaStream_t)stream, nullptr, cluster_part, 1, nullptr, 1);
}

extern "C" int aurora_expert_ffn_combine(const void* a_buf, const void* w13, const void* w2,
                                         void* h_buf, void* y_buf, const int32_t* m_rows, int G,
                                         int64_t cap, int H, int F, void* const* ret_bufs,
                                         const int32_t* counts, const int32_t* soff,
                                         const int32_t* roff, int n, int rank_base,
                                         int32_t* const* ctrs, int32_t* ticket, int sys,
                                         const int32_t* cluster_part, int32_t* landed, int arrival_pdl,
                                         int32_t* tile_ctr, int num_sms, void* stream) {
  if (!ret_bufs || !counts || !soff || !roff || !ctrs || !ticket) return AURORA_EINVAL;
  // landed != NULL: GEMM1 is arrival-driven -- a tile starts once the dispatch has landed its rows
  const AuroraArrivalArgs arr{landed, counts, roff, n, rank_base, sys ? 1 : 0, arrival_pdl ? 1 : 0};
  int rc = launch_grouped(a_buf, w13, h_buf, nullptr, m_rows, G, cap, 0, 2 * F, H, 1, tile_ctr, num_sms,
                          (cudaStream_t)stream, nullptr, cluster_part, 1, landed ? &arr : nullptr);
  if (rc != AURORA_OK) return rc;
  const AuroraScatterArgs sc{ret_bufs, counts, soff, roff, ctrs, ticket, n, rank_base, sys ? 1 : 0};
  return launch_grouped(h_buf, w2, y_buf, nullptr, m_rows, G, cap, 0, H, F, 0, tile_ctr, num_sms,
                        (cudaStream_t)stream, &sc, cluster_part, 1, nullptr, 1);
}

extern "C" int aurora_expert_ffn_packed_scatter(const void* a_buf, const void* w13, const void* w2, void* h_buf,
                                                void* y_buf, const int32_t* g_off, const int32_t* g_rows, int G,
                                                int64_t a_rows, int H, int F, const void* ginfo, int experts_per_rank,
                                                void* const* ret_bufs, const int32_t* counts, const int32_t* soff,
                                                const int32_t* roff, int n, int rank_base, void* ybuf,
                                                int64_t ycap, int to_ret, int sys, const int32_t* cluster_part,
                                                int32_t* tile_ctr, int num_sms, void* stream) {
  if (!ginfo || !ret_bufs || !counts || !soff || !roff || !ybuf || experts_per_rank < 1) return AURORA_EINVAL;
  int rc = launch_grouped(a_buf, w13, h_buf, g_off, g_rows, G, 0, a_rows, 2 * F, H, 1, tile_ctr, num_sms,
                          (cudaStream_t)stream, nullptr, cluster_part, experts_per_rank);
  if (rc != AURORA_OK) return rc;
  AuroraScatterArgs sc{ret_bufs, counts, soff, roff, nullptr, nullptr, n, rank_base, sys ? 1 : 0};
  sc.ginfo = ginfo;
  sc.G = experts_per_rank;
  sc.ybuf = ybuf;
  sc.ycap = ycap;
  sc.to_ret = to_ret ? 1 : 0;
  return launch_grouped(h_buf, w2, y_buf, g_off, g_rows, G, 0, a_rows, H, F, 0, tile_ctr, num_sms,
                        (cudaStream_t)stream, &sc, cluster_part, experts_per_rank, nullptr, 1);
}

extern "C" int aurora_expert_ffn_packed(const void* a_buf, const void* w13, const void* w2,
                                        void* h_buf, void* y_buf, const int32_t* g_off,
                                        const int32_t* g_rows, int G, int64_t a_rows, int H, int F,
                                        const int32_t* cluster_part, int part_groups, int32_t* tile_ctr,
                                        int num_sms, void* stream) {
  int rc = launch_grouped(a_buf, w13, h_buf, g_off, g_rows, G, 0, a_rows, 2 * F, H, 1, tile_ctr, num_sms,
                          (cudaStream_t)stream, nullptr, cluster_part, part_groups);
  if (rc != AURORA_OK) return rc;
  return launch_grouped(h_buf, w2, y_buf, g_off, g_rows, G, 0, a_rows, H, F, 0, tile_ctr, num_sms,
                        (cudaStream_t)stream, nullptr, cluster_part, part_groups, nullptr, 1);
}
