// Several experts per rank (E > n, config C5; two models' experts on one GPU,
// config C3): after the dispatch a received row may belong to up to k of the
// rank's local experts (a token crosses the network once per destination).
//   aurora_expert_sort    group the received rows by local expert (counting sort)
//   aurora_gather_rows    materialise each expert's rows contiguously for the GEMM
//   aurora_expert_reduce  pre-reduce: y_row = sum over its local experts of w * FFN_e(row),
//                         so the combine returns ONE row per (token, rank) and the
//                         reversed traffic matrix stays the dispatch transpose
//                         (LayerProfile.d_second, reference core.py:219-221).
#include "common.cuh"

namespace {

constexpr int ROWS_PER_BLOCK = 256;
constexpr int MAX_SLOTS = 8;

__device__ __forceinline__ bool row_valid(long long row, long long cap, const int32_t* rtot,
                                          int rank_base, int& r_local, int& i) {
  r_local = (int)(row / cap);
  i = (int)(row - (long long)r_local * cap);
  return i < rtot[rank_base + r_local];
}

// pass 1: per-block histogram of (local rank, local expert) groups
__global__ void sort_count_kernel(const uint8_t* __restrict__ meta, long long cap, int meta_bytes,
                                  const int32_t* __restrict__ rtot, int n_local, int rank_base,
                                  int k, int G, int32_t* __restrict__ blk_hist) {
  extern __shared__ int hist[];
  const int Gt = n_local * G;
  for (int g = threadIdx.x; g < Gt; g += blockDim.x) hist[g] = 0;
  __syncthreads();
  const long long row = (long long)blockIdx.x * ROWS_PER_BLOCK + threadIdx.x;
  int r, i;
  if (row < (long long)n_local * cap && row_valid(row, cap, rtot, rank_base, r, i)) {
    const int2* m = reinterpret_cast<const int2*>(meta + row * meta_bytes);
    for (int s = 0; s < k; s++) {
      const int e = m[s].x;
      if (e >= 0) atomicAdd(&hist[r * G + e], 1);
    }
  }
  __syncthreads();
  for (int g = threadIdx.x; g < Gt; g += blockDim.x) blk_hist[(size_t)blockIdx.x * Gt + g] = hist[g];
}

// pass 2 (one CTA): group sizes, packed offsets, and every block's base per group
__global__ void sort_scan_kernel(int32_t* __restrict__ blk_hist, int blocks, int Gt,
                                 int32_t* __restrict__ g_off, int32_t* __restrict__ g_rows) {
  __shared__ int rows_s[1024];
  const int g = threadIdx.x;
  int tot = 0;
  if (g < Gt)
    for (int b = 0; b < blocks; b++) tot += blk_hist[(size_t)b * Gt + g];
  rows_s[g] = tot;
  __syncthreads();
  if (g == 0) {  // Gt <= 1024: a short serial scan
    int acc = 0;
    for (int q = 0; q < Gt; q++) {
      const int v = rows_s[q];
      rows_s[q] = acc;
      acc += v;
    }
    g_off[Gt] = acc;
  }
  __syncthreads();
  if (g < Gt) {
    g_rows[g] = tot;
    int base = rows_s[g];
    g_off[g] = base;
    for (int b = 0; b < blocks; b++) {
      const int v = blk_hist[(size_t)b * Gt + g];
      blk_hist[(size_t)b * Gt + g] = base;
      base += v;
    }
  }
}

// pass 3: scatter each (row, slot) to its group position; inv[row][slot] = position
__global__ void sort_scatter_kernel(const uint8_t* __restrict__ meta, long long cap,
                                    int meta_bytes, const int32_t* __restrict__ rtot,
                                    int n_local, int rank_base, int k, int G,
                                    const int32_t* __restrict__ blk_base,
                                    int32_t* __restrict__ g_src, int32_t* __restrict__ inv) {
  extern __shared__ int cursor[];
  const int Gt = n_local * G;
  for (int g = threadIdx.x; g < Gt; g += blockDim.x) cursor[g] = blk_base[(size_t)blockIdx.x * Gt + g];
  __syncthreads();
  const long long row = (long long)blockIdx.x * ROWS_PER_BLOCK + threadIdx.x;
  if (row >= (long long)n_local * cap) return;
  int r, i;
  const bool valid = row_valid(row, cap, rtot, rank_base, r, i);
  const int2* m = reinterpret_cast<const int2*>(meta + row * meta_bytes);
  for (int s = 0; s < k; s++) {
    const int e = valid ? m[s].x : -1;
    int p = -1;
    if (e >= 0) {
      p = atomicAdd(&cursor[r * G + e], 1);
      g_src[p] = (int)row;
    }
    inv[row * k + s] = p;
  }
}

__global__ void gather_rows_kernel(const char* __restrict__ src, char* __restrict__ dst,
                                   const int32_t* __restrict__ idx, const int32_t* __restrict__ count,
                                   int row_bytes) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  const int nwarps = (gridDim.x * blockDim.x) >> 5;
  const int total = *count, vec = row_bytes >> 4;
  for (int p = warp; p < total; p += nwarps) {
    const int4* s = reinterpret_cast<const int4*>(src + (long long)idx[p] * row_bytes);
    int4* d = reinterpret_cast<int4*>(dst + (long long)p * row_bytes);
    for (int u0 = 0; u0 < vec; u0 += 256) {
      int4 v[8];
#pragma unroll
      for (int q = 0; q < 8; q++)
        if (u0 + q * 32 + lane < vec) v[q] = ld_nc_v4(s + u0 + q * 32 + lane);
#pragma unroll
      for (int q = 0; q < 8; q++)
        if (u0 + q * 32 + lane < vec) st_na_v4(d + u0 + q * 32 + lane, v[q]);
    }
  }
}

// one received row: the pre-reduction over its local experts; with the fused
// combine the row is stored straight into its sender's return buffer
__device__ __forceinline__ void reduce_row(const __nv_bfloat16* __restrict__ yg, const int32_t* __restrict__ inv,
                                           const uint8_t* __restrict__ meta, long long row, int r, int i,
                                           int meta_bytes, int rank_base, int k, int H,
                                           __nv_bfloat16* __restrict__ ybuf, const AuroraScatterArgs& sc,
                                           int lane, bool skip_single) {
  const int2* m = reinterpret_cast<const int2*>(meta + row * meta_bytes);
  const int4* src[MAX_SLOTS];
  float w[MAX_SLOTS];
  int ns = 0;
  for (int s = 0; s < k; s++) {
    const int p = inv ? inv[row * k + s] : m[s].x;  // grouped dispatch: the position is in the record
    if (p >= 0) {
      src[ns] = reinterpret_cast<const int4*>(yg + (long long)p * H);
      w[ns] = __int_as_float(m[s].y);
      ns++;
    }
  }
  if (skip_single && ns == 1) return;  // finished by GEMM2's epilogue (packed scatter)
  int4* o = reinterpret_cast<int4*>(ybuf + row * H);
  if (sc.n) {  // sender of this row: lane q tests sender q's block of rank r's receive buffer
    const int rr = rank_base + r;
    const int lo = lane < sc.n ? sc.roff[lane * sc.n + rr] : 0;
    const bool hit = lane < sc.n && i >= lo && i < lo + sc.counts[lane * sc.n + rr];
    const int src = __ffs(__ballot_sync(0xffffffffu, hit)) - 1;
    const int dst_row = __shfl_sync(0xffffffffu, lane < sc.n ? sc.soff[lane * sc.n + rr] + i - lo : 0, src);
    if (src != rr)
      o = reinterpret_cast<int4*>(reinterpret_cast<__nv_bfloat16* const*>(sc.ret)[src] + (long long)dst_row * H);
  }
  // U vectors per lane per step with every slot's loads issued before the math (C5, ncu:
  // U = 2 / 4 / 8 with 8 CTAs per SM 225 / 194 / 233 us)
  constexpr int U = 4;
  const int hv = H / 8;
  for (int u0 = lane; u0 < hv; u0 += 32 * U) {
    float acc[U][8];
#pragma unroll
    for (int uu = 0; uu < U; uu++)
#pragma unroll
      for (int e = 0; e < 8; e++) acc[uu][e] = 0.0f;
    for (int q = 0; q < ns; q++) {  // slot order fixed: fp32 sum in slot order
      int4 v[U];
#pragma unroll
      for (int uu = 0; uu < U; uu++)
        if (u0 + 32 * uu < hv) v[uu] = ld_nc_v4(src[q] + u0 + 32 * uu);
#pragma unroll
      for (int uu = 0; uu < U; uu++) {
        const __nv_bfloat162* b = reinterpret_cast<const __nv_bfloat162*>(&v[uu]);
#pragma unroll
        for (int e = 0; e < 4; e++) {
          float2 f = __bfloat1622float2(b[e]);
          acc[uu][2 * e] = fmaf(w[q], f.x, acc[uu][2 * e]);
          acc[uu][2 * e + 1] = fmaf(w[q], f.y, acc[uu][2 * e + 1]);
        }
      }
    }
#pragma unroll
    for (int uu = 0; uu < U; uu++) {
      if (u0 + 32 * uu >= hv) break;
      int4 res;
      __nv_bfloat162* rb = reinterpret_cast<__nv_bfloat162*>(&res);
#pragma unroll
      for (int e = 0; e < 4; e++) rb[e] = __floats2bfloat162_rn(acc[uu][2 * e], acc[uu][2 * e + 1]);
      st_na_v4(o + u0 + 32 * uu, res);
    }
  }
}

// y_row = sum_s w_s * yg[inv[row][s]] (fp32) -> bf16, warp per received row
__global__ void expert_reduce_kernel(const __nv_bfloat16* __restrict__ yg,
                                     const int32_t* __restrict__ inv,
                                     const uint8_t* __restrict__ meta, long long cap,
                                     int meta_bytes, const int32_t* __restrict__ rtot, int n_local,
                                     int rank_base, int k, int H, __nv_bfloat16* __restrict__ ybuf,
                                     const AuroraScatterArgs sc, int skip_single) {
  // persistent warps over the received rows only (rank r's first rtot rows of its cap): a warp
  // per row, grid-strided, so the completion ticket below is paid once per CTA, not per row slot
  __shared__ int pre_s[AUR_MAXN + 1];
  if (threadIdx.x == 0) {
    int acc = 0;
    for (int q = 0; q < n_local; q++) {
      pre_s[q] = acc;
      acc += (int)min((long long)rtot[rank_base + q], cap);
    }
    pre_s[n_local] = acc;
  }
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int warps = (int)(gridDim.x * (blockDim.x >> 5));
  const int total = pre_s[n_local];
  for (int v = (int)(blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5)); v < total; v += warps) {
    int r = 0;
    while (v >= pre_s[r + 1]) r++;
    const int i = v - pre_s[r];
    reduce_row(yg, inv, meta, (long long)r * cap + i, r, i, meta_bytes, rank_base, k, H, ybuf, sc, lane,
               skip_single != 0);
  }
  if (sc.n) {  // fused combine: grid completion -> one arrival per local rank on every sender
    if (sc.sys) __threadfence_system();
    else __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence();
      if (atomicAdd(sc.ticket, 1) == (int)gridDim.x - 1) {
        __threadfence();
        *sc.ticket = 0;
        for (int src = 0; src < sc.n; src++) {
          if (sc.sys) red_release_sys_add(sc.ctrs[src] + 1, n_local);
          else red_release_gpu_add(sc.ctrs[src] + 1, n_local);
        }
      }
    }
  }
}

}  // namespace

extern "C" int aurora_expert_sort(const void* meta, int64_t cap, int meta_bytes,
                                  const int32_t* rtot, int n_local, int rank_base, int k, int G,
                                  int32_t* g_off, int32_t* g_rows, int32_t* g_src, int32_t* inv,
                                  int32_t* scratch, int scratch_ints, void* stream) {
  const int Gt = n_local * G;
  if (!meta || cap < 1 || meta_bytes < 8 * k || meta_bytes % 16 || !rtot || n_local < 1 ||
      k < 1 || k > MAX_SLOTS || G < 1 || Gt > 1024 || !g_off || !g_rows || !g_src || !inv ||
      !scratch)
    return AURORA_EINVAL;
  const long long rows = (long long)n_local * cap;
  const int blocks = (int)((rows + ROWS_PER_BLOCK - 1) / ROWS_PER_BLOCK);
  if ((long long)blocks * Gt > scratch_ints) return AURORA_EINVAL;
  cudaStream_t s = (cudaStream_t)stream;
  const uint8_t* mb = (const uint8_t*)meta;
  sort_count_kernel<<<blocks, ROWS_PER_BLOCK, Gt * sizeof(int), s>>>(mb, cap, meta_bytes, rtot,
                                                                      n_local, rank_base, k, G,
                                                                      scratch);
  sort_scan_kernel<<<1, 1024, 0, s>>>(scratch, blocks, Gt, g_off, g_rows);
  sort_scatter_kernel<<<blocks, ROWS_PER_BLOCK, Gt * sizeof(int), s>>>(
      mb, cap, meta_bytes, rtot, n_local, rank_base, k, G, scratch, g_src, inv);
  AUR_CHECK_LAUNCH();
  return AURORA_OK;
}

extern "C" int aurora_gather_rows(const void* src, void* dst, const int32_t* idx,
                                  const int32_t* count, int64_t max_rows, int row_bytes,
                                  void* stream) {
  if (!src || !dst || !idx || !count || row_bytes % 16 || max_rows < 0) return AURORA_EINVAL;
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  gather_rows_kernel<<<sms * 4, 256, 0, (cudaStream_t)stream>>>((const char*)src, (char*)dst, idx,
                                                                count, row_bytes);
  AUR_CHECK_LAUNCH();
  return AURORA_OK;
}

namespace {
int launch_reduce(const void* yg, const int32_t* inv, const void* meta, int64_t cap, int meta_bytes,
                  const int32_t* rtot, int n_local, int rank_base, int k, int H, void* ybuf,
                  const AuroraScatterArgs& sc, int skip_single, void* stream) {
  if (!yg || !meta || cap < 1 || !rtot || k < 1 || k > MAX_SLOTS || H % 8 || !ybuf)
    return AURORA_EINVAL;
  if (n_local < 1 || n_local > AUR_MAXN) return AURORA_EINVAL;
  const long long rows = (long long)n_local * cap;
  // persistent: 8 CTAs of 8 warps per SM (a warp per received row, grid-strided)
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int blocks = (int)min((rows * 32 + 255) / 256, (long long)sms * 8);  // 4 per SM: 223 us
  expert_reduce_kernel<<<blocks, 256, 0, (cudaStream_t)stream>>>(
      (const __nv_bfloat16*)yg, inv, (const uint8_t*)meta, cap, meta_bytes, rtot, n_local,
      rank_base, k, H, (__nv_bfloat16*)ybuf, sc, skip_single);
  AUR_CHECK_LAUNCH();
  return AURORA_OK;
}
}  // namespace

extern "C" int aurora_expert_reduce(const void* yg, const int32_t* inv, const void* meta,
                                    int64_t cap, int meta_bytes, const int32_t* rtot, int n_local,
                                    int rank_base, int k, int H, void* ybuf, int skip_single, void* stream) {
  return launch_reduce(yg, inv, meta, cap, meta_bytes, rtot, n_local, rank_base, k, H, ybuf,
                       AuroraScatterArgs{}, skip_single, stream);
}

extern "C" int aurora_expert_reduce_combine(const void* yg, const int32_t* inv, const void* meta,
                                            int64_t cap, int meta_bytes, const int32_t* rtot,
                                            int n_local, int rank_base, int k, int H, void* ybuf,
                                            void* const* ret_bufs, const int32_t* counts,
                                            const int32_t* soff, const int32_t* roff, int n,
                                            int32_t* const* ctrs, int32_t* ticket, int sys,
                                            int skip_single, void* stream) {
  if (!ret_bufs || !counts || !soff || !roff || !ctrs || !ticket || n < 1 || n > 32 || n_local < 1 ||
      rank_base < 0 || rank_base + n_local > n)
    return AURORA_EINVAL;
  const AuroraScatterArgs sc{ret_bufs, counts, soff, roff, ctrs, ticket, n, rank_base, sys ? 1 : 0};
  return launch_reduce(yg, inv, meta, cap, meta_bytes, rtot, n_local, rank_base, k, H, ybuf, sc,
                       skip_single, stream);
}
