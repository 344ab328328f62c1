// K4 dispatch / K6 combine: the Aurora schedule executed as in-kernel stores
// into peer memory (NVSwitch is the paper's big switch).
//
// Schedule semantics (reference pkg/src/moeplan/commsched.py:112-162): in
// phase k sender i transmits `duration` tokens of its pair (i, j) while no
// other sender targets j and i targets nobody else. Instead of a global
// barrier per phase, every copy CTA runs its sender's entries in phase order
// and starts a run (consecutive phases of one pair) once ALL earlier runs into
// the same receiver have landed (per-receiver arrival counter, release/acquire
// at system scope); continuation entries of a run need no hand-over. Each
// GPU's send order and receive order are exactly the schedule's, so the
// execution stays contention-free while never waiting longer than the
// phase-aligned timeline would. Correctness does not depend on pacing: every
// entry owns a disjoint, precomputed region of the peer buffer.
//
// The dispatch consumes the schedule while K2 is still producing it: phase k
// is used as soon as K2's progress word says its entries are final, so the
// scheduler's latency hides behind the first phases' copies.
//
// Combine (mode 1) replays the same phases with directions flipped -- the
// reference's CommSchedule.reversed() (commsched.py:310-319) -- from the
// rchunks table, sending expert outputs back to the token owners.
#include "common.cuh"

namespace {

constexpr int THREADS = 256;
constexpr int WARPS = THREADS / 32;

struct EngineParams {
  int mode, n, n_local, rank_base;
  const int32_t* counts;
  const int4* chunks;
  const int4* rchunks;
  const int32_t* progress;  // K2's progress word (AURORA_PROGRESS_*)
  const int32_t* n_in;
  const int32_t* n_out;
  const int32_t* soff;
  const int32_t* roff;
  const int32_t* send_list;
  int send_list_stride;
  const char* const* src_bufs;
  char* const* dst_bufs;
  int row_bytes;
  const char* const* src2_bufs;  // optional second plane (dispatch): per-row expert metadata
  char* const* dst2_bufs;
  int row2_bytes;
  int32_t* const* ctrs;
  int C;
  int max_phases;
  long long spin_limit;
  int32_t* status;
};

// wait until *ctr >= target (thread 0), bounded. `sys`: the counter is written
// by other GPUs (system scope); otherwise every rank lives on this GPU.
__device__ __forceinline__ bool wait_ge(const int32_t* ctr, int target, long long limit, bool sys) {
  long long spins = 0;
  while ((sys ? ld_acquire_sys(ctr) : ld_acquire_gpu(ctr)) < target) {
    if (limit && ++spins > limit) return false;
    if (spins > 64) __nanosleep(20);
  }
  return true;
}

// copy rows [r0, r1) of one chunk: warp per row, 16-byte vectors, up to 16
// loads in flight per lane (one 8 KiB row per warp per batch at hidden 4096,
// 64 KiB per CTA) so a pair's CTAs keep enough bytes in flight to cover
// HBM / NVLink latency.
template <bool GATHER>
__device__ __forceinline__ void copy_rows(int row_bytes, const char* src_base,
                                          const int32_t* gather, int src_row0, char* dst_base,
                                          int dst_row0, int r0, int r1) {
  constexpr int U = 16;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int vec = row_bytes >> 4;
  for (int r = r0 + warp; r < r1; r += WARPS) {
    const long long srow = GATHER ? (long long)gather[src_row0 + r] : (long long)(src_row0 + r);
    const int4* s = reinterpret_cast<const int4*>(src_base + srow * row_bytes);
    int4* d = reinterpret_cast<int4*>(dst_base + (long long)(dst_row0 + r) * row_bytes);
    for (int u0 = 0; u0 < vec; u0 += 32 * U) {
      int4 v[U];
#pragma unroll
      for (int q = 0; q < U; q++) {
        const int u = u0 + q * 32 + lane;
        if (u < vec) v[q] = ld_nc_v4(s + u);
      }
#pragma unroll
      for (int q = 0; q < U; q++) {
        const int u = u0 + q * 32 + lane;
        if (u < vec) st_na_v4(d + u, v[q]);
      }
    }
  }
}

__device__ __forceinline__ void signal(int32_t* ctr, bool sys) {
  __syncthreads();  // every thread's stores of this slice are issued
  if (threadIdx.x == 0) {
    if (sys) {
      __threadfence_system();  // cumulative: orders the CTA's stores (observed via bar.sync)
      red_release_sys_add(ctr, 1);
    } else {
      __threadfence();
      red_release_gpu_add(ctr, 1);
    }
  }
}

__global__ void __launch_bounds__(THREADS, 2) engine_kernel(EngineParams p) {
  const int r_local = blockIdx.x / p.C, c = blockIdx.x % p.C;
  const int g = p.rank_base + r_local;  // this CTA's rank (sender in this mode)
  const int n = p.n;
  const bool dispatch = (p.mode & 1) == 0;
  const bool sys = (p.mode & 2) != 0;          // peers on other GPUs: system-scope ordering
  const bool do_remote = (p.mode & 4) == 0;    // bit 2: local rows only
  const bool do_local = (p.mode & 8) == 0;     // bit 3: scheduled (remote) chunks only
  const bool paced = (p.mode & 16) == 0;       // bit 4: ablation, every pair at once (no schedule)
  const char* src = p.src_bufs[r_local];
  const int32_t* list = p.send_list + (size_t)r_local * p.send_list_stride;
  const int4* table = dispatch ? p.chunks : p.rchunks;
  __shared__ int abort_s, avail_s, done_s;
  if (threadIdx.x == 0) abort_s = 0;
  __syncthreads();

  // local (diagonal) rows never cross the network (TrafficMatrix zeroes them,
  // core.py:95) and need no schedule: copy them while K2 is still running
  if (do_local) {
    const int nloc = p.counts[g * n + g];
    const int per = (nloc + p.C - 1) / p.C;
    const int r0 = min(nloc, c * per), r1 = min(nloc, r0 + per);
    if (dispatch) {
      copy_rows<true>(p.row_bytes, src, list, p.soff[g * n + g], p.dst_bufs[g], p.roff[g * n + g], r0, r1);
      if (p.src2_bufs)
        copy_rows<false>(p.row2_bytes, p.src2_bufs[r_local], nullptr, p.soff[g * n + g], p.dst2_bufs[g],
                         p.roff[g * n + g], r0, r1);
    } else {
      copy_rows<false>(p.row_bytes, src, nullptr, p.roff[g * n + g], p.dst_bufs[g], p.soff[g * n + g], r0, r1);
    }
  }
  if (!do_remote) return;

  // wait until phase `need` is final (or the schedule is complete)
  int avail = 0;
  bool done = false;
  auto refresh = [&](int need) {
    if (threadIdx.x == 0) {
      long long spins = 0;
      int pr;
      for (;;) {
        pr = ld_acquire_gpu(p.progress);
        if ((pr & AURORA_PROGRESS_COUNT) > need || (pr & AURORA_PROGRESS_DONE)) break;
        if (p.spin_limit && ++spins > p.spin_limit) {
          atomicExch(p.status, AURORA_ETIMEOUT);
          abort_s = 1;
          break;
        }
        if (spins > 16) __nanosleep(32);
      }
      avail_s = min(pr & AURORA_PROGRESS_COUNT, p.max_phases);
      done_s = (pr & AURORA_PROGRESS_DONE) != 0;
    }
    __syncthreads();
    avail = avail_s;
    done = done_s;
  };

  for (int k = 0;; k++) {
    if (k >= avail) {
      if (done) break;
      refresh(k);
      if (abort_s) return;
      if (k >= avail) break;
    }
    // dispatch: entry of sender g; combine: entry of the reversed schedule where g sends back
    const int4 ch = __ldcg(&table[k * n + g]);
    const int peer = ch.x;  // dispatch: receiver j; combine: original sender i (now receiver)
    if (peer < 0) continue;
    const int first = ch.y, ntok = ch.z;
    const bool cont = ch.w < 0;
    if (paced && !cont) {  // a run starts once every earlier run into `peer` has landed
      if (threadIdx.x == 0 && !wait_ge(p.ctrs[peer], ch.w * p.C, p.spin_limit, sys)) {
        abort_s = 1;
        atomicExch(p.status, AURORA_ETIMEOUT);
      }
      __syncthreads();
      if (abort_s) return;
    }
    const int per = (ntok + p.C - 1) / p.C;
    const int r0 = min(ntok, c * per), r1 = min(ntok, r0 + per);
    if (dispatch) {
      // x rows of list(g, peer) -> recv_buf[peer] rows roff[g][peer] + first ...
      copy_rows<true>(p.row_bytes, src, list, p.soff[g * n + peer] + first, p.dst_bufs[peer],
                      p.roff[g * n + peer] + first, r0, r1);
      if (p.src2_bufs)
        copy_rows<false>(p.row2_bytes, p.src2_bufs[r_local], nullptr, p.soff[g * n + peer] + first,
                         p.dst2_bufs[peer], p.roff[g * n + peer] + first, r0, r1);
    } else {
      // y rows of pair (peer, g) at roff[peer][g] -> ret_buf[peer] rows soff[peer][g] ...
      copy_rows<false>(p.row_bytes, src, nullptr, p.roff[peer * n + g] + first, p.dst_bufs[peer],
                       p.soff[peer * n + g] + first, r0, r1);
    }
    // the run ends unless this sender's next entry continues it
    if (k + 1 >= avail && !done) {
      refresh(k + 1);
      if (abort_s) return;
    }
    bool run_end = true;
    if (k + 1 < avail) {
      const int4 nx = __ldcg(&table[(k + 1) * n + g]);
      run_end = !(nx.x == peer && nx.w < 0);
    }
    if (run_end) signal(p.ctrs[peer], sys);
  }

  // completion: CTA 0 of each rank waits for all of its arrivals, then rearms its counter
  if (c == 0 && threadIdx.x == 0) {
    const int expect = (dispatch ? __ldcg(&p.n_in[g]) : __ldcg(&p.n_out[g])) * p.C;
    if (!wait_ge(p.ctrs[g], expect, p.spin_limit, sys)) {
      atomicExch(p.status, AURORA_ETIMEOUT);
    } else {
      *(volatile int32_t*)p.ctrs[g] = 0;
      __threadfence_system();
    }
  }
}

// K7: out[t] = sum over slots of (w *) returned rows, fp32 accumulate, bf16 out. Warp per token.
__global__ void __launch_bounds__(THREADS) aggregate_kernel(
    const __nv_bfloat16* __restrict__ ret, long long ret_stride_rows, const int32_t* __restrict__ soff,
    const int32_t* __restrict__ pos, const int32_t* __restrict__ slot_dst,
    const float* __restrict__ topk_w, int T, int k, int H, int n, int rank_base,
    int tokens_per_rank, int pre_weighted, __nv_bfloat16* __restrict__ out) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int t = blockIdx.x * WARPS + warp;
  if (t >= T) return;
  const int i_local = t / tokens_per_rank, i = rank_base + i_local;
  const __nv_bfloat16* base = ret + (size_t)i_local * ret_stride_rows * H;
  const int4* rows[8];
  float w[8];
  int ns = 0;
  for (int s = 0; s < k; s++) {
    const int v = slot_dst[(size_t)t * k + s];
    if (pre_weighted && v < 0) continue;  // duplicate slot: row already pre-reduced
    const int j = v >= 0 ? v : -(v + 1);
    rows[ns] = reinterpret_cast<const int4*>(base + (size_t)(soff[i * n + j] + pos[(size_t)t * k + s]) * H);
    w[ns] = pre_weighted ? 1.0f : topk_w[(size_t)t * k + s];
    ns++;
  }
  int4* o = reinterpret_cast<int4*>(out + (size_t)t * H);
  for (int u = lane; u < H / 8; u += 32) {
    float acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    for (int q = 0; q < ns; q++) {
      int4 v = ld_nc_v4(rows[q] + u);
      const __nv_bfloat162* b = reinterpret_cast<const __nv_bfloat162*>(&v);
#pragma unroll
      for (int e = 0; e < 4; e++) {
        float2 f = __bfloat1622float2(b[e]);
        acc[2 * e] = fmaf(w[q], f.x, acc[2 * e]);
        acc[2 * e + 1] = fmaf(w[q], f.y, acc[2 * e + 1]);
      }
    }
    int4 r;
    __nv_bfloat162* rb = reinterpret_cast<__nv_bfloat162*>(&r);
#pragma unroll
    for (int e = 0; e < 4; e++) rb[e] = __floats2bfloat162_rn(acc[2 * e], acc[2 * e + 1]);
    o[u] = r;
  }
}

}  // namespace

extern "C" int aurora_engine(int mode, int n, int n_local, int rank_base, const int32_t* counts,
                             const int32_t* chunks, const int32_t* rchunks,
                             const int32_t* progress, const int32_t* n_in, const int32_t* n_out,
                             const int32_t* soff, const int32_t* roff, const int32_t* send_list,
                             int send_list_stride, const void* const* src_bufs,
                             void* const* dst_bufs, int row_bytes, const void* const* src2_bufs,
                             void* const* dst2_bufs, int row2_bytes, int32_t* const* ctrs,
                             int ctas_per_rank, int max_phases, int64_t spin_limit,
                             int32_t* status, void* stream) {
  if (mode < 0 || mode > 63 || (mode & 12) == 12 || n < 1 || n > AUR_MAXN || n_local < 1 ||
      rank_base < 0 ||
      rank_base + n_local > n || row_bytes % 16 || ctas_per_rank < 1 || !counts || !chunks ||
      !rchunks || !progress || !soff || !roff || !src_bufs || !dst_bufs || !ctrs || !status ||
      ((mode & 1) == 0 && !send_list))
    return AURORA_EINVAL;
  int dev = 0, sms = 0, occ = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, engine_kernel, THREADS, 0) != cudaSuccess ||
      occ < 1)
    return AURORA_ECUDA;
  // every copy CTA spins on flags written by others: all of them must be
  // co-resident. Clamp deterministically (every process computes the same C).
  ctas_per_rank = min(ctas_per_rank, (occ * sms) / n_local);
  if (ctas_per_rank < 1) return AURORA_EINVAL;
  EngineParams p;
  p.mode = mode;
  p.n = n;
  p.n_local = n_local;
  p.rank_base = rank_base;
  p.counts = counts;
  p.chunks = reinterpret_cast<const int4*>(chunks);
  p.rchunks = reinterpret_cast<const int4*>(rchunks);
  p.progress = progress;
  p.n_in = n_in;
  p.n_out = n_out;
  p.soff = soff;
  p.roff = roff;
  p.send_list = send_list;
  p.send_list_stride = send_list_stride;
  p.src_bufs = reinterpret_cast<const char* const*>(src_bufs);
  p.dst_bufs = reinterpret_cast<char* const*>(dst_bufs);
  p.row_bytes = row_bytes;
  p.src2_bufs = reinterpret_cast<const char* const*>(src2_bufs);
  p.dst2_bufs = reinterpret_cast<char* const*>(dst2_bufs);
  p.row2_bytes = row2_bytes;
  if (src2_bufs && (!dst2_bufs || row2_bytes <= 0 || row2_bytes % 16)) return AURORA_EINVAL;
  p.ctrs = ctrs;
  p.C = ctas_per_rank;
  p.max_phases = max_phases;
  p.spin_limit = spin_limit;
  p.status = status;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(n_local * ctas_per_rank);
  cfg.blockDim = dim3(THREADS);
  cfg.stream = (cudaStream_t)stream;
  cudaLaunchAttribute attr[1];
  if (mode & 32) {  // programmatic dependent of the preceding K2 launch: start while it runs
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
  }
  if (cudaLaunchKernelEx(&cfg, engine_kernel, p) != cudaSuccess) return AURORA_ECUDA;
  AUR_CHECK_LAUNCH();
  return AURORA_OK;
}

extern "C" int aurora_aggregate(const void* ret_buf, int64_t ret_rank_stride_rows,
                                const int32_t* soff, const int32_t* pos, const int32_t* slot_dst,
                                const float* topk_w, int T, int k, int H, int n, int rank_base,
                                int tokens_per_rank, int pre_weighted, void* out, void* stream) {
  if (T <= 0 || k < 1 || k > 8 || H % 8 || n < 1 || n > AUR_MAXN || tokens_per_rank < 1)
    return AURORA_EINVAL;
  aggregate_kernel<<<(T + WARPS - 1) / WARPS, THREADS, 0, (cudaStream_t)stream>>>(
      (const __nv_bfloat16*)ret_buf, ret_rank_stride_rows, soff, pos, slot_dst, topk_w, T, k, H,
      n, rank_base, tokens_per_rank, pre_weighted, (__nv_bfloat16*)out);
  AUR_CHECK_LAUNCH();
  return AURORA_OK;
}
