// K4 dispatch / K6 combine: the Aurora schedule executed as in-kernel stores
// into peer memory (NVSwitch is the paper's big switch).
//
// Schedule semantics (reference pkg/src/moeplan/commsched.py:113-162): in
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
// reference's CommSchedule.reversed() (commsched.py:153-162) -- from the
// rchunks table, sending expert outputs back to the token owners.
#include "common.cuh"
#include "tc_helpers.cuh"
#include "apportion.cuh"

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
  int C;                 // copy CTAs per local rank at launch (grid = n_local * C)
  int split;             // apportion.cuh mode: how the grid is split among local ranks
  const double* bw;      // rank bandwidths (split mode 2) or nullptr
  int max_phases;
  long long spin_limit;
  int32_t* status;
  int meta_k;            // grouped dispatch (mode bit 8): expert records per meta row
  int4* const* ginfo;    // grouped dispatch: per-rank {recv row, weight, single, 0} arrays (nullable)
  // arrival-driven expert GEMM (LSU dispatch only; nullable): landed[j][i] = rows of block
  // (sender i -> receiver j) stored and visible, credited per CTA at every run end (and after the
  // local rows); the GEMM starts a tile once every block under it is complete
  int32_t* const* landed;
  // deadline pacing (TMA engine; phase_dur nullable = off): a run also starts once the schedule's
  // own clock reaches its phase -- t0 (the copy CTA's first remote entry) + start(k) * unit_ns,
  // start(k) = the durations of phases 0..k-1 -- whichever comes first with the hand-over
  const double* phase_dur;
  float unit_ns;
};

// This CTA's rank (local index), its index among the rank's CTAs and the
// rank's CTA count, from the same apportioning K2 used for the thresholds.
__device__ void cta_assign(const EngineParams& p, int* cs /* smem [AUR_MAXN] */, int& r_local, int& c,
                           int& C) {
  __shared__ long long w_s[AUR_MAXN];
  if (p.split == 0 || p.n_local == 1) {  // nothing to weigh
    if (threadIdx.x < p.n_local) cs[threadIdx.x] = p.C;
  } else {
    for (int i = threadIdx.x; i < p.n; i += blockDim.x)
      w_s[i] = aur_weight(p.counts, p.n, p.bw, p.n, i, p.split, (p.mode & 1) != 0);
    __syncthreads();
    if (threadIdx.x == 0) {
      int all[AUR_MAXN];
      aur_apportion_w(w_s, p.n, p.n_local, p.n_local * p.C, all);
      for (int r = 0; r < p.n_local; r++) cs[r] = all[p.rank_base + r];
    }
  }
  __syncthreads();
  int b = blockIdx.x, r = 0;
  while (r < p.n_local - 1 && b >= cs[r]) b -= cs[r++];
  r_local = r;
  c = b;
  C = cs[r];
}

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

// wait until *ctr >= target or the %globaltimer reaches `due` (deadline pacing), bounded
__device__ __forceinline__ bool wait_ge_or_until(const int32_t* ctr, int target, long long due, long long limit,
                                                 bool sys) {
  long long spins = 0;
  while ((sys ? ld_acquire_sys(ctr) : ld_acquire_gpu(ctr)) < target) {
    long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    if (t >= due) return true;
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

// landed: optional arrival credit (rows of this CTA's run now visible at the receiver)
__device__ __forceinline__ void signal(int32_t* ctr, bool sys, int32_t* landed = nullptr, int rows = 0) {
  __syncthreads();  // every thread's stores of this slice are issued
  if (threadIdx.x == 0) {
    if (sys) {
      __threadfence_system();  // cumulative: orders the CTA's stores (observed via bar.sync)
      if (landed && rows) red_release_sys_add(landed, rows);
      red_release_sys_add(ctr, 1);      // pace
      red_release_sys_add(ctr + 1, 1);  // done last: once the receiver sees every done, every pace is in
    } else {
      __threadfence();
      if (landed && rows) red_release_gpu_add(landed, rows);
      red_release_gpu_add(ctr, 1);
      red_release_gpu_add(ctr + 1, 1);
    }
  }
}

// diagnostics: per copy CTA {start, local rows done, end} in %globaltimer ns
__device__ long long* g_engine_trace = nullptr;
__device__ __forceinline__ long long eng_ns0() {
  long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__global__ void __launch_bounds__(THREADS, 2) engine_kernel(EngineParams p) {
  // a programmatically dependent launch (the arrival-driven expert GEMM) may start beside this grid
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  __shared__ int cs[AUR_MAXN];
  int r_local, c, C;
  cta_assign(p, cs, r_local, c, C);
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
  if (threadIdx.x == 0 && g_engine_trace) g_engine_trace[blockIdx.x * 4] = eng_ns0();
  __syncthreads();

  // local (diagonal) rows never cross the network (TrafficMatrix zeroes them,
  // core.py:95) and need no schedule: copy them while K2 is still running
  if (do_local) {
    const int nloc = p.counts[g * n + g];
    const int per = (nloc + C - 1) / C;
    const int r0 = min(nloc, c * per), r1 = min(nloc, r0 + per);
    if (dispatch) {
      copy_rows<true>(p.row_bytes, src, list, p.soff[g * n + g], p.dst_bufs[g], p.roff[g * n + g], r0, r1);
      if (p.src2_bufs)
        copy_rows<false>(p.row2_bytes, p.src2_bufs[r_local], nullptr, p.soff[g * n + g], p.dst2_bufs[g],
                         p.roff[g * n + g], r0, r1);
    } else {
      copy_rows<false>(p.row_bytes, src, nullptr, p.roff[g * n + g], p.dst_bufs[g], p.soff[g * n + g], r0, r1);
    }
    if (dispatch && p.landed && r1 > r0) {  // the local block's rows of this CTA are in place
      __syncthreads();
      if (threadIdx.x == 0) {
        __threadfence();
        red_release_gpu_add(p.landed[g] + g, r1 - r0);
      }
    }
  }
  if (threadIdx.x == 0 && g_engine_trace) g_engine_trace[blockIdx.x * 4 + 1] = eng_ns0();
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

  int run_rows = 0;  // rows this CTA moved in the open run (arrival credit)
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
      if (threadIdx.x == 0 && !wait_ge(p.ctrs[peer], ch.w, p.spin_limit, sys)) {
        abort_s = 1;
        atomicExch(p.status, AURORA_ETIMEOUT);
      }
      __syncthreads();
      if (abort_s) return;
    }
    const int per = (ntok + C - 1) / C;
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
    run_rows += r1 - r0;
    if (run_end) {
      signal(p.ctrs[peer], sys, (dispatch && p.landed) ? p.landed[peer] + g : nullptr, run_rows);
      run_rows = 0;
    }
  }

  if (threadIdx.x == 0 && g_engine_trace) g_engine_trace[blockIdx.x * 4 + 2] = eng_ns0();
  // completion: CTA 0 of each rank waits for all of its arrivals, then rearms its counter
  if (c == 0 && threadIdx.x == 0) {
    const int expect = dispatch ? __ldcg(&p.n_in[g]) : __ldcg(&p.n_out[g]);
    if (!wait_ge(p.ctrs[g] + 1, expect, p.spin_limit, sys)) {
      atomicExch(p.status, AURORA_ETIMEOUT);
    } else {
      ((volatile int32_t*)p.ctrs[g])[0] = 0;
      ((volatile int32_t*)p.ctrs[g])[1] = 0;
      __threadfence_system();
    }
  }
}

// ============================================================================
// TMA engine (default): the same schedule semantics, rows moved by the bulk
// copy engine -- cp.async.bulk global -> shared (the sender's rows, gathered
// through the send list) and cp.async.bulk shared -> global (the receiver's
// buffer, peer memory over NVSwitch at N > 1). Two warps per CTA:
//   warp 0 (producer) walks the CTA's rows in schedule order and keeps up to
//          S row slots of shared memory filling; it never waits for a
//          receiver, so the next run's rows are already on chip while the
//          previous sender into that receiver finishes (prefetch across the
//          hand-over);
//   warp 1 (consumer) waits for the hand-over at each run start, stores the
//          landed rows with bulk stores, recycles slots once a store has read
//          them, and at each run end waits for its stores to complete and
//          signals the receiver's arrival counter.
// A row's slot holds the row and its optional second-plane record.
// ============================================================================
constexpr int TMA_THREADS = 64;

__device__ __forceinline__ void bulk_load(uint32_t dst_smem, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   dst_smem),
               "l"(src), "r"(bytes), "r"(tc::smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void bulk_store(void* dst, uint32_t src_smem, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(src_smem), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
template <int N>
__device__ __forceinline__ void bulk_wait() {
  asm volatile("cp.async.bulk.wait_group %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(tc::smem_u32(bar)) : "memory");
}
// bounded wait: false if *abort was raised meanwhile
__device__ __forceinline__ bool mbar_wait_or_abort(uint64_t* bar, uint32_t parity, volatile int* abort) {
  for (;;) {
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred P1;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, P1;\n\t}"
        : "=r"(ok)
        : "r"(tc::smem_u32(bar)), "r"(parity)
        : "memory");
    if (ok) return true;
    if (*abort) return false;
  }
}

// One warp's view of the schedule: entries of sender g in phase order, read 32
// at a time (one L2 round trip per window) as K2 publishes them.
struct EntryWindow {
  int4* win;      // [32] shared
  int base, cnt;  // window covers entries [base, base + cnt)
  int avail;      // phases known final
  bool done;
};

// warp-collective. Returns false at the end of the schedule (or on timeout).
__device__ bool entry_at(const EngineParams& p, const int4* table, int g, int k, EntryWindow& w, int4& e,
                         volatile int* abort) {
  const int lane = threadIdx.x & 31;
  if (k >= w.base + w.cnt) {
    if (k >= w.avail && !w.done) {
      int pr = 0, fail = 0;
      if (lane == 0) {
        long long spins = 0;
        for (;;) {
          pr = ld_acquire_gpu(p.progress);
          if ((pr & AURORA_PROGRESS_COUNT) > k || (pr & AURORA_PROGRESS_DONE)) break;
          if (*abort) { fail = 1; break; }
          if (p.spin_limit && ++spins > p.spin_limit) {
            atomicExch(p.status, AURORA_ETIMEOUT);
            *abort = 1;
            fail = 1;
            break;
          }
          if (spins > 16) __nanosleep(32);
        }
      }
      pr = __shfl_sync(0xffffffffu, pr, 0);
      if (__shfl_sync(0xffffffffu, fail, 0)) return false;
      w.avail = min(pr & AURORA_PROGRESS_COUNT, p.max_phases);
      w.done = (pr & AURORA_PROGRESS_DONE) != 0;
    }
    if (k >= w.avail) return false;  // done and exhausted
    w.base = k;
    w.cnt = min(32, w.avail - k);
    if (lane < w.cnt) w.win[lane] = __ldcg(&table[(size_t)(k + lane) * p.n + g]);
    __syncwarp();
  }
  e = w.win[k - w.base];
  return true;
}

constexpr int RING = 128;


__device__ int g_early_rows = 2;  // rows before a run's end at which its pace signal goes out

__device__ __forceinline__ long long eng_ns() {
  long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}  // schedule entries the producer may run ahead of the consumer

struct TmaShared {
  uint64_t full[16], empty[16];
  int4 win[32];     // producer's window of global entries
  int4 ring[RING];  // entries handed to the consumer (producer -> consumer, in order)
  float ring_t[RING];  // deadline pacing: schedule time (units) at which entry k's phase starts
  float wdur[32];      // deadline pacing: durations of the producer's window of phases
  volatile int known, known_done, cons_k;
  int32_t idx[32];
  // per-call metadata staged once: every per-entry lookup is a shared-memory read
  char* dst[AUR_MAXN];
  char* dst2[AUR_MAXN];
  int32_t* ctr[AUR_MAXN];
  int nloc;
  int abort;
  long long issued, consumed;
  int runs_to[AUR_MAXN];  // runs this CTA ended into each receiver (done signals owed)
};

__global__ void __launch_bounds__(TMA_THREADS) engine_tma_kernel(EngineParams p, int S, int slot_bytes) {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  extern __shared__ __align__(128) unsigned char slots[];
  __shared__ TmaShared sh;
  // per-call buffer offsets behind the row slots (n x n each): every per-entry lookup is a shared read
  int32_t* soff_s = reinterpret_cast<int32_t*>(slots + (size_t)S * slot_bytes);
  int32_t* roff_s = soff_s + p.n * p.n;
  __shared__ int cs[AUR_MAXN];
  int r_local, c, C;
  cta_assign(p, cs, r_local, c, C);
  const int g = p.rank_base + r_local;
  const int n = p.n;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const bool dispatch = (p.mode & 1) == 0;
  const bool sys = (p.mode & 2) != 0;
  const bool do_remote = (p.mode & 4) == 0;
  const bool do_local = (p.mode & 8) == 0;
  const bool paced = (p.mode & 16) == 0;
  const int rb = p.row_bytes, rb2 = p.src2_bufs ? p.row2_bytes : 0;
  const bool grouped = (p.mode & 256) && rb2 && !(p.mode & 1);  // dispatch with the meta plane only
  const int4* table = dispatch ? p.chunks : p.rchunks;
  volatile int* abort = &sh.abort;
  for (int q = threadIdx.x; q < n * n; q += TMA_THREADS) {
    soff_s[q] = p.soff[q];
    roff_s[q] = p.roff[q];
  }
  for (int q = threadIdx.x; q < n; q += TMA_THREADS) {
    sh.dst[q] = p.dst_bufs[q];
    sh.dst2[q] = rb2 ? p.dst2_bufs[q] : nullptr;
    sh.ctr[q] = p.ctrs[q];
  }
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; s++) {
      tc::mbar_init(&sh.full[s], 1);
      tc::mbar_init(&sh.empty[s], 1);
    }
    sh.abort = 0;
    sh.nloc = p.counts[g * n + g];
    sh.issued = sh.consumed = 0;
    sh.known = 0;
    sh.known_done = 0;
    sh.cons_k = 0;
    for (int q = 0; q < AUR_MAXN; q++) sh.runs_to[q] = 0;
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0 && g_engine_trace) g_engine_trace[blockIdx.x * 4] = eng_ns();
  const uint32_t slot0 = tc::smem_u32(slots);

  // item = the local rows (k = -1) or schedule entry k; this CTA's rows [r0, r1)
  auto slice = [&](int ntok, int& r0, int& r1) {
    const int per = (ntok + C - 1) / C;
    r0 = min(ntok, c * per);
    r1 = min(ntok, r0 + per);
  };

  if (warp == 0) {
    // ------------------------------------------------------------ producer
    EntryWindow w{sh.win, 0, 0, 0, false};
    long long t = 0;  // rows issued
    int s = 0;        // slot of row t
    uint32_t u = 0;   // fill round of slot s (t / S)
    const char* src = p.src_bufs[r_local];
    const char* src2 = rb2 ? p.src2_bufs[r_local] : nullptr;
    const int32_t* list = p.send_list + (size_t)r_local * p.send_list_stride;
    const double* ddur = p.phase_dur;
    double tcum = 0.0;  // deadline pacing: schedule time at the start of phase k
    for (int k = do_local ? -1 : 0; do_remote || k < 0; k++) {
      int peer, first, ntok;
      if (k < 0) {
        peer = g, first = 0, ntok = sh.nloc;
      } else {
        int4 e;
        const int wb = w.base + w.cnt;
        if (!entry_at(p, table, g, k, w, e, abort)) break;
        if (ddur && w.base + w.cnt != wb) {  // a new window: its phases' durations
          if (lane < w.cnt) sh.wdur[lane] = (float)__ldcg(&ddur[w.base + lane]);
          __syncwarp();
        }
        // hand the entry to the consumer (it never reads the global table itself)
        if (lane == 0) {
          while (k - sh.cons_k >= RING - 1 && !*abort) {
          }
          sh.ring[k & (RING - 1)] = e;
          if (ddur) {
            sh.ring_t[k & (RING - 1)] = (float)tcum;
            tcum += sh.wdur[k - w.base];
          }
          __threadfence_block();
          sh.known = k + 1;
        }
        __syncwarp();
        if (e.x < 0) continue;
        peer = e.x, first = e.y, ntok = e.z;
      }
      int r0, r1;
      slice(ntok, r0, r1);
      // source rows: dispatch gathers x rows through the send list (pair (g, peer)
      // starts at soff[g][peer]); combine reads expert outputs of pair (peer, g)
      const int base = dispatch ? soff_s[g * n + peer] + first : roff_s[peer * n + g] + first;
      for (int b = r0; b < r1; b += 32) {
        const int cnt = min(32, r1 - b);
        if (dispatch) {
          if (lane < cnt) sh.idx[lane] = __ldg(&list[base + b + lane]);
          __syncwarp();
        }
        if (lane == 0) {
          for (int q = 0; q < cnt; q++) {
            if (u > 0 && !mbar_wait_or_abort(&sh.empty[s], (u - 1) & 1, abort)) break;
            const long long row = dispatch ? sh.idx[q] : (long long)(base + b + q);
            const uint32_t dst = slot0 + (uint32_t)(s * slot_bytes);
            tc::mbar_expect_tx(&sh.full[s], rb + rb2);
            bulk_load(dst, src + row * rb, rb, &sh.full[s]);
            if (rb2) bulk_load(dst + rb, src2 + (long long)(base + b + q) * rb2, rb2, &sh.full[s]);
            t++;
            if (++s == S) { s = 0; u++; }
          }
        }
        __syncwarp();
        if (*abort) break;
      }
      if (*abort) break;
    }
    if (lane == 0) {
      sh.issued = t;
      __threadfence_block();
      sh.known_done = 1;
    }
  } else {
    // ------------------------------------------------------------ consumer
    long long t = 0, released = 0;
    int s = 0, rs = 0;  // slot of row t; slot of row `released`
    uint32_t u = 0;
    auto release_upto = [&](long long upto) {  // slots of rows < upto may be refilled
      for (; released < upto; released++) {
        mbar_arrive(&sh.empty[rs]);
        if (++rs == S) rs = 0;
      }
    };
    int prev_peer = -1;    // peer of the open run (-1: none)
    bool paced_out = false;  // this CTA already released the open run's receiver (early pace)
    // early pace: release the receiver when this CTA has only EARLY rows of the
    // run left to issue -- about the flag's round trip -- so the next sender's
    // first stores follow this run's last ones instead of waiting a hand-over
    const int EARLY = (p.mode & 128) ? g_early_rows : 0;  // mode bit 7
    const float unit_ns = p.phase_dur ? p.unit_ns : 0.0f;
    long long t0 = 0;  // deadline pacing: this CTA's clock origin (its first remote entry)
    auto pace = [&](int peer_) {
      if (sys) red_relaxed_sys_add(sh.ctr[peer_], 1);
      else red_relaxed_gpu_add(sh.ctr[peer_], 1);
    };
    // does entry k end the open run into `peer_`? 1 yes, 0 no, -1 not known yet
    auto run_ends_at = [&](int k_, int peer_) -> int {
      if (k_ + 1 < sh.known) {
        __threadfence_block();  // acquire side of the producer's fence + `known` store
        const int4 nx = sh.ring[(k_ + 1) & (RING - 1)];
        return (nx.x == peer_ && nx.w < 0) ? 0 : 1;
      }
      return sh.known_done ? 1 : -1;
    };
    for (int k = do_local ? -1 : 0; do_remote || k < 0; k++) {
      int peer, first, ntok;
      if (k < 0) {
        peer = g, first = 0, ntok = sh.nloc;
      } else {
        int4 e = make_int4(-1, 0, 0, 0);
        if (lane == 0) {
          if (k == 0 && unit_ns > 0.0f) t0 = eng_ns();
          while (k >= sh.known && !sh.known_done && !*abort) {
          }
          sh.cons_k = k;
        }
        __syncwarp();
        __threadfence_block();
        const bool more = k < sh.known && !*abort;
        if (more) e = sh.ring[k & (RING - 1)];
        // a run ends where this sender's entries stop continuing it
        const bool cont = more && e.x >= 0 && e.x == prev_peer && e.w < 0;
        if (prev_peer >= 0 && !cont) {
          // the run's stores are all issued: the next run into prev_peer may start
          // (pace); completion (done) is owed until this CTA's final drain
          if (lane == 0) {
            if (!paced_out) pace(prev_peer);
            sh.runs_to[prev_peer]++;
          }
          prev_peer = -1;
          paced_out = false;
        }
        if (!more) break;
        if (e.x < 0) continue;
        peer = e.x, first = e.y, ntok = e.z;
        if (!cont) {  // run start: every earlier run into `peer` must have landed
          prev_peer = peer;
          if (paced && lane == 0) {
            bool ok;
            if (unit_ns > 0.0f) {  // ... or the schedule's clock has reached this phase
              if (!t0) t0 = eng_ns();
              const long long due = t0 + (long long)(sh.ring_t[k & (RING - 1)] * unit_ns);
              ok = wait_ge_or_until(sh.ctr[peer], e.w, due, p.spin_limit, sys);
            } else {
              ok = wait_ge(sh.ctr[peer], e.w, p.spin_limit, sys);
            }
            if (!ok) {
              atomicExch(p.status, AURORA_ETIMEOUT);
              *abort = 1;
            }
          }
          __syncwarp();
          if (*abort) break;
        }
      }
      int r0, r1;
      slice(ntok, r0, r1);
      const long long drow0 = dispatch ? (long long)roff_s[g * n + peer] + first : (long long)soff_s[peer * n + g] + first;
      char* dst = sh.dst[peer];
      char* dst2 = sh.dst2[peer];
      if (lane == 0) {
        const int early_at = r1 - EARLY;  // signal before issuing row early_at (or now)
        if (EARLY && k >= 0 && paced && !paced_out && early_at <= r0 && run_ends_at(k, peer) == 1) {
          pace(peer);
          paced_out = true;
        }
        for (int r = r0; r < r1; r++) {
          if (EARLY && k >= 0 && paced && !paced_out && r == early_at && run_ends_at(k, peer) == 1) {
            pace(peer);
            paced_out = true;
          }
          if (!mbar_wait_or_abort(&sh.full[s], u & 1, abort)) break;
          const uint32_t sp = slot0 + (uint32_t)(s * slot_bytes);
          if (grouped) {
            // the row goes to its position in every local-expert group it belongs to:
            // the positions are the x fields of its meta records, landed in this slot
            int nq = 0;
            if (p.ginfo)
              for (int q = 0; q < p.meta_k; q++) {
                int gp;
                asm volatile("ld.shared.b32 %0, [%1];" : "=r"(gp) : "r"(sp + rb + 8 * q) : "memory");
                nq += gp >= 0;
              }
            for (int q = 0; q < p.meta_k; q++) {
              int gp, wb;
              asm volatile("ld.shared.v2.b32 {%0, %1}, [%2];" : "=r"(gp), "=r"(wb) : "r"(sp + rb + 8 * q) : "memory");
              if (gp >= 0) {
                bulk_store(dst + (long long)gp * rb, sp, rb);
                if (p.ginfo) p.ginfo[peer][gp] = make_int4((int)(drow0 + r), wb, nq == 1 ? 1 : 0, 0);
              }
            }
          } else {
            bulk_store(dst + (drow0 + r) * rb, sp, rb);
          }
          if (rb2) bulk_store(dst2 + (drow0 + r) * rb2, sp + rb, rb2);
          bulk_commit();
          t++;
          if (++s == S) { s = 0; u++; }
          // keep a few stores reading their slots; older slots go back to the producer
          if (S >= 8) {
            bulk_wait_read<4>();
            release_upto(t - 4);
          } else {
            bulk_wait_read<1>();
            release_upto(t - 1);
          }
        }
      }
      __syncwarp();
      if (k < 0 && lane == 0 && g_engine_trace) g_engine_trace[blockIdx.x * 4 + 1] = eng_ns();
      if (*abort) break;
    }
    if (lane == 0) {
      bulk_wait_all();
      release_upto(t);
      sh.consumed = t;
      // every store of this CTA has completed: pay the done signals (release, cumulative)
      asm volatile("fence.proxy.async.global;" ::: "memory");
      for (int j = 0; j < n; j++)
        if (sh.runs_to[j]) {
          if (sys) red_release_sys_add(sh.ctr[j] + 1, sh.runs_to[j]);
          else red_release_gpu_add(sh.ctr[j] + 1, sh.runs_to[j]);
        }
      if (g_engine_trace) g_engine_trace[blockIdx.x * 4 + 2] = eng_ns();
    }
    // completion: CTA 0 of each rank waits for all of its arrivals, then rearms its counter
    if (do_remote && !*abort && c == 0 && lane == 0) {
      const int expect = dispatch ? __ldcg(&p.n_in[g]) : __ldcg(&p.n_out[g]);
      if (!wait_ge(sh.ctr[g] + 1, expect, p.spin_limit, sys)) {
        atomicExch(p.status, AURORA_ETIMEOUT);
      } else {  // every pace signal precedes its sender's done signal (release): both are final
        ((volatile int32_t*)sh.ctr[g])[0] = 0;
        ((volatile int32_t*)sh.ctr[g])[1] = 0;
        __threadfence_system();
      }
    }
  }
  // on abort: let every issued load land before the CTA's shared memory is released
  __syncthreads();
  if (threadIdx.x == 0 && sh.abort)
    for (long long q = sh.consumed; q < sh.issued; q++) tc::mbar_wait(&sh.full[q % S], (uint32_t)(q / S) & 1);
}

// K7: out[t] = sum over slots of (w *) returned rows, fp32 accumulate, bf16 out. Warp per token.
template <int U>
__global__ void __launch_bounds__(THREADS) aggregate_kernel(
    const __nv_bfloat16* __restrict__ ret, long long ret_stride_rows, const int32_t* __restrict__ soff,
    const int32_t* __restrict__ pos, const int32_t* __restrict__ slot_dst,
    const float* __restrict__ topk_w, int T, int k, int H, int n, int rank_base,
    int tokens_per_rank, int pre_weighted, __nv_bfloat16* __restrict__ out,
    const __nv_bfloat16* __restrict__ ybuf, long long y_stride_rows, const int32_t* __restrict__ roff) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int t = blockIdx.x * WARPS + warp;
  if (t >= T) return;
  const int i_local = t / tokens_per_rank, i = rank_base + i_local;
  const __nv_bfloat16* base = ret + (size_t)i_local * ret_stride_rows * H;
  // local slots (expert on the token's own rank): straight from the expert output
  const __nv_bfloat16* ybase = ybuf ? ybuf + (size_t)i_local * y_stride_rows * H : nullptr;
  const int4* rows[8];
  float w[8];
  int ns = 0;
  for (int s = 0; s < k; s++) {
    const int v = slot_dst[(size_t)t * k + s];
    if (pre_weighted && v < 0) continue;  // duplicate slot: row already pre-reduced
    const int j = v >= 0 ? v : -(v + 1);
    rows[ns] = (ybase && j == i)
                   ? reinterpret_cast<const int4*>(ybase + (size_t)(roff[i * n + i] + pos[(size_t)t * k + s]) * H)
                   : reinterpret_cast<const int4*>(base + (size_t)(soff[i * n + j] + pos[(size_t)t * k + s]) * H);
    w[ns] = pre_weighted ? 1.0f : topk_w[(size_t)t * k + s];
    ns++;
  }
  int4* o = reinterpret_cast<int4*>(out + (size_t)t * H);
  // U vectors per lane per step, every slot's loads issued before the math:
  // up to U * k 16-byte loads in flight per lane (HBM latency x bandwidth)
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
        if (u0 + 32 * uu < hv) v[uu] = ld_nc_v4(rows[q] + u0 + 32 * uu);
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
      int4 r;
      __nv_bfloat162* rb = reinterpret_cast<__nv_bfloat162*>(&r);
#pragma unroll
      for (int e = 0; e < 4; e++) rb[e] = __floats2bfloat162_rn(acc[uu][2 * e], acc[uu][2 * e + 1]);
      st_na_v4(o + u0 + 32 * uu, r);
    }
  }
}

}  // namespace

// Copy CTAs per local rank after clamping to co-residency (every copy CTA
// spins on flags written by others, so all must be resident); also the TMA
// engine's slot geometry. Returns the clamped count, 0 if none fit, -1 on a
// CUDA error. Deterministic: every process computes the same value.
static int engine_ctas(int n, int n_local, int ctas_per_rank, int row_bytes, int rb2, bool lsu, int* S_out,
                       int* slot_out, size_t* dyn_out) {
  int dev = 0, sms = 0, occ = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int slot_bytes = ((row_bytes + rb2 + 127) / 128) * 128;
  // 48 KB of row slots: four TMA-engine CTAs fit per SM -- more copy CTAs beat deeper rings
  // (loopback C2, paced dispatch: 2 CTAs/SM x 12 slots 204 us, 3 x 8 170 us, 4 x 6 155 us, 6 x 4 159 us)
  const int S = max(2, min(16, (48 * 1024) / slot_bytes));
  const size_t dyn = lsu ? 0 : (size_t)S * slot_bytes + 2 * (size_t)n * n * sizeof(int32_t);
  if (!lsu && dyn > 200 * 1024) return 0;
  if (!lsu && cudaFuncSetAttribute(engine_tma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn) !=
                  cudaSuccess)
    return -1;
  // the LSU engine needs almost no shared memory, but it shares SMs with the arrival-driven
  // expert GEMM (N1): an SM's L1 / shared split is fixed while CTAs are resident, so ask for the
  // largest shared carveout or the GEMM's CTAs could not land beside it
  if (lsu && cudaFuncSetAttribute(engine_kernel, cudaFuncAttributePreferredSharedMemoryCarveout,
                                  (int)cudaSharedmemCarveoutMaxShared) != cudaSuccess)
    return -1;
  const cudaError_t oe = lsu ? cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, engine_kernel, THREADS, 0)
                             : cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, engine_tma_kernel,
                                                                             TMA_THREADS, dyn);
  if (oe != cudaSuccess || occ < 1) return -1;
  if (S_out) *S_out = S;
  if (slot_out) *slot_out = slot_bytes;
  if (dyn_out) *dyn_out = dyn;
  // one SM stays free for K2, which runs beside the PDL-launched dispatch (it
  // reserves most of its SM's shared memory); every copy CTA must be resident
  return min(ctas_per_rank, (occ * (sms - 1)) / n_local);
}

extern "C" int aurora_engine_ctas(int n, int n_local, int ctas_per_rank, int row_bytes, int row2_bytes, int lsu) {
  if (n < 1 || n > AUR_MAXN || n_local < 1 || n_local > n || ctas_per_rank < 1 || row_bytes < 16 ||
      row_bytes % 16 || row2_bytes < 0 || row2_bytes % 16)
    return -AURORA_EINVAL;
  const int c = engine_ctas(n, n_local, ctas_per_rank, row_bytes, row2_bytes, lsu != 0, nullptr, nullptr, nullptr);
  return c > 0 ? c : (c == 0 ? -AURORA_EINVAL : -AURORA_ECUDA);
}

extern "C" int aurora_engine(int mode, int n, int n_local, int rank_base, const int32_t* counts,
                             const int32_t* chunks, const int32_t* rchunks,
                             const int32_t* progress, const int32_t* n_in, const int32_t* n_out,
                             const int32_t* soff, const int32_t* roff, const int32_t* send_list,
                             int send_list_stride, const void* const* src_bufs,
                             void* const* dst_bufs, int row_bytes, const void* const* src2_bufs,
                             void* const* dst2_bufs, int row2_bytes, int32_t* const* ctrs,
                             int ctas_per_rank, int max_phases, int64_t spin_limit,
                             int32_t* status, int split, const double* bw, void* const* ginfo_bufs,
                             int32_t* const* landed, const double* phase_dur, float unit_ns, void* stream) {
  if (split < 0 || split > 2) return AURORA_EINVAL;
  if (mode < 0 || mode > 511 || (mode & 12) == 12 || n < 1 || n > AUR_MAXN || n_local < 1 ||
      ((mode & 256) && ((mode & 65) || !src2_bufs || !dst2_bufs || row2_bytes < 8)) ||
      rank_base < 0 ||
      rank_base + n_local > n || row_bytes % 16 || ctas_per_rank < 1 || !counts || !chunks ||
      !rchunks || !progress || !soff || !roff || !src_bufs || !dst_bufs || !ctrs || !status ||
      ((mode & 1) == 0 && !send_list))
    return AURORA_EINVAL;
  const bool lsu = (mode & 64) != 0;
  const int rb2 = src2_bufs ? row2_bytes : 0;
  int S = 0, slot_bytes = 0;
  size_t dyn = 0;
  const int c_clamped = engine_ctas(n, n_local, ctas_per_rank, row_bytes, rb2, lsu, &S, &slot_bytes, &dyn);
  if (c_clamped < 1) return c_clamped == 0 ? AURORA_EINVAL : AURORA_ECUDA;
  ctas_per_rank = c_clamped;
  EngineParams p;
  p.mode = mode;
  p.n = n;
  p.n_local = n_local;
  p.rank_base = rank_base;
  p.meta_k = row2_bytes / 8;
  p.ginfo = reinterpret_cast<int4* const*>(ginfo_bufs);
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
  p.split = split;
  p.bw = bw;
  p.max_phases = max_phases;
  p.spin_limit = spin_limit;
  p.status = status;
  p.landed = landed;
  if (unit_ns < 0.0f || !(unit_ns == unit_ns)) return AURORA_EINVAL;
  p.phase_dur = unit_ns > 0.0f ? phase_dur : nullptr;
  p.unit_ns = unit_ns;
  if (landed && (!lsu || (mode & 1))) return AURORA_EINVAL;  // arrival credits: LSU dispatch only
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(n_local * ctas_per_rank);
  cfg.blockDim = dim3(lsu ? THREADS : TMA_THREADS);
  cfg.dynamicSmemBytes = dyn;
  cfg.stream = (cudaStream_t)stream;
  cudaLaunchAttribute attr[1];
  if (mode & 32) {  // programmatic dependent of the preceding K2 launch: start while it runs
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
  }
  const cudaError_t le = lsu ? cudaLaunchKernelEx(&cfg, engine_kernel, p)
                             : cudaLaunchKernelEx(&cfg, engine_tma_kernel, p, S, slot_bytes);
  if (le != cudaSuccess) return AURORA_ECUDA;
  AUR_CHECK_LAUNCH();
  return AURORA_OK;
}

// Traffic-matrix exchange over peer memory (SURVEY 8(e) pre-step): every process
// stores its ranks' rows of counts into every peer's copy, then releases one flag
// per local rank (value = the call's epoch); it returns once every other rank's
// flag reached the epoch. counts are double-buffered by epoch parity, so a peer
// one step ahead never overwrites rows this process may still read.
__global__ void exchange_counts_kernel(int32_t* counts2, int32_t* const* peer_counts2, int32_t* rows2,
                                       int32_t* const* peer_rows2, int w2, int32_t* xflag,
                                       int32_t* const* peer_xflag, int32_t* epoch, int n, int rank_base,
                                       int n_local, long long spin_limit, int32_t* status) {
  __shared__ int e_s;
  const int q = threadIdx.x;
  if (q == 0) {
    const int e = *epoch + 1;
    *epoch = e;
    e_s = e;
  }
  __syncthreads();
  const int e = e_s, par = (e - 1) & 1;
  const bool local_q = q >= rank_base && q < rank_base + n_local;
  // one writer per peer process: the lowest non-local rank of that process
  bool first = q < n && !local_q;
  for (int q2 = 0; first && q2 < q; q2++)
    if (!(q2 >= rank_base && q2 < rank_base + n_local) && peer_counts2[q2] == peer_counts2[q]) first = false;
  if (first) {
    const int32_t* src = counts2 + (size_t)par * n * n + (size_t)rank_base * n;
    int32_t* dst = peer_counts2[q] + (size_t)par * n * n + (size_t)rank_base * n;
    for (int v = 0; v < n_local * n; v++) dst[v] = src[v];
    if (rows2) {  // second matrix [2][n][w2] (per-expert token counts), same rows
      const int32_t* src2 = rows2 + (size_t)par * n * w2 + (size_t)rank_base * w2;
      int32_t* dst2 = peer_rows2[q] + (size_t)par * n * w2 + (size_t)rank_base * w2;
      for (int v = 0; v < n_local * w2; v++) dst2[v] = src2[v];
    }
    __threadfence_system();
    for (int r = 0; r < n_local; r++) st_release_sys(peer_xflag[q] + rank_base + r, e);
  }
  if (q < n && !local_q && !wait_ge(xflag + q, e, spin_limit, true)) atomicExch(status, AURORA_ETIMEOUT);
}

extern "C" int aurora_exchange_counts(int32_t* counts2, int32_t* const* peer_counts2, int32_t* rows2,
                                      int32_t* const* peer_rows2, int w2, int32_t* xflag,
                                      int32_t* const* peer_xflag, int32_t* epoch, int n, int rank_base,
                                      int n_local, int64_t spin_limit, int32_t* status, void* stream) {
  if (!counts2 || !peer_counts2 || !xflag || !peer_xflag || !epoch || !status || n < 1 || n > AUR_MAXN ||
      n_local < 1 || rank_base < 0 || rank_base + n_local > n || (rows2 && (!peer_rows2 || w2 < 1)))
    return AURORA_EINVAL;
  exchange_counts_kernel<<<1, 32, 0, (cudaStream_t)stream>>>(counts2, peer_counts2, rows2, peer_rows2, w2, xflag,
                                                             peer_xflag, epoch, n, rank_base, n_local, spin_limit,
                                                             status);
  AUR_CHECK_LAUNCH();
  return AURORA_OK;
}

// the fused combine's receiving side: wait for every expert rank's arrival on
// this process's senders, then re-arm the counters for the next layer step
__global__ void combine_wait_kernel(int32_t* const* ctrs, int rank_base, int n_local, int expect, int sys,
                                    long long spin_limit, int32_t* status) {
  const int r = threadIdx.x;
  if (r >= n_local) return;
  int32_t* c = ctrs[rank_base + r];
  if (!wait_ge(c + 1, expect, spin_limit, sys)) {
    atomicExch(status, AURORA_ETIMEOUT);
    return;
  }
  ((volatile int32_t*)c)[0] = 0;
  ((volatile int32_t*)c)[1] = 0;
  if (sys) __threadfence_system();  // peers on other GPUs see the re-arm before our next exchange
}

extern "C" int aurora_combine_wait(int32_t* const* ctrs, int rank_base, int n_local, int expect, int sys,
                                   int64_t spin_limit, int32_t* status, void* stream) {
  if (!ctrs || !status || n_local < 1 || n_local > AUR_MAXN || rank_base < 0 || expect < 1) return AURORA_EINVAL;
  combine_wait_kernel<<<1, 32, 0, (cudaStream_t)stream>>>(ctrs, rank_base, n_local, expect, sys, spin_limit,
                                                          status);
  AUR_CHECK_LAUNCH();
  return AURORA_OK;
}

extern "C" int aurora_debug_set_early_rows(int rows) {
  if (rows < 0) return AURORA_EINVAL;
  return cudaMemcpyToSymbol(g_early_rows, &rows, sizeof(rows)) == cudaSuccess ? AURORA_OK : AURORA_ECUDA;
}

extern "C" int aurora_debug_set_engine_trace(long long* trace) {
  return cudaMemcpyToSymbol(g_engine_trace, &trace, sizeof(trace)) == cudaSuccess ? AURORA_OK : AURORA_ECUDA;
}

extern "C" int aurora_aggregate(const void* ret_buf, int64_t ret_rank_stride_rows,
                                const int32_t* soff, const int32_t* pos, const int32_t* slot_dst,
                                const float* topk_w, int T, int k, int H, int n, int rank_base,
                                int tokens_per_rank, int pre_weighted, void* out,
                                const void* y_buf, int64_t y_rank_stride_rows, const int32_t* roff,
                                void* stream) {
  if (T <= 0 || k < 1 || k > 8 || H % 8 || n < 1 || n > AUR_MAXN || tokens_per_rank < 1 ||
      (y_buf && !roff))
    return AURORA_EINVAL;
  // 2 vectors per lane per slot in flight: measured best of 1 / 2 / 4 / 8 (C2 67 vs 73 us at 4)
  aggregate_kernel<2><<<(T + WARPS - 1) / WARPS, THREADS, 0, (cudaStream_t)stream>>>(
      (const __nv_bfloat16*)ret_buf, ret_rank_stride_rows, soff, pos, slot_dst, topk_w, T, k, H,
      n, rank_base, tokens_per_rank, pre_weighted, (__nv_bfloat16*)out, (const __nv_bfloat16*)y_buf,
      y_rank_stride_rows, roff);
  AUR_CHECK_LAUNCH();
  return AURORA_OK;
}
