// K5, CTA-pair variant: the expert grouped GEMM on tcgen05.mma.cta_group::2.
//
// A cluster of two CTAs (one TPC) computes a 256 x 256 output tile: CTA r
// stages A rows [m0 + 128 r, +128) and weight rows [n0 + 128 r, +128) (the
// instruction reads A's M halves and B's N halves from the two CTAs' shared
// memory at the same offsets) and keeps output rows m0 + 128 r .. +127, all
// 256 columns, in its own TMEM. Per CTA a pipeline stage is 32 KB instead of
// 48 KB, so six stages fit, and each SM reads half as many B bytes per FLOP.
//
// Roles per CTA: warp 0 TMA producer (both CTAs; bytes land on the leader's
// full barrier), warp 1 TMEM allocator (both, cta_group::2) and MMA issuer
// (leader only), warps 2-5 epilogue (both; arrive on the leader's tmem_empty).
// Same grouped tiling, rasterisation, epilogues and C ABI as gemm.cu.
#include <map>
#include <mutex>
#include <utility>

#include "tc_helpers.cuh"

namespace {

constexpr int BMP = 256, BN = 256, BK = 64, STAGES = 6, UMMA_K = 16;
constexpr int HALF = 128;                        // rows per CTA of A and of B
constexpr int THREADS = 192;
constexpr int A_BYTES = HALF * BK * 2;           // 16 KB
constexpr int B_BYTES = HALF * BK * 2;           // 16 KB
constexpr int STAGE_BYTES = A_BYTES + B_BYTES;   // 32 KB per CTA
constexpr int TMEM_COLS = 512;                   // 2 accumulators x 256 columns
constexpr int MAX_GROUPS = 64;
constexpr int OUT_CHUNK = 32 * 32 * 2;              // epilogue staging: 32 rows x 32 columns bf16
constexpr int OUT_BYTES = 4 * 2 * OUT_CHUNK;         // 4 epilogue warps x 2 buffers
constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + 1024 + 1024 + OUT_BYTES;
constexpr uint32_t IDESC = tc::idesc_bf16(BMP, BN);
constexpr int SC_MAXN = 16;
constexpr int TRING = 8;                         // tile-index ring (dynamic schedule)
// readers of a ring slot that arrive on the leader's tr_empty: the peer's
// producer, the MMA issuer and the 4 epilogue warps of each CTA
constexpr int TR_READERS = 1 + 1 + 8;                      // fused combine: ranks / local groups

// Fused combine (epilogue 0 with n > 0): group g is expert rank rank_base + g;
// its received rows come in per-sender blocks (roff / counts); the epilogue
// stores each output row straight into the sender's return buffer (peer memory
// over NVSwitch) at the row the combine engine would have written, local rows
// into c. The last CTA to finish releases one arrival per local group on every
// sender's {pace, done} counter (done slot).
struct Scatter {
  __nv_bfloat16* const* ret;  // [n] return buffers (peer addresses), rows of N
  const int32_t* counts;      // [n][n]
  const int32_t* soff;        // [n][n]
  const int32_t* roff;        // [n][n]
  int32_t* const* ctrs;       // [n] {pace, done} counters of the senders
  int32_t* ticket;            // grid completion ticket (zero; re-armed by the last CTA)
  int n, rank_base, sys;
  // packed groups (several experts per rank): ginfo[row] = {recv row, weight bits, single, -}
  // per packed row (written by the grouped dispatch). A row whose (token, rank) has one
  // local expert is finished here -- w * y, stored into its sender's return buffer (to_ret,
  // other ranks) or into ybuf -- instead of going through the pre-reduction. No arrivals:
  // the pre-reduction that follows signals the senders.
  const int4* ginfo;
  int G;                      // experts per rank (groups per local rank)
  __nv_bfloat16* ybuf;        // [n_local][ycap] rows of N
  long long ycap;
  int to_ret;
};

struct TileIter2 {
  int n_tiles_n, total, nseg;
  // tile order = segments (group, first m-tile, m-tiles) back to back; one per group, or with
  // arrival-driven tiles two per group: the m-tiles holding only local rows first (all groups),
  // then the rest
  int seg_g[2 * MAX_GROUPS], seg_m0[2 * MAX_GROUPS], seg_mt[2 * MAX_GROUPS + 1], seg_prefix[2 * MAX_GROUPS + 1];
  int pg, plc, pnc, plo, phi;  // partitioned mode: this cluster's partition, index among its
                               // clusters, their count, its tile range [plo, phi)
  int prefix[MAX_GROUPS + 1];
  int mt[MAX_GROUPS];
  int ms[MAX_GROUPS];
  int rows[MAX_GROUPS];
};

__device__ __forceinline__ void tile_coords2(const TileIter2& it, int G, int gm, int t, int& g,
                                             int& mt, int& nt) {
  // segment of tile t: the last q with seg_prefix[q] <= t (binary search: up to 128 segments)
  int lo = 0, hi = it.nseg - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (it.seg_prefix[mid] <= t) lo = mid;
    else hi = mid - 1;
  }
  g = it.seg_g[lo];
  const int local = t - it.seg_prefix[lo];
  const int per_block = gm * it.n_tiles_n;
  const int sb = local / per_block, rem = local - sb * per_block;
  const int rows = min(gm, it.seg_mt[lo] - sb * gm);
  mt = it.seg_m0[lo] + sb * gm + rem % rows;
  nt = rem / rows;
}

// diagnostics (aurora_debug_set_gemm_trace): per CTA {entry, first tile's loads issued} in
// %globaltimer ns -- shows the arrival-driven GEMM1 running beside the dispatch
__device__ long long* g_gemm_trace = nullptr;
__device__ __forceinline__ long long gemm_ns() {
  long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// Arrival-driven GEMM1 (N1): the receive buffer of local group g (rank rank_base + g) holds the
// rank's local rows first, then each sender's block at roff[i][j]; landed[g * n + i] counts the
// rows of block (i -> j) the dispatch has made visible. A tile waits until every block under its
// rows is complete.
struct Arrival {
  int32_t* landed;        // [n_local][n] (this process's receivers), re-armed by the last cluster
  const int32_t* counts;  // [n][n]
  const int32_t* roff;    // [n][n]
  int n, rank_base, sys;
};

__device__ __forceinline__ void wait_rows_landed(const Arrival& ar, int g, int r_lo, int r_hi) {
  const int j = ar.rank_base + g;
  for (int i = 0; i < ar.n; i++) {
    const int c = ar.counts[i * ar.n + j];
    const int b0 = ar.roff[i * ar.n + j];
    if (c == 0 || b0 >= r_hi || b0 + c <= r_lo) continue;
    const int32_t* f = ar.landed + g * ar.n + i;
    int spins = 0;
    while ((ar.sys ? ld_acquire_sys(f) : ld_acquire_gpu(f)) < c)
      if (++spins > 8) __nanosleep(64);
  }
  // the rows were written through the generic proxy; the tile loads are TMA (async proxy)
  asm volatile("fence.proxy.async.global;" ::: "memory");
}

__device__ __forceinline__ float silu_mul(float g, float u) { return g / (1.0f + __expf(-g)) * u; }

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(THREADS, 1)
    grouped_gemm_2sm_kernel(const __grid_constant__ CUtensorMap map_a,
                            const __grid_constant__ CUtensorMap map_b,
                            __nv_bfloat16* __restrict__ c, const int32_t* __restrict__ m_start,
                            const int32_t* __restrict__ m_rows, int G, long long cap, int N, int K,
                            int epilogue, int group_m, const Scatter sc,
                            int32_t* __restrict__ tile_ctr, const __grid_constant__ CUtensorMap map_c,
                            int tma_out, const int32_t* __restrict__ part, int part_gp, const Arrival ar,
                            int pdl_wait) {
  // the next GEMM of the same FFN (a programmatic dependent launch) may start its prologue as CTAs exit
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  extern __shared__ uint8_t smem_raw[];
  // first launch after arming wins (GEMM1; GEMM2's CTAs find the slots taken)
  if (threadIdx.x == 0 && g_gemm_trace)
    atomicCAS(reinterpret_cast<unsigned long long*>(g_gemm_trace + blockIdx.x * 2), 0ull,
              (unsigned long long)gemm_ns());
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_base_s = reinterpret_cast<uint32_t*>(tempty + 2);
  // epilogue staging for the TMA stores (1 KB-aligned, 64-byte swizzle)
  uint8_t* out_stage = smem + STAGES * STAGE_BYTES + 1024;
  __shared__ TileIter2 it;
  // dynamic tile order (tile_ctr != NULL): the leader's producer takes the next
  // tile index from a global counter and publishes it to both CTAs' rings
  __shared__ int tile_ring[TRING];
  __shared__ __align__(8) uint64_t tr_full[TRING], tr_empty[TRING];
  __shared__ int sc_lo[SC_MAXN * SC_MAXN], sc_cnt[SC_MAXN * SC_MAXN], sc_dst[SC_MAXN * SC_MAXN];

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = tc::cluster_rank();
  const bool leader = rank == 0;
  const int cluster_id = blockIdx.x >> 1, n_clusters = gridDim.x >> 1;

  if (threadIdx.x == 0) {
    it.n_tiles_n = N / BN;
    int acc = 0;
    for (int g = 0; g < G; g++) {
      const int m = m_rows[g];
      it.rows[g] = m;
      it.mt[g] = (m + BMP - 1) / BMP;
      it.ms[g] = m_start ? m_start[g] : 0;
      it.prefix[g] = acc;
      acc += it.mt[g] * it.n_tiles_n;
    }
    it.prefix[G] = acc;
    it.total = acc;
    int ns = 0, sacc = 0;
    auto add_seg = [&](int g, int m0, int mtn) {
      if (mtn <= 0) return;
      it.seg_g[ns] = g;
      it.seg_m0[ns] = m0;
      it.seg_mt[ns] = mtn;
      it.seg_prefix[ns] = sacc;
      sacc += mtn * it.n_tiles_n;
      ns++;
    };
    if (ar.landed) {  // local-only m-tiles of every group first: they need no network row
      for (int g = 0; g < G; g++) add_seg(g, 0, min(it.mt[g], ar.counts[(ar.rank_base + g) * (ar.n + 1)] / BMP));
      for (int g = 0; g < G; g++) {
        const int l = min(it.mt[g], ar.counts[(ar.rank_base + g) * (ar.n + 1)] / BMP);
        add_seg(g, l, it.mt[g] - l);
      }
    } else {
      for (int g = 0; g < G; g++) add_seg(g, 0, it.mt[g]);
    }
    if (ns == 0) {  // no tiles: keep the search well-defined
      it.seg_g[0] = 0;
      it.seg_m0[0] = it.seg_mt[0] = it.seg_prefix[0] = 0;
      ns = 1;
    }
    it.seg_prefix[ns] = sacc;
    it.nseg = ns;
    // partitioned mode (emulated per-rank compute): clusters [part[q], part[q+1]) serve partition q
    // only -- groups [q * part_gp, (q + 1) * part_gp), one rank's experts -- round robin over its tiles
    it.pg = -1;
    if (part) {
      for (int q = 0; q < G / part_gp; q++)
        if (part[q] <= cluster_id && cluster_id < part[q + 1]) {
          it.pg = q;
          it.plc = cluster_id - part[q];
          it.pnc = part[q + 1] - part[q];
          it.plo = it.prefix[q * part_gp];
          it.phi = it.prefix[(q + 1) * part_gp];
        }
    }
    const int sc_ranks = sc.ginfo ? G / sc.G : G;   // local ranks the table covers
    for (int q = 0; q < (sc.n ? sc_ranks * sc.n : 0); q++) {  // (local rank, sender) -> row block
      const int g = q / sc.n, src = q - g * sc.n, r = sc.rank_base + g;
      sc_lo[q] = sc.roff[src * sc.n + r];
      sc_cnt[q] = sc.counts[src * sc.n + r];
      sc_dst[q] = sc.soff[src * sc.n + r];
    }
    for (int s = 0; s < STAGES; s++) {
      tc::mbar_init(&full[s], 1);   // leader: its expect_tx arrive + both CTAs' bytes
      tc::mbar_init(&empty[s], 1);  // the leader's MMA commit, multicast to both CTAs
    }
    for (int q = 0; q < TRING; q++) {
      tc::mbar_init(&tr_full[q], 1);
      tc::mbar_init(&tr_empty[q], TR_READERS);
    }
    for (int a = 0; a < 2; a++) {
      tc::mbar_init(&tfull[a], 1);
      tc::mbar_init(&tempty[a], 2 * 128);  // every epilogue thread of both CTAs
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     tc::smem_u32(tmem_base_s)),
                 "r"(TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  tc::fence_before();
  __syncthreads();
  tc::cluster_sync();
  tc::fence_after();
  const uint32_t tmem_base = *tmem_base_s;
  // GEMM2 launched as a programmatic dependent of GEMM1: barriers, TMEM and the tile tables are set
  // up while GEMM1's last tiles run; wait for GEMM1's grid (its h and the re-armed tile counter)
  if (pdl_wait) asm volatile("griddepcontrol.wait;" ::: "memory");
  const int k_blocks = K / BK;
  const bool dyn = tile_ctr != nullptr && part == nullptr;
  // i-th tile of this cluster (-1: done). Static: round robin over clusters.
  // Dynamic: ring slot i % TRING, published by the leader's producer.
  auto next_tile = [&](int i, bool arrive) -> int {
    if (!dyn) {
      if (part) {  // round robin over the partition's own clusters
        if (it.pg < 0) return -1;
        const int t = it.plo + it.plc + i * it.pnc;
        return t < it.phi ? t : -1;
      }
      const int t = cluster_id + i * n_clusters;
      return t < it.total ? t : -1;
    }
    const int q = i % TRING;
    tc::mbar_wait_cluster(&tr_full[q], (uint32_t)(i / TRING) & 1u);
    const int t = *(volatile int*)&tile_ring[q];
    if (arrive) tc::mbar_arrive_cluster(tc::mapa(tc::smem_u32(&tr_empty[q]), 0));
    return t;
  };

  if (warp == 0) {
    if (lane == 0) {  // ---------------- TMA producer (both CTAs)
      const uint32_t full0 = tc::mapa(tc::smem_u32(&full[0]), 0);
      int s = 0;
      uint32_t ph = 0;
      bool ended = false;
      // leader: publish tile j (index t from the global counter) to both CTAs' rings
      auto publish = [&](int j, int t) {
        const int q = j % TRING;
        if (j >= TRING) tc::mbar_wait_cluster(&tr_empty[q], (uint32_t)(j / TRING - 1) & 1u);
        if (ended || t >= it.total) t = -1;
        ended = ended || t < 0;
        tile_ring[q] = t;
        const uint32_t peer_slot = tc::mapa(tc::smem_u32(&tile_ring[q]), 1);
        asm volatile("st.shared::cluster.u32 [%0], %1;" ::"r"(peer_slot), "r"(t) : "memory");
        tc::mbar_arrive_cluster(tc::smem_u32(&tr_full[q]));
        tc::mbar_arrive_cluster(tc::mapa(tc::smem_u32(&tr_full[q]), 1));
      };
      if (dyn && leader) {
        publish(0, atomicAdd(tile_ctr, 1));
        publish(1, atomicAdd(tile_ctr, 1));
      }
      for (int i = 0;; i++) {
        int t, ahead = -1;
        if (dyn && leader) {
          // two tiles of lookahead: tile i + 2's counter fetch is issued now and its
          // result consumed after this tile's loads, so neither CTA waits on it
          ahead = ended ? -1 : atomicAdd(tile_ctr, 1);
          t = tile_ring[i % TRING];
        } else {
          t = next_tile(i, dyn);
        }
        if (t < 0) break;
        int g, mt, nt;
        tile_coords2(it, G, group_m, t, g, mt, nt);
        if (ar.landed) {  // N1: this CTA's 128 rows of the tile must have arrived
          const int r_lo = mt * BMP + (int)rank * HALF;
          if (r_lo < it.rows[g]) wait_rows_landed(ar, g, r_lo, min(r_lo + HALF, it.rows[g]));
        }
        if (i == 0 && g_gemm_trace)
          atomicCAS(reinterpret_cast<unsigned long long*>(g_gemm_trace + blockIdx.x * 2 + 1), 0ull,
                    (unsigned long long)gemm_ns());
        const int a_row = (int)(g * cap) + it.ms[g] + mt * BMP + (int)rank * HALF;
        const int b_row = g * N + nt * BN + (int)rank * HALF;
        for (int kb = 0; kb < k_blocks; kb++) {
          tc::mbar_wait(&empty[s], ph ^ 1);
          uint8_t* sa = smem + s * STAGE_BYTES;
          if (leader) tc::mbar_expect_tx(&full[s], 2 * STAGE_BYTES);
          const uint32_t fb = full0 + s * 8;
          tc::tma_load_2d_pair(sa, &map_a, fb, kb * BK, a_row);
          tc::tma_load_2d_pair(sa + A_BYTES, &map_b, fb, kb * BK, b_row);
          if (++s == STAGES) { s = 0; ph ^= 1; }
        }
        if (dyn && leader) publish(i + 2, ahead);
      }
    }
  } else if (warp == 1) {
    if (leader && lane == 0) {  // ---------------- MMA issuer (leader only)
      int s = 0;
      uint32_t ph = 0;
      for (int local = 0;; local++) {
        if (next_tile(local, true) < 0) break;
        const int acc = local & 1;
        tc::mbar_wait_cluster(&tempty[acc], ((local >> 1) & 1) ^ 1);
        tc::fence_after();
        const uint32_t d = tmem_base + acc * BN;
        for (int kb = 0; kb < k_blocks; kb++) {
          tc::mbar_wait(&full[s], ph);
          tc::fence_after();
          uint8_t* sa = smem + s * STAGE_BYTES;
          const uint64_t ad = tc::sw128_desc(sa), bd = tc::sw128_desc(sa + A_BYTES);
#pragma unroll
          for (int k = 0; k < BK / UMMA_K; k++)
            tc::umma_bf16_pair(d, ad + 2 * k, bd + 2 * k, IDESC, (kb | k) != 0);
          tc::umma_commit_pair(&empty[s], 0x3);  // frees the stage in both CTAs
          if (++s == STAGES) { s = 0; ph ^= 1; }
        }
        tc::umma_commit_pair(&tfull[acc], 0x3);
      }
    }
  } else {  // ---------------- epilogue warps 2..5 (both CTAs)
    const int quarter = warp & 3;
    const uint32_t tempty0 = tc::mapa(tc::smem_u32(&tempty[0]), 0);
    // Output of one 32-column chunk of the warp's 32 rows (lane = row, 64 B each). With
    // tma_out and every row live: staged in shared memory (64-byte swizzle, two buffers)
    // and written by one TMA store of the 32 x 32 box -- whole 64-byte row segments
    // instead of 32 rows x 16 B per store instruction. Otherwise plain stores.
    const uint32_t stage_w = tc::smem_u32(out_stage) + quarter * 2 * OUT_CHUNK;
    int chunk_no = 0;
    auto emit = [&](const uint32_t (&packed)[16], bool live, __nv_bfloat16* out_row, int col, long long row0) {
      if (tma_out && __all_sync(0xffffffffu, live)) {
        const uint32_t buf = stage_w + (chunk_no & 1) * OUT_CHUNK;
        if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
        __syncwarp();
#pragma unroll
        for (int q = 0; q < 4; q++) {
          const uint32_t a = buf + lane * 64 + ((q ^ ((lane >> 1) & 3)) << 4);
          asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(a), "r"(packed[4 * q]),
                       "r"(packed[4 * q + 1]), "r"(packed[4 * q + 2]), "r"(packed[4 * q + 3])
                       : "memory");
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
        if (lane == 0) {
          asm volatile(
              "cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(
                  reinterpret_cast<uint64_t>(&map_c)),
              "r"(col), "r"((int)row0), "r"(buf)
              : "memory");
          asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        }
        chunk_no++;
      } else if (live) {
        int4* o = reinterpret_cast<int4*>(out_row);
#pragma unroll
        for (int q = 0; q < 4; q++)
          o[q] = make_int4(packed[4 * q], packed[4 * q + 1], packed[4 * q + 2], packed[4 * q + 3]);
      }
    };
    for (int local = 0;; local++) {
      // one reader arrival per epilogue warp: lane 0 after the warp has the index
      int t = 0;
      if (lane == 0) t = next_tile(local, false);
      t = __shfl_sync(0xffffffffu, t, 0);
      if (dyn && lane == 0)  // t is consumed (shuffled) above: the slot has been read
        tc::mbar_arrive_cluster_relaxed(tc::mapa(tc::smem_u32(&tr_empty[local % TRING]), 0));
      if (t < 0) break;
      int g, mt, nt;
      tile_coords2(it, G, group_m, t, g, mt, nt);
      const int acc = local & 1;
      tc::mbar_wait(&tfull[acc], (local >> 1) & 1);
      tc::fence_after();
      const int row_in_group = mt * BMP + (int)rank * HALF + quarter * 32 + lane;
      const bool live = row_in_group < it.rows[g];
      const long long row = g * cap + it.ms[g] + row_in_group;
      const uint32_t tbase = tmem_base + ((uint32_t)(quarter * 32) << 16) + acc * BN;
      const long long row0 = row - lane;  // the warp's first row
      if (epilogue == 1) {
        __nv_bfloat16* out = c + row * (long long)(N / 2) + nt * (BN / 2);
        for (int c0 = 0; c0 < BN / 2; c0 += 32) {
          uint32_t gr[32], ur[32];
          TC_TMEM_LD32(tbase + c0, gr);
          TC_TMEM_LD32(tbase + BN / 2 + c0, ur);
          tc::tmem_ld_wait();
          uint32_t packed[16];
#pragma unroll
          for (int q = 0; q < 16; q++) {
            float a0 = silu_mul(__uint_as_float(gr[2 * q]), __uint_as_float(ur[2 * q]));
            float a1 = silu_mul(__uint_as_float(gr[2 * q + 1]), __uint_as_float(ur[2 * q + 1]));
            __nv_bfloat162 h2 = __floats2bfloat162_rn(a0, a1);
            packed[q] = *reinterpret_cast<uint32_t*>(&h2);
          }
          emit(packed, live, out + c0, nt * (BN / 2) + c0, row0);
        }
      } else {
        __nv_bfloat16* out = c + row * (long long)N + nt * BN;
        bool weighted = false;
        float wsc = 0.0f;
        if (sc.n && live && sc.ginfo) {  // packed groups: single-expert rows are finished here
          const int4 rec = sc.ginfo[row];
          if (rec.z) {
            weighted = true;
            wsc = __int_as_float(rec.y);
            const int rl = g / sc.G, rr = sc.rank_base + rl, recv_row = rec.x;
            out = sc.ybuf + ((long long)rl * sc.ycap + recv_row) * N + nt * BN;
            if (sc.to_ret)
              for (int src = 0; src < sc.n; src++) {
                const int q = rl * sc.n + src, off = recv_row - sc_lo[q];
                if (off >= 0 && off < sc_cnt[q]) {
                  if (src != rr) out = sc.ret[src] + (long long)(sc_dst[q] + off) * N + nt * BN;
                  break;
                }
              }
          }
        } else if (sc.n && live) {  // fused combine: the row goes back to its sender
          for (int src = 0; src < sc.n; src++) {
            const int q = g * sc.n + src, off = row_in_group - sc_lo[q];
            if (off >= 0 && off < sc_cnt[q]) {
              if (src != sc.rank_base + g)
                out = sc.ret[src] + (long long)(sc_dst[q] + off) * N + nt * BN;
              break;
            }
          }
        }
        for (int c0 = 0; c0 < BN; c0 += 32) {
          uint32_t r[32];
          TC_TMEM_LD32(tbase + c0, r);
          tc::tmem_ld_wait();
          uint32_t packed[16];
#pragma unroll
          for (int q = 0; q < 16; q++) {
            __nv_bfloat162 h2 = __floats2bfloat162_rn(__uint_as_float(r[2 * q]), __uint_as_float(r[2 * q + 1]));
            if (weighted) {  // the pre-reduction's arithmetic: fmaf(w, bf16(y), 0) in fp32, then bf16
              const float2 f = __bfloat1622float2(h2);
              h2 = __floats2bfloat162_rn(fmaf(wsc, f.x, 0.0f), fmaf(wsc, f.y, 0.0f));
            }
            packed[q] = *reinterpret_cast<uint32_t*>(&h2);
          }
          emit(packed, live, out + c0, nt * BN + c0, row0);
        }
      }
      // the accumulator may be overwritten once every tcgen05.ld of it has completed
      // (tmem_ld_wait above); the epilogue's global stores need no ordering here
      tc::fence_before();
      tc::mbar_arrive_cluster_relaxed(tempty0 + acc * 8);
    }
    if (tma_out && lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  }
  if (sc.n) {
    if (sc.sys) __threadfence_system();
    else __threadfence();
  }
  tc::fence_before();
  __syncthreads();
  tc::cluster_sync();
  if (dyn && leader && threadIdx.x == 0) {  // last cluster out re-arms the tile counter
    if (atomicAdd(tile_ctr + 1, 1) == n_clusters - 1) {
      tile_ctr[0] = 0;
      tile_ctr[1] = 0;
      if (ar.landed)  // every tile has passed its arrival wait: re-arm for the next dispatch
        for (int q = 0; q < G * ar.n; q++) ar.landed[q] = 0;
      __threadfence();
    }
  }
  if (sc.n && !sc.ginfo && threadIdx.x == 0) {  // grid completion -> one arrival per group on every sender
    __threadfence();
    if (atomicAdd(sc.ticket, 1) == (int)gridDim.x - 1) {
      __threadfence();
      *sc.ticket = 0;
      for (int src = 0; src < sc.n; src++) {
        if (sc.sys) red_release_sys_add(sc.ctrs[src] + 1, G);
        else red_release_gpu_add(sc.ctrs[src] + 1, G);
      }
    }
  }
  if (warp == 1) {
    __syncwarp();
    tc::fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                 "r"(TMEM_COLS));
  }
}

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                  const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                  const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

bool make_map_2d(CUtensorMap* m, const void* base, uint64_t rows, uint64_t cols, uint32_t box_rows) {
  static EncodeTiledFn fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) !=
            cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      return false;
    fn = reinterpret_cast<EncodeTiledFn>(p);
  }
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {cols * 2};
  cuuint32_t box[2] = {BK, box_rows};
  cuuint32_t estr[2] = {1, 1};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box,
            estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// output map for the epilogue's TMA stores: 32 x 32 boxes, 64-byte swizzle
bool make_map_out(CUtensorMap* m, const void* base, uint64_t rows, uint64_t cols) {
  static EncodeTiledFn fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      return false;
    fn = reinterpret_cast<EncodeTiledFn>(p);
  }
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {cols * 2};
  cuuint32_t box[2] = {32, 32};
  cuuint32_t estr[2] = {1, 1};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, estr,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_NONE,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

}  // namespace

// C-ABI-internal launcher used by gemm.cu when the pair kernel is selected.
int aurora_launch_grouped_2sm(const void* a, const void* b, void* c, const int32_t* m_start,
                              const int32_t* m_rows, int G, int64_t cap, int64_t map_rows, int N,
                              int K, int epilogue, int32_t* tile_ctr, int num_sms, cudaStream_t stream,
                              const AuroraScatterArgs* scatter, const int32_t* cluster_part, int part_gp,
                              const AuroraArrivalArgs* arrival, int after_gemm) {
  Scatter sc{};
  if (scatter) {
    const bool packed = scatter->ginfo != nullptr;
    const int ranks = packed ? (scatter->G > 0 ? G / scatter->G : 0) : G;
    if (epilogue != 0 || scatter->n < 1 || scatter->n > SC_MAXN || ranks < 1 || ranks > SC_MAXN ||
        scatter->rank_base < 0 || scatter->rank_base + ranks > scatter->n || !scatter->ret || !scatter->counts ||
        !scatter->soff || !scatter->roff ||
        (packed ? (cap != 0 || !m_start || G % scatter->G || !scatter->ybuf || scatter->ycap < 1)
                : (m_start || cap <= 0 || !scatter->ctrs || !scatter->ticket)))
      return AURORA_EINVAL;
    sc.ginfo = reinterpret_cast<const int4*>(scatter->ginfo);
    sc.G = scatter->G;
    sc.ybuf = reinterpret_cast<__nv_bfloat16*>(scatter->ybuf);
    sc.ycap = scatter->ycap;
    sc.to_ret = scatter->to_ret;
    sc.ret = reinterpret_cast<__nv_bfloat16* const*>(scatter->ret);
    sc.counts = scatter->counts;
    sc.soff = scatter->soff;
    sc.roff = scatter->roff;
    sc.ctrs = scatter->ctrs;
    sc.ticket = scatter->ticket;
    sc.n = scatter->n;
    sc.rank_base = scatter->rank_base;
    sc.sys = scatter->sys;
  }
  if (cap < 0 || (cap == 0 && (map_rows <= 0 || !m_start))) return AURORA_EINVAL;
  if (cluster_part && (part_gp < 1 || G % part_gp)) return AURORA_EINVAL;
  if (map_rows <= 0) map_rows = (int64_t)G * cap;
  if (G < 1 || G > MAX_GROUPS || N % BN || K % BK || N <= 0 || K <= 0 ||
      (epilogue != 0 && epilogue != 1) || !a || !b || !c || !m_rows)
    return AURORA_EINVAL;
  CUtensorMap ma, mb, mc;
  if (!make_map_2d(&ma, a, (uint64_t)map_rows, K, HALF) ||
      !make_map_2d(&mb, b, (uint64_t)G * N, K, HALF))
    return AURORA_ECUDA;
  // TMA-stored epilogue for plain outputs (rows go where the tile is); scattered
  // outputs (fused combine, packed scatter) keep per-row stores
  static const bool tma_env = !getenv("AURORA_GEMM_TMA_STORE") || atoi(getenv("AURORA_GEMM_TMA_STORE")) != 0;
  const int n_out = epilogue == 1 ? N / 2 : N;
  const int tma_out = (tma_env && !scatter) ? 1 : 0;
  if (!make_map_out(&mc, c, (uint64_t)map_rows, (uint64_t)n_out)) return AURORA_ECUDA;
  static bool attr_set = false;
  if (!attr_set) {
    if (cudaFuncSetAttribute(grouped_gemm_2sm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             SMEM_BYTES) != cudaSuccess)
      return AURORA_ECUDA;
    attr_set = true;
  }
  // dynamic tile order (default): clusters take tiles from a global counter, so the
  // tiles in flight stay a window of consecutive indices and each operand tile is
  // read from DRAM about once (8-expert C2 GEMM1: 8.1 -> 2.2 GB for 2.15 GB of
  // operands); AURORA_GEMM_STATIC=1: round robin (clusters drift apart over the
  // persistent loop and the window -- the L2 working set -- grows with the drift)
  // The counter pair {next tile, clusters done} is the caller's (zero before first use, re-armed by
  // the kernel's last cluster): one per stream of launches that may run concurrently. NULL = round robin.
  static const bool dyn_sched = !getenv("AURORA_GEMM_STATIC") || atoi(getenv("AURORA_GEMM_STATIC")) == 0;
  if (!dyn_sched) tile_ctr = nullptr;
  int group_m = (int)max(1LL, min(64LL, (32LL << 20) / ((long long)BMP * K * 2)));
  // long K (GEMM2, K = F): blocks of 8 m-tiles -- the weight slab of an n-tile serves 8 consecutive
  // tiles; measured C2 GEMM2 DRAM reads 5.8 GB (4) / 5.0 (6) / 5.0 (8) / 5.3 (12) / 6.6 GB (16)
  // at equal duration (tools/gemm2_gm_sweep.sh), and ~1.5 % faster sustained steps with 8
  if (K > 8192) group_m = max(group_m, 8);
  // experiment hook: AURORA_GEMM_GM_LONGK=g sets the m-block of long-K launches (K > 8192, GEMM2)
  static const int gm_longk = getenv("AURORA_GEMM_GM_LONGK") ? atoi(getenv("AURORA_GEMM_GM_LONGK")) : 0;
  if (gm_longk > 0 && K > 8192) group_m = gm_longk;
  if (num_sms <= 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&num_sms, cudaDevAttrMultiProcessorCount, dev);
  }
  const int grid = num_sms & ~1;
  Arrival ar{};
  if (arrival) {
    // arrival-driven tiles need the dynamic order (its last cluster re-arms `landed`), whole
    // receive buffers (m_start 0) and one expert per rank
    if (!tile_ctr || cluster_part || m_start || scatter || !arrival->landed || !arrival->counts ||
        !arrival->roff || arrival->n < 1 || arrival->rank_base < 0 || arrival->rank_base + G > arrival->n)
      return AURORA_EINVAL;
    ar = Arrival{arrival->landed, arrival->counts, arrival->roff, arrival->n, arrival->rank_base, arrival->sys};
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(THREADS);
  cfg.dynamicSmemBytes = SMEM_BYTES;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  // programmatic dependent launch: of the dispatch (N1: runs beside it, gated by `landed`), or of
  // the FFN's previous GEMM (after_gemm: prologue overlaps its tail, then griddepcontrol.wait)
  static const bool gemm_pdl = !getenv("AURORA_GEMM_PDL") || atoi(getenv("AURORA_GEMM_PDL")) != 0;
  if (!gemm_pdl) after_gemm = 0;
  if ((arrival && arrival->pdl) || after_gemm) {
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
  }
  if (cudaLaunchKernelEx(&cfg, grouped_gemm_2sm_kernel, ma, mb, (__nv_bfloat16*)c, m_start, m_rows, G,
                         (long long)cap, N, K, epilogue, group_m, sc, tile_ctr, mc, tma_out, cluster_part,
                         part_gp > 0 ? part_gp : 1, ar, after_gemm ? 1 : 0) != cudaSuccess)
    return AURORA_ECUDA;
  AUR_CHECK_LAUNCH();
  return AURORA_OK;
}

extern "C" int aurora_debug_set_gemm_trace(long long* trace) {
  return cudaMemcpyToSymbol(g_gemm_trace, &trace, sizeof(trace)) == cudaSuccess ? AURORA_OK : AURORA_ECUDA;
}
