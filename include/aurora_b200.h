/*
 * aurora_b200.h -- C ABI of the B200-native Aurora MoE-layer hot path.
 *
 * One shared library (paper_2410_17043_b200/libaurora_b200.so, built for
 * sm_100a) exports these entry points. Plain pointers and sizes only; every
 * pointer named d_* / "device" is a CUDA device pointer, `stream` is a
 * cudaStream_t passed as void*. Calls are asynchronous on `stream`; results
 * that the reference returns synchronously (status words, phase counts) are
 * written to device memory and read by the host shim only on the drop-in /
 * debug path -- the MoE layer itself never synchronises with the host.
 *
 * The reference (arxiv 2410.17043, package `moeplan`) is pure Python with
 * no FFI; each entry point below names the reference function it replaces
 * (file:line under pkg/src/moeplan/). The Python binding a maintainer would
 * add on the reference side is in INTEGRATION.md.
 */
#ifndef AURORA_B200_H
#define AURORA_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Return / status codes. Map to the reference's exception types:
 *   AURORA_EINVAL    -> ValueError           (core.py:88-94, commsched.py:56-59, 95-101)
 *   AURORA_EOVERFLOW -> DecompositionError   (commsched.py:260-264, phase bound n^2-2n+2)
 *   AURORA_ENOMATCH  -> DecompositionError   (commsched.py:267-272, no perfect matching)   */
#define AURORA_OK 0
#define AURORA_EINVAL 1
#define AURORA_EOVERFLOW 2
#define AURORA_ENOMATCH 3
#define AURORA_ECUDA 10
#define AURORA_EUNSUPPORTED 11
#define AURORA_ETIMEOUT 12

#define AURORA_MAX_RANKS 32

int aurora_version(void);

/* Table capacities: raw permutation phases (commsched.py:253, n^2-2n+2) and
 * stripped phases (each of the <= n(n-1) real pairs can split one raw phase:
 * 2n^2-3n+2). */
int aurora_raw_phase_cap(int n);
int aurora_phase_cap(int n);

/* ---------------------------------------------------------------- K2 ----
 * aurora_schedule_f64: replaces moeplan.commsched.build_schedule
 * (commsched.py:291-324) including decompose's raw permutations
 * (commsched.py:237-278). Bit-exact with the reference for n <= 32.
 *   d[n*n]   traffic matrix, row-major, float64 (TrafficMatrix.entries, core.py:75-97)
 *   bw[n]    ClusterSpec.bandwidths (core.py:179-181); NULL == all 1.0
 *   raw_perm[(n^2-2n+2)*n], raw_dur[n^2-2n+2], n_raw[1]       (decompose output)
 *   phase_recv[(2n^2-3n+2)*n]  receiver of sender i in phase k, or -1
 *   phase_dur[2n^2-3n+2], n_phases[1], b_max[1] (bmax_heterogeneous)
 *   status[1] AURORA_OK / EINVAL / EOVERFLOW / ENOMATCH
 * The makespan is math.fsum(phase_dur) (commsched.py:323), done by the shim. */
int aurora_schedule_f64(const double* d, const double* bw, int n, int32_t* raw_perm,
                        double* raw_dur, int32_t* n_raw, int32_t* phase_recv, double* phase_dur,
                        int32_t* n_phases, double* b_max, int32_t* status, void* stream);

/* aurora_schedule_counts: the in-layer variant. Same schedule, computed from
 * the router's int32 GPU x GPU token counts (diagonal = local tokens,
 * ignored by the schedule like TrafficMatrix does, core.py:95), plus the
 * engine tables, one entry per (coalesced) phase:
 *   chunks[P][n][4]   per phase k and sender i: {receiver j (-1: idle), first
 *                     token of pair (i,j) in this phase, token count, run code}.
 *                     A run is a maximal stretch of consecutive phases in which
 *                     i sends to j; run code = r (index of the run among the
 *                     runs into j) on a run's first entry, -1-r on its
 *                     continuation entries (no hand-over needed: nobody else
 *                     sends to j in between).
 *   rchunks[P][n][4]  the same entries indexed by receiver j: {sender, first,
 *                     count, run code of the reversed run into the sender} (the
 *                     combine runs CommSchedule.reversed(), commsched.py:153-162)
 *   n_in[n], n_out[n] arrival signals each rank receives in the dispatch / combine
 *   Hand-over thresholds and n_in / n_out count arrival signals: every copy CTA of
 *   the sending rank signals once per run. The copy CTAs are the engine's
 *   (aurora_engine_ctas): each process drives n_local ranks with ctas_dispatch /
 *   ctas_combine CTAs in total, split among them by `split` (AURORA_SPLIT_*,
 *   csrc/apportion.cuh). ctas_dispatch == 0: thresholds in runs (one signal per run).
 *   progress[1]       (nullable) written while the kernel runs: the number of
 *                     leading phases whose entries are final, then
 *                     n_phases | AURORA_PROGRESS_DONE once every output is
 *                     written. The engine polls it, so dispatch can start on
 *                     phase 0 while later phases are still being computed. The
 *                     caller zeroes it (stream-ordered) before the launch.
 * (the buffer layout soff / roff the chunk offsets refer to comes from aurora_pack)
 * Heterogeneous durations (time units, commsched.py:181-190) are converted to
 * whole tokens per entry by rounding each pair's cumulative time x
 * min(B_i,B_j) (the pair's final cumulative time lands on its exact count; a
 * pair that would need a correction is reported as AURORA_EINVAL). */
#define AURORA_PROGRESS_DONE (1 << 20)
#define AURORA_SPLIT_EVEN 0
#define AURORA_SPLIT_VOLUME 1
#define AURORA_SPLIT_BANDWIDTH 2
#define AURORA_PROGRESS_COUNT ((1 << 20) - 1)
int aurora_schedule_counts(const int32_t* counts, const double* bw, int n, int32_t* phase_recv,
                           double* phase_dur, int32_t* n_phases, int32_t* chunks,
                           int32_t* rchunks, int32_t* n_in, int32_t* n_out, int32_t* status,
                           int32_t* progress, int n_local, int ctas_dispatch, int ctas_combine,
                           int split, void* stream);

/* ---------------------------------------------------------------- K1 ----
 * aurora_route: top-k gating + GPU x GPU traffic matrix. No reference
 * function: the reference models the gate as LayerProfile.gate_work
 * (core.py:194-221) and consumes its output as TrafficMatrix (core.py:75-117)
 * relabelled by deploy_to_gpus (core.py:337-345).
 *   x[T][H] bf16; gate_prep = the bf16 gate w_gate[E][H] prepared once by
 *   aurora_route_prepare_gate; bias[E] f32; H % 256 == 0, E <= 64, k <= 8
 *   gpu_of_expert[E]  rank hosting expert e (DeploymentPlan.assignment_a, core.py:253-304)
 *   tokens are grouped by rank: token t (local index) lives on rank
 *   rank_base + t / tokens_per_rank (workload.py:59-61)
 * Outputs: topk_idx[T][k], topk_w[T][k] (softmax over the selected logits),
 *   slot_dst[T][k] (destination rank g of the slot, or -(g+1) when an earlier
 *   slot of the same token already goes to g: a token crosses the network
 *   once per destination), blk_cnt[T/64][n] per-64-token-block histogram,
 *   counts[n][n] += this call's rows (must be zeroed by the caller).
 * logits (nullable): [T][E] fp32 workspace; with E > 8 the (64-token tile,
 *   8-expert pass) units are balanced over a persistent grid and the logits
 *   (+ bias) are left there; NULL (or E <= 8) = one CTA per tile, all passes. */
int aurora_route(const void* x, const float* gate_prep, const float* bias, int T, int H, int E,
                 int k, const int32_t* gpu_of_expert, int n, int rank_base, int tokens_per_rank,
                 int32_t* topk_idx, float* topk_w, int32_t* slot_dst, int32_t* blk_cnt,
                 int32_t* counts, float* logits, void* stream);
/* aurora_route_gate_floats: floats of the prepared gate (ceil(E/8) * 8 * H, + 4 * H when
 *   E <= 8), or -AURORA_E*.
 * aurora_route_prepare_gate: w_gate[E][H] bf16 -> gate_prep: widened to fp32 (exact) in the
 *   router's shared-memory order (per 8-expert pass and 256-h chunk, lane-major expert pairs;
 *   experts past E zero); for E <= 8 followed by the bf16 rows [8][H] (zero past E) that the
 *   E <= 8 router reads with TMA. Once per layer (the gate is a weight). */
int aurora_route_gate_floats(int E, int H);
/* aurora_route_tc: the same router output (bit-exact top-k, weights, slot_dst, blk_cnt,
 *   counts) for 8 < E <= 64 with the gate's contraction on the tensor cores: approximate
 *   logits La = x W^T by the CTA-pair grouped GEMM into la_buf ([T][256] bf16 workspace;
 *   t_rows: one device int32 of workspace, set to T here; tile_ctr as for aurora_grouped_gemm,
 *   nullable), then per token
 *   the min(k + 2, E) largest approximate logits recomputed in the defined order and a
 *   certificate that no other expert can reach the k-th (bound: 2^-8 |La| + 2^-20 (|a| + 1)
 *   + 2^-13 sum_h |x_h| max_e |w_eh|); uncertified tokens get every logit exactly
 *   (n_fallback += their number, nullable). logits[T][E] (required) ends exact for the
 *   candidates / fallback tokens, approximate elsewhere (strictly below the selected k).
 *   gate_tc: aurora_route_tc_bytes(E, H) bytes prepared by aurora_route_prepare_gate_tc
 *   (padded / chunked bf16 copies of w_gate and max_e |w_eh|); H <= 8192.
 *   Replaces the FMA-bound logits of aurora_route (the reference models the gate only as
 *   LayerProfile.gate_work, core.py:194-221). */
int aurora_route_tc_bytes(int E, int H);
int aurora_route_prepare_gate_tc(const void* w_gate, int E, int H, void* gate_tc, void* stream);
int aurora_route_tc(const void* x, const void* w_gate, const void* gate_tc, const float* bias, int T, int H,
                    int E, int k, const int32_t* gpu_of_expert, int n, int rank_base, int tokens_per_rank,
                    int32_t* topk_idx, float* topk_w, int32_t* slot_dst, int32_t* blk_cnt, int32_t* counts,
                    float* logits, void* la_buf, int32_t* t_rows, int32_t* tile_ctr, int32_t* n_fallback,
                    void* stream);
int aurora_route_prepare_gate(const void* w_gate, int E, int H, float* gate_prep, void* stream);

/* ---------------------------------------------------------------- K3 ----
 * aurora_pack: the token permutation. For each local source rank i and
 * destination j, list(i,j) = the rank's tokens routed to j in ascending token
 * order; send_list[i_local][soff[i][j] + p] = local token index of the p-th
 * entry; pos[t][s] = p for the slot's destination (same p for deduplicated
 * slots). Needs counts complete (every row, for the layout).
 * Buffer layout (all [n] / [n][n] int32, written for every rank):
 *   soff[i][j]  start of list(i,j) in sender i's send list / return buffer (row prefix)
 *   roff[i][j]  start of list(i,j) in receiver j's buffer: the local rows
 *               list(j,j) first (roff[j][j] = 0), then the other senders in
 *               index order, so the local expert work can start before the schedule
 *   rtot[j]     rows receiver j holds; rloc[j] = counts[j][j]; rrem[j] = rtot - rloc
 * meta (nullable; needed when a rank hosts several experts): per send-list row
 * a record of k {int32 local expert on the destination or -1, float gate
 * weight}, padded to a multiple of 16 bytes (meta_bytes = roundup(8k, 16));
 * [n_local][T/n * k] records. local_of_expert[E] = expert index within its rank. */
/* Grouped placement (several experts per rank, engine mode bit 8): the receiver
 * keeps its rows grouped by local expert -- the packed layout aurora_expert_ffn_packed
 * runs on: groups (r_local, local expert) of a process back to back, each ordered
 * by (sender rank, token) -- and every dispatched row lands directly at its position
 * in each local-expert group it belongs to, so no receiver-side sort / gather runs.
 *   aurora_expert_hist: blk_cnt_e[T/64][E] tokens of each 64-token tile choosing each
 *     expert; cnt_e[n][E] += per sender rank (rows of the caller's ranks zeroed by the
 *     caller; exchanged like counts).
 *   aurora_pack_grouped: aurora_pack, plus (cnt_e complete) meta records whose x field
 *     is the row's position in its process's packed group buffer (-1: not on that
 *     rank; padding records -1), and this process's g_off[n_local*G + 1] / g_rows[n_local*G]
 *     (group g = r_local*G + local expert). Experts e live on gpu_of_expert[e]; every
 *     process drives n_local consecutive ranks; E = n*G. */
int aurora_expert_hist(const int32_t* topk_idx, int T, int k, int E, int rank_base, int tokens_per_rank,
                       int32_t* blk_cnt_e, int32_t* cnt_e, void* stream);
int aurora_pack_grouped(const int32_t* slot_dst, const int32_t* blk_cnt, const int32_t* counts, int T, int k,
                        int n, int rank_base, int tokens_per_rank, int32_t* send_list, int32_t* pos,
                        int32_t* soff, int32_t* roff, int32_t* rtot, int32_t* rloc, int32_t* rrem,
                        const int32_t* topk_idx, const float* topk_w, const int32_t* local_of_expert, void* meta,
                        const int32_t* blk_cnt_e, const int32_t* cnt_e, const int32_t* gpu_of_expert, int E,
                        int G, int n_local, int32_t* g_off, int32_t* g_rows, void* const* ginfo_bufs,
                        void* stream);
/* ginfo_bufs (nullable): per rank the base of its process's [rows] int4 array; every row
 * position also gets {receiver-layout row, gate weight bits, single (the token's only
 * expert on that rank), 0} (aurora_expert_ffn_packed_scatter). Peer stores: the
 * receiver reads them after its dispatch completes (the senders' done signals follow). */
int aurora_pack(const int32_t* slot_dst, const int32_t* blk_cnt, const int32_t* counts, int T,
                int k, int n, int rank_base, int tokens_per_rank, int32_t* send_list,
                int32_t* pos, int32_t* soff, int32_t* roff, int32_t* rtot, int32_t* rloc,
                int32_t* rrem, const int32_t* topk_idx, const float* topk_w,
                const int32_t* local_of_expert, void* meta, void* stream);

/* ------------------------------------------------------------ K4 / K6 ----
 * aurora_engine: executes the schedule as in-kernel stores into peer
 * memory, self-timed per run (a run i->j starts once every earlier run into j
 * has landed), replacing a single NCCL alltoallv. mode bit 0: 0 =
 * dispatch (CommSchedule phases, commsched.py:113-132), 1 = combine (the
 * reversed schedule, commsched.py:153-162: same phases, directions flipped);
 * mode bit 1: peers live on other GPUs (system-scope flag ordering) -- clear
 * when every rank of the call shares this GPU (gpu scope suffices);
 * mode bit 2: local (diagonal) rows only -- no schedule needed, so it can run
 * while K2 is still computing; mode bit 3: scheduled remote chunks only;
 * mode bit 4: ablation -- no pacing, every sender pushes all of its chunks at
 * once (the unscheduled all-pairs-concurrent all-to-all);
 * mode bit 8 (dispatch, TMA engine, meta plane required): grouped placement -- dst_bufs[j]
 * is the base of rank j's process's packed group buffer and every row is stored at
 * the positions in its meta record (aurora_pack_grouped), one store per local expert
 * (ginfo_bufs below: optional, the records can come from aurora_pack_grouped instead);
 * mode bit 5: launch as a programmatic dependent (PDL) of the immediately
 * preceding aurora_schedule_counts on the same stream -- the engine starts
 * while K2 runs (K2 triggers its dependents on entry, so it is resident first)
 * and consumes phases through `progress`; mode bit 6: copy with 256-thread
 * CTAs of 16-byte vector loads/stores instead of the default TMA engine (two
 * warps per CTA: a producer streaming rows into shared-memory slots with
 * cp.async.bulk, a consumer bulk-storing them into the receiver once its
 * run may start -- the next run's rows are prefetched across the hand-over).
 * Continuation entries of a run need no hand-over, so a handshake only
 * happens where the schedule changes partners. Local (diagonal) rows are
 * copied first; then phase k is executed as soon as progress (K2's progress
 * word) covers it, so the engine may run concurrently with K2 on another
 * stream of the same device.
 *   tables + progress from aurora_schedule_counts; counts[n][n] from aurora_route;
 *   n_local ranks [rank_base, rank_base+n_local) are served by this call
 *   dispatch: src rows = x_local[i_local] gathered through send_list,
 *             dst = recv_buf[j] rows roff[i][j] + first ...
 *   combine:  src rows = out_buf[j_local] rows roff[i][j] + first ...,
 *             dst = ret_buf[i] rows soff[i][j] + first ...
 *   optional second plane (dispatch only; NULL to skip): src2_bufs[n_local] rows
 *   of row2_bytes in send-list order (aurora_pack's meta), landing beside the
 *   token rows in dst2_bufs[n] at the same row index;
 *   src_bufs[n_local], dst_bufs[n] (peer-mapped), ctrs[n] (peer-mapped pairs of
 *   int32 arrival counters {pace, done}, zero on entry, left zero on exit), all
 *   device arrays. The TMA engine signals `pace` as soon as a run's last store
 *   is issued (the next run into that receiver may start; runs own disjoint
 *   rows, so only pacing depends on it) and `done` once its stores completed;
 *   the receiver's exit waits on `done`. The LSU engine signals both at once.
 *   ctas_per_rank copy CTAs per local rank; all must be co-resident.
 *   spin_limit bounds every flag wait (0 = unbounded); on expiry status = ETIMEOUT. */
int aurora_engine(int mode, int n, int n_local, int rank_base, const int32_t* counts,
                  const int32_t* chunks, const int32_t* rchunks, const int32_t* progress,
                  const int32_t* n_in, const int32_t* n_out, const int32_t* soff,
                  const int32_t* roff, const int32_t* send_list, int send_list_stride,
                  const void* const* src_bufs, void* const* dst_bufs, int row_bytes,
                  const void* const* src2_bufs, void* const* dst2_bufs, int row2_bytes,
                  int32_t* const* ctrs, int ctas_per_rank, int max_phases, int64_t spin_limit,
                  int32_t* status, int split, const double* bw, void* const* ginfo_bufs,
                  int32_t* const* landed, const double* phase_dur, float unit_ns, void* stream);
/* ginfo_bufs (mode bit 8, nullable): per rank the base of its process's [rows] int4
 * array; every grouped store of a row also writes {receiver-layout row, gate weight,
 * single (the row's only local expert), 0} at the row's group position
 * (aurora_expert_ffn_packed_scatter).
 * landed (nullable; LSU dispatch, mode bit 6, only): per receiver j the address of its row
 * landed[j][0..n) (peer memory at N > 1); every copy CTA adds the rows it moved for block
 * (i -> j) after they are visible -- at each run end and after its share of the local rows
 * (release) -- the arrival signal of aurora_expert_ffn_combine's arrival-driven GEMM1. The
 * engine triggers griddepcontrol.launch_dependents at entry, so that GEMM may be a
 * programmatic dependent launch running beside it.
 * phase_dur / unit_ns (TMA engine; phase_dur NULL or unit_ns 0 = off): deadline pacing. A run
 * also starts once the schedule's own clock reaches its phase -- the copy CTA's first remote
 * entry + (phase_dur[0] + ... + phase_dur[k-1]) * unit_ns ns -- whichever comes first with the
 * hand-over, so a late flag no longer delays the chain. phase_dur = aurora_schedule_counts'
 * output (the combine replays the same phases); unit_ns = ns per schedule time unit of a pair
 * (row bytes / link bytes per ns). Pacing only: rows and completion are unchanged. */
/* aurora_engine_ctas: copy CTAs per local rank the engine will actually use
 * (ctas_per_rank clamped so every copy CTA is co-resident), or -AURORA_E* on
 * error. K2 needs n_local x this value to count hand-over thresholds. The
 * engine's grid (n_local x that value) is split among its ranks by `split`
 * (csrc/apportion.cuh; bw: rank bandwidths for AURORA_SPLIT_BANDWIDTH). */
int aurora_engine_ctas(int n, int n_local, int ctas_per_rank, int row_bytes, int row2_bytes, int lsu);

/* aurora_exchange_counts: the traffic-matrix all-gather over peer memory (SURVEY
 * 8(e) pre-step; the reference has one process and a complete TrafficMatrix,
 * core.py:75-117). counts2 [2][n][n] int32 (this process; buffer (epoch-1) & 1 of
 * the call is used, its rows [rank_base, rank_base + n_local) filled by
 * aurora_route); peer_counts2[n] = base of the [2][n][n] buffer of rank q's
 * process, xflag[n] (this process, zero-initialised, monotonic), peer_xflag[n] =
 * base of rank q's process's xflag, epoch: one int32 of this process (zero at
 * first call; every process must make the same sequence of calls). Stores this
 * process's rows into every peer's buffer, releases xflag[r] = epoch for its
 * ranks, and completes once every other rank's flag has arrived (system scope).
 * The caller alternates the counts buffer it passes to the other kernels with
 * the same parity. spin_limit bounds the wait; on expiry status = ETIMEOUT. */
int aurora_exchange_counts(int32_t* counts2, int32_t* const* peer_counts2, int32_t* rows2,
                           int32_t* const* peer_rows2, int w2, int32_t* xflag,
                           int32_t* const* peer_xflag, int32_t* epoch, int n, int rank_base, int n_local,
                           int64_t spin_limit, int32_t* status, void* stream);
/* (rows2 / peer_rows2 / w2, nullable: a second [2][n][w2] matrix exchanged the same way --
 * the per-expert token counts of aurora_expert_hist for the grouped dispatch.) */

/* aurora_combine_wait: the receiving side of the fused combine
 * (aurora_expert_ffn_combine). One thread per local sender rank
 * r in [rank_base, rank_base + n_local) waits until its {pace, done} pair
 * ctrs[r] (the combine's peer-mapped counter table, device array [n]) has
 * done >= expect arrivals (one per expert rank: n), then re-arms the pair to
 * zero. spin_limit bounds the wait (0 = unbounded); on expiry status =
 * ETIMEOUT. sys: peers on other GPUs. */
int aurora_combine_wait(int32_t* const* ctrs, int rank_base, int n_local, int expect, int sys,
                        int64_t spin_limit, int32_t* status, void* stream);

/* ---------------------------------------------------------------- K7 ----
 * aurora_aggregate: out[t] = sum_s topk_w[t][s] * ret_i[soff[i][dst_s] + pos[t][s]]
 * (with y_buf: slots whose expert lives on the token's own rank i are read from
 * the expert output y_i[roff[i][i] + pos[t][s]] instead, so the combine can skip
 * the local rows -- engine mode bit 3)
 * in fp32, bf16 out (pre_weighted = 0; every slot must have its own destination),
 * or the plain sum of the rows of the non-duplicate slots when the expert side
 * already applied the gate weights and pre-reduced its local experts
 * (pre_weighted = 1). ret_i = ret_buf + i_local * ret_rank_stride_rows rows.
 * The reference's LayerProfile.agg_work (core.py:194-221). */
int aurora_aggregate(const void* ret_buf, int64_t ret_rank_stride_rows, const int32_t* soff,
                     const int32_t* pos, const int32_t* slot_dst, const float* topk_w, int T,
                     int k, int H, int n, int rank_base, int tokens_per_rank, int pre_weighted,
                     void* out, const void* y_buf, int64_t y_rank_stride_rows,
                     const int32_t* roff, void* stream);

/* ---------------------------------------------------------------- K5 ----
 * aurora_expert_ffn: SwiGLU experts as tcgen05/TMEM grouped GEMMs fed by TMA
 * (the reference's ffn_work_per_token, core.py:194-221 / sim.py:71-89).
 *   groups G (one per local expert); group g owns rows g*cap .. g*cap+cap-1 of
 *   a_buf [G*cap][H] bf16 and processes rows g*cap + m_start[g] + [0, m_rows[g])
 *   (device arrays; m_start may be NULL = 0) -- so the local rows and the
 *   network rows of one receive buffer can run as two launches.
 *   w13[G][2F][H] bf16: rows interleaved in 128-row blocks (gate block b at
 *   rows 256b..256b+127, up block at 256b+128..256b+255) -- see DESIGN.md
 *   w2[G][H][F] bf16; h_buf [G*cap][F] bf16 scratch; y_buf [G*cap][H] bf16 out.
 *   y = (silu(x W1^T) * (x W3^T)) W2^T, fp32 accumulate. */
int aurora_expert_ffn(const void* a_buf, const void* w13, const void* w2, void* h_buf,
                      void* y_buf, const int32_t* m_start, const int32_t* m_rows, int G,
                      int64_t cap, int H, int F, const int32_t* cluster_part, int32_t* tile_ctr,
                      int num_sms, void* stream);

/* aurora_expert_ffn_combine: the same FFN (one expert per rank: group g is
 * expert rank rank_base + g, all received rows) with the combine fused into
 * GEMM2's epilogue -- the K6 + K5 pair written as one kernel over peer memory
 * (reference: ffn_work_per_token, core.py:194-221, then the reversed all-to-all,
 * CommSchedule.reversed commsched.py:153-162, as sequenced by sim.py:130-154):
 * every output row of sender i's block (recv rows roff[i][j] + [0, counts[i][j]))
 * is stored straight into ret_bufs[i] row soff[i][j] + offset (the row the
 * combine engine would write; NVSwitch stores overlap the GEMM tile by tile),
 * rows of the rank's own tokens (i == j) into y_buf as with local-direct
 * aggregation. The last CTA to finish adds G arrivals (release) to the done
 * slot of every sender's {pace, done} pair ctrs[i] (the combine table);
 * aurora_combine_wait on the sender consumes them. ticket: one int32, zero
 * on first use (re-armed by the kernel). counts/soff/roff [n][n], ret_bufs[n],
 * ctrs[n]: device arrays. sys: peers on other GPUs. n, G <= 16. */
int aurora_expert_ffn_combine(const void* a_buf, const void* w13, const void* w2, void* h_buf,
                              void* y_buf, const int32_t* m_rows, int G, int64_t cap, int H, int F,
                              void* const* ret_bufs, const int32_t* counts, const int32_t* soff,
                              const int32_t* roff, int n, int rank_base, int32_t* const* ctrs,
                              int32_t* ticket, int sys, const int32_t* cluster_part, int32_t* landed,
                              int arrival_pdl, int32_t* tile_ctr, int num_sms, void* stream);
/* landed (nullable): arrival-driven GEMM1 (N1). landed[g * n + i] = rows of block (sender i ->
 * local rank rank_base + g) the dispatch has made visible (aurora_engine's landed credits); a
 * GEMM1 tile starts once every block under its rows is complete, the m-tiles holding only local
 * rows first. GEMM1's last cluster re-arms landed to zero. arrival_pdl: GEMM1 is launched as a
 * programmatic dependent of the preceding dispatch launch, so its tiles run beside the copy CTAs
 * (an LSU dispatch leaves each SM's shared memory to the GEMM). Needs tile_ctr and no
 * cluster_part. */

/* aurora_expert_ffn_packed_scatter: the packed FFN of the grouped dispatch with the
 * pre-reduction of single-expert rows folded into GEMM2's epilogue. ginfo [a_rows]
 * int4 per packed row = {receiver-layout row, gate weight bits, single, -} (written by
 * the grouped dispatch, engine mode bit 8). A single row's output is w * y (the
 * pre-reduction's fp32 arithmetic on the bf16 y) stored into ybuf row
 * r_local * ycap + recv row, or with to_ret (fused combine) straight into its
 * sender's return buffer (ret_bufs / counts / soff / roff as in
 * aurora_expert_ffn_combine; rank = rank_base + group / experts_per_rank). Other
 * rows go to y_buf for aurora_expert_reduce(_combine) with skip_single = 1. */
int aurora_expert_ffn_packed_scatter(const void* a_buf, const void* w13, const void* w2, void* h_buf,
                                     void* y_buf, const int32_t* g_off, const int32_t* g_rows, int G,
                                     int64_t a_rows, int H, int F, const void* ginfo, int experts_per_rank,
                                     void* const* ret_bufs, const int32_t* counts, const int32_t* soff,
                                     const int32_t* roff, int n, int rank_base, void* ybuf, int64_t ycap,
                                     int to_ret, int sys, const int32_t* cluster_part, int32_t* tile_ctr,
                                     int num_sms, void* stream);

/* Same FFN with the groups packed back to back (a rank hosting several
 * experts): group g's rows are a_buf rows [g_off[g], g_off[g] + g_rows[g]);
 * a_rows = rows allocated in a_buf / h_buf / y_buf. */
int aurora_expert_ffn_packed(const void* a_buf, const void* w13, const void* w2, void* h_buf,
                             void* y_buf, const int32_t* g_off, const int32_t* g_rows, int G,
                             int64_t a_rows, int H, int F, const int32_t* cluster_part, int part_groups,
                             int32_t* tile_ctr, int num_sms, void* stream);

/* Several experts per rank (E > n). After the dispatch, receiver rows of the
 * local ranks (rank r_local: rows r_local*cap + [0, rtot[rank_base+r_local]))
 * carry aurora_pack's meta records (copied by the engine's second plane).
 *   aurora_expert_sort: group g = r_local*G + local expert; g_rows[g], packed
 *     offsets g_off[0..n_local*G] (g_off[n_local*G] = total), g_src[p] = the
 *     received row of grouped position p, inv[row][slot] = p or -1.
 *     scratch >= ceil(n_local*cap/256) * n_local*G ints.
 *   aurora_gather_rows: dst[p] = src[idx[p]] for p < *count (device count).
 *   aurora_expert_reduce: ybuf[row] = sum_slots w * yg[inv[row][slot]] (fp32 -> bf16)
 *     (inv NULL: the position is the meta record's x field -- grouped dispatch),
 *     the pre-reduction that returns one row per (token, rank) to the combine. */
int aurora_expert_sort(const void* meta, int64_t cap, int meta_bytes, const int32_t* rtot,
                       int n_local, int rank_base, int k, int G, int32_t* g_off, int32_t* g_rows,
                       int32_t* g_src, int32_t* inv, int32_t* scratch, int scratch_ints,
                       void* stream);
int aurora_gather_rows(const void* src, void* dst, const int32_t* idx, const int32_t* count,
                       int64_t max_rows, int row_bytes, void* stream);
int aurora_expert_reduce(const void* yg, const int32_t* inv, const void* meta, int64_t cap,
                         int meta_bytes, const int32_t* rtot, int n_local, int rank_base, int k, int H,
                         void* ybuf, int skip_single, void* stream);
/* aurora_expert_reduce_combine: the pre-reduction with the combine fused into it
 * (several experts per rank): each reduced row of sender i's block is stored
 * straight into ret_bufs[i] row soff[i][j] + offset (rows of the rank's own tokens
 * into ybuf), then the last CTA adds n_local arrivals to every sender's combine
 * counter; same contract as aurora_expert_ffn_combine's scatter / signal half. */
int aurora_expert_reduce_combine(const void* yg, const int32_t* inv, const void* meta, int64_t cap,
                                 int meta_bytes, const int32_t* rtot, int n_local, int rank_base, int k,
                                 int H, void* ybuf, void* const* ret_bufs, const int32_t* counts,
                                 const int32_t* soff, const int32_t* roff, int n, int32_t* const* ctrs,
                                 int32_t* ticket, int sys, int skip_single, void* stream);
/* skip_single (both): rows whose (token, rank) has exactly one local expert were
 * finished by aurora_expert_ffn_packed_scatter; only the others are reduced. */

/* cluster_part (expert FFN entry points; NULL = off): emulated per-rank compute for heterogeneous
 * clusters (configs C4, C3 on C4's cluster) -- R + 1 ints for R ranks, clusters (CTA pairs,
 * num_sms / 2 of them) [cluster_part[r], cluster_part[r + 1]) serve rank r's groups only (its
 * experts: groups r * Gp .. r * Gp + Gp - 1, Gp = 1, experts_per_rank or part_groups), round robin
 * over their tiles, so a rank's GEMM time follows its share of the GPU like experts on a GPU of that
 * speed (ClusterSpec compute_scale, reference core.py:135-191; placement.py:46-60 / 129-157 decide
 * which experts land where). cluster_part[R] <= num_sms / 2: pairs past it stay idle (a process
 * emulating slower GPUs than the fastest one).
 * tile_ctr (every expert FFN / grouped GEMM entry point): two int32 owned by the caller,
 * zero before first use and re-armed by each launch's last cluster -- the dynamic tile
 * order's {next tile, clusters done} pair. One per stream whose GEMM launches may run
 * concurrently with another's (a layer keeps one per stream it launches on); NULL
 * selects the static round-robin tile order. No allocation or host sync happens inside. */

/* Plain grouped GEMM (tests / building block): C[g] = A[g] B[g]^T, bf16 in,
 * fp32 accumulate, bf16 out; epilogue 0 = store, 1 = SwiGLU pairs (N/2 cols). */
int aurora_grouped_gemm(const void* a, const void* b, void* c, const int32_t* m_start,
                        const int32_t* m_rows, int G, int64_t cap, int N, int K, int epilogue,
                        int32_t* tile_ctr, int num_sms, void* stream);

/* ------------------------------------------------------- peer memory ----
 * CUDA IPC for the multi-GPU layer (one process per GPU). aurora_ipc_get
 * returns the handle of the allocation containing `ptr` (handle buffer of
 * aurora_ipc_handle_bytes() bytes) and ptr's offset inside it; a peer process
 * maps it with aurora_ipc_open(handle, offset, &peer_ptr). */
int aurora_ipc_handle_bytes(void);
int aurora_ipc_get(const void* ptr, void* handle, int64_t* offset);
int aurora_ipc_open(const void* handle, int64_t offset, void** out);
int aurora_ipc_close(void* base);

/* Diagnostics: one K2 run with per-section cycle counters
 * prof[5] = {snap+masks, matching, update, strip, decompose total};
 * scratch >= (n^2-2n+2)*n + 3 + (2n^2-3n+2)*n int32, dscratch >= 3n^2 doubles. */
int aurora_debug_schedule_cycles(const double* d, int n, long long* prof, int32_t* scratch,
                                 double* dscratch, void* stream);
/* Diagnostics: every later K2 launch (any entry point) writes its section
 * cycles to the device array prof[8] = {snap+masks, matching, update, strip,
 * decompose, prologue, whole kernel, chunk pass}; NULL turns it off. */
int aurora_debug_set_schedule_profile(long long* prof);
/* Diagnostics: the in-layer K2 path (int32 counts, uniform cluster, n <= 8):
 * 0 (default) cell-lane decomposition and strip (FastMatch8d, two cells of
 * the matrix per lane, support / preferred / active sets as ballots); 1
 * FastMatch8b with per-step masks; 2 cell-lane decomposition with the
 * row-lane strip; 3 row-lane incremental decomposition (lane i = row i) with
 * the row-lane strip. Same results. */
int aurora_debug_set_schedule_variant(int generic);
/* Diagnostics timelines (%globaltimer ns; NULL switches off): K2 records the
 * time each phase is published at trace[count & 511]; the TMA engine records
 * per copy CTA {start, local rows done, end, -} at trace[4 * cta]. */
int aurora_debug_set_schedule_trace(long long* trace);
int aurora_debug_set_engine_trace(long long* trace);
/* per expert-GEMM CTA {entry, first tile's loads issued} (%globaltimer ns) at trace[2 * cta] */
int aurora_debug_set_gemm_trace(long long* trace);
/* aurora_debug_set_early_rows: rows before the end of a CTA's share of a run at
 * which the TMA engine sends the run's pace signal (engine mode bit 7; default 2). */
int aurora_debug_set_early_rows(int rows);

#ifdef __cplusplus
}
#endif
#endif /* AURORA_B200_H */
