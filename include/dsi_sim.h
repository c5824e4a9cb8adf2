/*
 * dsi_sim.h -- C ABI of the B200-native Monte Carlo latency simulator of
 * Distributed Speculative Inference (DSI, arXiv 2405.14105).
 *
 * For every grid point (target latency, drafter latency, acceptance rate,
 * lookahead k, SP degree, N tokens) the library runs n_trials independent
 * trials on sm_100a GPUs.  One trial draws the acceptance indicators
 * A_1..A_{N-1} (i.i.d. Bernoulli(a) per draft token)
 * from a counter-based Philox4x32-10 stream and computes three latencies in
 * integer ticks:
 *   non-SI  N * t_target
 *   SI      the draft-then-verify loop of App. F.4
 *   DSI     Algorithm 1 with the App. D lookahead:
 *           a verification task every k drafts on SP FIFO target servers,
 *           a rejection terminates all threads and restarts.
 * Per configuration it returns exact integer sums over trials and FP64 means.
 * DESIGN.md lists the readings of the paper this ABI commits to (R1-R22).
 *
 * Random-number contract (bit-exact, any device count and partition):
 *   key = (seed & 0xffffffff, seed >> 32)
 *   counter = (q, 0, trial, stream_id), q = (p-1) >> 2, output word (p-1) & 3
 *   A_p = [word < floor(a * 2^32)]   (a = 1 always accepts, a = 0 never)
 * trial runs over 0..n_trials-1 of its configuration.
 *
 * Conventions
 *  - Every function returns dsi_status; no C++ exception crosses the ABI.
 *  - A failing call writes nothing to caller-owned outputs.
 *  - All validation happens in dsi_sim_create, before any device work.
 *  - dsi_sim_create copies cfg[]; the library owns all device memory, streams
 *    and NCCL communicators until dsi_sim_destroy.  Output arrays are
 *    caller-owned host memory.
 *  - A handle is used by one host thread at a time; handles are independent.
 *  - Eq. 1 violation is legal (FIFO queueing is simulated, R7)
 *    unless DSI_F_STRICT_EQ1 is set.
 */
#ifndef DSI_SIM_H
#define DSI_SIM_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define DSI_ABI_VERSION 2u

/* every entry point is exported with default visibility (the library hides the rest) */
#if defined(__GNUC__)
#define DSI_API __attribute__((visibility("default")))
#else
#define DSI_API
#endif

typedef enum {
  DSI_OK = 0,
  DSI_E_NULL = 1,       /* a required pointer was NULL                                   */
  DSI_E_RANGE = 2,      /* a not in [0,1]; k < 1; SP < 1; N not in [1, 32768]; n_trials not
                           in [1, 2^32]; latency <= 0 or not finite; t_drafter > t_target
                           (Assumption 2); bad option field; n_cfg == 0        */
  DSI_E_TICK = 3,       /* latency / tick not within 1e-9 (relative) of an integer >= 1  */
  DSI_E_OVERFLOW = 4,   /* N*(k*t_d + t_t) >= 2^31 ticks, or n_trials*bound^2 >= 2^64     */
  DSI_E_STRICT_EQ1 = 5, /* DSI_F_STRICT_EQ1 set and ceil(t_t/(k*t_d)) > SP                */
  DSI_E_DEVICE = 6,     /* CUDA error, or fewer usable sm_100 devices than requested      */
  DSI_E_COMM = 7,       /* NCCL could not be loaded or an NCCL call failed                */
  DSI_E_STATE = 8,      /* call order violated (reduce before run, trials without
                           DSI_F_PER_TRIAL, hist without DSI_F_HIST, ...)                 */
  DSI_E_NOMEM = 9       /* host or device allocation failed                               */
} dsi_status;

/* Option flags */
#define DSI_F_PER_TRIAL 0x1u  /* keep per-trial records {acc, m, I, L_SI, L_DSI} (test mode) */
#define DSI_F_HIST 0x2u       /* per-config histograms: segment lengths (64 bins, last = >=63)
                                 and SI accepted drafts per iteration (k+1 bins, iterations
                                 whose k-draft window lies in 1..N-1 only)                   */
#define DSI_F_PATTERN 0x4u    /* enumeration mode: A_p = bit (p-1) of the trial index; N <= 33 */
#define DSI_F_STRICT_EQ1 0x8u /* reject configs violating Eq. 1                               */
#define DSI_F_TIMING 0x10u    /* record CUDA events around the trial kernels of each run      */
#define DSI_F_SHARED_STREAMS 0x20u /* configs with equal (stream_id, floor(a 2^32), N, n_trials)
                                 draw identical indicators (the RNG contract): generate each
                                 trial's stream once per group and evaluate every config of the
                                 group on it.  Results are bit-identical to the default mode.
                                 TTFT configs join no group: the per-config kernel runs them in
                                 the same dsi_sim_run.  Not with PER_TRIAL, HIST or PATTERN;
                                 N <= 2048.                                                     */
#define DSI_F_FRESH_VERIFIER 0x40u /* fresh-verifier DSI variant (R24; Thm 2's proof
                                 P:445, "DSI either invokes a new current verifier thread or
                                 labels an existing thread"): whenever the committed prefix
                                 grows to p at time tau and no started target thread settles
                                 p+1 by tau + t_t, a fresh target forward starts at tau on an
                                 extra server, on the committed prefix plus the drafts done by
                                 tau (at most k).  Identical to the default when k t_d <= t_t;
                                 otherwise L_DSI <= N t_t on every trial (Thm 1).
                                 Every mode (per-config, SHARED_STREAMS, MEANS_ONLY, heatmap)
                                 gives the same integers under it.  Not with TTFT configs.
                                 DESIGN.md 2.1: the reading the paper's theorems and figures
                                 require when k t_d > t_t; the bench and CLI products use it. */

#define DSI_F_MEANS_ONLY 0x80u /* means only ("aggregate H[g]"): per group of
                                 configs drawing identical indicators (as SHARED_STREAMS), one
                                 pass builds the histogram H[g] of segment lengths over all
                                 trials, and each config's sums follow by linearity over
                                 segments: sum L_DSI = sum_g H[g] C(g), sum I = sum_g H[g]
                                 ceil(g/(k+1)), sum m = sum_g H[g] -- the same integers as the
                                 default mode, so sums, means and dsi_sim_heatmap are
                                 bit-identical.  Second moments and per-trial counters are not
                                 produced: sumsq_* = 0, std_* = NaN, n_dsi_gt_* = -1.  TTFT
                                 configs add sum_g H1[g] D1(g), H1 the first-segment lengths.
                                 Not with PER_TRIAL, HIST, PATTERN or SHARED_STREAMS;
                                 dsi_sim_update keeps (stream_id, a, N, n_trials) and which
                                 configs use TTFT.                                              */

#define DSI_F_REDUCE_TO_ROOT 0x100u /* multi-process: dsi_sim_reduce returns the results on rank 0
                                 only; the other ranks contribute to the all-reduce and return
                                 without the device-to-host copy and FP64 finalize (out may be
                                 NULL there).  Without it every rank gets every result.       */

#define DSI_F_RNG_HALVES 0x200u /* the "halves" layout of the indicator stream (R26):
                                 call q = (p-1) >> 3 of Philox counter (q, 0, trial, stream_id)
                                 serves positions 8q+1..8q+8, offset j = (p-1) & 7 reading
                                 v = the high 16 bits of output word j (j < 4) or the low 16
                                 bits of word j-4; with thr = floor(a 2^32) = T 2^16 + R,
                                 A_p = [v < T], or on a tie (v == T) [w < R], w the same half of
                                 the same word of call (q, 1, trial, stream_id).  So A_p =
                                 [v 2^16 + w < thr]: the same Bernoulli(thr / 2^32) law as the
                                 default layout from half the Philox calls, but different
                                 indicators (results are not comparable trial by trial with
                                 the default layout).  Every mode (per-config, SHARED_STREAMS,
                                 MEANS_ONLY, the heatmap) gives the same integers under it.
                                 dsi_multi_simulate takes it too: drafter j on counter word 1
                                 = 2(j-1), its tie-break on 2(j-1)+1 (drafter 1 draws exactly
                                 the single-drafter stream).                                  */

/* One grid point: the paper's quantities (Table 2 columns P:249-256; Sec. 3.1). */
typedef struct {
  double t_target;    /* target forward latency (t_2, "Target Latency"), user units > 0   */
  double t_drafter;   /* drafter forward latency (t_1), 0 < t_drafter <= t_target          */
  double accept_rate; /* a in [0,1]: P(draft token accepted), i.i.d. per token             */
  int32_t lookahead;  /* k >= 1: drafts per verification task (App. D)               */
  int32_t sp_degree;  /* SP >= 1: concurrent target servers                        */
  int32_t n_tokens;   /* N in [1, 32768]: tokens to generate                               */
  uint32_t stream_id; /* Philox counter word 3; equal ids => common random numbers         */
  uint64_t n_trials;  /* T in [1, 2^32]                                                    */
  double ttft_target; /* TTFT variant: the target pool's first-ever forward
                         (thread 0 of the first segment; non-SI's and SI's first target
                         forward) costs this; 0 = same as t_target                         */
  double ttft_drafter;/* the drafter's first forward costs this; 0 = same as t_drafter;
                         ttft_drafter <= ttft_target (Assumption 2 for first forwards)     */
} dsi_config;         /* 64 bytes */

typedef struct {
  uint32_t abi_version;   /* must equal DSI_ABI_VERSION                                     */
  uint32_t flags;         /* DSI_F_* */
  double tick;            /* time quantum in latency units, > 0 (e.g. 0.01 relative, 0.1 ms) */
  uint64_t seed;          /* Philox key                                                     */
  int32_t device;         /* first CUDA device ordinal of this process (e.g. LOCAL_RANK)    */
  int32_t n_devices;      /* must be 1: one process drives one GPU; several GPUs run one
                             process each (torchrun), ranks joined by NCCL  */
  int32_t rank, world;    /* multi-process mode: this process is rank of world (world >= 1) */
  const uint8_t *nccl_id; /* 128-byte ncclUniqueId shared by all ranks; required when
                             world > 1.  With one device, a
                             non-NULL id still routes the reduction through a one-rank NCCL
                             communicator.  Obtain it with dsi_nccl_unique_id on one rank
                             and broadcast it; use a fresh id for every handle (an id serves
                             one communicator: a second init with it fails with DSI_E_COMM,
                             profiles/nccl_id_reuse.py).                                    */
  int32_t n_shards;       /* 0 or 1: normal.  > 1 (test only, single device): split the work
                             into n_shards cost-balanced shards run back to back on one
                             device, exercising the same partition code as multi-GPU.     */
  int32_t block_threads;  /* 0 = default (128); else 32..128, multiple of 32 (trial kernel)  */
  void *stream;           /* cudaStream_t for the first device, or NULL (library-owned)    */
} dsi_options;

/* Per configuration, after dsi_sim_reduce.  Integers are exact; doubles derive from them. */
typedef struct {
  uint64_t trials;
  int64_t t_target_ticks, t_drafter_ticks;
  int64_t nonsi_ticks;              /* ttft_t + (N-1) t_t per trial (N t_t without TTFT)   */
  int64_t sum_si_ticks, sum_dsi_ticks;
  uint64_t sumsq_si_ticks, sumsq_dsi_ticks;
  int64_t sum_si_iters;             /* sum of I = SI target forwards                       */
  int64_t sum_accepts;              /* sum of acc = #{p <= N-1 : A_p = 1}                  */
  int64_t sum_segments;             /* sum of m = #rejections + 1                          */
  int64_t n_dsi_gt_nonsi;           /* trials with L_DSI > L_non (Thm 1 counter)           */
  int64_t n_dsi_gt_si;              /* trials with L_DSI > L_SI  (Thm 2 counter)           */
  uint64_t threshold;               /* floor(a * 2^32)                                     */
  int32_t eq1_feasible;             /* ceil(t_t/(k t_d)) <= SP  (Eq. 1)                    */
  int32_t min_lookahead;            /* smallest k with ceil(t_t/(k t_d)) <= SP             */
  double mean_nonsi, mean_si, mean_dsi; /* user units: ((double)sum / (double)T) * tick    */
  double std_si, std_dsi;           /* population std, user units, from the exact integer
                                       numerator T*sumsq - sum^2 (128-bit)                  */
} dsi_result;

typedef struct dsi_sim dsi_sim; /* opaque handle */

/* Validate options and configs, convert to ticks, plan shards, allocate device
 * memory, upload the config table, initialise NCCL when world*n_devices > 1
 * (collective: every rank must call it).  On error *out is set to NULL. */
DSI_API dsi_status dsi_sim_create(const dsi_options *opt, const dsi_config *cfg, size_t n_cfg,
                          dsi_sim **out);

/* Replace the configuration values of an existing handle (same n_cfg, same
 * n_trials per config; with DSI_F_HIST also the same min(k, N)).  Validates like
 * create.  Device path (one device, no test-mode flag): the configurations are copied as
 * given (straight from a page-locked cfg, else through pinned staging) and validated and
 * converted on the GPU, ordered after any previous run on the library's stream; committed when
 * every config is valid, the launch limits (max N, max min(k, N), TTFT / fresh-verifier
 * present) are unchanged and no plan below needs rebuilding -- otherwise, and always for the
 * test modes, the host path validates, re-plans and uploads (and reports any error with its
 * message).  N may grow (shared-memory tables are sized per launch).  With
 * DSI_F_SHARED_STREAMS the plan is kept when (stream_id, threshold, N, n_trials, k,
 * t_target, t_drafter, SP) are unchanged, else rebuilt; an update that changes the
 * number of groups or units returns DSI_E_RANGE ("create a new handle").  On error
 * the handle keeps its previous configs. */
DSI_API dsi_status dsi_sim_update(dsi_sim *h, const dsi_config *cfg, size_t n_cfg);

/* Enqueue one full simulation on every device of this process (asynchronous). */
DSI_API dsi_status dsi_sim_run(dsi_sim *h);

/* Wait for the run, sum the per-config integer moments across devices and ranks
 * (one NCCL all-reduce), check on the device that every trial was simulated exactly
 * once (DSI_E_DEVICE otherwise, nothing written), copy the moments to the host in
 * chunks and derive FP64 means/std (overlapped).  n must equal n_cfg.  Blocking.
 * Every rank must call it. */
DSI_API dsi_status dsi_sim_reduce(dsi_sim *h, dsi_result *out, size_t n);

/* The exchange step of dsi_sim_reduce without bringing anything to the host: the cross-rank
 * all-reduce of the moments and the device-side partition check, enqueued on the library's
 * stream (asynchronous; every rank must call it).  The exact per-config moments stay in device
 * memory; dsi_sim_fetch derives any range of results, dsi_sim_heatmap the cells, without a
 * second all-reduce.  P:531's averaging is deferred to what the caller reads.  DSI_E_STATE
 * before dsi_sim_run or with DSI_F_HIST (histograms come back with dsi_sim_reduce). */
DSI_API dsi_status dsi_sim_reduce_device(dsi_sim *h);

/* Results [first, first + count) after dsi_sim_reduce_device (or dsi_sim_reduce): blocks, checks
 * the partition flag (DSI_E_DEVICE, nothing written), copies those configs' moments to the host
 * and derives the FP64 fields exactly as dsi_sim_reduce does -- out[i] is config first + i.
 * DSI_E_RANGE if the range exceeds n_cfg; DSI_E_STATE before a reduce, or on a rank != 0 with
 * DSI_F_REDUCE_TO_ROOT. */
DSI_API dsi_status dsi_sim_fetch(dsi_sim *h, size_t first, size_t count, dsi_result *out);

/* Per-trial records of trials [first, first+count) of config cfg (needs
 * DSI_F_PER_TRIAL, one device, world == 1).  Any output pointer may be NULL. */
DSI_API dsi_status dsi_sim_trials(dsi_sim *h, size_t cfg, uint64_t first, uint64_t count,
                          int32_t *acc, int32_t *m, int32_t *iters, int32_t *si_ticks,
                          int32_t *dsi_ticks);

/* Histograms of config cfg after reduce (needs DSI_F_HIST).  seg_hist: 64 bins,
 * bin g = segments of length g (bin 63 = length >= 63, bin 0 unused).
 * si_hist: si_bins must be k+1; bin j = SI iterations with j accepted drafts. */
DSI_API dsi_status dsi_sim_hist(dsi_sim *h, size_t cfg, int64_t *seg_hist, int64_t *si_hist,
                        size_t si_bins);

/* CUDA stream of the i-th device of this handle (cudaStream_t as void*). */
DSI_API dsi_status dsi_sim_stream(dsi_sim *h, int32_t device_index, void **stream);

/* Environment: DSI_TRACE=1 makes create / update / run / reduce / heatmap print their host-side
 * phases (wall clock, ms) to stderr on return. */

/* Kernel launches enqueued on this process since the last dsi_sim_run began: its trial
 * kernels, plus the partition check of dsi_sim_reduce and the heatmap kernel of
 * dsi_sim_heatmap when those were called. */
DSI_API dsi_status dsi_sim_launches(dsi_sim *h, int32_t *launches);

/* With DSI_F_TIMING: device time (ms) of the trial kernels of the last run on
 * device_index, measured with CUDA events on the launching stream (blocks). */
DSI_API dsi_status dsi_sim_kernel_ms(dsi_sim *h, int32_t device_index, float *ms);

/* Host<->device bytes moved per update+run+reduce on this process: what dsi_sim_update uploads
 * (h2d: the configurations as given, validated on the device, or -- with DSI_F_PER_TRIAL,
 * DSI_F_HIST or DSI_F_PATTERN -- the host-built device table) and the per-config moments (and
 * histograms) dsi_sim_reduce reads back (d2h). */
DSI_API dsi_status dsi_sim_io_bytes(dsi_sim *h, uint64_t *h2d, uint64_t *d2h);

/* Work units (config, trial tile) of this process: [first, first+count) of total. */
DSI_API dsi_status dsi_sim_units(dsi_sim *h, uint64_t *first, uint64_t *count, uint64_t *total);

/* The cross-rank exchange of this handle: *nranks and *rank as the NCCL
 * communicator itself reports them (ncclCommCount / ncclCommUserRank), *transport 1 = NCCL,
 * 2 = the test build's host all-reduce hook, 0 = none (one rank: nothing to exchange, *nranks
 * = 1, *rank = 0).  Lets a caller check that a multi-process run formed one communicator of
 * the expected size.  *cell_local (may be NULL) = 1 when every heatmap cell's configs are
 * simulated by one part (the shards are snapped to cell or group starts), so dsi_sim_heatmap
 * evaluates each part's cells from its own moments and exchanges only the 64-byte cells; 0 when
 * it all-reduces every config's moments first (the cells are planned on first use: query after
 * a dsi_sim_heatmap call for the handle's final answer). */
DSI_API dsi_status dsi_sim_comm_info(dsi_sim *h, int32_t *nranks, int32_t *rank, int32_t *transport,
                                     int32_t *cell_local);

DSI_API void dsi_sim_destroy(dsi_sim *h); /* NULL-safe */

DSI_API const char *dsi_status_str(dsi_status s);
DSI_API const char *dsi_sim_last_error(const dsi_sim *h); /* handle-owned; "" if none */
DSI_API const char *dsi_last_create_error(void);          /* thread-local message of the last failed
                                                     dsi_sim_create                          */
DSI_API uint32_t dsi_abi_version(void);

/* 128-byte NCCL unique id for multi-GPU runs (call on one rank, broadcast); one per handle
 * (or per dsi_multi_simulate call). */
DSI_API dsi_status dsi_nccl_unique_id(uint8_t id[128]);

/* Pure planner helpers of Eq. 1, exact integers.
 * Return -1 on invalid input (ticks < 1, sp < 1, k < 1). */
/* R15's time quantisation, the one create applies to every latency: *out = round(x / tick) when
 * x and tick are finite and positive and x / tick is within 1e-9 (relative) of an integer >= 1;
 * else DSI_E_RANGE (x or tick not finite / not positive), DSI_E_TICK (not a whole number of
 * ticks) or DSI_E_OVERFLOW, and *out is not written. */
DSI_API dsi_status dsi_ticks(double x, double tick, int64_t *out);
DSI_API int32_t dsi_min_lookahead(int64_t t_target_ticks, int64_t t_drafter_ticks, int32_t sp);
DSI_API int32_t dsi_required_processors(int64_t t_target_ticks, int64_t t_drafter_ticks, int32_t k);
DSI_API int32_t dsi_eq1_feasible(int64_t t_target_ticks, int64_t t_drafter_ticks, int32_t k, int32_t sp);

/* ---- Heatmap product (Fig. 3 / Fig. 5) ----------------
 * A cell is a maximal run of consecutive configs with equal (t_target, t_drafter,
 * accept_rate, sp_degree, n_tokens): the lookahead grid of one (drafter latency,
 * acceptance rate) point.  Per cell: SI = the minimal mean SI latency over the cell's
 * lookaheads ("the minimal average latency among all the lookahead values"),
 * DSI = the minimal mean DSI latency over the lookaheads satisfying Eq. 1 at the
 * config's SP, ties to the smallest k.  Panel "X/Y" is the run time of X divided
 * by the run time of Y: r_nonsi_si = nonSI/SI, r_si_dsi = SI/DSI,
 * r_nonsi_dsi = nonSI/DSI, r_min_dsi = min(SI, nonSI)/DSI (Fig. 3(a)-(d));
 * a ratio above 1 is a speedup of Y.  Cells with no feasible
 * DSI lookahead get dsi_lookahead = -1 and NaN DSI fields. */
typedef struct {
  double t_target, t_drafter, accept_rate; /* user units, copied from the configs */
  int32_t sp_degree, n_tokens;
  int32_t si_lookahead;   /* argmin k of mean SI                                    */
  int32_t dsi_lookahead;  /* argmin Eq.-1-feasible k of mean DSI, or -1             */
  double nonsi, si, dsi;  /* mean latencies, user units                             */
  double r_nonsi_si, r_si_dsi, r_nonsi_dsi, r_min_dsi;
  uint64_t first_cfg;     /* index of the cell's first config                       */
  uint64_t n_cfg;         /* number of configs (lookaheads) in the cell             */
} dsi_heatmap_cell;       /* 112 bytes */

/* Host-only.  cells may be NULL to count: *n_cells receives the number of cells;
 * otherwise at most cap cells are written (DSI_E_RANGE if cap is too small). */
DSI_API dsi_status dsi_heatmap(const dsi_config *cfg, const dsi_result *res, size_t n,
                       dsi_heatmap_cell *cells, size_t cap, size_t *n_cells);

/* On-device form: after dsi_sim_run, sums the moments across devices and
 * ranks (the all-reduce of dsi_sim_reduce; every rank must call it), evaluates every cell on
 * device 0 -- one warp per cell -- and copies only the cells back (64 B each instead of
 * 64 B per config).  With DSI_F_MEANS_ONLY and one device per process the ranks' config
 * ranges hold whole cells: each rank evaluates its own cells and only the cell records are
 * all-reduced (while the cells keep the layout they had at create).  Cells group consecutive configs with equal (t_target, t_drafter,
 * accept_rate, sp_degree, n_tokens) as given to create/update; the values are bit-identical
 * to dsi_heatmap over dsi_sim_reduce's results.  cells == NULL: *n_cells receives the
 * count (no device work).  DSI_E_RANGE if cap is too small, DSI_E_STATE before a run. */
DSI_API dsi_status dsi_sim_heatmap(dsi_sim *h, dsi_heatmap_cell *cells, size_t cap, size_t *n_cells);

/* CSV of cells (SPEC S:450-458 columns; fixed formatting, %.6f; rows in input order). */
DSI_API dsi_status dsi_heatmap_csv(const dsi_heatmap_cell *cells, size_t n, const char *path);

/* ---- Multi-drafter DSI: Algorithm 1 with m > 2 models ------------------
 * Algorithm 1 as stated: models f_1..f_m, f_m the target, lookahead 1 ("set to 1
 * for simplicity"), every finished thread initiates m threads (line 6), no bound on
 * concurrent threads (the abstract form).  The verifier at position p (a target
 * thread) keeps the sibling with the smallest index j* whose token equals the target's
 * (lines 8-11), so position p costs t_{j*(p)} and the run takes
 *     L_DSI = t_m + sum_{p=1}^{N-1} t_{j*(p)}       (P:418 with j_N = m),
 * non-SI N t_m.  Readings (R25):
 *   - drafters are ordered by latency, t_1 <= ... <= t_{m-1} <= t_m (Assumption 2);
 *   - drafter j's token at position p equals the target's with probability a_j,
 *     independently over j and p: A_{j,p} = [u < floor(a_j 2^32)], u = word (p-1) & 3 of
 *     Philox4x32-10 at counter ((p-1) >> 2, j-1, trial, stream_id) -- drafter 1 draws
 *     exactly the single-drafter stream of this library;
 *   - equal finish ticks: a drafter's token is compared before the target's (tie rule only
 *     affects which j is credited, never L_DSI);
 *   - DSI_F_PATTERN: trial i enumerates outcomes, digit p-1 of i in base m is j*(p) - 1
 *     (A_{j,p} = [j >= j*(p)]); run m^(N-1) trials for all of them.
 * The paper never measures m > 2; App. D's lookahead > 1 form for m > 2 and a
 * bounded SP are not modelled. */
#define DSI_MAX_DRAFTERS 7

typedef struct {
  double t_target;                      /* t_m: target forward latency, user units > 0      */
  double t_drafter[DSI_MAX_DRAFTERS];   /* t_1..t_{m-1}: 0 < t_1 <= ... <= t_{m-1} <= t_m    */
  double accept_rate[DSI_MAX_DRAFTERS]; /* a_j in [0,1]                                      */
  int32_t n_drafters;                   /* m - 1 in 1..7; entries beyond it are ignored      */
  int32_t n_tokens;                     /* N in [1, 32768]                                   */
  uint32_t stream_id;                   /* Philox counter word 3                             */
  uint32_t reserved;                    /* must be 0                                         */
  uint64_t n_trials;                    /* T in [1, 2^32]                                    */
} dsi_multi_config;                     /* 144 bytes */

typedef struct {
  uint64_t trials;
  int64_t t_target_ticks;
  int64_t nonsi_ticks;                           /* N t_m per trial                      */
  int64_t sum_dsi_ticks;
  uint64_t sumsq_dsi_ticks;
  int64_t sum_settled[DSI_MAX_DRAFTERS + 1];     /* [j-1]: sum over trials of
                                                    #{p in 1..N-1 : j*(p) = j}, j = 1..m;
                                                    entries >= m are 0                  */
  int64_t n_dsi_gt_nonsi;                        /* trials with L_DSI > N t_m (Thm 1: 0) */
  double mean_nonsi, mean_dsi;                   /* ((double)sum / (double)T) * tick     */
  double std_dsi;                                /* population std from exact integers   */
} dsi_multi_result;                              /* 136 bytes */

/* Simulate every config, blocking.  One device per process (opt->device, n_devices = 1).
 * Multi-GPU: with world > 1 each rank runs a contiguous, cost-balanced share of the units
 * (config, tile of trials) and the per-config integer moments are summed with one NCCL
 * all-reduce over a communicator created for the call from opt->nccl_id (a fresh id per
 * call: an NCCL id serves one communicator; every rank must call it with the same configs;
 * results are bit-identical for any world).  A non-NULL
 * nccl_id with world == 1 runs the same path on a one-rank communicator; n_shards > 1
 * (world == 1, tests) runs the partition's shards back to back.  Options used: abi_version,
 * tick, seed, device, rank, world, nccl_id, n_shards, stream, flags (DSI_F_PER_TRIAL (world
 * == 1), DSI_F_PATTERN, DSI_F_TIMING, DSI_F_MEANS_ONLY only).  out[n_cfg] is written on success.
 * DSI_F_MEANS_ONLY: j*(p) depends on the indicators only, so configs with equal (stream_id, N,
 * n_trials, thresholds) share one kernel pass and every config's sum_dsi_ticks = t_m (T +
 * sum_settled[m-1]) + sum_j t_j sum_settled[j] exactly (bit-identical sums and means, e.g. for a
 * latency grid); sumsq_dsi_ticks = 0 and std_dsi = NaN (n_dsi_gt_nonsi stays exact: 0).  With DSI_F_PER_TRIAL (else both must be NULL): trial_dsi[i] and
 * trial_settled[8 i + j-1] for i = the trial's position in config-major order (config c's
 * trials follow those of configs < c), either pointer may be NULL.  Validation as
 * dsi_sim_create (DSI_E_RANGE, DSI_E_TICK, DSI_E_OVERFLOW when N t_m >= 2^31 ticks or
 * T (N t_m)^2 >= 2^64); the message is in dsi_last_create_error(). */
DSI_API dsi_status dsi_multi_simulate(const dsi_options *opt, const dsi_multi_config *cfg, size_t n_cfg,
                              dsi_multi_result *out, int32_t *trial_dsi, int32_t *trial_settled);

/* With DSI_F_TIMING: device time (ms) of the kernel of the last dsi_multi_simulate on this
 * host thread (CUDA events on the launching stream); launches of it in *launches. */
DSI_API dsi_status dsi_multi_last_kernel(float *ms, int32_t *launches);

/* Build identity: the SHA-256 (hex) of the sources and flags this library was compiled from
 * (paper_2405_14105_b200/build.py embeds it), e.g. to prove a test ran a build of HEAD.
 * Static storage, never NULL. */
DSI_API const char *dsi_build_id(void);


/* Pure sharder (host only, no device): split per-unit costs into `parts`
 * contiguous ranges of near-equal total cost.  cost_units[i] >= 0.
 * bounds must hold parts+1 entries; bounds[0] = 0, bounds[parts] = n.
 * Used by dsi_sim_create for devices x ranks x shards; exported for tests. */
DSI_API dsi_status dsi_shard_bounds(const double *cost_units, uint64_t n, int32_t parts,
                            uint64_t *bounds);

#ifdef __cplusplus
}
#endif
#endif /* DSI_SIM_H */
