// dsi_device.h -- layout shared by the host runtime (dsi_*.cpp) and the
// sm_100a trial kernel (dsi_kernel.cu).  Internal: not part of the C ABI.
#pragma once
#include <stddef.h>
#include <stdint.h>

// Bounds checks of the kernels' computed indices: compiled in only by the checked test build
// (libdsi_sim_checked.so, -DDSI_BOUNDS_CHECK; tests/test_bounds_checked.py), which traps with the
// failing line -- the substitute for compute-sanitizer memcheck where the GPU pool has it closed.
#ifdef DSI_BOUNDS_CHECK
#include <cstdio>
#define DSI_CHECK(c)                                                            \
  do {                                                                          \
    if (!(c)) {                                                                 \
      printf("DSI_CHECK failed: %s at %s:%d\n", #c, __FILE__, __LINE__);       \
      __trap();                                                                 \
    }                                                                           \
  } while (0)
#else
#define DSI_CHECK(c) \
  do {               \
  } while (0)
#endif

namespace dsi {

// Indicator mode of a configuration (uniform per block).
enum : uint32_t {
  MODE_STREAM = 0,      // Philox stream, A_p = [u < thr]
  MODE_ALL_ACCEPT = 1,  // thr == 2^32: every draft accepted, no random numbers needed
  MODE_ALL_REJECT = 2,  // thr == 0: every draft rejected, no random numbers needed
};
enum : uint32_t {
  CFG_NOQUEUE = 1u << 8,  // S(b) = b*k*t_d (Eq. 1 holds or SP >= N)
  CFG_TTFT = 1u << 9,     // first forwards cost TTFT: first-segment correction table
  CFG_FRESH = 1u << 10,   // fresh-verifier variant and k t_d > t_t (else it equals the default)
  CFG_EQ1 = 1u << 11,     // Eq. 1 holds: ceil(t_t / (k t_d)) <= SP (heatmap DSI argmin)
};

// One configuration in ticks, as the kernel reads it (112 bytes).
struct alignas(16) DevCfg {
  uint32_t thr;        // floor(a * 2^32) when mode == MODE_STREAM
  uint32_t flags;      // mode (low byte) | CFG_NOQUEUE
  int32_t n_tokens;    // N
  int32_t k_eff;       // min(k, N): same ceil-divisions for every g <= N
  int32_t sp_eff;      // min(SP, N): b <= N-1, so larger SP never queues
  int32_t t_t;         // target latency, ticks
  int32_t kd;          // k * t_d, ticks
  int32_t si_cost;     // k * t_d + t_t: one SI iteration
  uint32_t stream_id;  // Philox counter word 3
  uint32_t m_si;       // ceil(2^32 / (k_eff+1))           : x / (k_eff+1)
  uint32_t m_k_lo;     // ceil(2^32 / k_eff) mod 2^32       : x / k_eff
  uint32_t m_k_hi;     //   ... and its bit 32 (k_eff == 1)
  uint32_t m_sp_lo;    // ceil(2^32 / sp_eff) mod 2^32      : x / sp_eff
  uint32_t m_sp_hi;
  uint32_t si_hist_off;  // first SI-histogram bin of this config (DSI_F_HIST)
  int32_t s1;            // S(1): DSI cost of any segment with 2 <= g <= k+1 beyond t_t
  uint64_t rec_off;      // first per-trial record of this config (DSI_F_PER_TRIAL)
  uint64_t n_trials;
  int32_t nonsi;         // t_t1 + (N-1) t_t: non-SI latency (first forward TTFT)
  int32_t e_si;          // (t_d1 - t_d) + (t_t1 - t_t): SI's first-iteration surcharge
  int32_t t_t1;          // the target's first-forward latency (TTFT variant), ticks
  int32_t ttft_shift;    // t_d1 - t_d: first-segment drafts are late by this (TTFT variant)
  int32_t t_d;           // drafter latency, ticks (fresh-verifier variant)
  int32_t k;             // the lookahead as given (heatmap argmin reports it)
  uint32_t m_tt;         // floor(x / t_t) = (umulhi(x, m_tt) + x) >> sh_tt for x < 2^31
  int32_t sh_tt;         //   (Granlund-Montgomery; fresh-verifier savings, dsi_common.cuh)
};
static_assert(sizeof(DevCfg) == 112, "DevCfg layout");

// Per-config integer moments accumulated by the kernel (u64 each).
enum Field : int {
  F_M = 0,       // sum of segments m
  F_I,           // sum of SI iterations I
  F_I2,          // sum of I^2            (L_SI = I * si_cost)
  F_DSI,         // sum of L_DSI
  F_DSI2,        // sum of L_DSI^2
  F_GT_NONSI,    // #trials with L_DSI > N t_t
  F_GT_SI,       // #trials with L_DSI > L_SI
  F_TRIALS,      // trials simulated (checks the partition covers every trial once)
  NF
};

struct Keys {
  uint32_t k0[10];  // key word 0 of rounds 0..9: seed_lo + r * 0x9E3779B9
  uint32_t k1[10];  // key word 1 of rounds 0..9: seed_hi + r * 0xBB67AE85
};

struct LaunchParams {
  const DevCfg *cfg;
  const uint64_t *tile_prefix;  // n_cfg + 1: first unit of each config
  uint32_t n_cfg;
  uint32_t tile_trials;         // trials per unit (the last unit of a config is ragged)
  uint64_t unit_begin;          // first unit of this launch; block b runs unit_begin + b
  unsigned long long *acc;      // n_cfg * NF
  int32_t *rec_acc, *rec_m, *rec_iters, *rec_si, *rec_dsi;  // DSI_F_PER_TRIAL
  unsigned long long *seg_hist;  // n_cfg * 64              (DSI_F_HIST)
  unsigned long long *si_hist;   // sum over configs of (k_eff + 1)
  int32_t max_n;                 // largest N over all configs (shared-memory sizing)
  int32_t max_keff;              // largest min(k, N) over all configs
  int32_t any_ttft;              // some config uses the TTFT variant (first-segment tables)
  int32_t any_fresh;             // some config has CFG_FRESH (every segment walked)
  int32_t k1_fast;               // launch the variant with the k = 1 no-queue fast path (VAR 3)
  int32_t halves;                // DSI_F_RNG_HALVES: the halves layout of the indicator stream
  int32_t pad_[2];               // keeps keys 16-byte aligned in the parameter bank (LDCU.128 loads)
  Keys keys;
};

// ---- shared-stream mode (DSI_F_SHARED_STREAMS, dsi_crn.cu)
struct CrnGroup {      // configs drawing identical indicators: equal (stream, threshold, N, T)
  uint32_t first;      // first position in perm
  uint32_t count;      // configs in the group
  int32_t n_tokens;
  uint32_t stream_id;
  uint32_t thr;        // threshold low word (mode says whether the stream is used)
  uint32_t mode;       // MODE_*
  uint64_t n_trials;
};
struct CrnUnit {       // one block: a slice of one group's configs over a range of its trials
  uint32_t group;
  uint32_t begin;      // position in perm
  uint32_t count;      // <= cfg_per_block
  uint32_t kind;       // 1: every config has k_eff = 1 and no queueing (no run lists needed)
  uint64_t t0, t1;     // trials [t0, t1)
};
struct CrnTile {       // two-pass mode, pass 1: one block per (group, tile of trials)
  uint32_t group;
  uint32_t tile;
};
struct CrnParams {
  const DevCfg *cfg;
  const uint32_t *perm;  // processing order of the configs (grouped, lookahead-major)
  const CrnGroup *groups;
  const CrnUnit *units;
  uint64_t unit_begin;
  unsigned long long *acc;  // n_cfg * NF, integer atomics (a config may span trial ranges)
  int32_t max_n, max_nq, max_runs, cfg_per_block;
  // two-pass mode (dsi_crn2.cu): trial records written by pass 1, streamed by pass 2
  unsigned char *records;      // record of (group g, tile t) at (group_tile0[g] + t) * rec_bytes
  const uint64_t *group_tile0;
  const CrnTile *tiles;        // pass-1 work list of this device
  uint64_t tile_begin;
  uint32_t rec_bytes;
  int32_t any_fresh;  // some config of the launch has CFG_FRESH (template FRESH variants)
  int32_t halves;     // DSI_F_RNG_HALVES: the halves layout of the indicator stream
  int32_t pad_[2];
  Keys keys;
};
// On-device heatmap product: one warp per cell, a cell being a run of
// consecutive configs (the lookahead grid of one (t_d, a) point).
struct HeatCell {
  uint64_t first;
  uint32_t count;
  uint32_t pad;
};
struct HeatOut {  // 64 bytes: the computed part of dsi_heatmap_cell
  double nonsi, si, dsi, r_nonsi_si, r_si_dsi, r_nonsi_dsi, r_min_dsi;
  int32_t si_k, dsi_k;  // argmin lookaheads (-1: no Eq.-1-feasible lookahead)
};
struct HeatParams {
  const DevCfg *cfg;
  const unsigned long long *acc;  // n_cfg * NF global sums
  const HeatCell *cells;
  const uint32_t *idx;  // NULL: cells [0, n_cells); else the n_cells cell indices to evaluate
  uint32_t n_cells;
  double tick;
  HeatOut *out;
  unsigned int *bad;  // set when a config's trial count differs from n_trials
};
int launch_heatmap_kernel(const HeatParams &p, void *stream);
// *bad |= 1 if some config's F_TRIALS differs from its n_trials
int launch_check_trials(const DevCfg *cfg, const unsigned long long *acc, uint64_t n, unsigned int *bad,
                        void *stream);

size_t crn_kernel_smem(int max_n, int block_threads, int cfg_per_block, int max_runs, bool fresh);
size_t crn_record_bytes(int max_runs, int threads, bool fresh);
size_t crn_eval_smem(int max_runs, int threads, bool fresh);
// pass 1 over n_tiles records (p.tiles from p.tile_begin), then pass 2 over n_units units
int launch_crn_two_pass(const CrnParams &p, uint64_t n_tiles, uint64_t n_units, int threads, void *stream);
int launch_crn_kernel(const CrnParams &p, uint64_t n_units, int block_threads, void *stream,
                      bool sums_only = false);

// ---- means-only mode (dsi_seg.cu, DSI_F_MEANS_ONLY): segment-length histograms per group
struct SegGroup {      // configs drawing identical indicators: equal (stream, threshold, N, T)
  uint64_t n_trials;
  uint64_t hist_off;   // H of this group: hist[hist_off .. hist_off + N]
  int32_t n_tokens;
  uint32_t stream_id;
  uint32_t thr;
  uint32_t mode;       // MODE_*
};
struct SegParams {
  const DevCfg *cfg;
  const SegGroup *groups;
  const uint64_t *unit_prefix;  // n_groups + 1: first hist unit of each group
  const uint32_t *cfg_group;    // group of each config
  uint32_t n_groups;
  uint32_t tile_trials;
  uint64_t unit_begin;          // pass 1: first unit of this launch
  uint64_t cfg_begin, cfg_end;  // pass 2: configs evaluated by this launch
  unsigned long long *hist;     // sum over groups of (N + 1) bins; bin 0 = trials
  unsigned long long *pre;      // prefix sums of hist (same offsets), for the bucketed evaluation
  unsigned long long *hist1;    // TTFT: first-segment lengths per group (same offsets; or NULL)
  const uint32_t *ttft_cfgs;    // TTFT: sorted indices of the TTFT configs of this launch
  unsigned long long *acc;      // n_cfg * NF
  int32_t max_n;
  int32_t halves;               // DSI_F_RNG_HALVES: the halves layout of the indicator stream
  int32_t pad_[2];
  Keys keys;
};
size_t seg_hist_smem(int max_n);
int launch_seg_hist(const SegParams &p, uint64_t n_units, void *stream);
int launch_seg_eval(const SegParams &p, void *stream);
int launch_seg_prefix(const SegParams &p, void *stream);
// TTFT correction of the configs ttft_cfgs[begin, end): F_DSI += sum_g H1[g] D1(g)
int launch_seg_ttft(const SegParams &p, uint64_t begin, uint64_t end, void *stream);

// ---- multi-drafter DSI (dsi_multi.cu)
struct alignas(16) MultiCfg {  // 112 bytes
  uint32_t thr[7];      // floor(a_j 2^32) when mode[j] == MODE_STREAM
  uint8_t mode[8];      // MODE_* per drafter
  int32_t t_d[7];       // drafter latencies, ticks (nondecreasing)
  int32_t t_t;          // target latency, ticks
  int32_t n_drafters;   // m - 1
  int32_t n_tokens;     // N
  uint32_t stream_id;
  uint64_t n_trials;
  uint64_t rec_off;     // first per-trial record of this config (DSI_F_PER_TRIAL)
  uint8_t width[8];     // drafter j >= 2 is called per group of width[j] quads (4, 2 or 1)
                        // when any of them is open: wide when quads are rarely all settled
  uint32_t pad[2];
};
static_assert(sizeof(MultiCfg) == 112, "MultiCfg layout");
enum MField : int { MF_DSI = 0, MF_DSI2, MF_GT_NONSI, MF_TRIALS, MF_SETTLED, MF = MF_SETTLED + 7 };
struct MultiParams {
  const MultiCfg *cfg;
  const uint64_t *tile_prefix;  // n_cfg + 1
  uint32_t n_cfg;
  uint32_t tile_trials;
  uint64_t unit_begin;
  unsigned long long *acc;      // n_cfg * MF
  int32_t *rec_dsi;             // per trial (or NULL)
  int32_t *rec_settled;         // 8 per trial (or NULL)
  int32_t max_n;
  int32_t max_drafters;
  int32_t halves;  // DSI_F_RNG_HALVES: drafter j on counter word 1 = 2j, its tie-break on 2j + 1
  int32_t pad_[3];
  Keys keys;
};
int launch_multi_kernel(const MultiParams &p, uint64_t n_units, bool pattern, void *stream);

// Dynamic shared memory of the variant chosen for (max_n, max_keff, hist).
size_t trial_kernel_smem(int max_n, int max_keff, bool hist, bool ttft);

// Launch the trial kernel variant for (per_trial, hist, pattern) on `stream`
// over units [p.unit_begin, p.unit_begin + n_units).  Returns a cudaError_t.
int launch_trial_kernel(const LaunchParams &p, uint64_t n_units, int block_threads,
                        bool per_trial, bool hist, bool pattern, void *stream);

}  // namespace dsi
