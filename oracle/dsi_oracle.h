/*
 * dsi_oracle.h -- the CPU oracle of the DSI Monte Carlo latency simulator.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library.
 * The product path (include/dsi_sim.h, paper_2405_14105_b200/) never links,
 * imports or executes anything under oracle/, and the oracle shares no code
 * with it (no headers, no helpers, no tables).
 *
 * What it computes, for one configuration (target latency t_t, drafter latency
 * t_d, acceptance rate a, lookahead k, SP degree, N tokens) and one trial:
 *   - the acceptance indicators A_1..A_{N-1} (paper P:434: i.i.d.
 *     Bernoulli(a) per draft token) drawn from a Philox4x32-10 stream, one
 *     32-bit word per position or (rng_halves) 16 bits plus a tie-break draw;
 *   - non-SI latency  N*t_t;
 *   - SI latency by the literal pseudocode loop;
 *   - DSI latency by a literal event simulation of Algorithm 1
 *     with the lookahead generalisation of Appendix D on SP
 *     FIFO target servers.
 * Times are integer ticks.  See DESIGN.md "Readings" for every place where the
 * paper is silent and the reading adopted (R1..R22 of SURVEY.md 8(c).4).
 */
#ifndef DSI_ORACLE_H
#define DSI_ORACLE_H
#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
  int64_t  t_target;     /* target forward latency t_2, integer ticks >= 1      */
  int64_t  t_drafter;    /* drafter forward latency t_1, 1 <= t_d <= t_t ticks  */
  double   accept_rate;  /* a in [0,1]                                          */
  int32_t  lookahead;    /* k >= 1                                              */
  int32_t  sp_degree;    /* SP >= 1 target servers                              */
  int32_t  n_tokens;     /* N >= 1                                              */
  uint32_t stream_id;    /* Philox counter word 3                               */
  /* TTFT variant: the first forward of each model costs
     its time-to-first-token -- the drafter's first draft and the target pool's
     first-ever forward (thread 0 of the first segment); 0 = same as the TPOT. */
  int64_t  t_target_first;
  int64_t  t_drafter_first;
  /* Fresh-verifier variant (R24; Thm 2's proof P:445:
     "DSI either invokes a new current verifier thread or labels an existing thread
     as the current verifier"): non-zero enables it.  Not with the TTFT variant. */
  int32_t  fresh_verifier;
  /* Indicator-stream layout: 0 = one 32-bit word per position; 1 = the
     "halves" layout (R26): 16 bits per position plus a tie-break draw. */
  int32_t  rng_halves;
} oracle_config;

typedef struct {
  int32_t acc;       /* #{p in 1..N-1 : A_p = 1}                            */
  int32_t m;         /* #segments = #rejections in 1..N-1 + 1              */
  int32_t iters;     /* SI iterations I (= SI target forwards)             */
  int64_t nonsi;     /* N * t_t                                            */
  int64_t si;        /* SI latency, ticks                                  */
  int64_t dsi;       /* DSI latency, ticks                                 */
  /* debug counters of the DSI event simulation */
  int32_t dsi_segments;        /* restarts + 1, must equal m                 */
  int32_t dsi_peak_busy;       /* max concurrently busy target servers       */
  int32_t dsi_max_queue;       /* max FIFO queue length (0 <=> never waited) */
  int32_t dsi_forwards;        /* target forwards started                    */
} oracle_trial_out;

typedef struct {
  uint64_t trials;
  int64_t  sum_acc, sum_m, sum_iters;
  int64_t  sum_si, sum_dsi;
  uint64_t sumsq_si, sumsq_dsi;
  int64_t  n_dsi_gt_nonsi, n_dsi_gt_si;
} oracle_sums;

/* Philox4x32-10 block function (Salmon et al., SC'11, "Parallel random
 * numbers: as easy as 1, 2, 3").  ctr[4], key[2] -> out[4]. */
void oracle_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]);

/* Bernoulli threshold thr = floor(a * 2^32) in [0, 2^32]; A_p = [u_p < thr]. */
uint64_t oracle_threshold(double a);

/* One trial.  pattern != 0: A_p = bit (p-1) of `trial` (enumeration mode, N <= 33).
 * si_hist (k+1 bins, may be NULL): SI accepted-drafts-per-iteration counts,
 *   only iterations whose k-draft window lies in positions <= N-1.
 * seg_hist (64 bins, may be NULL): segment lengths g, bin min(g, 63).
 * Returns 0, or -1 on invalid input / internal assertion failure. */
int oracle_trial(const oracle_config *cfg, uint64_t seed, uint64_t trial, int pattern,
                 oracle_trial_out *out, int64_t *si_hist, int64_t *seg_hist);

/* oracle_trial with the DSI event simulation's trace: one JSON object per line, kinds
   SegmentStart, VerifyDispatch, VerifyQueued, VerifyDone, ServerFreed, FreshDispatch, DraftDone,
   Accept, Reject, TokenEmitted (time in ticks, position, verification thread, segment), in
   processing order.  Debug output only; -2 when cap is too small. */
int oracle_trace_trial(const oracle_config *cfg, uint64_t seed, uint64_t trial, int pattern,
                       oracle_trial_out *out, char *buf, size_t cap, size_t *len);

/* Trials first..first+count-1: optional per-trial arrays (may be NULL),
 * sums accumulated into *sums (zero it first).  Returns 0 or -1. */
int oracle_run(const oracle_config *cfg, uint64_t seed, uint64_t first, uint64_t count,
               int pattern, oracle_sums *sums,
               int32_t *acc, int32_t *m, int32_t *iters, int64_t *si, int64_t *dsi,
               int64_t *si_hist, int64_t *seg_hist);

/* ------------------------------------------------------------------------ */
/* Multi-drafter DSI (dsi_oracle_multi.c).  Algorithm 1 as    */
/* stated: m models f_1..f_m, f_m the target, lookahead 1 (P:150 */
/* "set to 1 for simplicity"), every finished thread spawns m children, no   */
/* bound on concurrent threads.  Readings (R25):                   */
/*   - latencies t_1 <= t_2 <= ... <= t_{m-1} <= t_m (Assumption 2;   */
/*     j* = the smallest agreeing index is then the fastest agreeing model); */
/*   - on the verified prefix, drafter j's token at position p equals the    */
/*     target's with probability a_j, independently over j and p:            */
/*     A_{j,p} = [u < floor(a_j 2^32)], u = word (p-1)&3 of Philox at counter */
/*     (q = (p-1)>>2, j-1, trial, stream_id) -- drafter 1 draws exactly the   */
/*     single-drafter stream;                                                */
/*   - pattern mode: trial index i holds j*(p) - 1 as base-m digit p-1, and   */
/*     A_{j,p} = [j >= j*(p)];                                               */
/*   - equal finish ticks: drafters before targets, lower levels first;      */
/*   - RETURN (line 17) is taken by the current verifier at level N (a target */
/*     thread on an unverified prefix is never returned).                    */
/* ------------------------------------------------------------------------ */
#define ORACLE_MAX_MODELS 8

typedef struct {
  int64_t  t_target;                          /* t_m, ticks >= 1                     */
  int64_t  t_drafter[ORACLE_MAX_MODELS - 1];  /* t_1..t_{m-1}: 1 <= t_1 <= ... <= t_m  */
  double   accept_rate[ORACLE_MAX_MODELS - 1];/* a_j in [0,1]                         */
  int32_t  n_drafters;                        /* m - 1 in 1..7                        */
  int32_t  n_tokens;                          /* N >= 1                               */
  uint32_t stream_id;
  /* 0: drafter j's indicator at p is word (p-1)&3 of counter (q=(p-1)>>2, j-1, trial, stream);
     1: the halves layout (R26) with drafter j on counter word 1 = 2(j-1) and its
     tie-break on 2(j-1)+1 -- drafter 1 draws exactly the single-drafter halves stream */
  int32_t  rng_halves;
} oracle_multi_config;

typedef struct {
  int64_t nonsi;                       /* N t_m                                         */
  int64_t dsi;                         /* return time of Algorithm 1                    */
  int32_t settled[ORACLE_MAX_MODELS];  /* settled[j-1] = #{p in 1..N-1 : j*(p) = j}      */
  int64_t threads;                     /* tree simulation: threads started (0 in chain)  */
} oracle_multi_out;

typedef struct {
  uint64_t trials;
  int64_t  sum_dsi;
  uint64_t sumsq_dsi;
  int64_t  sum_settled[ORACLE_MAX_MODELS];
  int64_t  n_dsi_gt_nonsi;
} oracle_multi_sums;

/* A_{j,p} for drafter j in 1..m-1 and position p in 1..N-1 (0/1), -1 on bad input. */
int oracle_multi_indicator(const oracle_multi_config *cfg, uint64_t seed, uint64_t trial,
                           int pattern, int32_t j, int32_t p);

/* Literal thread-tree event simulation of Algorithm 1 (exponential in N; for pins).
 * Returns 0, -1 on invalid input / internal assertion, -2 if more than max_threads
 * threads would be started. */
int oracle_multi_tree(const oracle_multi_config *cfg, uint64_t seed, uint64_t trial, int pattern,
                      int64_t max_threads, oracle_multi_out *out);

/* The same schedule followed only along the verified prefix: threads on a rejected
 * prefix never change the verified chain's times when threads are unbounded, so the
 * chain is simulated level by level (spawn m siblings, the target sibling verifies,
 * j* = first agreeing model, its target child becomes the verifier).  Linear in N. */
int oracle_multi_chain(const oracle_multi_config *cfg, uint64_t seed, uint64_t trial, int pattern,
                       oracle_multi_out *out);

/* Trials first..first+count-1 with the chain simulation; optional per-trial arrays
 * (dsi[count], settled[count * m], m = n_drafters + 1); sums accumulated into *sums. */
int oracle_multi_run(const oracle_multi_config *cfg, uint64_t seed, uint64_t first, uint64_t count,
                     int pattern, oracle_multi_sums *sums, int64_t *dsi, int32_t *settled);

#ifdef __cplusplus
}
#endif
#endif
