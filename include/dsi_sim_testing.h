/*
 * dsi_sim_testing.h -- test-only entry points of the DSI simulator library.
 *
 * They exist only in the TEST build, paper_2405_14105_b200/libdsi_sim_test.so (compiled with
 * -DDSI_TEST_HOOKS from the same sources as libdsi_sim.so); the product library exports none
 * of them and reads no developer knobs.  Include after dsi_sim.h.
 */
#ifndef DSI_SIM_TESTING_H
#define DSI_SIM_TESTING_H

#include "dsi_sim.h"

#ifdef __cplusplus
extern "C" {
#endif

/* Test hook: cross-rank sums through a host function instead of NCCL.  While set (fn != NULL),
 * handles and dsi_multi_simulate calls created with world > 1 need no nccl_id and one device per
 * process; every cross-rank sum (moments, histograms, heatmap cells) copies the u64 words to the
 * host, calls fn(buf, n, user) -- which must replace buf by the element-wise sum over all ranks
 * and return 0 -- and copies them back.  It lets several ranks share one GPU (which NCCL refuses),
 * e.g. with a torch.distributed gloo all_reduce.  Process-global; pass NULL to clear. */
typedef int (*dsi_host_allreduce_fn)(uint64_t *buf, size_t n, void *user);
DSI_API dsi_status dsi_set_host_allreduce(dsi_host_allreduce_fn fn, void *user);

/* Developer A/B knobs of the launch planner (defaults in brackets; every value gives the same
 * results bit for bit, only the kernel variant or launch shape changes):
 *   "k1_fast"        trial kernel with the k = 1 no-queue fast path: -1 automatic [-1], 0, 1
 *   "crn_two_pass"   shared-stream two-pass form: -1 automatic [-1], 0 off
 *   "crn_threads"    shared-stream block size: 0 automatic [0], 128, 256
 *   "crn_sums_split" shared-stream sums-only slices: 1 [1], 0
 *   "tile_r"         trial tiles of 128 * tile_r trials: 0 automatic [0], 1..1024
 * Process-global; read by dsi_sim_create / dsi_sim_update.  DSI_E_RANGE for an unknown name. */
DSI_API dsi_status dsi_test_set_knob(const char *name, int32_t value);

#ifdef __cplusplus
}
#endif
#endif /* DSI_SIM_TESTING_H */
