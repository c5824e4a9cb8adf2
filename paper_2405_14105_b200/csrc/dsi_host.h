// dsi_host.h -- internal declarations of the host runtime behind include/dsi_sim.h
// (not installed, not part of the ABI).  The runtime is split by concern:
//   dsi_validate.cpp   validation, tick conversion, Eq. 1 planner helpers, launch limits
//   dsi_plan.cpp       work plans (per-config tiles, shared-stream groups, means-only
//                      histograms, heatmap cells) and the device config table
//   dsi_collective.cpp NCCL (dlopen), the cross-device sums, test-build hooks
//   dsi_runtime.cpp    handle lifetime, create/update/run/reduce/heatmap and accessors
//   dsi_multi_host.cpp the multi-drafter call (dsi_multi_simulate)
// All arithmetic of the method runs in the CUDA kernels (dsi_*.cu); the host prepares
// inputs and combines exact integer sums.
#pragma once
#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>  // NVTX ranges of the API calls (header-only, see Trace)
#include <nccl.h>  // types and enums only; libnccl is loaded with dlopen at first use

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <condition_variable>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <map>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "../../include/dsi_sim.h"
#include "../../include/dsi_sim_testing.h"
#include "dsi_convert.h"
#include "dsi_device.h"

namespace dsih {

using dsi::CfgTicks;
using dsi::DevCfg;
using dsi::LaunchParams;
using dsi::kMaxTokens;
using dsi::kMaxTrials;
constexpr int kDefaultThreads = 128;
constexpr int kCrnThreads = 128;   // dsi_crn_kernel block size when 256 does not fit (see plan_shared)
constexpr size_t kReduceChunks = 8;  // dsi_sim_reduce: D2H chunks overlapped with the finalize
constexpr int kMeansMaxN = kMaxTokens;  // means-only mode (smem histograms up to N 8192, global above)
constexpr int kCrnMaxN = 2048;     // shared-stream mode: 128 per-trial run lists of <= N/3+2
                                   // u16 entries fit shared memory (209 KB at N 2048)

// ----------------------------------------------------------------------------- NCCL (dlopen)
struct NcclApi {
  void *lib = nullptr;
  ncclResult_t (*GetUniqueId)(ncclUniqueId *) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t *, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*AllReduce)(const void *, void *, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char *(*GetErrorString)(ncclResult_t) = nullptr;
  ncclResult_t (*CommCount)(const ncclComm_t, int *) = nullptr;     // optional (comm info)
  ncclResult_t (*CommUserRank)(const ncclComm_t, int *) = nullptr;  // optional (comm info)
  bool ok = false;
};

NcclApi &nccl();

// ----------------------------------------------------------------------------- helpers
inline int64_t ceil_div(int64_t a, int64_t b) { return dsi::ceil_div64(a, b); }

template <class T>
struct Pinned {  // page-locked host buffer (true async DMA for H2D/D2H)
  T *p = nullptr;
  size_t n = 0;
  cudaError_t alloc(size_t count) {
    release();
    n = count;
    return cudaMallocHost((void **)&p, std::max<size_t>(1, count) * sizeof(T));
  }
  void release() {
    if (p) cudaFreeHost(p);
    p = nullptr;
    n = 0;
  }
};

// Developer A/B knobs.  The product library always uses the defaults below; only the test
// build (-DDSI_TEST_HOOKS, libdsi_sim_test.so) lets dsi_test_set_knob change them.
struct Knobs {
  int k1_fast = -1;          // trial kernel k = 1 fast path: -1 automatic (work share), 0 off, 1 on
  int crn_two_pass = -1;     // shared-stream two-pass form: -1 automatic, 0 off
  int crn_threads = 0;       // shared-stream block size: 0 automatic, 128 or 256
  int crn_sums_split = 1;    // shared-stream sums-only slices: 1 on, 0 off
  int tile_r = 0;            // trial tiles of 128 * tile_r trials: 0 automatic
};
const Knobs &knobs();

}  // namespace dsih

// the handle types below use the internal ones (this header is private to the library)
using namespace dsih;

// ----------------------------------------------------------------------------- handle
struct DeviceState {
  int ordinal = -1;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  DevCfg *d_cfg = nullptr;
  uint64_t *d_prefix = nullptr;
  unsigned long long *d_acc = nullptr;
  unsigned long long *d_red = nullptr;
  unsigned long long *d_seg = nullptr, *d_seg_red = nullptr;
  unsigned long long *d_si = nullptr, *d_si_red = nullptr;
  int32_t *d_rec = nullptr;  // 5 arrays of total_trials
  uint32_t *d_perm = nullptr;            // shared-stream mode: processing order
  dsi::CrnGroup *d_groups = nullptr;     //   groups of configs sharing a stream
  dsi::CrnUnit *d_crn_units = nullptr;   //   one block per unit
  unsigned char *d_records = nullptr;    //   two-pass mode: trial records (pass 1 -> pass 2)
  uint64_t *d_group_tile0 = nullptr;
  dsi::CrnTile *d_tiles = nullptr;       //   pass-1 work list of this device
  size_t tiles_cap = 0, records_cap = 0, group_tile0_cap = 0;  // tiles: entries; others: bytes
  std::vector<dsi::CrnTile> tiles;
  dsi::HeatCell *d_heat_cells = nullptr; // on-device heatmap product (device 0 only)
  dsi::HeatOut *d_heat_out = nullptr;
  unsigned int *d_heat_bad = nullptr;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  ncclComm_t comm = nullptr;
  std::vector<std::pair<uint64_t, uint64_t>> ranges;  // [begin, end) units, one per shard
  std::vector<std::pair<uint64_t, uint64_t>> ttft_ranges;  // shared-stream mode: per-config units of the TTFT configs
  dsi::SegGroup *d_seg_groups = nullptr;  // means-only mode: groups, unit prefix, config -> group,
  uint64_t *d_seg_prefix = nullptr;       //   segment-length histograms (bin 0 = trials)
  uint32_t *d_cfg_group = nullptr;
  unsigned long long *d_hist = nullptr;   // H | prefix of H | (TTFT) H1, hist_len each
  uint32_t *d_ttft_cfgs = nullptr;
  std::vector<std::pair<uint64_t, uint64_t>> cfg_ranges;  // means-only: configs evaluated here
  std::vector<uint32_t> owned_cells;      // cell-local heatmap: the cells this device's parts own
  uint32_t *d_owned = nullptr;            //   ... on the device
  size_t owned_cap = 0;
  // device path of dsi_sim_update (dsi_stage.cu): the configurations as given, current and spare,
  // the spare device table and the staging status
  dsi_config *d_raw = nullptr, *d_raw_next = nullptr;
  DevCfg *d_cfg_next = nullptr;
  dsi::StageStatus *d_stage = nullptr;
};

struct dsi_sim {
  dsi_options opt{};
  size_t n_cfg = 0;
  std::vector<CfgTicks> ticks;
  std::vector<CfgTicks> ticks_next;      // dsi_sim_update validates into this, then swaps
  Pinned<DevCfg> dev_cfg;                // staging of the device config table
  std::vector<uint64_t> prefix;          // n_cfg + 1 units
  uint64_t total_units = 0;
  uint64_t total_trials = 0;
  uint32_t tile_trials = 0;
  int block_threads = kDefaultThreads;
  int32_t max_n = 1, max_keff = 1;
  bool any_ttft = false;
  bool any_fresh = false;                 // DSI_F_FRESH_VERIFIER and some k t_d > t_t
  bool k1_fast = false;                   // trial kernel variant with the k = 1 no-queue fast path
  uint64_t si_bins_total = 0;
  bool shared = false;                    // DSI_F_SHARED_STREAMS
  bool means_only = false;                // DSI_F_MEANS_ONLY (dsi_seg.cu)
  std::vector<dsi::SegGroup> seg_groups;
  std::vector<uint64_t> seg_prefix;       // groups + 1 histogram units
  std::vector<uint32_t> cfg_group;
  uint64_t hist_len = 0;
  std::vector<uint32_t> ttft_cfgs;        // means-only + TTFT: configs with a first-segment correction
  std::vector<uint64_t> cfg_bounds;       // means-only: parts' config ranges (all ranks), cell-aligned
  std::vector<uint64_t> part_bounds;      // every part's unit range [b[p], b[p+1]) (all ranks)
  bool cell_local = false;                // every heatmap cell's configs lie in one part (plan_cell_owners)
  bool use_nccl = false;                  // per-config moments summed across devices/ranks
  bool host_coll = false;                 // ... through the host all-reduce hook instead of NCCL
  std::vector<uint32_t> perm;
  std::vector<uint32_t> shared_ttft;      // shared-stream mode: the TTFT configs (not shared; per-config kernel)
  uint64_t ttft_units = 0;                //   their (config, tile) units, h->prefix / h->tile_trials
  std::vector<dsi::CrnGroup> groups;
  std::vector<dsi::CrnUnit> crn_units;
  int32_t cfg_per_block = 0, max_runs = 0;
  bool two_pass = false;                  // shared-stream mode in two passes (dsi_crn2.cu)
  uint64_t n_sums_units = 0;              // the first units need no run lists (plan_shared)
  int32_t max_runs_normal = 0;            // run-list slots the other units need
  uint32_t rec_bytes = 0;
  uint64_t total_records = 0;
  std::vector<uint64_t> group_tile0;
  std::vector<DeviceState> dev;
  Pinned<unsigned long long> host_acc, host_seg, host_si;  // D2H targets
  bool ran = false, reduced = false;
  bool raw_valid = false;    // dev[0].d_raw holds the current configurations (device update path)
  bool ticks_stale = false;  // a device update committed: ticks / dev_cfg staging refreshed on demand
  Pinned<dsi_config> raw_pinned;        // staging of configurations (H2D from pageable memory, D2H)
  Pinned<dsi::StageStatus> stage_host;
  bool reduced_device = false;  // the moments of the last run are summed (dsi_sim_reduce[_device])
  std::vector<dsi::HeatCell> heat_cells;  // heatmap cells (planned on first use, reset by update)
  bool heat_planned = false, heat_uploaded = false;
  Pinned<dsi::HeatOut> heat_out;
  Pinned<unsigned int> host_bad;         // partition-check flag (D2H)
  cudaEvent_t chunk_ev[8] = {};          // reduce: one event per D2H chunk
  int launches = 0;
  std::string err;
};

namespace dsih {

extern thread_local std::string g_create_error;

inline dsi_status fail(dsi_sim *h, dsi_status s, const std::string &msg) {
  if (h) h->err = msg; else g_create_error = msg;
  return s;
}

inline dsi_status cuda_fail(dsi_sim *h, cudaError_t e, const char *what) {
  return fail(h, e == cudaErrorMemoryAllocation ? DSI_E_NOMEM : DSI_E_DEVICE,
              std::string(what) + ": " + cudaGetErrorString(e));
}

#define CUDA_TRY(h, call)                                  \
  do {                                                     \
    cudaError_t e_ = (call);                               \
    if (e_ != cudaSuccess) return cuda_fail(h, e_, #call); \
  } while (0)

// Cross-rank sums through the test build's host hook (several ranks on one GPU).
bool host_hook_set();
bool host_hook_sum(uint64_t *buf, size_t count);  // true on success
dsi_status host_allreduce(dsi_sim *h, cudaStream_t st, const void *src, void *dst, size_t count);

dsi_status to_ticks(double x, double tick, int64_t *out);
dsi_status convert(const dsi_options &opt, const dsi_config &c, size_t i, CfgTicks &o, std::string &msg);
std::string convert_message(size_t i, int code);
using dsi::config_noqueue;
using dsi::make_dev_cfg;
double unit_cost(const CfgTicks &t, uint64_t trials);
double shared_eval_cost(const CfgTicks &t, bool fresh, bool two_pass);

// Every API call is an NVTX range (nvtx3, header-only: a no-op unless a profiler such as
// ncu or nsys injects its NVTX handler), and each phase an NVTX mark; with DSI_TRACE=1 in the
// environment each call also prints its phases (host wall clock, ms) to stderr on return --
// e.g. where dsi_sim_update's time goes.
class Trace {
 public:
  explicit Trace(const char *call) : call_(call), on_(enabled()) {
    nvtxRangePushA(call);
    if (on_) t0_ = last_ = std::chrono::steady_clock::now();
  }
  Trace(const Trace &) = delete;
  Trace &operator=(const Trace &) = delete;
  void mark(const char *phase) {
    nvtxMarkA(phase);
    if (!on_) return;
    const auto t = std::chrono::steady_clock::now();
    char b[96];
    std::snprintf(b, sizeof b, " %s=%.3f", phase, std::chrono::duration<double, std::milli>(t - last_).count());
    phases_ += b;
    last_ = t;
  }
  ~Trace() {
    nvtxRangePop();
    if (!on_) return;
    const double total =
        std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0_).count();
    std::fprintf(stderr, "[dsi] %s %.3f ms:%s\n", call_, total, phases_.c_str());
  }

 private:
  static bool enabled() {
    static const bool e = [] {
      const char *v = std::getenv("DSI_TRACE");
      return v && std::atoi(v) != 0;
    }();
    return e;
  }
  const char *call_;
  bool on_;
  std::chrono::steady_clock::time_point t0_, last_;
  std::string phases_;
};

// Process-wide pool of host worker threads (created on first use, kept for the life of
// the process): the O(n_cfg) host passes -- validation, staging, finalize -- run on it
// without spawning threads per call.  One job at a time; the calling thread helps.
class WorkerPool {
 public:
  static WorkerPool &get() {
    static WorkerPool *pool = new WorkerPool();  // never destroyed: workers idle at exit
    return *pool;
  }
  size_t threads() const { return workers_.size() + 1; }
  void run(uint32_t n_chunks, const std::function<void(size_t)> &job) {
    std::lock_guard<std::mutex> one_job(submit_mu_);
    {
      std::lock_guard<std::mutex> lk(mu_);
      ++gen_;
      job_.store(&job);
      // tickets are (generation << 32 | chunk): a worker holding a ticket of an older job
      // sees a different generation in info_ and drops it, so no chunk runs twice
      info_.store(gen_ << 32 | n_chunks);
      pending_.store(n_chunks);
      next_.store(gen_ << 32);
    }
    cv_.notify_all();
    work();
    std::unique_lock<std::mutex> lk(mu_);
    done_cv_.wait(lk, [&] { return pending_.load() == 0; });
  }

 private:
  WorkerPool() {
    size_t nt = std::thread::hardware_concurrency();
    nt = std::min<size_t>(std::max<size_t>(nt, 1), 32);
    for (size_t i = 1; i < nt; ++i) workers_.emplace_back([this] { loop(); });
  }
  void work() {
    for (;;) {
      const uint64_t t = next_.fetch_add(1);
      const uint64_t info = info_.load();
      if ((t >> 32) != (info >> 32) || (t & 0xffffffffu) >= (info & 0xffffffffu)) return;
      (*job_.load())((size_t)(t & 0xffffffffu));  // a valid ticket: its job is still running
      if (pending_.fetch_sub(1) == 1) {
        std::lock_guard<std::mutex> lk(mu_);
        done_cv_.notify_all();
      }
    }
  }
  void loop() {
    uint64_t seen = 0;
    for (;;) {
      {
        std::unique_lock<std::mutex> lk(mu_);
        cv_.wait(lk, [&] { return gen_ != seen; });
        seen = gen_;
      }
      work();
    }
  }
  std::vector<std::thread> workers_;
  std::mutex submit_mu_, mu_;
  std::condition_variable cv_, done_cv_;
  std::atomic<const std::function<void(size_t)> *> job_{nullptr};
  std::atomic<uint64_t> info_{0}, next_{0};
  std::atomic<uint32_t> pending_{0};
  uint64_t gen_ = 0;  // guarded by mu_
};

// Run fn(begin, end) over [0, n) on the worker pool (large grids only: the per-config
// host work is O(1) and independent).
template <class Fn>
inline void parallel_for(size_t n, Fn fn, size_t min_parallel = (1u << 15)) {
  WorkerPool &pool = WorkerPool::get();
  if (n < min_parallel || n < 2 || pool.threads() == 1) {
    fn((size_t)0, n);
    return;
  }
  const size_t chunks = std::min(n, pool.threads() * 4);
  const std::function<void(size_t)> job = [&](size_t c) { fn(n * c / chunks, n * (c + 1) / chunks); };
  pool.run((uint32_t)chunks, job);
}

// What an update keeps (validate_all with prev): the shared-stream plan's keys (stream, a, N, T, k,
// t_t, t_d, SP), the means-only groups' keys (stream, a, N, T, TTFT or not), the heatmap cells' keys
// (t_target, t_drafter, a as given, SP, N).
struct UpdateKeys {
  bool plan_same = false, groups_same = false, cells_same = false;
};
dsi_status validate_all(dsi_sim *h, const dsi_config *cfg, size_t n, std::vector<CfgTicks> &out,
                        const std::vector<CfgTicks> *prev = nullptr, UpdateKeys *keys = nullptr);
cudaError_t fill_dev_cfg(dsi_sim *h, bool upload_chunks = false);
void free_device(DeviceState &d);
void free_handle(dsi_sim *h);
dsi_status upload(dsi_sim *h, bool plan = true, bool cfg_table = true);
dsi_status plan_means(dsi_sim *h, std::vector<double> &cost, uint64_t target_units);
dsi_status derive_limits(dsi_sim *h, const std::vector<CfgTicks> &ticks);
dsi_status sum_across(dsi_sim *h, bool hist);
dsi_status plan_two_pass(dsi_sim *h);
dsi_status alloc_two_pass(dsi_sim *h);
dsi_status plan_shared(dsi_sim *h, std::vector<double> &cost);
void plan_heat_cells(dsi_sim *h);
bool snap_bounds(std::vector<uint64_t> &bounds, const std::vector<double> &cost, const std::vector<uint64_t> &cand,
                 double slack);
void plan_cell_owners(dsi_sim *h);
dsi_status ensure_ticks(dsi_sim *h);
bool cells_aligned(const dsi_sim *h);

}  // namespace dsih
