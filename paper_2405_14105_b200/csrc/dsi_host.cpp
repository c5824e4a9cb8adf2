// dsi_host.cpp -- host runtime behind include/dsi_sim.h.
//
// Validation and tick conversion, Eq. 1 planner helpers, the cost-balanced
// sharder, per-device state (streams, buffers, pinned staging of the config
// table and results), the NCCL all-reduce of the per-config integer moments,
// and FP64 finalisation.  All arithmetic of the method runs in dsi_kernel.cu;
// this file only prepares inputs and combines exact integer sums.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>  // types and enums only; libnccl is loaded with dlopen at first use

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <condition_variable>
#include <functional>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <new>
#include <map>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "../../include/dsi_sim.h"
#include "dsi_device.h"

using dsi::DevCfg;
using dsi::LaunchParams;

namespace {

thread_local std::string g_create_error;

constexpr int kMaxTokens = 32768;  // keeps every magic division exact (x * d <= 2^32)
constexpr uint64_t kMaxTrials = 1ull << 32;
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
  bool ok = false;
};

NcclApi &nccl() {
  static NcclApi api;
  static bool tried = false;
  if (!tried) {
    tried = true;
    // Reuse a libnccl already mapped into the process (e.g. torch's), else load one.
    void *h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (h) {
      api.lib = h;
      api.GetUniqueId = (decltype(api.GetUniqueId))dlsym(h, "ncclGetUniqueId");
      api.CommInitRank = (decltype(api.CommInitRank))dlsym(h, "ncclCommInitRank");
      api.CommDestroy = (decltype(api.CommDestroy))dlsym(h, "ncclCommDestroy");
      api.AllReduce = (decltype(api.AllReduce))dlsym(h, "ncclAllReduce");
      api.GroupStart = (decltype(api.GroupStart))dlsym(h, "ncclGroupStart");
      api.GroupEnd = (decltype(api.GroupEnd))dlsym(h, "ncclGroupEnd");
      api.GetErrorString = (decltype(api.GetErrorString))dlsym(h, "ncclGetErrorString");
      api.ok = api.GetUniqueId && api.CommInitRank && api.CommDestroy && api.AllReduce &&
               api.GroupStart && api.GroupEnd && api.GetErrorString;
    }
  }
  return api;
}

// ----------------------------------------------------------------------------- helpers
struct CfgTicks {
  int64_t t_t, t_d, kd;
  int64_t t_t1, t_d1;  // first-forward latencies (TTFT variant; equal to t_t, t_d when off)
  uint64_t thr;
  int32_t k, sp, n;
  uint32_t stream_id;
  uint64_t trials;
  double a;
  double ut, ud;  // t_target, t_drafter as given (heatmap cells group on the user values)
  int32_t eq1, min_k;  // Eq. 1 holds at (k, SP); the minimal lookahead at SP
};

// ceil(2^32 / d) split into low word and bit 32 (d >= 1).
void magic(uint32_t d, uint32_t &lo, uint32_t &hi) {
  // divisors below 2^16 (every lookahead, SP and N the planner sees in practice) come from a
  // table built once: make_dev_cfg needs three per config, millions of times per update
  static const std::vector<uint64_t> table = [] {
    std::vector<uint64_t> t(1u << 16, 0);
    for (uint32_t x = 1; x < (1u << 16); ++x) t[x] = ((1ull << 32) + x - 1) / x;
    return t;
  }();
  const uint64_t m = d < (1u << 16) ? table[d] : ((1ull << 32) + d - 1) / d;
  lo = (uint32_t)m;
  hi = (uint32_t)(m >> 32);
}

int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

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

}  // namespace

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
  size_t tiles_cap = 0, records_cap = 0;
  std::vector<dsi::CrnTile> tiles;
  dsi::HeatCell *d_heat_cells = nullptr; // on-device heatmap product (device 0 only)
  dsi::HeatOut *d_heat_out = nullptr;
  unsigned int *d_heat_bad = nullptr;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  ncclComm_t comm = nullptr;
  std::vector<std::pair<uint64_t, uint64_t>> ranges;  // [begin, end) units, one per shard
  dsi::SegGroup *d_seg_groups = nullptr;  // means-only mode: groups, unit prefix, config -> group,
  uint64_t *d_seg_prefix = nullptr;       //   segment-length histograms (bin 0 = trials)
  uint32_t *d_cfg_group = nullptr;
  unsigned long long *d_hist = nullptr;   // H | prefix of H | (TTFT) H1, hist_len each
  uint32_t *d_ttft_cfgs = nullptr;
  std::vector<std::pair<uint64_t, uint64_t>> cfg_ranges;  // means-only: configs evaluated here
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
  bool use_nccl = false;                  // per-config moments summed across devices/ranks
  bool host_coll = false;                 // ... through the host all-reduce hook instead of NCCL
  std::vector<uint32_t> perm;
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
  std::vector<dsi::HeatCell> heat_cells;  // heatmap cells (planned on first use, reset by update)
  bool heat_planned = false, heat_uploaded = false;
  Pinned<dsi::HeatOut> heat_out;
  Pinned<unsigned int> host_bad;         // partition-check flag (D2H)
  cudaEvent_t chunk_ev[8] = {};          // reduce: one event per D2H chunk
  int launches = 0;
  std::string err;
};

namespace {
// Test hook (dsi_set_host_allreduce): cross-rank sums through a caller-supplied host function
// instead of NCCL, so multi-rank runs can be exercised where NCCL cannot form a communicator
// (several ranks on one GPU).
dsi_host_allreduce_fn g_host_ar = nullptr;
void *g_host_ar_user = nullptr;
}  // namespace

namespace {

dsi_status fail(dsi_sim *h, dsi_status s, const std::string &msg) {
  if (h) h->err = msg; else g_create_error = msg;
  return s;
}

dsi_status cuda_fail(dsi_sim *h, cudaError_t e, const char *what) {
  return fail(h, e == cudaErrorMemoryAllocation ? DSI_E_NOMEM : DSI_E_DEVICE,
              std::string(what) + ": " + cudaGetErrorString(e));
}

#define CUDA_TRY(h, call)                                  \
  do {                                                     \
    cudaError_t e_ = (call);                               \
    if (e_ != cudaSuccess) return cuda_fail(h, e_, #call); \
  } while (0)

// In-place-or-copy sum of count u64 words across the ranks through the host hook (one device per
// process): device -> host, hook, host -> device, synchronous on the stream.
dsi_status host_allreduce(dsi_sim *h, cudaStream_t st, const void *src, void *dst, size_t count) {
  std::vector<uint64_t> buf;
  try {
    buf.resize(count);
  } catch (...) {
    return fail(h, DSI_E_NOMEM, "host all-reduce buffer");
  }
  CUDA_TRY(h, cudaMemcpyAsync(buf.data(), src, count * sizeof(uint64_t), cudaMemcpyDeviceToHost, st));
  CUDA_TRY(h, cudaStreamSynchronize(st));
  if (!g_host_ar || g_host_ar(buf.data(), count, g_host_ar_user) != 0)
    return fail(h, DSI_E_COMM, "host all-reduce hook failed");
  CUDA_TRY(h, cudaMemcpyAsync(dst, buf.data(), count * sizeof(uint64_t), cudaMemcpyHostToDevice, st));
  CUDA_TRY(h, cudaStreamSynchronize(st));
  return DSI_OK;
}

dsi_status to_ticks(double x, double tick, int64_t *out) {
  if (!std::isfinite(x) || x <= 0.0) return DSI_E_RANGE;
  const double r = x / tick;
  if (!(r < 9.0e18)) return DSI_E_OVERFLOW;
  const int64_t t = std::llround(r);
  if (t < 1 || std::fabs(r - (double)t) > 1e-9 * std::fabs(r)) return DSI_E_TICK;
  *out = t;
  return DSI_OK;
}

dsi_status convert(const dsi_options &opt, const dsi_config &c, size_t i, CfgTicks &o,
                   std::string &msg) {
  char buf[256];
  auto bad = [&](dsi_status s, const char *what) {
    std::snprintf(buf, sizeof buf, "config %zu: %s", i, what);
    msg = buf;
    return s;
  };
  if (!(c.accept_rate >= 0.0 && c.accept_rate <= 1.0))
    return bad(DSI_E_RANGE, "accept_rate must be in [0, 1]");
  if (c.lookahead < 1) return bad(DSI_E_RANGE, "lookahead must be >= 1");
  if (c.sp_degree < 1) return bad(DSI_E_RANGE, "sp_degree must be >= 1");
  if (c.n_tokens < 1 || c.n_tokens > kMaxTokens)
    return bad(DSI_E_RANGE, "n_tokens must be in [1, 32768]");
  if (c.n_trials < 1 || c.n_trials > kMaxTrials)
    return bad(DSI_E_RANGE, "n_trials must be in [1, 2^32]");
  if ((opt.flags & DSI_F_PATTERN) && c.n_tokens > 33)
    return bad(DSI_E_RANGE, "DSI_F_PATTERN needs n_tokens <= 33");
  dsi_status s = to_ticks(c.t_target, opt.tick, &o.t_t);
  if (s != DSI_OK) return bad(s, "t_target is not a positive whole number of ticks");
  s = to_ticks(c.t_drafter, opt.tick, &o.t_d);
  if (s != DSI_OK) return bad(s, "t_drafter is not a positive whole number of ticks");
  if (o.t_d > o.t_t) return bad(DSI_E_RANGE, "t_drafter > t_target violates Assumption 2 (P:187-189)");
  o.t_t1 = o.t_t;
  o.t_d1 = o.t_d;
  if (c.ttft_target != 0.0) {
    s = to_ticks(c.ttft_target, opt.tick, &o.t_t1);
    if (s != DSI_OK) return bad(s, "ttft_target is not 0 or a positive whole number of ticks");
  }
  if (c.ttft_drafter != 0.0) {
    s = to_ticks(c.ttft_drafter, opt.tick, &o.t_d1);
    if (s != DSI_OK) return bad(s, "ttft_drafter is not 0 or a positive whole number of ticks");
  }
  if (o.t_d1 > o.t_t1) return bad(DSI_E_RANGE, "ttft_drafter > ttft_target violates Assumption 2");
  if ((opt.flags & DSI_F_SHARED_STREAMS) && (o.t_t1 != o.t_t || o.t_d1 != o.t_d))
    return bad(DSI_E_RANGE, "DSI_F_SHARED_STREAMS does not support the TTFT variant");
  if ((opt.flags & DSI_F_FRESH_VERIFIER) && (o.t_t1 != o.t_t || o.t_d1 != o.t_d))
    return bad(DSI_E_RANGE, "DSI_F_FRESH_VERIFIER does not support the TTFT variant");
  // every per-trial latency is <= N (k t_d + t_t) plus the first-forward surcharges
  // (kernel overflow bound)
  const unsigned __int128 kd = (unsigned __int128)c.lookahead * (uint64_t)o.t_d;
  const unsigned __int128 bound = (unsigned __int128)c.n_tokens * (kd + (uint64_t)o.t_t) +
                                  (uint64_t)std::max<int64_t>(0, o.t_t1 - o.t_t) +
                                  (uint64_t)std::max<int64_t>(0, o.t_d1 - o.t_d);
  if (bound >= ((unsigned __int128)1 << 31))
    return bad(DSI_E_OVERFLOW, "N*(k*t_drafter + t_target) must stay below 2^31 ticks");
  if ((unsigned __int128)c.n_trials * bound * bound >= ((unsigned __int128)1 << 64))
    return bad(DSI_E_OVERFLOW, "n_trials * bound^2 must stay below 2^64");
  o.kd = (int64_t)kd;
  if ((opt.flags & DSI_F_STRICT_EQ1) && ceil_div(o.t_t, o.kd) > c.sp_degree)
    return bad(DSI_E_STRICT_EQ1, "Eq. 1 violated: ceil(t_t/(k t_d)) > SP");
  o.a = c.accept_rate;
  o.ut = c.t_target;
  o.ud = c.t_drafter;
  o.eq1 = dsi_eq1_feasible(o.t_t, o.t_d, c.lookahead, c.sp_degree);
  o.min_k = dsi_min_lookahead(o.t_t, o.t_d, c.sp_degree);
  o.thr = (uint64_t)(c.accept_rate * 4294967296.0);  // exact: a * 2^32, then floor
  o.k = c.lookahead;
  o.sp = c.sp_degree;
  o.n = c.n_tokens;
  o.stream_id = c.stream_id;
  o.trials = c.n_trials;
  return DSI_OK;
}

// S(b) = b k t_d for every b: Eq. 1 holds at min(SP, N), or SP >= N (no thread ever waits).
bool config_noqueue(const CfgTicks &t) {
  const int32_t sp_eff = std::min(t.sp, t.n);
  return (t.t_t <= (int64_t)sp_eff * t.kd) || sp_eff >= t.n;
}

DevCfg make_dev_cfg(const CfgTicks &t, bool pattern, bool fresh) {
  DevCfg d{};
  uint32_t mode = dsi::MODE_STREAM;
  if (!pattern) {
    if (t.thr >= (1ull << 32)) mode = dsi::MODE_ALL_ACCEPT;
    else if (t.thr == 0) mode = dsi::MODE_ALL_REJECT;
  }
  const int32_t k_eff = std::min(t.k, t.n);
  const int32_t sp_eff = std::min(t.sp, t.n);
  const bool noqueue = config_noqueue(t);
  d.thr = (uint32_t)std::min<uint64_t>(t.thr, 0xffffffffull);
  const bool ttft = t.t_t1 != t.t_t || t.t_d1 != t.t_d;
  // fresh-verifier variant: with k t_d <= t_t a fresh forward never finishes sooner than
  // the regular thread (R24), so only k t_d > t_t configs take its cost table
  const bool fresh_cfg = fresh && t.kd > t.t_t;
  d.flags = mode | (noqueue ? dsi::CFG_NOQUEUE : 0u) | (ttft ? dsi::CFG_TTFT : 0u) |
            (fresh_cfg ? dsi::CFG_FRESH : 0u);
  d.t_d = (int32_t)t.t_d;
  d.k = t.k;
  if (t.eq1 == 1) d.flags |= dsi::CFG_EQ1;
  d.nonsi = (int32_t)(t.t_t1 + (int64_t)(t.n - 1) * t.t_t);
  d.e_si = (int32_t)((t.t_d1 - t.t_d) + (t.t_t1 - t.t_t));
  d.t_t1 = (int32_t)t.t_t1;
  d.ttft_shift = (int32_t)(t.t_d1 - t.t_d);
  d.n_tokens = t.n;
  d.k_eff = k_eff;
  d.sp_eff = sp_eff;
  d.t_t = (int32_t)t.t_t;
  d.kd = (int32_t)t.kd;
  d.si_cost = (int32_t)(t.kd + t.t_t);
  // S(1) = max(k t_d, (1 mod SP) k t_d + floor(1/SP) t_t): k t_d, or max(k t_d, t_t) if SP = 1
  d.s1 = (int32_t)(t.sp >= 2 ? t.kd : std::max(t.kd, t.t_t));
  d.stream_id = t.stream_id;
  uint32_t hi;
  magic((uint32_t)k_eff + 1u, d.m_si, hi);  // k_eff + 1 >= 2: hi == 0
  magic((uint32_t)k_eff, d.m_k_lo, d.m_k_hi);
  magic((uint32_t)sp_eff, d.m_sp_lo, d.m_sp_hi);
  d.n_trials = t.trials;
  return d;
}

// Relative cost of one trial-token: Philox (~10 instr) + compare (~1) + segment walk
// (~10 instr per rejection, expected (1-a) per token), SURVEY 8(d).4.
double unit_cost(const CfgTicks &t, uint64_t trials) {
  return (double)trials * (double)t.n * (11.0 + 10.0 * (1.0 - t.a));
}

// DSI_TRACE=1 in the environment: each API call prints its phases (host wall clock, ms)
// to stderr on return -- e.g. where dsi_sim_update's time goes.
class Trace {
 public:
  explicit Trace(const char *call) : call_(call), on_(enabled()) {
    if (on_) t0_ = last_ = std::chrono::steady_clock::now();
  }
  void mark(const char *phase) {
    if (!on_) return;
    const auto t = std::chrono::steady_clock::now();
    char b[96];
    std::snprintf(b, sizeof b, " %s=%.3f", phase, std::chrono::duration<double, std::milli>(t - last_).count());
    phases_ += b;
    last_ = t;
  }
  ~Trace() {
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
void parallel_for(size_t n, Fn fn, size_t min_parallel = (1u << 15)) {
  WorkerPool &pool = WorkerPool::get();
  if (n < min_parallel || n < 2 || pool.threads() == 1) {
    fn((size_t)0, n);
    return;
  }
  const size_t chunks = std::min(n, pool.threads() * 4);
  const std::function<void(size_t)> job = [&](size_t c) { fn(n * c / chunks, n * (c + 1) / chunks); };
  pool.run((uint32_t)chunks, job);
}

// Validate every config into ticks; on failure h->err names the first bad config.
// Validate every config into `out`; on failure h->err names the first bad config.  With
// `prev` (dsi_sim_update), also checks what an update must keep: n_trials, and with
// DSI_F_HIST min(k, N) (the histogram layout).
dsi_status validate_all(dsi_sim *h, const dsi_config *cfg, size_t n, std::vector<CfgTicks> &out,
                        const std::vector<CfgTicks> *prev = nullptr) {
  std::mutex mu;
  size_t bad = n;
  dsi_status bad_s = DSI_OK;
  std::string bad_msg;
  const bool hist = h->opt.flags & DSI_F_HIST;
  parallel_for(n, [&](size_t b, size_t e) {
    for (size_t i = b; i < e; ++i) {
      std::string msg;
      dsi_status s = convert(h->opt, cfg[i], i, out[i], msg);
      if (s == DSI_OK && prev) {
        const CfgTicks &o = (*prev)[i], &t = out[i];
        if (t.trials != o.trials || (hist && std::min(t.k, t.n) != std::min(o.k, o.n))) {
          s = DSI_E_RANGE;
          msg = "config " + std::to_string(i) + ": n_trials (and, with DSI_F_HIST, min(k, N)) must not change";
        }
      }
      if (s != DSI_OK) {
        std::lock_guard<std::mutex> lock(mu);
        if (i < bad) {
          bad = i;
          bad_s = s;
          bad_msg = msg;
        }
        return;
      }
    }
  });
  if (bad < n) return fail(h, bad_s, bad_msg);
  return DSI_OK;
}

// Fill the pinned device-config staging table from h->ticks.
void fill_dev_cfg(dsi_sim *h) {
  const bool pattern = h->opt.flags & DSI_F_PATTERN;
  const bool fresh = h->opt.flags & DSI_F_FRESH_VERIFIER;
  const size_t n = h->n_cfg;
  // prefix offsets (per-trial records, SI-histogram bins) in two passes over fixed chunks
  constexpr size_t K = 64;
  uint64_t rec[K + 1] = {}, sib[K + 1] = {};
  parallel_for(K, [&](size_t b, size_t e) {
    for (size_t c = b; c < e; ++c) {
      uint64_t r = 0, q = 0;  // in registers: the neighbouring chunks' sums share cache lines
      for (size_t i = n * c / K; i < n * (c + 1) / K; ++i) {
        r += h->ticks[i].trials;
        q += (uint64_t)std::min(h->ticks[i].k, h->ticks[i].n) + 1;
      }
      rec[c + 1] = r;
      sib[c + 1] = q;
    }
  }, 1);
  for (size_t c = 0; c < K; ++c) {
    rec[c + 1] += rec[c];
    sib[c + 1] += sib[c];
  }
  parallel_for(K, [&](size_t b, size_t e) {
    for (size_t c = b; c < e; ++c) {
      uint64_t r = rec[c], q = sib[c];
      for (size_t i = n * c / K; i < n * (c + 1) / K; ++i) {
        DevCfg &d = h->dev_cfg.p[i];
        d = make_dev_cfg(h->ticks[i], pattern, fresh);
        d.rec_off = r;
        r += h->ticks[i].trials;
        d.si_hist_off = (uint32_t)q;
        q += (uint64_t)d.k_eff + 1;
      }
    }
  }, 1);
}

void free_device(DeviceState &d) {
  if (d.ordinal < 0) return;
  cudaSetDevice(d.ordinal);
  if (d.comm && nccl().ok) nccl().CommDestroy(d.comm);
  cudaFree(d.d_cfg);
  cudaFree(d.d_prefix);
  cudaFree(d.d_acc);
  cudaFree(d.d_red);
  cudaFree(d.d_seg);
  cudaFree(d.d_seg_red);
  cudaFree(d.d_si);
  cudaFree(d.d_si_red);
  cudaFree(d.d_rec);
  cudaFree(d.d_perm);
  cudaFree(d.d_groups);
  cudaFree(d.d_crn_units);
  cudaFree(d.d_records);
  cudaFree(d.d_group_tile0);
  cudaFree(d.d_tiles);
  cudaFree(d.d_heat_cells);
  cudaFree(d.d_heat_out);
  cudaFree(d.d_heat_bad);
  cudaFree(d.d_seg_groups);
  cudaFree(d.d_seg_prefix);
  cudaFree(d.d_cfg_group);
  cudaFree(d.d_hist);
  cudaFree(d.d_ttft_cfgs);
  if (d.ev0) cudaEventDestroy(d.ev0);
  if (d.ev1) cudaEventDestroy(d.ev1);
  if (d.own_stream && d.stream) cudaStreamDestroy(d.stream);
  d = DeviceState{};
}

void free_handle(dsi_sim *h) {
  for (auto &d : h->dev) free_device(d);
  h->dev_cfg.release();
  h->host_acc.release();
  h->host_seg.release();
  h->host_si.release();
  h->heat_out.release();
  h->host_bad.release();
  for (auto &ev : h->chunk_ev)
    if (ev) cudaEventDestroy(ev);
  delete h;
}

// Upload the staging table to every device (async on each device's stream).
dsi_status upload(dsi_sim *h, bool plan = true) {
  for (auto &d : h->dev) {
    CUDA_TRY(h, cudaSetDevice(d.ordinal));
    CUDA_TRY(h, cudaMemcpyAsync(d.d_cfg, h->dev_cfg.p, h->n_cfg * sizeof(DevCfg),
                                cudaMemcpyHostToDevice, d.stream));
    if (h->means_only && plan) {
      CUDA_TRY(h, cudaMemcpyAsync(d.d_seg_groups, h->seg_groups.data(), h->seg_groups.size() * sizeof(dsi::SegGroup),
                                  cudaMemcpyHostToDevice, d.stream));
      CUDA_TRY(h, cudaMemcpyAsync(d.d_seg_prefix, h->seg_prefix.data(), h->seg_prefix.size() * sizeof(uint64_t),
                                  cudaMemcpyHostToDevice, d.stream));
      CUDA_TRY(h, cudaMemcpyAsync(d.d_cfg_group, h->cfg_group.data(), h->cfg_group.size() * sizeof(uint32_t),
                                  cudaMemcpyHostToDevice, d.stream));
      if (!h->ttft_cfgs.empty())
        CUDA_TRY(h, cudaMemcpyAsync(d.d_ttft_cfgs, h->ttft_cfgs.data(), h->ttft_cfgs.size() * sizeof(uint32_t),
                                    cudaMemcpyHostToDevice, d.stream));
      CUDA_TRY(h, cudaStreamSynchronize(d.stream));
    }
    if (h->shared && plan) {  // the shared-stream plan (unchanged by an update that keeps its keys)
      CUDA_TRY(h, cudaMemcpyAsync(d.d_perm, h->perm.data(), h->perm.size() * sizeof(uint32_t),
                                  cudaMemcpyHostToDevice, d.stream));
      CUDA_TRY(h, cudaMemcpyAsync(d.d_groups, h->groups.data(), h->groups.size() * sizeof(dsi::CrnGroup),
                                  cudaMemcpyHostToDevice, d.stream));
      CUDA_TRY(h, cudaMemcpyAsync(d.d_crn_units, h->crn_units.data(),
                                  h->crn_units.size() * sizeof(dsi::CrnUnit), cudaMemcpyHostToDevice,
                                  d.stream));
      if (h->two_pass) {
        CUDA_TRY(h, cudaMemcpyAsync(d.d_group_tile0, h->group_tile0.data(), h->group_tile0.size() * sizeof(uint64_t),
                                    cudaMemcpyHostToDevice, d.stream));
        if (!d.tiles.empty())
          CUDA_TRY(h, cudaMemcpyAsync(d.d_tiles, d.tiles.data(), d.tiles.size() * sizeof(dsi::CrnTile),
                                      cudaMemcpyHostToDevice, d.stream));
      }
      CUDA_TRY(h, cudaStreamSynchronize(d.stream));  // the host vectors are pageable and may change
    }
  }
  return DSI_OK;
}

// Shared-stream plan: group configs by (stream_id, threshold, N, n_trials) -- equal keys
// draw identical indicators -- ordered lookahead-major inside a group (so the lanes of a
// warp mostly share k), then cut each group into slices of cfg_per_block configs.
// Launch-shape limits that follow from the configs (max N, max min(k, N), TTFT present),
// and the shared-memory bounds they imply.  Called by create and again by update, whose
// new configs may change them (the kernels size shared memory from these values).
// Means-only plan: groups of configs with equal (stream_id, threshold, N, n_trials) -- they
// draw identical indicators -- each with its segment-length histogram; histogram units are
// (group, tile of tile_trials trials).  cost[u] feeds the sharder.
dsi_status plan_means(dsi_sim *h, std::vector<double> &cost, uint64_t target_units) {
  const size_t n = h->n_cfg;
  std::vector<uint32_t> order(n);
  for (size_t i = 0; i < n; ++i) order[i] = (uint32_t)i;
  auto key = [&](uint32_t i) {
    const CfgTicks &t = h->ticks[i];
    return std::make_tuple(t.stream_id, t.thr, t.n, t.trials);
  };
  std::stable_sort(order.begin(), order.end(), [&](uint32_t a, uint32_t b) { return key(a) < key(b); });
  h->seg_groups.clear();
  h->cfg_group.assign(n, 0u);
  uint64_t off = 0, trials = 0;
  for (size_t i = 0; i < n;) {
    size_t j = i + 1;
    while (j < n && key(order[j]) == key(order[i])) ++j;
    const CfgTicks &t = h->ticks[order[i]];
    dsi::SegGroup g{};
    g.n_trials = t.trials;
    g.hist_off = off;
    g.n_tokens = t.n;
    g.stream_id = t.stream_id;
    g.thr = (uint32_t)std::min<uint64_t>(t.thr, 0xffffffffull);
    g.mode = t.thr >= (1ull << 32) ? dsi::MODE_ALL_ACCEPT : (t.thr == 0 ? dsi::MODE_ALL_REJECT : dsi::MODE_STREAM);
    for (size_t q = i; q < j; ++q) h->cfg_group[order[q]] = (uint32_t)h->seg_groups.size();
    h->seg_groups.push_back(g);
    off += (uint64_t)t.n + 1;
    trials += t.trials;
    i = j;
  }
  h->hist_len = off;
  h->ttft_cfgs.clear();
  for (size_t i = 0; i < n; ++i)
    if (h->ticks[i].t_t1 != h->ticks[i].t_t || h->ticks[i].t_d1 != h->ticks[i].t_d) h->ttft_cfgs.push_back((uint32_t)i);
  // tiles: multiples of 128 trials, enough units to fill the devices
  uint64_t r = trials / (128ull * std::max<uint64_t>(1, target_units));
  r = std::min<uint64_t>(128, std::max<uint64_t>(1, r));
  h->tile_trials = (uint32_t)(128 * r);
  h->seg_prefix.assign(h->seg_groups.size() + 1, 0);
  for (size_t gi = 0; gi < h->seg_groups.size(); ++gi)
    h->seg_prefix[gi + 1] = h->seg_prefix[gi] + (h->seg_groups[gi].n_trials + h->tile_trials - 1) / h->tile_trials;
  h->total_units = h->seg_prefix.back();
  cost.assign(h->total_units, 0.0);
  for (size_t gi = 0; gi < h->seg_groups.size(); ++gi) {
    const dsi::SegGroup &g = h->seg_groups[gi];
    const double a = (double)g.thr / 4294967296.0;
    for (uint64_t u = h->seg_prefix[gi]; u < h->seg_prefix[gi + 1]; ++u) {
      const uint64_t t0 = (u - h->seg_prefix[gi]) * h->tile_trials;
      const double tr = (double)std::min<uint64_t>(h->tile_trials, g.n_trials - t0);
      cost[u] = tr * (double)g.n_tokens * (g.mode == dsi::MODE_STREAM ? 11.0 + 10.0 * (1.0 - a) : 1.0);
    }
  }
  return DSI_OK;
}

dsi_status derive_limits(dsi_sim *h, const std::vector<CfgTicks> &ticks) {
  struct Lim {
    int32_t max_n = 1, max_keff = 1;
    bool ttft = false, fresh = false;
    double work = 0.0, work_k1 = 0.0;  // trial-tokens in all configs / in k = 1 configs without queueing
  } lim;
  std::mutex mu;
  const bool fresh = h->opt.flags & DSI_F_FRESH_VERIFIER;
  parallel_for(ticks.size(), [&](size_t b, size_t e) {
    Lim l;
    for (size_t i = b; i < e; ++i) {
      const CfgTicks &t = ticks[i];
      l.max_n = std::max(l.max_n, t.n);
      l.max_keff = std::max(l.max_keff, std::min(t.k, t.n));
      l.ttft = l.ttft || t.t_t1 != t.t_t || t.t_d1 != t.t_d;
      l.fresh = l.fresh || (fresh && t.kd > t.t_t);
      const double w = (double)t.trials * (double)t.n;
      l.work += w;
      if (std::min(t.k, t.n) == 1 && config_noqueue(t)) l.work_k1 += w;
    }
    std::lock_guard<std::mutex> lock(mu);
    lim.max_n = std::max(lim.max_n, l.max_n);
    lim.max_keff = std::max(lim.max_keff, l.max_keff);
    lim.ttft = lim.ttft || l.ttft;
    lim.fresh = lim.fresh || l.fresh;
    lim.work += l.work;
    lim.work_k1 += l.work_k1;
  });
  if (lim.ttft && lim.max_n > 4096) return fail(h, DSI_E_RANGE, "the TTFT variant supports n_tokens <= 4096");
  if (dsi::trial_kernel_smem(lim.max_n, lim.max_keff, h->opt.flags & DSI_F_HIST, lim.ttft) > 200 * 1024)
    return fail(h, DSI_E_RANGE, "DSI_F_HIST needs (64 + k + 1) * 4 bytes of shared memory <= 200 KiB");
  if (h->shared && lim.max_n > kCrnMaxN)
    return fail(h, DSI_E_RANGE, "DSI_F_SHARED_STREAMS supports n_tokens <= " + std::to_string(kCrnMaxN));
  h->max_n = lim.max_n;
  h->max_keff = lim.max_keff;
  h->any_ttft = lim.ttft;
  h->any_fresh = lim.fresh;
  // the k = 1 fast path (dsi_kernel.cu, VAR 3) pays for its extra code only when such configs carry
  // a good share of the work (measured: config 5, 86% of its configs, -14%; config 3, 0.5%, +2% if on)
  h->k1_fast = !lim.ttft && !lim.fresh && lim.work_k1 >= 0.25 * lim.work;
  if (const char *f = std::getenv("DSI_K1_FAST")) h->k1_fast = !lim.ttft && !lim.fresh && std::atoi(f) != 0;
  return DSI_OK;
}

// The shared-stream plan orders configs by these fields (plan_shared): an update that
// keeps all of them keeps the plan.
bool same_plan_keys(const std::vector<CfgTicks> &a, const std::vector<CfgTicks> &b) {
  std::atomic<bool> same{true};
  parallel_for(a.size(), [&](size_t lo, size_t hi) {
    for (size_t i = lo; i < hi && same.load(std::memory_order_relaxed); ++i) {
      const CfgTicks &x = a[i], &y = b[i];
      if (x.stream_id != y.stream_id || x.thr != y.thr || x.n != y.n || x.trials != y.trials || x.k != y.k ||
          x.t_t != y.t_t || x.t_d != y.t_d || x.sp != y.sp)
        same = false;
    }
  });
  return same;
}

// Sum the per-config moments (and, with hist, the histograms) over every device of
// every rank: one grouped ncclAllReduce into the *_red buffers.  No-op on one device.
dsi_status sum_across(dsi_sim *h, bool hist) {
  if (!h->use_nccl) return DSI_OK;
  const size_t n_cfg = h->n_cfg;
  if (h->host_coll) {
    DeviceState &d = h->dev[0];
    dsi_status st = host_allreduce(h, d.stream, d.d_acc, d.d_red, n_cfg * dsi::NF);
    if (st == DSI_OK && hist) st = host_allreduce(h, d.stream, d.d_seg, d.d_seg_red, n_cfg * 64);
    if (st == DSI_OK && hist) st = host_allreduce(h, d.stream, d.d_si, d.d_si_red, h->si_bins_total);
    return st;
  }
  NcclApi &api = nccl();
  ncclResult_t r = api.GroupStart();
  for (auto &d : h->dev) {
    if (r != ncclSuccess) break;
    cudaSetDevice(d.ordinal);
    r = api.AllReduce(d.d_acc, d.d_red, n_cfg * dsi::NF, ncclUint64, ncclSum, d.comm, d.stream);
    if (r == ncclSuccess && hist) {
      r = api.AllReduce(d.d_seg, d.d_seg_red, n_cfg * 64, ncclUint64, ncclSum, d.comm, d.stream);
      if (r == ncclSuccess)
        r = api.AllReduce(d.d_si, d.d_si_red, h->si_bins_total, ncclUint64, ncclSum, d.comm, d.stream);
    }
  }
  const ncclResult_t r2 = api.GroupEnd();
  if (r != ncclSuccess || r2 != ncclSuccess)
    return fail(h, DSI_E_COMM, std::string("ncclAllReduce: ") + api.GetErrorString(r != ncclSuccess ? r : r2));
  return DSI_OK;
}

// Two-pass shared-stream mode (dsi_crn2.cu): records of (group, tile of TH trials), and
// for every device the tiles its units read (pass 1 writes exactly those).  Requires
// h->crn_units and the devices' unit ranges.
dsi_status plan_two_pass(dsi_sim *h) {
  const int th = h->cfg_per_block;
  h->two_pass = th == 256 && dsi::crn_eval_smem(h->max_runs, th) <= 76 * 1024;
  if (const char *force = std::getenv("DSI_CRN_TWO_PASS"))  // developer A/B runs only
    h->two_pass = h->two_pass && std::atoi(force) != 0;
  if (!h->two_pass) return DSI_OK;
  try {
    h->rec_bytes = (uint32_t)dsi::crn_record_bytes(h->max_runs, th);
    h->group_tile0.assign(h->groups.size() + 1, 0);
    for (size_t g = 0; g < h->groups.size(); ++g)
      h->group_tile0[g + 1] = h->group_tile0[g] + (h->groups[g].n_trials + th - 1) / th;
    h->total_records = h->group_tile0.back();
    for (auto &d : h->dev) {
      std::vector<char> seen(h->total_records, 0);
      d.tiles.clear();
      for (const auto &rg : d.ranges)
        for (uint64_t u = rg.first; u < rg.second; ++u) {
          const dsi::CrnUnit &un = h->crn_units[u];
          for (uint64_t t = un.t0 / th; t * th < un.t1; ++t) {
            const uint64_t r = h->group_tile0[un.group] + t;
            if (!seen[r]) {
              seen[r] = 1;
              d.tiles.push_back(dsi::CrnTile{un.group, (uint32_t)t});
            }
          }
        }
    }
  } catch (...) {
    return fail(h, DSI_E_NOMEM, "two-pass plan");
  }
  return DSI_OK;
}

// Device buffers of the two-pass mode (sized by plan_two_pass; grown if an update needs more).
dsi_status alloc_two_pass(dsi_sim *h) {
  if (!h->two_pass) return DSI_OK;
  for (auto &d : h->dev) {
    CUDA_TRY(h, cudaSetDevice(d.ordinal));
    if (h->total_records > d.records_cap || !d.d_records) {
      cudaFree(d.d_records);
      cudaFree(d.d_group_tile0);
      d.d_records = nullptr;
      d.d_group_tile0 = nullptr;
      CUDA_TRY(h, cudaMalloc((void **)&d.d_records, std::max<uint64_t>(1, h->total_records) * h->rec_bytes));
      CUDA_TRY(h, cudaMalloc((void **)&d.d_group_tile0, h->group_tile0.size() * sizeof(uint64_t)));
      d.records_cap = h->total_records;
    }
    if (d.tiles.size() > d.tiles_cap) {
      cudaFree(d.d_tiles);
      d.d_tiles = nullptr;
      CUDA_TRY(h, cudaMalloc((void **)&d.d_tiles, d.tiles.size() * sizeof(dsi::CrnTile)));
      d.tiles_cap = d.tiles.size();
    }
  }
  return DSI_OK;
}

dsi_status plan_shared(dsi_sim *h, std::vector<double> &cost) {
  const size_t n = h->n_cfg;
  try {
    h->perm.resize(n);
    for (size_t i = 0; i < n; ++i) h->perm[i] = (uint32_t)i;
    const auto &t = h->ticks;
    std::stable_sort(h->perm.begin(), h->perm.end(), [&](uint32_t a, uint32_t b) {
      const CfgTicks &x = t[a], &y = t[b];
      if (x.stream_id != y.stream_id) return x.stream_id < y.stream_id;
      if (x.thr != y.thr) return x.thr < y.thr;
      if (x.n != y.n) return x.n < y.n;
      if (x.trials != y.trials) return x.trials < y.trials;
      if (x.k != y.k) return x.k < y.k;
      if (x.t_t != y.t_t) return x.t_t < y.t_t;
      if (x.t_d != y.t_d) return x.t_d < y.t_d;
      return x.sp < y.sp;
    });
    h->max_runs = h->max_n / 3 + 2;  // runs of >= 2 accepted drafts in one trial
    // groups first, then the block shape: configs per block follow the typical group size
    h->groups.clear();
    for (size_t i = 0; i < n;) {
      const CfgTicks &k0 = t[h->perm[i]];
      size_t j = i + 1;
      while (j < n) {
        const CfgTicks &kj = t[h->perm[j]];
        if (kj.stream_id != k0.stream_id || kj.thr != k0.thr || kj.n != k0.n || kj.trials != k0.trials) break;
        ++j;
      }
      dsi::CrnGroup g{};
      g.first = (uint32_t)i;
      g.count = (uint32_t)(j - i);
      g.n_tokens = k0.n;
      g.stream_id = k0.stream_id;
      g.thr = (uint32_t)std::min<uint64_t>(k0.thr, 0xffffffffull);
      g.mode = k0.thr >= (1ull << 32) ? dsi::MODE_ALL_ACCEPT : (k0.thr == 0 ? dsi::MODE_ALL_REJECT : dsi::MODE_STREAM);
      g.n_trials = k0.trials;
      h->groups.push_back(g);
      i = j;
    }
    // one config per thread, one trial per thread per tile; 256-thread blocks halve the
    // phase-1 (Philox) passes per trial of a group -- worth it when groups are large (>= 256
    // configs on average) and the shared memory still leaves room for 4 blocks per SM; else
    // 128 (profiles/r01_ab_crn_th.jsonl: cfg3 30.5 -> 26.0 ms; forced on cfg2/cfg4/cfg5, whose
    // groups hold 3 / 140 / 100 configs, 1.8-1.9x slower; 2 or 4 configs per thread were
    // slower too, profiles/r01_ab_crn*.jsonl)
    const bool big_groups = n >= 256 * h->groups.size();
    int th = (big_groups && dsi::crn_kernel_smem(h->max_n, 256, 256, h->max_runs) <= 48 * 1024) ? 256 : kCrnThreads;
    if (const char *force = std::getenv("DSI_CRN_THREADS")) {  // developer A/B runs only
      const int f = std::atoi(force);
      if (f == 128 || f == 256) th = f;
    }
    h->cfg_per_block = th;
    h->block_threads = th;
    // units: (group, slice of cfg_per_block configs, range of trials); trials are split
    // until there are enough blocks to fill every SM of every device a few times.  With
    // 128-thread blocks a group's configs are first cut into maximal runs of "sums-only"
    // configs (k_eff = 1 and no queueing: every run of >= 2 accepted drafts is long and
    // the corrections are linear in per-trial sums, no run list needed) and the others;
    // sums-only units go first and run a kernel variant without run lists in shared memory
    // (so many more blocks fit an SM; large N, e.g. config 5, gains most).
    const bool split_sums = th == kCrnThreads && !std::getenv("DSI_CRN_NO_SUMS_SPLIT");
    auto sums_only = [&](uint32_t pos) {
      const CfgTicks &c = t[h->perm[pos]];
      return split_sums && std::min(c.k, c.n) == 1 && config_noqueue(c);
    };
    struct Slice {
      uint32_t group, begin, count;
      bool sums;
    };
    std::vector<Slice> slices_v;
    for (uint32_t gi = 0; gi < h->groups.size(); ++gi) {
      const dsi::CrnGroup &g = h->groups[gi];
      for (uint32_t b = g.first; b < g.first + g.count;) {
        const bool kind = sums_only(b);
        uint32_t e = b + 1;
        while (e < g.first + g.count && e - b < (uint32_t)th && sums_only(e) == kind) ++e;
        slices_v.push_back(Slice{gi, b, e - b, kind});
        b = e;
      }
    }
    const size_t slices = slices_v.size();
    const int total_devices = h->opt.world * h->opt.n_devices;
    const uint64_t target = 148ull * 4 * 4 * (uint64_t)total_devices;
    const uint64_t split = std::max<uint64_t>(1, (target + slices - 1) / slices);
    h->crn_units.clear();
    cost.clear();
    h->n_sums_units = 0;
    h->max_runs_normal = 1;
    for (int pass = 0; pass < 2; ++pass) {  // sums-only units first
      for (const Slice &sl : slices_v) {
        if (sl.sums != (pass == 0)) continue;
        const dsi::CrnGroup &g = h->groups[sl.group];
        const uint64_t tiles = (g.n_trials + th - 1) / th;
        const uint64_t nchunks = std::min<uint64_t>(split, tiles);
        for (uint64_t c = 0; c < nchunks; ++c) {
          dsi::CrnUnit u{};
          u.group = sl.group;
          u.begin = sl.begin;
          u.count = sl.count;
          u.kind = sl.sums ? 1u : 0u;
          u.t0 = (tiles * c / nchunks) * th;
          u.t1 = std::min<uint64_t>((tiles * (c + 1) / nchunks) * th, g.n_trials);
          h->crn_units.push_back(u);
          if (sl.sums) ++h->n_sums_units;
          else {  // stored runs have L > the slice's smallest k_eff: each takes >= kmin + 2 positions
            int32_t kmin = 1 << 30;
            for (uint32_t q = sl.begin; q < sl.begin + sl.count; ++q)
              kmin = std::min(kmin, std::min(t[h->perm[q]].k, t[h->perm[q]].n));
            h->max_runs_normal = std::max<int32_t>(h->max_runs_normal, (g.n_tokens - 1) / (kmin + 2) + 1);
          }
          // phase 1 (one stream pass per trial) + phase 2 (each config on every trial)
          cost.push_back((double)(u.t1 - u.t0) * ((double)g.n_tokens * 12.0 + (double)sl.count * 25.0));
        }
      }
    }
  } catch (...) {
    return fail(h, DSI_E_NOMEM, "shared-stream plan");
  }
  h->total_units = h->crn_units.size();
  return DSI_OK;
}

}  // namespace

// ============================================================================= C ABI
// Heatmap cells: maximal runs of consecutive configs with equal (t_target, t_drafter, a, SP, N).
static void plan_heat_cells(dsi_sim *h) {
  h->heat_cells.clear();
  const auto &t = h->ticks;
  for (size_t i = 0; i < h->n_cfg;) {
    size_t j = i + 1;
    while (j < h->n_cfg && t[j].ut == t[i].ut && t[j].ud == t[i].ud && t[j].a == t[i].a && t[j].sp == t[i].sp &&
           t[j].n == t[i].n)
      ++j;
    h->heat_cells.push_back(dsi::HeatCell{(uint64_t)i, (uint32_t)(j - i), 0u});
    i = j;
  }
}

// Means-only, one device per process: every part's config range starts at a cell, so each
// part's cells can be evaluated from its own moments (no all-reduce of the moments).
static bool cells_aligned(const dsi_sim *h) {
  if (!h->means_only || h->opt.n_devices != 1 || h->cfg_bounds.empty()) return false;
  size_t ci = 0;
  for (const uint64_t b : h->cfg_bounds) {
    while (ci < h->heat_cells.size() && h->heat_cells[ci].first < b) ++ci;
    if (b < h->n_cfg && (ci == h->heat_cells.size() || h->heat_cells[ci].first != b)) return false;
  }
  return true;
}

extern "C" {

uint32_t dsi_abi_version(void) { return DSI_ABI_VERSION; }

const char *dsi_status_str(dsi_status s) {
  switch (s) {
    case DSI_OK: return "DSI_OK";
    case DSI_E_NULL: return "DSI_E_NULL: required pointer was NULL";
    case DSI_E_RANGE: return "DSI_E_RANGE: argument out of range";
    case DSI_E_TICK: return "DSI_E_TICK: latency is not a whole number of ticks";
    case DSI_E_OVERFLOW: return "DSI_E_OVERFLOW: tick sums would overflow";
    case DSI_E_STRICT_EQ1: return "DSI_E_STRICT_EQ1: Eq. 1 violated under DSI_F_STRICT_EQ1";
    case DSI_E_DEVICE: return "DSI_E_DEVICE: CUDA error or missing sm_100 device";
    case DSI_E_COMM: return "DSI_E_COMM: NCCL error";
    case DSI_E_STATE: return "DSI_E_STATE: call order violated";
    case DSI_E_NOMEM: return "DSI_E_NOMEM: allocation failed";
  }
  return "unknown dsi_status";
}

const char *dsi_sim_last_error(const dsi_sim *h) { return h ? h->err.c_str() : ""; }
const char *dsi_last_create_error(void) { return g_create_error.c_str(); }

int32_t dsi_eq1_feasible(int64_t t_t, int64_t t_d, int32_t k, int32_t sp) {
  if (t_t < 1 || t_d < 1 || k < 1 || sp < 1) return -1;
  return ceil_div(t_t, (int64_t)k * t_d) <= sp ? 1 : 0;
}

int32_t dsi_min_lookahead(int64_t t_t, int64_t t_d, int32_t sp) {
  if (t_t < 1 || t_d < 1 || sp < 1) return -1;
  // smallest k with ceil(t_t/(k t_d)) <= sp  <=>  k t_d sp >= t_t
  const int64_t k = ceil_div(t_t, t_d * (int64_t)sp);
  return (int32_t)std::max<int64_t>(1, k);
}

int32_t dsi_required_processors(int64_t t_t, int64_t t_d, int32_t k) {
  if (t_t < 1 || t_d < 1 || k < 1) return -1;
  return (int32_t)(1 + ceil_div(t_t, (int64_t)k * t_d));
}

dsi_status dsi_shard_bounds(const double *cost, uint64_t n, int32_t parts, uint64_t *bounds) {
  if (!bounds || (!cost && n)) return DSI_E_NULL;
  if (parts < 1) return DSI_E_RANGE;
  double total = 0.0;
  for (uint64_t i = 0; i < n; ++i) {
    if (!(cost[i] >= 0.0)) return DSI_E_RANGE;
    total += cost[i];
  }
  bounds[0] = 0;
  uint64_t i = 0;
  double run = 0.0;
  for (int32_t j = 1; j < parts; ++j) {
    const double target = total * (double)j / (double)parts;
    // advance while taking unit i keeps the prefix closer to the target
    while (i < n && run + 0.5 * cost[i] <= target) run += cost[i++];
    bounds[j] = i;
  }
  bounds[parts] = n;
  return DSI_OK;
}

dsi_status dsi_nccl_unique_id(uint8_t id[128]) {
  if (!id) return DSI_E_NULL;
  NcclApi &api = nccl();
  if (!api.ok) return DSI_E_COMM;
  ncclUniqueId u;
  if (api.GetUniqueId(&u) != ncclSuccess) return DSI_E_COMM;
  static_assert(sizeof(u) == 128, "ncclUniqueId is 128 bytes");
  std::memcpy(id, &u, 128);
  return DSI_OK;
}

dsi_status dsi_sim_create(const dsi_options *opt, const dsi_config *cfg, size_t n_cfg,
                          dsi_sim **out) {
  Trace tr("dsi_sim_create");
  g_create_error.clear();
  if (!out) return fail(nullptr, DSI_E_NULL, "out is NULL");
  *out = nullptr;
  if (!opt || !cfg) return fail(nullptr, DSI_E_NULL, "opt or cfg is NULL");
  if (opt->abi_version != DSI_ABI_VERSION) return fail(nullptr, DSI_E_RANGE, "abi_version mismatch");
  if (n_cfg == 0 || n_cfg >= (1ull << 31)) return fail(nullptr, DSI_E_RANGE, "n_cfg out of range");
  if (!(std::isfinite(opt->tick) && opt->tick > 0.0)) return fail(nullptr, DSI_E_RANGE, "tick must be > 0");
  const uint32_t known = DSI_F_PER_TRIAL | DSI_F_HIST | DSI_F_PATTERN | DSI_F_STRICT_EQ1 | DSI_F_TIMING |
                         DSI_F_SHARED_STREAMS | DSI_F_FRESH_VERIFIER | DSI_F_MEANS_ONLY |
                         DSI_F_REDUCE_TO_ROOT;
  if (opt->flags & ~known) return fail(nullptr, DSI_E_RANGE, "unknown flag");
  if (opt->n_devices < 1 || opt->n_devices > 8) return fail(nullptr, DSI_E_RANGE, "n_devices must be 1..8");
  if (opt->world < 1 || opt->rank < 0 || opt->rank >= opt->world)
    return fail(nullptr, DSI_E_RANGE, "need 0 <= rank < world");
  if (opt->device < 0) return fail(nullptr, DSI_E_RANGE, "device must be >= 0");
  if (opt->n_shards < 0 || opt->n_shards > 4096) return fail(nullptr, DSI_E_RANGE, "n_shards out of range");
  if (opt->n_shards > 1 && (opt->n_devices > 1 || opt->world > 1))
    return fail(nullptr, DSI_E_RANGE, "n_shards > 1 is single-device only");
  if (opt->block_threads != 0 &&
      (opt->block_threads < 32 || opt->block_threads > 128 || opt->block_threads % 32))
    return fail(nullptr, DSI_E_RANGE, "block_threads must be a multiple of 32 in [32, 128]");
  const int total_devices = opt->world * opt->n_devices;
  const bool host_coll = g_host_ar != nullptr && opt->world > 1;
  if (host_coll && opt->n_devices != 1)
    return fail(nullptr, DSI_E_RANGE, "the host all-reduce hook needs one device per process");
  if (total_devices > 1 && !opt->nccl_id && !host_coll)
    return fail(nullptr, DSI_E_NULL, "nccl_id is required when world*n_devices > 1");
  // NCCL whenever several devices take part, or when the caller passes an id for a
  // one-rank communicator (exercises the collective path on one GPU)
  const bool use_nccl = total_devices > 1 || opt->nccl_id != nullptr;
  const bool per_trial = opt->flags & DSI_F_PER_TRIAL;
  if (per_trial && total_devices > 1)
    return fail(nullptr, DSI_E_RANGE, "DSI_F_PER_TRIAL needs a single device and world == 1");
  const bool shared = opt->flags & DSI_F_SHARED_STREAMS;
  if (shared && (opt->flags & (DSI_F_PER_TRIAL | DSI_F_HIST | DSI_F_PATTERN | DSI_F_FRESH_VERIFIER)))
    return fail(nullptr, DSI_E_RANGE,
                "DSI_F_SHARED_STREAMS excludes PER_TRIAL, HIST, PATTERN and FRESH_VERIFIER");

  const bool means_only = opt->flags & DSI_F_MEANS_ONLY;
  if (means_only && (opt->flags & (DSI_F_PER_TRIAL | DSI_F_HIST | DSI_F_PATTERN | DSI_F_SHARED_STREAMS)))
    return fail(nullptr, DSI_E_RANGE, "DSI_F_MEANS_ONLY excludes PER_TRIAL, HIST, PATTERN and SHARED_STREAMS");

  dsi_sim *h = new (std::nothrow) dsi_sim;
  if (!h) return fail(nullptr, DSI_E_NOMEM, "handle allocation");
  auto abort_create = [&](dsi_status s) {
    g_create_error = h->err;
    free_handle(h);
    return s;
  };
  h->opt = *opt;
  h->opt.nccl_id = nullptr;
  h->n_cfg = n_cfg;
  h->shared = shared;
  h->means_only = means_only;
  h->use_nccl = use_nccl;
  h->host_coll = host_coll;
  h->block_threads = shared ? kCrnThreads : (opt->block_threads ? opt->block_threads : kDefaultThreads);
  try {
    h->ticks.resize(n_cfg);
    h->prefix.resize(n_cfg + 1);
  } catch (...) {
    h->err = "host tables";
    return abort_create(DSI_E_NOMEM);
  }

  // ---- validation and tick conversion (before any device work)
  dsi_status s = validate_all(h, cfg, n_cfg, h->ticks);
  if (s != DSI_OK) return abort_create(s);
  uint64_t sib = 0;
  for (size_t i = 0; i < n_cfg; ++i) {
    h->total_trials += h->ticks[i].trials;
    sib += (uint64_t)std::min(h->ticks[i].k, h->ticks[i].n) + 1;
  }
  if (per_trial && h->total_trials > (1ull << 31)) {
    h->err = "DSI_F_PER_TRIAL supports at most 2^31 trials in total";
    return abort_create(DSI_E_RANGE);
  }
  if (sib >= (1ull << 32)) {
    h->err = "too many SI histogram bins";
    return abort_create(DSI_E_RANGE);
  }
  h->si_bins_total = sib;
  s = derive_limits(h, h->ticks);
  if (s != DSI_OK) return abort_create(s);
  tr.mark("validate+limits");

  // ---- work units: (config, tile of tile_trials trials), or shared-stream (group, config slice)
  std::vector<double> crn_cost;
  if (means_only) {
    if (h->max_n > kMeansMaxN) {
      h->err = "DSI_F_MEANS_ONLY: N too large";
      return abort_create(DSI_E_RANGE);
    }
    s = plan_means(h, crn_cost, 148ull * 16 * (uint64_t)total_devices);
    if (s != DSI_OK) return abort_create(s);
  } else if (shared) {
    s = plan_shared(h, crn_cost);
    if (s != DSI_OK) return abort_create(s);
  } else {
    const uint64_t threads = (uint64_t)h->block_threads;
    const uint64_t target_blocks = 148ull * 16 * 8 * (uint64_t)total_devices;
    uint64_t r = h->total_trials / (threads * target_blocks);
    // up to 128 x 128 trials per unit: whole configs of the paper's grids in one unit
    // (measured, profiles/r01_ab_tile.jsonl: cap 32 -> 128 is 0.65% faster on cfg3)
    r = std::min<uint64_t>(128, std::max<uint64_t>(1, r));
    if (const char *force = std::getenv("DSI_TILE_R")) {  // developer A/B runs only
      const int fr = std::atoi(force);
      if (fr >= 1 && fr <= 1024) r = (uint64_t)fr;
    }
    h->tile_trials = (uint32_t)(threads * r);
    h->prefix[0] = 0;
    for (size_t i = 0; i < n_cfg; ++i)
      h->prefix[i + 1] = h->prefix[i] + (h->ticks[i].trials + h->tile_trials - 1) / h->tile_trials;
    h->total_units = h->prefix[n_cfg];
  }

  // ---- shards: world x n_devices x n_shards contiguous unit ranges of equal cost
  const int shards_per_dev = std::max(1, opt->n_shards);
  const int parts = total_devices * shards_per_dev;
  std::vector<uint64_t> bounds(parts + 1);
  {
    std::vector<double> cost;
    try {
      cost.resize(h->total_units);
    } catch (...) {
      h->err = "sharder cost table";
      return abort_create(DSI_E_NOMEM);
    }
    if (shared || means_only) {
      cost.swap(crn_cost);
    } else {
      for (size_t i = 0; i < n_cfg; ++i) {
        const uint64_t t = h->ticks[i].trials;
        for (uint64_t u = h->prefix[i]; u < h->prefix[i + 1]; ++u) {
          const uint64_t first = (u - h->prefix[i]) * h->tile_trials;  // the last tile is ragged
          cost[u] = unit_cost(h->ticks[i], std::min<uint64_t>(h->tile_trials, t - first));
        }
      }
    }
    dsi_shard_bounds(cost.data(), h->total_units, parts, bounds.data());
  }
  tr.mark("plan+shard");

  // means-only: the parts' config ranges, snapped to heatmap cell starts (dsi_sim_heatmap then
  // evaluates each part's cells from its own moments)
  if (means_only) {
    try {
      plan_heat_cells(h);
      h->cfg_bounds.assign(parts + 1, 0);
      size_t ci = 0;
      for (int q = 0; q <= parts; ++q) {
        const uint64_t want = (uint64_t)n_cfg * q / parts;
        while (ci + 1 < h->heat_cells.size() && h->heat_cells[ci + 1].first <= want) ++ci;
        uint64_t b = h->heat_cells.empty() ? want : h->heat_cells[ci].first;  // the cell start at or below
        if (q == parts) b = n_cfg;
        h->cfg_bounds[q] = std::max<uint64_t>(b, q ? h->cfg_bounds[q - 1] : 0);
      }
      h->heat_planned = true;
      h->heat_uploaded = false;
    } catch (...) {
      h->err = "host tables";
      return abort_create(DSI_E_NOMEM);
    }
  }

  // ---- devices
  int visible = 0;
  if (cudaGetDeviceCount(&visible) != cudaSuccess || visible < opt->device + opt->n_devices) {
    h->err = "not enough CUDA devices visible";
    return abort_create(DSI_E_DEVICE);
  }
  for (int di = 0; di < opt->n_devices; ++di) {
    int major = 0;
    const int ord = opt->device + di;
    if (cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, ord) != cudaSuccess || major != 10) {
      h->err = "device " + std::to_string(ord) + " is not an sm_100 (Blackwell) GPU";
      return abort_create(DSI_E_DEVICE);
    }
  }
  if (cudaSetDevice(opt->device) != cudaSuccess) {
    h->err = "cudaSetDevice failed";
    return abort_create(DSI_E_DEVICE);
  }
  // pinned staging: config table (H2D) and results (D2H)
  {
    cudaError_t e = h->dev_cfg.alloc(n_cfg);
    if (e == cudaSuccess) e = h->host_acc.alloc(n_cfg * dsi::NF);
    if (e == cudaSuccess) e = h->host_bad.alloc(1);
    if (e == cudaSuccess && (opt->flags & DSI_F_HIST)) {
      e = h->host_seg.alloc(n_cfg * 64);
      if (e == cudaSuccess) e = h->host_si.alloc(sib);
    }
    if (e != cudaSuccess) {
      h->err = std::string("pinned host buffers: ") + cudaGetErrorString(e);
      return abort_create(DSI_E_NOMEM);
    }
  }
  fill_dev_cfg(h);

  h->dev.resize(opt->n_devices);
  for (int di = 0; di < opt->n_devices; ++di) {
    DeviceState &d = h->dev[di];
    d.ordinal = opt->device + di;
    cudaError_t e = cudaSetDevice(d.ordinal);
    const int global_dev = opt->rank * opt->n_devices + di;
    for (int sh = 0; sh < shards_per_dev; ++sh) {
      const int part = global_dev * shards_per_dev + sh;
      d.ranges.emplace_back(bounds[part], bounds[part + 1]);
      // means-only: part p also evaluates configs [cfg_bounds[p], cfg_bounds[p+1])
      if (means_only) d.cfg_ranges.emplace_back(h->cfg_bounds[part], h->cfg_bounds[part + 1]);
    }
    if (e == cudaSuccess) {
      if (di == 0 && opt->stream) {
        d.stream = (cudaStream_t)opt->stream;
      } else {
        e = cudaStreamCreateWithFlags(&d.stream, cudaStreamNonBlocking);
        d.own_stream = true;
      }
    }
    const size_t acc_bytes = n_cfg * dsi::NF * sizeof(unsigned long long);
    if (e == cudaSuccess) e = cudaMalloc(&d.d_cfg, n_cfg * sizeof(DevCfg));
    if (e == cudaSuccess) e = cudaMalloc(&d.d_prefix, (n_cfg + 1) * sizeof(uint64_t));

    if (e == cudaSuccess) e = cudaMalloc(&d.d_acc, acc_bytes);
    if (e == cudaSuccess && use_nccl) e = cudaMalloc(&d.d_red, acc_bytes);
    if (e == cudaSuccess && (opt->flags & DSI_F_HIST)) {
      e = cudaMalloc(&d.d_seg, n_cfg * 64 * sizeof(unsigned long long));
      if (e == cudaSuccess) e = cudaMalloc(&d.d_si, sib * sizeof(unsigned long long));
      if (e == cudaSuccess && use_nccl) {
        e = cudaMalloc(&d.d_seg_red, n_cfg * 64 * sizeof(unsigned long long));
        if (e == cudaSuccess) e = cudaMalloc(&d.d_si_red, sib * sizeof(unsigned long long));
      }
    }
    if (e == cudaSuccess && per_trial) e = cudaMalloc(&d.d_rec, 5 * h->total_trials * sizeof(int32_t));
    if (e == cudaSuccess && means_only) {
      e = cudaMalloc(&d.d_seg_groups, h->seg_groups.size() * sizeof(dsi::SegGroup));
      if (e == cudaSuccess) e = cudaMalloc(&d.d_seg_prefix, h->seg_prefix.size() * sizeof(uint64_t));
      if (e == cudaSuccess) e = cudaMalloc(&d.d_cfg_group, n_cfg * sizeof(uint32_t));
      if (e == cudaSuccess) e = cudaMalloc(&d.d_hist, 3 * h->hist_len * sizeof(unsigned long long));
      if (e == cudaSuccess && !h->ttft_cfgs.empty())
        e = cudaMalloc(&d.d_ttft_cfgs, h->ttft_cfgs.size() * sizeof(uint32_t));
    }
    if (e == cudaSuccess && shared) {
      e = cudaMalloc(&d.d_perm, n_cfg * sizeof(uint32_t));
      if (e == cudaSuccess) e = cudaMalloc(&d.d_groups, h->groups.size() * sizeof(dsi::CrnGroup));
      if (e == cudaSuccess) e = cudaMalloc(&d.d_crn_units, h->crn_units.size() * sizeof(dsi::CrnUnit));
    }
    if (e == cudaSuccess)
      e = cudaMemcpyAsync(d.d_prefix, h->prefix.data(), (n_cfg + 1) * sizeof(uint64_t),
                          cudaMemcpyHostToDevice, d.stream);
    if (e == cudaSuccess && (opt->flags & DSI_F_TIMING)) {
      e = cudaEventCreate(&d.ev0);
      if (e == cudaSuccess) e = cudaEventCreate(&d.ev1);
    }
    if (e != cudaSuccess) {
      h->err = std::string("device setup: ") + cudaGetErrorString(e);
      return abort_create(e == cudaErrorMemoryAllocation ? DSI_E_NOMEM : DSI_E_DEVICE);
    }
  }
  tr.mark("devices");
  if (shared) {
    s = plan_two_pass(h);
    if (s == DSI_OK) s = alloc_two_pass(h);
    if (s != DSI_OK) return abort_create(s);
  }
  s = upload(h);
  if (s != DSI_OK) return abort_create(s);
  for (auto &d : h->dev) {
    cudaSetDevice(d.ordinal);
    if (cudaStreamSynchronize(d.stream) != cudaSuccess) {
      h->err = "device setup: stream synchronize failed";
      return abort_create(DSI_E_DEVICE);
    }
  }

  tr.mark("upload");
  // ---- NCCL: one communicator per device over world * n_devices ranks
  if (use_nccl && !host_coll) {
    NcclApi &api = nccl();
    if (!api.ok) {
      h->err = "libnccl.so.2 could not be loaded";
      return abort_create(DSI_E_COMM);
    }
    ncclUniqueId uid;
    std::memcpy(&uid, opt->nccl_id, sizeof(uid));
    ncclResult_t r = api.GroupStart();
    for (int di = 0; di < opt->n_devices && r == ncclSuccess; ++di) {
      cudaSetDevice(h->dev[di].ordinal);
      r = api.CommInitRank(&h->dev[di].comm, total_devices, uid, opt->rank * opt->n_devices + di);
    }
    const ncclResult_t r2 = api.GroupEnd();
    if (r != ncclSuccess || r2 != ncclSuccess) {
      h->err = std::string("ncclCommInitRank: ") + api.GetErrorString(r != ncclSuccess ? r : r2);
      return abort_create(DSI_E_COMM);
    }
  }
  *out = h;
  return DSI_OK;
}

dsi_status dsi_sim_update(dsi_sim *h, const dsi_config *cfg, size_t n_cfg) {
  if (!h) return DSI_E_NULL;
  Trace tr("dsi_sim_update");
  h->err.clear();
  if (!cfg) return fail(h, DSI_E_NULL, "cfg is NULL");
  if (n_cfg != h->n_cfg) return fail(h, DSI_E_RANGE, "n_cfg must equal the handle's");
  // validate into the spare table; h->ticks (and the whole handle) stay as they are on failure
  try {
    h->ticks_next.resize(n_cfg);
  } catch (...) {
    return fail(h, DSI_E_NOMEM, "host tables");
  }
  const int32_t old_n = h->max_n, old_keff = h->max_keff;
  const bool old_ttft = h->any_ttft, old_fresh = h->any_fresh;
  dsi_status s = validate_all(h, cfg, n_cfg, h->ticks_next, &h->ticks);
  tr.mark("validate");
  if (s == DSI_OK) s = derive_limits(h, h->ticks_next);  // the new configs may need a larger launch shape
  if (s != DSI_OK) return s;                              // derive_limits only commits on success
  if (h->means_only) {  // the histogram groups are fixed at create: their keys must not change
    bool same = h->max_n <= kMeansMaxN;
    for (size_t i = 0; same && i < n_cfg; ++i) {
      const CfgTicks &a = h->ticks[i], &b = h->ticks_next[i];
      const bool ta = a.t_t1 != a.t_t || a.t_d1 != a.t_d, tb = b.t_t1 != b.t_t || b.t_d1 != b.t_d;
      same = a.stream_id == b.stream_id && a.thr == b.thr && a.n == b.n && a.trials == b.trials && ta == tb;
    }
    if (!same) {
      h->max_n = old_n;
      h->max_keff = old_keff;
      h->any_ttft = old_ttft;
      h->any_fresh = old_fresh;
      return fail(h, DSI_E_RANGE,
                  "DSI_F_MEANS_ONLY: (stream_id, accept_rate, N, n_trials) or the TTFT configs changed; "
                  "create a new handle");
    }
  }
  const bool replan = h->shared && !same_plan_keys(h->ticks, h->ticks_next);
  tr.mark("limits");
  if (replan) {
    // re-plan on the host first: the unit table's size is fixed at create
    const int32_t old_cpb = h->cfg_per_block, old_runs = h->max_runs;
    std::vector<uint32_t> old_perm;
    std::vector<dsi::CrnGroup> old_groups;
    std::vector<dsi::CrnUnit> old_units;
    h->ticks.swap(h->ticks_next);
    try {
      old_perm = h->perm;
      old_groups = h->groups;
      old_units = h->crn_units;
      std::vector<double> cost;
      s = plan_shared(h, cost);
    } catch (...) {
      s = fail(h, DSI_E_NOMEM, "host tables");
    }
    if (s == DSI_OK && (h->groups.size() != old_groups.size() || h->crn_units.size() != old_units.size()))
      s = fail(h, DSI_E_RANGE, "DSI_F_SHARED_STREAMS: the stream grouping changed; create a new handle");
    if (s == DSI_OK) s = plan_two_pass(h);
    if (s == DSI_OK) {  // the buffers may grow: wait for any run still reading them
      for (auto &d : h->dev) {
        CUDA_TRY(h, cudaSetDevice(d.ordinal));
        CUDA_TRY(h, cudaStreamSynchronize(d.stream));
      }
      s = alloc_two_pass(h);
    }
    if (s != DSI_OK) {  // the handle keeps its previous configs and plan
      if (!old_groups.empty()) {
        h->perm.swap(old_perm);
        h->groups.swap(old_groups);
        h->crn_units.swap(old_units);
      }
      h->cfg_per_block = old_cpb;
      h->max_runs = old_runs;
      h->block_threads = old_cpb;
      h->ticks.swap(h->ticks_next);
      const std::string msg = h->err;
      plan_two_pass(h);  // the old plan's pass-1 lists (the buffers only ever grow)
      h->err = msg;
      h->max_n = old_n;
      h->max_keff = old_keff;
      h->any_ttft = old_ttft;
      h->any_fresh = old_fresh;
      return s;
    }
  } else {
    h->ticks.swap(h->ticks_next);
  }
  // wait until no kernel of a previous run still reads the table, then restage it
  for (auto &d : h->dev) {
    CUDA_TRY(h, cudaSetDevice(d.ordinal));
    CUDA_TRY(h, cudaStreamSynchronize(d.stream));
  }
  tr.mark(replan ? "replan+sync" : "sync");
  fill_dev_cfg(h);
  tr.mark("fill");
  h->ran = h->reduced = false;
  h->heat_planned = h->heat_uploaded = false;
  const dsi_status su = upload(h, replan);
  tr.mark("upload");
  return su;
}

static dsi::SegParams seg_params(dsi_sim *h, DeviceState &d, const dsi::Keys &keys) {
  dsi::SegParams q{};
  q.cfg = d.d_cfg;
  q.groups = d.d_seg_groups;
  q.unit_prefix = d.d_seg_prefix;
  q.cfg_group = d.d_cfg_group;
  q.n_groups = (uint32_t)h->seg_groups.size();
  q.tile_trials = h->tile_trials;
  q.hist = d.d_hist;
  q.pre = d.d_hist + h->hist_len;
  q.hist1 = h->ttft_cfgs.empty() ? nullptr : d.d_hist + 2 * h->hist_len;
  q.ttft_cfgs = d.d_ttft_cfgs;
  q.acc = d.d_acc;
  q.max_n = h->max_n;
  q.keys = keys;
  return q;
}

dsi_status dsi_sim_run(dsi_sim *h) {
  if (!h) return DSI_E_NULL;
  Trace tr("dsi_sim_run (enqueue)");
  h->err.clear();
  const size_t n_cfg = h->n_cfg;
  const uint64_t tt = h->total_trials;
  h->launches = 0;
  for (auto &d : h->dev) {
    CUDA_TRY(h, cudaSetDevice(d.ordinal));
    CUDA_TRY(h, cudaMemsetAsync(d.d_acc, 0, n_cfg * dsi::NF * sizeof(unsigned long long), d.stream));
    if (d.d_seg) {
      CUDA_TRY(h, cudaMemsetAsync(d.d_seg, 0, n_cfg * 64 * sizeof(unsigned long long), d.stream));
      CUDA_TRY(h, cudaMemsetAsync(d.d_si, 0, h->si_bins_total * sizeof(unsigned long long), d.stream));
    }
    LaunchParams p{};
    p.cfg = d.d_cfg;
    p.tile_prefix = d.d_prefix;
    p.n_cfg = (uint32_t)n_cfg;
    p.tile_trials = h->tile_trials;
    p.acc = d.d_acc;
    if (d.d_rec) {
      p.rec_acc = d.d_rec;
      p.rec_m = d.d_rec + tt;
      p.rec_iters = d.d_rec + 2 * tt;
      p.rec_si = d.d_rec + 3 * tt;
      p.rec_dsi = d.d_rec + 4 * tt;
    }
    p.seg_hist = d.d_seg;
    p.si_hist = d.d_si;
    p.max_n = h->max_n;
    p.max_keff = h->max_keff;
    p.any_ttft = h->any_ttft ? 1 : 0;
    p.any_fresh = h->any_fresh ? 1 : 0;
    p.k1_fast = h->k1_fast ? 1 : 0;
    const uint32_t s_lo = (uint32_t)h->opt.seed, s_hi = (uint32_t)(h->opt.seed >> 32);
    for (int r = 0; r < 10; ++r) {
      p.keys.k0[r] = s_lo + (uint32_t)r * 0x9E3779B9u;
      p.keys.k1[r] = s_hi + (uint32_t)r * 0xBB67AE85u;
    }
    if (d.ev0) CUDA_TRY(h, cudaEventRecord(d.ev0, d.stream));
    if (h->means_only) {  // pass 1 here; the histogram all-reduce and pass 2 after the loop
      CUDA_TRY(h, cudaMemsetAsync(d.d_hist, 0, h->hist_len * sizeof(unsigned long long), d.stream));
      if (!h->ttft_cfgs.empty())
        CUDA_TRY(h, cudaMemsetAsync(d.d_hist + 2 * h->hist_len, 0, h->hist_len * sizeof(unsigned long long),
                                    d.stream));
      dsi::SegParams q = seg_params(h, d, p.keys);
      for (const auto &rg : d.ranges) {
        if (rg.second <= rg.first) continue;
        q.unit_begin = rg.first;
        const int e = dsi::launch_seg_hist(q, rg.second - rg.first, d.stream);
        if (e) return cuda_fail(h, (cudaError_t)e, "segment histogram launch");
        h->launches += 1;
      }
      continue;
    }
    if (h->shared) {
      dsi::CrnParams q{};
      q.cfg = d.d_cfg;
      q.perm = d.d_perm;
      q.groups = d.d_groups;
      q.units = d.d_crn_units;
      q.acc = d.d_acc;
      q.max_n = h->max_n;
      q.max_nq = (h->max_n - 1 + 3) / 4 + 1;
      q.max_runs = h->max_runs;
      q.cfg_per_block = h->cfg_per_block;
      q.keys = p.keys;
      if (h->two_pass) {
        q.records = d.d_records;
        q.group_tile0 = d.d_group_tile0;
        q.tiles = d.d_tiles;
        q.tile_begin = 0;
        q.rec_bytes = h->rec_bytes;
        if (!d.tiles.empty()) {  // pass 1: every record this device's units read
          const int e = dsi::launch_crn_two_pass(q, d.tiles.size(), 0, h->cfg_per_block, d.stream);
          if (e) return cuda_fail(h, (cudaError_t)e, "shared-stream pass-1 launch");
          h->launches += 1;
        }
      }
      for (const auto &rg : d.ranges) {
        if (rg.second <= rg.first) continue;
        if (h->two_pass) {
          q.unit_begin = rg.first;
          const int e = dsi::launch_crn_two_pass(q, 0, rg.second - rg.first, h->cfg_per_block, d.stream);
          if (e) return cuda_fail(h, (cudaError_t)e, "shared-stream kernel launch");
          h->launches += 1;
          continue;
        }
        // units [0, n_sums_units) are sums-only (no run lists), the rest are not
        const uint64_t mid = std::min(std::max(rg.first, h->n_sums_units), rg.second);
        for (int part = 0; part < 2; ++part) {
          const uint64_t b = part ? mid : rg.first, e_ = part ? rg.second : mid;
          if (e_ <= b) continue;
          q.unit_begin = b;
          q.max_runs = part == 0 ? h->max_runs : std::min(h->max_runs, h->max_runs_normal);
          const int e = dsi::launch_crn_kernel(q, e_ - b, h->cfg_per_block, d.stream, part == 0);
          if (e) return cuda_fail(h, (cudaError_t)e, "shared-stream kernel launch");
          h->launches += 1;
        }
      }
    }
    for (const auto &rg : d.ranges) {
      if (h->shared) break;
      if (rg.second <= rg.first) continue;
      p.unit_begin = rg.first;
      const int e = dsi::launch_trial_kernel(p, rg.second - rg.first, h->block_threads,
                                             h->opt.flags & DSI_F_PER_TRIAL, h->opt.flags & DSI_F_HIST,
                                             h->opt.flags & DSI_F_PATTERN, d.stream);
      if (e) return cuda_fail(h, (cudaError_t)e, "trial kernel launch");
      h->launches += 1;
    }
    if (d.ev1) CUDA_TRY(h, cudaEventRecord(d.ev1, d.stream));
  }
  if (h->means_only) {
    // every device needs every group's full histogram: one (grouped) all-reduce, in place
    if (h->use_nccl && h->host_coll) {
      DeviceState &d = h->dev[0];
      dsi_status st = host_allreduce(h, d.stream, d.d_hist, d.d_hist, h->hist_len);
      if (st == DSI_OK && !h->ttft_cfgs.empty())
        st = host_allreduce(h, d.stream, d.d_hist + 2 * h->hist_len, d.d_hist + 2 * h->hist_len, h->hist_len);
      if (st != DSI_OK) return st;
    } else if (h->use_nccl) {
      NcclApi &api = nccl();
      ncclResult_t r = api.GroupStart();
      for (auto &d : h->dev) {
        if (r != ncclSuccess) break;
        cudaSetDevice(d.ordinal);
        r = api.AllReduce(d.d_hist, d.d_hist, h->hist_len, ncclUint64, ncclSum, d.comm, d.stream);
        if (r == ncclSuccess && !h->ttft_cfgs.empty())
          r = api.AllReduce(d.d_hist + 2 * h->hist_len, d.d_hist + 2 * h->hist_len, h->hist_len, ncclUint64,
                            ncclSum, d.comm, d.stream);
      }
      const ncclResult_t r2 = api.GroupEnd();
      if (r != ncclSuccess || r2 != ncclSuccess)
        return fail(h, DSI_E_COMM, std::string("histogram all-reduce: ") +
                                       api.GetErrorString(r != ncclSuccess ? r : r2));
    }
    for (auto &d : h->dev) {
      CUDA_TRY(h, cudaSetDevice(d.ordinal));
      dsi::SegParams q = seg_params(h, d, dsi::Keys{});
      {
        const int e = dsi::launch_seg_prefix(q, d.stream);
        if (e) return cuda_fail(h, (cudaError_t)e, "segment prefix launch");
        h->launches += 1;
      }
      for (const auto &cr : d.cfg_ranges) {
        q.cfg_begin = cr.first;
        q.cfg_end = cr.second;
        const int e = dsi::launch_seg_eval(q, d.stream);
        if (e) return cuda_fail(h, (cudaError_t)e, "segment evaluation launch");
        h->launches += cr.second > cr.first;
        if (!h->ttft_cfgs.empty()) {  // first-segment corrections of this range's TTFT configs
          const auto &L = h->ttft_cfgs;
          const uint64_t b = std::lower_bound(L.begin(), L.end(), (uint32_t)cr.first) - L.begin();
          const uint64_t en = std::lower_bound(L.begin(), L.end(), (uint32_t)cr.second) - L.begin();
          const int e2 = dsi::launch_seg_ttft(q, b, en, d.stream);
          if (e2) return cuda_fail(h, (cudaError_t)e2, "TTFT correction launch");
          h->launches += en > b;
        }
      }
      if (d.ev1) CUDA_TRY(h, cudaEventRecord(d.ev1, d.stream));
    }
  }
  h->ran = true;
  h->reduced = false;
  return DSI_OK;
}

dsi_status dsi_sim_reduce(dsi_sim *h, dsi_result *out, size_t n) {
  if (!h) return DSI_E_NULL;
  Trace tr("dsi_sim_reduce");
  h->err.clear();
  const bool root_only = (h->opt.flags & DSI_F_REDUCE_TO_ROOT) && h->opt.rank != 0;
  if (!out && !root_only) return fail(h, DSI_E_NULL, "out is NULL");
  const size_t n_cfg = h->n_cfg;
  if (n != n_cfg) return fail(h, DSI_E_RANGE, "n must equal n_cfg");
  if (!h->ran) return fail(h, DSI_E_STATE, "dsi_sim_reduce before dsi_sim_run");
  const bool hist = h->opt.flags & DSI_F_HIST;
  dsi_status st = sum_across(h, hist);
  if (st != DSI_OK) return st;
  tr.mark("allreduce-enqueue");
  if (root_only) {  // DSI_F_REDUCE_TO_ROOT: this rank contributed its sums; rank 0 checks and finalizes
    for (auto &d : h->dev) {
      CUDA_TRY(h, cudaSetDevice(d.ordinal));
      CUDA_TRY(h, cudaStreamSynchronize(d.stream));
    }
    h->reduced = true;
    return DSI_OK;
  }
  // every device now holds the global sums (or there is one device): read device 0.
  // The partition check (every trial simulated exactly once) runs on the device before the
  // copies; the moments come back in chunks so the host finalizes chunk i while chunk i+1
  // is in flight.
  DeviceState &d0 = h->dev[0];
  CUDA_TRY(h, cudaSetDevice(d0.ordinal));
  const unsigned long long *src = h->use_nccl ? d0.d_red : d0.d_acc;
  if (!d0.d_heat_bad) CUDA_TRY(h, cudaMalloc((void **)&d0.d_heat_bad, sizeof(unsigned int)));
  if (!h->chunk_ev[0])
    for (auto &ev : h->chunk_ev) CUDA_TRY(h, cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
  CUDA_TRY(h, cudaMemsetAsync(d0.d_heat_bad, 0, sizeof(unsigned int), d0.stream));
  {
    const int e = dsi::launch_check_trials(d0.d_cfg, src, n_cfg, d0.d_heat_bad, d0.stream);
    if (e) return cuda_fail(h, (cudaError_t)e, "partition check launch");
    h->launches += 1;
  }
  CUDA_TRY(h, cudaMemcpyAsync(h->host_bad.p, d0.d_heat_bad, sizeof(unsigned int), cudaMemcpyDeviceToHost,
                              d0.stream));
  if (hist) {
    CUDA_TRY(h, cudaMemcpyAsync(h->host_seg.p, h->use_nccl ? d0.d_seg_red : d0.d_seg,
                                n_cfg * 64 * sizeof(unsigned long long), cudaMemcpyDeviceToHost, d0.stream));
    CUDA_TRY(h, cudaMemcpyAsync(h->host_si.p, h->use_nccl ? d0.d_si_red : d0.d_si,
                                h->si_bins_total * sizeof(unsigned long long), cudaMemcpyDeviceToHost,
                                d0.stream));
  }
  const size_t n_chunks = n_cfg < (1u << 16) ? 1 : kReduceChunks;
  for (size_t c = 0; c < n_chunks; ++c) {
    const size_t b = n_cfg * c / n_chunks, e = n_cfg * (c + 1) / n_chunks;
    CUDA_TRY(h, cudaMemcpyAsync(h->host_acc.p + b * dsi::NF, src + b * dsi::NF,
                                (e - b) * dsi::NF * sizeof(unsigned long long), cudaMemcpyDeviceToHost,
                                d0.stream));
    CUDA_TRY(h, cudaEventRecord(h->chunk_ev[c], d0.stream));
  }
  for (auto &d : h->dev) {  // the all-reduce ran on every device's stream
    if (d.ordinal == d0.ordinal) continue;
    CUDA_TRY(h, cudaSetDevice(d.ordinal));
    CUDA_TRY(h, cudaStreamSynchronize(d.stream));
  }
  CUDA_TRY(h, cudaSetDevice(d0.ordinal));
  CUDA_TRY(h, cudaEventSynchronize(h->chunk_ev[0]));  // the flag precedes chunk 0
  tr.mark("wait-run+check+chunk0");
  if (*h->host_bad.p) {
    CUDA_TRY(h, cudaStreamSynchronize(d0.stream));
    return fail(h, DSI_E_DEVICE, "trial count mismatch after reduce (partition error)");
  }
  const double tick = h->opt.tick;
  for (size_t c = 0; c < n_chunks; ++c) {
  const size_t cb = n_cfg * c / n_chunks, ce = n_cfg * (c + 1) / n_chunks;
  if (c) CUDA_TRY(h, cudaEventSynchronize(h->chunk_ev[c]));
  parallel_for(ce - cb, [&](size_t b, size_t e) {
  for (size_t i = cb + b; i < cb + e; ++i) {
    const unsigned long long *a = &h->host_acc.p[i * dsi::NF];
    const CfgTicks &t = h->ticks[i];
    dsi_result &r = out[i];
    const uint64_t T = t.trials;
    const uint64_t si_cost = (uint64_t)(t.kd + t.t_t);
    // L_SI = I (k t_d + t_t) + e, e = SI's first-iteration surcharge (TTFT variant, else 0)
    const __int128 e = (__int128)(t.t_d1 - t.t_d) + (__int128)(t.t_t1 - t.t_t);
    r.trials = T;
    r.t_target_ticks = t.t_t;
    r.t_drafter_ticks = t.t_d;
    r.nonsi_ticks = t.t_t1 + (int64_t)(t.n - 1) * t.t_t;
    r.sum_si_iters = (int64_t)a[dsi::F_I];
    r.sum_si_ticks = (int64_t)((__int128)si_cost * a[dsi::F_I] + (__int128)T * e);
    r.sumsq_si_ticks = (uint64_t)((__int128)si_cost * si_cost * a[dsi::F_I2] +
                                  2 * (__int128)si_cost * e * a[dsi::F_I] + (__int128)T * e * e);
    r.sum_dsi_ticks = (int64_t)a[dsi::F_DSI];
    r.sumsq_dsi_ticks = a[dsi::F_DSI2];
    r.sum_segments = (int64_t)a[dsi::F_M];
    // acc = (N-1) - (m-1) per trial
    r.sum_accepts = (int64_t)(T * (uint64_t)t.n) - (int64_t)a[dsi::F_M];
    r.n_dsi_gt_nonsi = (int64_t)a[dsi::F_GT_NONSI];
    r.n_dsi_gt_si = (int64_t)a[dsi::F_GT_SI];
    r.threshold = t.thr;
    r.eq1_feasible = t.eq1;
    r.min_lookahead = t.min_k;
    const double Td = (double)T;
    r.mean_nonsi = (double)r.nonsi_ticks * tick;
    r.mean_si = ((double)r.sum_si_ticks / Td) * tick;
    r.mean_dsi = ((double)r.sum_dsi_ticks / Td) * tick;
    auto stdev = [&](uint64_t s1, uint64_t s2) {
      const unsigned __int128 num = (unsigned __int128)T * s2 - (unsigned __int128)s1 * s1;
      return std::sqrt((double)num) / Td * tick;
    };
    if (h->means_only) {  // no per-trial values: no second moments, no per-trial counters
      r.sumsq_si_ticks = r.sumsq_dsi_ticks = 0;
      r.n_dsi_gt_nonsi = r.n_dsi_gt_si = -1;
      r.std_si = r.std_dsi = std::nan("");
    } else {
      r.std_si = stdev((uint64_t)r.sum_si_ticks, r.sumsq_si_ticks);
      r.std_dsi = stdev((uint64_t)r.sum_dsi_ticks, r.sumsq_dsi_ticks);
    }
  }
  });
  }
  CUDA_TRY(h, cudaStreamSynchronize(d0.stream));  // the histogram copies (HIST), if any
  tr.mark("finalize");
  h->reduced = true;
  return DSI_OK;
}

dsi_status dsi_sim_heatmap(dsi_sim *h, dsi_heatmap_cell *cells, size_t cap, size_t *n_cells) {
  if (!h) return DSI_E_NULL;
  Trace tr("dsi_sim_heatmap");
  h->err.clear();
  if (!n_cells) return fail(h, DSI_E_NULL, "n_cells is NULL");
  if (!h->heat_planned) {  // cells: maximal runs of equal (t_target, t_drafter, a, SP, N)
    try {
      plan_heat_cells(h);
    } catch (...) {
      return fail(h, DSI_E_NOMEM, "host tables");
    }
    h->heat_planned = true;
    h->heat_uploaded = false;
  }
  const size_t nc = h->heat_cells.size();
  *n_cells = nc;
  if (!cells) return DSI_OK;
  if (cap < nc) return fail(h, DSI_E_RANGE, "cap is smaller than the number of cells");
  if (!h->ran) return fail(h, DSI_E_STATE, "dsi_sim_heatmap before dsi_sim_run");
  const bool local = cells_aligned(h);
  if (!local) {
    dsi_status st = sum_across(h, false);
    if (st != DSI_OK) return st;
  }
  DeviceState &d0 = h->dev[0];
  CUDA_TRY(h, cudaSetDevice(d0.ordinal));
  if (!h->heat_uploaded) {
    if (h->heat_out.n < nc) {
      cudaFree(d0.d_heat_cells);
      cudaFree(d0.d_heat_out);
      d0.d_heat_cells = nullptr;
      d0.d_heat_out = nullptr;
      CUDA_TRY(h, cudaMalloc((void **)&d0.d_heat_cells, std::max<size_t>(1, nc) * sizeof(dsi::HeatCell)));
      CUDA_TRY(h, cudaMalloc((void **)&d0.d_heat_out, std::max<size_t>(1, nc) * sizeof(dsi::HeatOut)));
      CUDA_TRY(h, h->heat_out.alloc(nc));
    }
    if (!d0.d_heat_bad) CUDA_TRY(h, cudaMalloc((void **)&d0.d_heat_bad, sizeof(unsigned int)));
    CUDA_TRY(h, cudaMemcpyAsync(d0.d_heat_cells, h->heat_cells.data(), nc * sizeof(dsi::HeatCell),
                                cudaMemcpyHostToDevice, d0.stream));
    CUDA_TRY(h, cudaStreamSynchronize(d0.stream));  // the vector is pageable
    h->heat_uploaded = true;
  }
  CUDA_TRY(h, cudaMemsetAsync(d0.d_heat_bad, 0, sizeof(unsigned int), d0.stream));
  dsi::HeatParams p{};
  p.cfg = d0.d_cfg;
  p.acc = h->use_nccl ? d0.d_red : d0.d_acc;
  p.cells = d0.d_heat_cells;
  p.n_cells = (uint32_t)nc;
  p.tick = h->opt.tick;
  p.out = d0.d_heat_out;
  p.bad = d0.d_heat_bad;
  if (!local) {
    const int e = dsi::launch_heatmap_kernel(p, d0.stream);
    if (e) return cuda_fail(h, (cudaError_t)e, "heatmap kernel launch");
    h->launches += 1;
  } else {
    // this process's parts hold whole cells: evaluate them from the local moments, then (several
    // ranks) one all-reduce of the 64-byte cell records, zero where another rank owns the cell
    p.acc = d0.d_acc;
    if (h->use_nccl) CUDA_TRY(h, cudaMemsetAsync(d0.d_heat_out, 0, nc * sizeof(dsi::HeatOut), d0.stream));
    for (const auto &cr : d0.cfg_ranges) {
      const auto lo = std::lower_bound(h->heat_cells.begin(), h->heat_cells.end(), cr.first,
                                       [](const dsi::HeatCell &c, uint64_t v) { return c.first < v; });
      const auto hi = std::lower_bound(h->heat_cells.begin(), h->heat_cells.end(), cr.second,
                                       [](const dsi::HeatCell &c, uint64_t v) { return c.first < v; });
      if (hi <= lo) continue;
      dsi::HeatParams q = p;
      q.cells = d0.d_heat_cells + (lo - h->heat_cells.begin());
      q.out = d0.d_heat_out + (lo - h->heat_cells.begin());
      q.n_cells = (uint32_t)(hi - lo);
      const int e = dsi::launch_heatmap_kernel(q, d0.stream);
      if (e) return cuda_fail(h, (cudaError_t)e, "heatmap kernel launch");
      h->launches += 1;
    }
    if (h->use_nccl && h->host_coll) {
      const dsi_status st = host_allreduce(h, d0.stream, d0.d_heat_out, d0.d_heat_out, nc * 8);
      if (st != DSI_OK) return st;
    } else if (h->use_nccl) {
      static_assert(sizeof(dsi::HeatOut) == 64, "HeatOut is 8 words");
      NcclApi &api = nccl();
      const ncclResult_t r = api.AllReduce(d0.d_heat_out, d0.d_heat_out, nc * 8, ncclUint64, ncclSum, d0.comm,
                                           d0.stream);
      if (r != ncclSuccess) return fail(h, DSI_E_COMM, std::string("heatmap all-reduce: ") + api.GetErrorString(r));
    }
  }
  unsigned int bad = 0;
  CUDA_TRY(h, cudaMemcpyAsync(h->heat_out.p, d0.d_heat_out, nc * sizeof(dsi::HeatOut), cudaMemcpyDeviceToHost,
                              d0.stream));
  CUDA_TRY(h, cudaMemcpyAsync(&bad, d0.d_heat_bad, sizeof(unsigned int), cudaMemcpyDeviceToHost, d0.stream));
  for (auto &d : h->dev) {  // the all-reduce ran on every device's stream
    CUDA_TRY(h, cudaSetDevice(d.ordinal));
    CUDA_TRY(h, cudaStreamSynchronize(d.stream));
  }
  if (bad) return fail(h, DSI_E_DEVICE, "trial count mismatch after reduce (partition error)");
  for (size_t i = 0; i < nc; ++i) {
    const dsi::HeatCell &hc = h->heat_cells[i];
    const dsi::HeatOut &o = h->heat_out.p[i];
    const CfgTicks &t = h->ticks[hc.first];
    dsi_heatmap_cell &c = cells[i];
    c.t_target = t.ut;
    c.t_drafter = t.ud;
    c.accept_rate = t.a;
    c.sp_degree = t.sp;
    c.n_tokens = t.n;
    c.si_lookahead = o.si_k;
    c.dsi_lookahead = o.dsi_k;
    c.nonsi = o.nonsi;
    c.si = o.si;
    c.dsi = o.dsi;
    c.r_nonsi_si = o.r_nonsi_si;
    c.r_si_dsi = o.r_si_dsi;
    c.r_nonsi_dsi = o.r_nonsi_dsi;
    c.r_min_dsi = o.r_min_dsi;
    c.first_cfg = hc.first;
    c.n_cfg = hc.count;
  }
  return DSI_OK;
}

dsi_status dsi_sim_trials(dsi_sim *h, size_t cfg, uint64_t first, uint64_t count, int32_t *acc,
                          int32_t *m, int32_t *iters, int32_t *si_ticks, int32_t *dsi_ticks) {
  if (!h) return DSI_E_NULL;
  h->err.clear();
  if (!(h->opt.flags & DSI_F_PER_TRIAL)) return fail(h, DSI_E_STATE, "needs DSI_F_PER_TRIAL");
  if (!h->ran) return fail(h, DSI_E_STATE, "dsi_sim_trials before dsi_sim_run");
  if (cfg >= h->n_cfg) return fail(h, DSI_E_RANGE, "cfg out of range");
  const uint64_t T = h->ticks[cfg].trials;
  if (first > T || count > T - first) return fail(h, DSI_E_RANGE, "trial range out of bounds");
  DeviceState &d = h->dev[0];
  CUDA_TRY(h, cudaSetDevice(d.ordinal));
  CUDA_TRY(h, cudaStreamSynchronize(d.stream));
  const uint64_t tt = h->total_trials;
  const uint64_t off = h->dev_cfg.p[cfg].rec_off + first;
  int32_t *dst[5] = {acc, m, iters, si_ticks, dsi_ticks};
  for (int f = 0; f < 5; ++f) {
    if (!dst[f] || count == 0) continue;
    CUDA_TRY(h, cudaMemcpy(dst[f], d.d_rec + f * tt + off, count * sizeof(int32_t), cudaMemcpyDeviceToHost));
  }
  return DSI_OK;
}

dsi_status dsi_sim_hist(dsi_sim *h, size_t cfg, int64_t *seg_hist, int64_t *si_hist, size_t si_bins) {
  if (!h) return DSI_E_NULL;
  h->err.clear();
  if (!(h->opt.flags & DSI_F_HIST)) return fail(h, DSI_E_STATE, "needs DSI_F_HIST");
  if (!h->reduced) return fail(h, DSI_E_STATE, "dsi_sim_hist before dsi_sim_reduce");
  if (cfg >= h->n_cfg) return fail(h, DSI_E_RANGE, "cfg out of range");
  const size_t k = (size_t)h->ticks[cfg].k;
  if (si_hist && si_bins != k + 1) return fail(h, DSI_E_RANGE, "si_bins must equal k+1");
  if (seg_hist)
    for (int i = 0; i < 64; ++i) seg_hist[i] = (int64_t)h->host_seg.p[cfg * 64 + i];
  if (si_hist) {
    const DevCfg &dc = h->dev_cfg.p[cfg];
    for (size_t j = 0; j <= k; ++j)
      si_hist[j] = j <= (size_t)dc.k_eff ? (int64_t)h->host_si.p[dc.si_hist_off + j] : 0;
  }
  return DSI_OK;
}

dsi_status dsi_sim_stream(dsi_sim *h, int32_t i, void **stream) {
  if (!h || !stream) return DSI_E_NULL;
  if (i < 0 || i >= (int32_t)h->dev.size()) return fail(h, DSI_E_RANGE, "device index");
  *stream = (void *)h->dev[i].stream;
  return DSI_OK;
}

dsi_status dsi_sim_launches(dsi_sim *h, int32_t *launches) {
  if (!h || !launches) return DSI_E_NULL;
  *launches = h->launches;
  return DSI_OK;
}

dsi_status dsi_sim_kernel_ms(dsi_sim *h, int32_t i, float *ms) {
  if (!h || !ms) return DSI_E_NULL;
  if (!(h->opt.flags & DSI_F_TIMING)) return fail(h, DSI_E_STATE, "needs DSI_F_TIMING");
  if (!h->ran) return fail(h, DSI_E_STATE, "no run yet");
  if (i < 0 || i >= (int32_t)h->dev.size()) return fail(h, DSI_E_RANGE, "device index");
  DeviceState &d = h->dev[i];
  CUDA_TRY(h, cudaSetDevice(d.ordinal));
  CUDA_TRY(h, cudaEventSynchronize(d.ev1));
  CUDA_TRY(h, cudaEventElapsedTime(ms, d.ev0, d.ev1));
  return DSI_OK;
}

dsi_status dsi_sim_io_bytes(dsi_sim *h, uint64_t *h2d, uint64_t *d2h) {
  if (!h || !h2d || !d2h) return DSI_E_NULL;
  const uint64_t n = h->n_cfg;
  *h2d = (uint64_t)h->dev.size() * n * sizeof(DevCfg);
  uint64_t back = n * dsi::NF * sizeof(unsigned long long);
  if (h->opt.flags & DSI_F_HIST) back += (n * 64 + h->si_bins_total) * sizeof(unsigned long long);
  *d2h = back;
  return DSI_OK;
}

dsi_status dsi_sim_units(dsi_sim *h, uint64_t *first, uint64_t *count, uint64_t *total) {
  if (!h || !first || !count || !total) return DSI_E_NULL;
  uint64_t lo = UINT64_MAX, hi = 0;
  for (auto &d : h->dev)
    for (auto &r : d.ranges) {
      lo = std::min(lo, r.first);
      hi = std::max(hi, r.second);
    }
  *first = lo == UINT64_MAX ? 0 : lo;
  *count = hi > *first ? hi - *first : 0;
  *total = h->total_units;
  return DSI_OK;
}

void dsi_sim_destroy(dsi_sim *h) {
  if (!h) return;
  free_handle(h);
}

// ---- multi-drafter DSI: one-shot, one device -------------------------------
#ifndef DSI_MULTI_WARP_LANES
#define DSI_MULTI_WARP_LANES 32.0  // (A/B: 1.0 restores the per-lane rule)
#endif
#ifndef DSI_MULTI_TILE
#define DSI_MULTI_TILE 2048  // trials per block (1024..8192 within 3%, profiles/r01_ab_multi.txt)
#endif
namespace {
thread_local float g_multi_ms = 0.0f;
thread_local int32_t g_multi_launches = 0;

struct DevBuf {  // stream-ordered device allocation (the device's default pool keeps the memory
                 // between calls, so repeated calls do not pay cudaMalloc / cudaFree), freed on exit
  void *p = nullptr;
  cudaStream_t s = nullptr;
  cudaError_t alloc(size_t bytes, cudaStream_t st) {
    s = st;
    return cudaMallocAsync(&p, bytes, st);
  }
  ~DevBuf() { if (p) cudaFreeAsync(p, s); }
};
}  // namespace

dsi_status dsi_multi_simulate(const dsi_options *opt, const dsi_multi_config *cfg, size_t n_cfg,
                              dsi_multi_result *out, int32_t *trial_dsi, int32_t *trial_settled) {
  Trace tr("dsi_multi_simulate");
  g_create_error.clear();
  g_multi_ms = 0.0f;
  g_multi_launches = 0;
  if (!opt || !cfg || !out) return fail(nullptr, DSI_E_NULL, "opt, cfg or out is NULL");
  if (opt->abi_version != DSI_ABI_VERSION) return fail(nullptr, DSI_E_RANGE, "abi_version mismatch");
  if (n_cfg == 0 || n_cfg >= (1ull << 31)) return fail(nullptr, DSI_E_RANGE, "n_cfg out of range");
  if (!(std::isfinite(opt->tick) && opt->tick > 0.0)) return fail(nullptr, DSI_E_RANGE, "tick must be > 0");
  if (opt->flags & ~(DSI_F_PER_TRIAL | DSI_F_PATTERN | DSI_F_TIMING | DSI_F_MEANS_ONLY))
    return fail(nullptr, DSI_E_RANGE, "multi-drafter mode takes PER_TRIAL, PATTERN, TIMING and MEANS_ONLY only");
  const bool means = opt->flags & DSI_F_MEANS_ONLY;
  if (means && (opt->flags & DSI_F_PER_TRIAL))
    return fail(nullptr, DSI_E_RANGE, "DSI_F_MEANS_ONLY excludes DSI_F_PER_TRIAL");
  if (opt->n_devices != 1 || opt->device < 0)
    return fail(nullptr, DSI_E_RANGE, "multi-drafter mode drives one device per process (n_devices = 1)");
  if (opt->world < 1 || opt->rank < 0 || opt->rank >= opt->world)
    return fail(nullptr, DSI_E_RANGE, "need 0 <= rank < world");
  if (opt->n_shards < 0 || opt->n_shards > 4096 || (opt->n_shards > 1 && opt->world > 1))
    return fail(nullptr, DSI_E_RANGE, "n_shards must be 0..4096 and > 1 only with world == 1");
  const bool host_coll = g_host_ar != nullptr && opt->world > 1;
  if (opt->world > 1 && !opt->nccl_id && !host_coll)
    return fail(nullptr, DSI_E_NULL, "nccl_id is required when world > 1");
  const bool use_nccl = (opt->world > 1 || opt->nccl_id != nullptr) && !host_coll;
  const bool per_trial = opt->flags & DSI_F_PER_TRIAL;
  if (per_trial && opt->world > 1)
    return fail(nullptr, DSI_E_RANGE, "DSI_F_PER_TRIAL needs world == 1");
  if (!per_trial && (trial_dsi || trial_settled))
    return fail(nullptr, DSI_E_STATE, "per-trial outputs need DSI_F_PER_TRIAL");

  std::vector<dsi::MultiCfg> dc(n_cfg);
  std::vector<uint64_t> prefix(n_cfg + 1, 0);
  std::vector<int64_t> tt(n_cfg);
  uint64_t rec = 0;
  int32_t max_n = 1, max_d = 1;
  const uint32_t tile = DSI_MULTI_TILE;  // trials per block
  for (size_t i = 0; i < n_cfg; ++i) {
    const dsi_multi_config &c = cfg[i];
    char buf[160];
    auto bad = [&](dsi_status st, const char *what) {
      std::snprintf(buf, sizeof buf, "config %zu: %s", i, what);
      return fail(nullptr, st, buf);
    };
    if (c.n_drafters < 1 || c.n_drafters > DSI_MAX_DRAFTERS) return bad(DSI_E_RANGE, "n_drafters must be 1..7");
    if (c.reserved != 0) return bad(DSI_E_RANGE, "reserved must be 0");
    if (c.n_tokens < 1 || c.n_tokens > kMaxTokens) return bad(DSI_E_RANGE, "n_tokens out of [1, 32768]");
    if (c.n_trials < 1 || c.n_trials > kMaxTrials) return bad(DSI_E_RANGE, "n_trials out of [1, 2^32]");
    int64_t t_t = 0;
    dsi_status st = to_ticks(c.t_target, opt->tick, &t_t);
    if (st != DSI_OK) return bad(st, "t_target is not a positive whole number of ticks");
    dsi::MultiCfg &d = dc[i];
    std::memset(&d, 0, sizeof d);
    int64_t prev = 1;
    for (int j = 0; j < c.n_drafters; ++j) {
      int64_t t_d = 0;
      st = to_ticks(c.t_drafter[j], opt->tick, &t_d);
      if (st != DSI_OK) return bad(st, "t_drafter is not a positive whole number of ticks");
      if (t_d > t_t) return bad(DSI_E_RANGE, "t_drafter > t_target (Assumption 2, P:109)");
      if (t_d < prev) return bad(DSI_E_RANGE, "drafters must be ordered by latency (R25)");
      prev = t_d;
      const double a = c.accept_rate[j];
      if (!(a >= 0.0 && a <= 1.0)) return bad(DSI_E_RANGE, "accept_rate not in [0, 1]");
      const uint64_t thr = (uint64_t)(a * 4294967296.0);  // exact scaling, then floor
      d.thr[j] = (uint32_t)std::min<uint64_t>(thr, 0xffffffffull);
      d.mode[j] = thr >= (1ull << 32) ? dsi::MODE_ALL_ACCEPT : (thr == 0 ? dsi::MODE_ALL_REJECT : dsi::MODE_STREAM);
      d.t_d[j] = (int32_t)t_d;
    }
    const unsigned __int128 bound = (unsigned __int128)c.n_tokens * (uint64_t)t_t;
    if (bound >= ((unsigned __int128)1 << 31)) return bad(DSI_E_OVERFLOW, "N * t_target >= 2^31 ticks");
    if ((unsigned __int128)c.n_trials * bound * bound >= ((unsigned __int128)1 << 64))
      return bad(DSI_E_OVERFLOW, "n_trials * (N t_target)^2 >= 2^64");
    d.t_t = (int32_t)t_t;
    {
      // P(a quad still has an open position when drafter j is reached) = 1 - (1 - r)^4,
      // r = prod_{i<j} (1 - a_i) the chance a position is open.  A warp makes a call when any
      // of its 32 lanes needs it, so calling per quad saves work only when open quads are rare
      // in the whole warp; otherwise 4 independent calls at once (ILP) win.
      double r = 1.0;
      for (int j = 0; j < c.n_drafters; ++j) {
        const double open = 1.0 - std::pow(1.0 - r, 4.0);
        const double warp_needs = 1.0 - std::pow(1.0 - open, DSI_MULTI_WARP_LANES);
        d.width[j] = warp_needs >= 0.9 ? 4 : (warp_needs >= 0.5 ? 2 : 1);
        r *= d.mode[j] == dsi::MODE_ALL_ACCEPT ? 0.0 : 1.0 - (double)d.thr[j] / 4294967296.0;
      }
    }
    d.n_drafters = c.n_drafters;
    d.n_tokens = c.n_tokens;
    d.stream_id = c.stream_id;
    d.n_trials = c.n_trials;
    d.rec_off = rec;
    rec += c.n_trials;
    tt[i] = t_t;
    prefix[i + 1] = prefix[i] + (c.n_trials + tile - 1) / tile;
    max_n = std::max(max_n, c.n_tokens);
    max_d = std::max(max_d, c.n_drafters);
  }
  // Means-only: j*(p) depends on the indicators only, never on the latencies, so configs with
  // equal (stream_id, N, T, thresholds) have equal settled-by counts per trial.  The kernel runs
  // one representative per such group; every config's sum of L = t_m (T + sum S_m) +
  // sum_j t_j sum S_j follows from the representative's exact sums (no second moments).
  std::vector<uint32_t> rep_of(n_cfg);
  for (size_t i = 0; i < n_cfg; ++i) rep_of[i] = (uint32_t)i;
  size_t nk = n_cfg;  // configs the kernel runs
  std::vector<dsi::MultiCfg> orig;  // means-only: every config's latencies (dc then holds the representatives)
  if (means) {
    std::map<std::vector<uint64_t>, uint32_t> seen;
    std::vector<dsi::MultiCfg> kc;
    std::vector<uint64_t> kprefix(1, 0);
    for (size_t i = 0; i < n_cfg; ++i) {
      const dsi::MultiCfg &d = dc[i];
      std::vector<uint64_t> key = {d.stream_id, (uint64_t)d.n_tokens, d.n_trials, (uint64_t)d.n_drafters};
      for (int j = 0; j < d.n_drafters; ++j) key.push_back(((uint64_t)d.mode[j] << 32) | d.thr[j]);
      auto it = seen.find(key);
      if (it == seen.end()) {
        it = seen.emplace(key, (uint32_t)kc.size()).first;
        kc.push_back(d);
        kprefix.push_back(kprefix.back() + (d.n_trials + tile - 1) / tile);
      }
      rep_of[i] = it->second;
    }
    nk = kc.size();
    orig.swap(dc);
    dc.swap(kc);
    prefix.swap(kprefix);
  }
  // units (config, tile of trials) split into world x shards contiguous ranges of equal expected
  // cost (trials x Philox calls a drafter must make, as bench.py's multi_alg_multiplies); this
  // rank runs its ranges, the per-config moments are summed with one NCCL all-reduce
  const uint64_t n_units = prefix[nk];
  const int shards = std::max(1, opt->n_shards);
  const int parts = opt->world * shards;
  std::vector<uint64_t> bounds(parts + 1, 0);
  {
    std::vector<double> cost(n_units);
    for (size_t i = 0; i < nk; ++i) {
      const dsi::MultiCfg &d = dc[i];
      const int npos = d.n_tokens - 1;
      double open = 1.0, calls = 0.0;
      for (int j = 0; j < d.n_drafters; ++j) {
        if (d.mode[j] == dsi::MODE_STREAM) calls += (double)((npos + 3) / 4) * (1.0 - std::pow(1.0 - open, 4.0));
        open *= d.mode[j] == dsi::MODE_ALL_ACCEPT ? 0.0 : 1.0 - (double)d.thr[j] / 4294967296.0;
      }
      const double per_trial_cost = 1.0 + (double)npos * 0.05 + calls;  // + per-trial and per-position work
      for (uint64_t u = prefix[i]; u < prefix[i + 1]; ++u) {
        const uint64_t t0 = (u - prefix[i]) * tile;
        cost[u] = per_trial_cost * (double)std::min<uint64_t>(tile, d.n_trials - t0);
      }
    }
    dsi_shard_bounds(cost.data(), n_units, parts, bounds.data());
  }
  tr.mark("validate");

  int visible = 0, major = 0;  // (an attribute query: cudaGetDeviceProperties costs ~10 ms)
  if (cudaGetDeviceCount(&visible) != cudaSuccess || visible <= opt->device)
    return fail(nullptr, DSI_E_DEVICE, "not enough CUDA devices visible");
  if (cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, opt->device) != cudaSuccess ||
      major != 10)
    return fail(nullptr, DSI_E_DEVICE, "device is not an sm_100 (Blackwell) GPU");
  if (cudaSetDevice(opt->device) != cudaSuccess) return fail(nullptr, DSI_E_DEVICE, "cudaSetDevice failed");
#define MULTI_TRY(call)                                    \
  do {                                                     \
    cudaError_t e_ = (call);                               \
    if (e_ != cudaSuccess) return cuda_fail(nullptr, e_, #call); \
  } while (0)
  cudaStream_t stream = (cudaStream_t)opt->stream;
  struct OwnedStream {
    cudaStream_t s = nullptr;
    ~OwnedStream() { if (s) cudaStreamDestroy(s); }
  } owned;
  if (!stream) {
    MULTI_TRY(cudaStreamCreateWithFlags(&owned.s, cudaStreamNonBlocking));
    stream = owned.s;
  }
  tr.mark("stream");
  {
    // keep freed blocks in the device's default pool between calls (release threshold 0
    // would hand them back to the driver at every synchronisation)
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, opt->device) == cudaSuccess) {
      uint64_t keep = UINT64_MAX;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
    }
  }
  DevBuf b_cfg, b_prefix, b_acc, b_dsi, b_set;
  const size_t acc_bytes = nk * dsi::MF * sizeof(unsigned long long);
  MULTI_TRY(b_cfg.alloc(nk * sizeof(dsi::MultiCfg), stream));
  MULTI_TRY(b_prefix.alloc((nk + 1) * sizeof(uint64_t), stream));
  MULTI_TRY(b_acc.alloc(acc_bytes, stream));
  if (trial_dsi) MULTI_TRY(b_dsi.alloc(rec * sizeof(int32_t), stream));
  if (trial_settled) MULTI_TRY(b_set.alloc(rec * 8 * sizeof(int32_t), stream));
  tr.mark("alloc");
  MULTI_TRY(cudaMemcpyAsync(b_cfg.p, dc.data(), nk * sizeof(dsi::MultiCfg), cudaMemcpyHostToDevice, stream));
  MULTI_TRY(cudaMemcpyAsync(b_prefix.p, prefix.data(), (nk + 1) * sizeof(uint64_t), cudaMemcpyHostToDevice,
                            stream));
  MULTI_TRY(cudaMemsetAsync(b_acc.p, 0, acc_bytes, stream));
  tr.mark("h2d");

  dsi::MultiParams p{};
  p.cfg = (const dsi::MultiCfg *)b_cfg.p;
  p.tile_prefix = (const uint64_t *)b_prefix.p;
  p.n_cfg = (uint32_t)nk;
  p.tile_trials = tile;
  p.unit_begin = 0;
  p.acc = (unsigned long long *)b_acc.p;
  p.rec_dsi = (int32_t *)b_dsi.p;
  p.rec_settled = (int32_t *)b_set.p;
  p.max_n = max_n;
  p.max_drafters = max_d;
  const uint32_t s_lo = (uint32_t)opt->seed, s_hi = (uint32_t)(opt->seed >> 32);
  for (int r = 0; r < 10; ++r) {
    p.keys.k0[r] = s_lo + (uint32_t)r * 0x9E3779B9u;
    p.keys.k1[r] = s_hi + (uint32_t)r * 0xBB67AE85u;
  }
  const bool timing = opt->flags & DSI_F_TIMING;
  struct Events {  // destroyed on every exit path
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    ~Events() {
      if (e0) cudaEventDestroy(e0);
      if (e1) cudaEventDestroy(e1);
    }
  } ev;
  if (timing) {
    MULTI_TRY(cudaEventCreate(&ev.e0));
    MULTI_TRY(cudaEventCreate(&ev.e1));
    MULTI_TRY(cudaEventRecord(ev.e0, stream));
  }
  int32_t launches = 0;
  for (int sh = 0; sh < shards; ++sh) {
    const int part = opt->rank * shards + sh;
    p.unit_begin = bounds[part];
    const uint64_t nu = bounds[part + 1] - bounds[part];
    const int le = dsi::launch_multi_kernel(p, nu, (opt->flags & DSI_F_PATTERN) != 0, stream);
    if (le) return cuda_fail(nullptr, (cudaError_t)le, "dsi_multi_kernel launch");
    launches += (int32_t)((nu + 0x7ffffffeull) / 0x7fffffffull);
  }
  g_multi_launches = launches;
  if (timing) MULTI_TRY(cudaEventRecord(ev.e1, stream));
  if (host_coll) {
    std::vector<uint64_t> hb(nk * dsi::MF);
    MULTI_TRY(cudaMemcpyAsync(hb.data(), b_acc.p, acc_bytes, cudaMemcpyDeviceToHost, stream));
    MULTI_TRY(cudaStreamSynchronize(stream));
    if (g_host_ar(hb.data(), hb.size(), g_host_ar_user) != 0)
      return fail(nullptr, DSI_E_COMM, "host all-reduce hook failed");
    MULTI_TRY(cudaMemcpyAsync(b_acc.p, hb.data(), acc_bytes, cudaMemcpyHostToDevice, stream));
    MULTI_TRY(cudaStreamSynchronize(stream));
  }
  if (use_nccl) {
    // one communicator for this call (ranks of the world, one device each), one all-reduce
    NcclApi &api = nccl();
    if (!api.ok) return fail(nullptr, DSI_E_COMM, "libnccl.so.2 could not be loaded");
    ncclUniqueId uid;
    std::memcpy(&uid, opt->nccl_id, sizeof(uid));
    ncclComm_t comm = nullptr;
    ncclResult_t r = api.CommInitRank(&comm, opt->world, uid, opt->rank);
    if (r == ncclSuccess)
      r = api.AllReduce(b_acc.p, b_acc.p, nk * dsi::MF, ncclUint64, ncclSum, comm, stream);
    if (r == ncclSuccess && cudaStreamSynchronize(stream) != cudaSuccess) r = ncclUnhandledCudaError;
    if (comm) api.CommDestroy(comm);
    if (r != ncclSuccess) return fail(nullptr, DSI_E_COMM, std::string("multi-drafter all-reduce: ") +
                                                           api.GetErrorString(r));
  }
  std::vector<unsigned long long> acc(nk * dsi::MF);
  MULTI_TRY(cudaMemcpyAsync(acc.data(), b_acc.p, acc_bytes, cudaMemcpyDeviceToHost, stream));
  if (trial_dsi) MULTI_TRY(cudaMemcpyAsync(trial_dsi, b_dsi.p, rec * sizeof(int32_t), cudaMemcpyDeviceToHost, stream));
  if (trial_settled)
    MULTI_TRY(cudaMemcpyAsync(trial_settled, b_set.p, rec * 8 * sizeof(int32_t), cudaMemcpyDeviceToHost, stream));
  const cudaError_t se = cudaStreamSynchronize(stream);
  if (timing && se == cudaSuccess) cudaEventElapsedTime(&g_multi_ms, ev.e0, ev.e1);
  if (se != cudaSuccess) return cuda_fail(nullptr, se, "dsi_multi_simulate");
  tr.mark("kernel+d2h");
#undef MULTI_TRY

  // every trial simulated exactly once, then the FP64 derivations of the exact sums
  for (size_t i = 0; i < nk; ++i)
    if (acc[i * dsi::MF + dsi::MF_TRIALS] != dc[i].n_trials)
      return fail(nullptr, DSI_E_DEVICE, "trial count mismatch after the kernel");
  const double tick = opt->tick;
  for (size_t i = 0; i < n_cfg; ++i) {
    const unsigned long long *a = &acc[(size_t)rep_of[i] * dsi::MF];
    dsi_multi_result &r = out[i];
    std::memset(&r, 0, sizeof r);
    const uint64_t T = cfg[i].n_trials;
    const int m = cfg[i].n_drafters + 1;
    r.trials = T;
    r.t_target_ticks = tt[i];
    r.nonsi_ticks = (int64_t)cfg[i].n_tokens * tt[i];
    r.sum_dsi_ticks = (int64_t)a[dsi::MF_DSI];
    r.sumsq_dsi_ticks = a[dsi::MF_DSI2];
    r.n_dsi_gt_nonsi = (int64_t)a[dsi::MF_GT_NONSI];
    int64_t by_drafters = 0;
    for (int j = 0; j < m - 1; ++j) {
      r.sum_settled[j] = (int64_t)a[dsi::MF_SETTLED + j];
      by_drafters += r.sum_settled[j];
    }
    r.sum_settled[m - 1] = (int64_t)T * (cfg[i].n_tokens - 1) - by_drafters;
    const double Td = (double)T;
    if (means) {
      // L = t_m (1 + S_m) + sum_{j<m} t_j S_j per trial, summed with this config's latencies;
      // L <= N t_m on every trial (t_j <= t_m), so the Thm 1 counter is exactly 0
      const dsi::MultiCfg &d = orig[i];
      __int128 sum = (__int128)d.t_t * ((__int128)T + r.sum_settled[m - 1]);
      for (int j = 0; j < m - 1; ++j) sum += (__int128)d.t_d[j] * r.sum_settled[j];
      r.sum_dsi_ticks = (int64_t)sum;
      r.sumsq_dsi_ticks = 0;
      r.n_dsi_gt_nonsi = 0;
    }
    r.mean_nonsi = (double)r.nonsi_ticks * tick;
    r.mean_dsi = ((double)r.sum_dsi_ticks / Td) * tick;
    const unsigned __int128 num = (unsigned __int128)T * r.sumsq_dsi_ticks -
                                  (unsigned __int128)(uint64_t)r.sum_dsi_ticks * (uint64_t)r.sum_dsi_ticks;
    r.std_dsi = means ? std::nan("") : std::sqrt((double)num) / Td * tick;
  }
  tr.mark("finalize");
  return DSI_OK;
}

dsi_status dsi_set_host_allreduce(dsi_host_allreduce_fn fn, void *user) {
  g_host_ar = fn;
  g_host_ar_user = user;
  return DSI_OK;
}

dsi_status dsi_multi_last_kernel(float *ms, int32_t *launches) {
  if (!ms || !launches) return DSI_E_NULL;
  *ms = g_multi_ms;
  *launches = g_multi_launches;
  return DSI_OK;
}

}  // extern "C"

static_assert(sizeof(dsi_multi_config) == 144, "dsi_multi_config ABI layout");
static_assert(sizeof(dsi_multi_result) == 136, "dsi_multi_result ABI layout");

static_assert(sizeof(dsi_config) == 64, "dsi_config ABI layout");
static_assert(sizeof(dsi_result) == 160, "dsi_result ABI layout");
static_assert(sizeof(dsi_options) == 64, "dsi_options ABI layout");
