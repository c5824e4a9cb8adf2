// dsi_multi_host.cpp -- multi-drafter DSI: dsi_multi_simulate, one
// device per process, one kernel per call, exact sums and FP64 means.
#include "dsi_host.h"

using namespace dsih;

extern "C" {

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
  if (opt->flags & ~(DSI_F_PER_TRIAL | DSI_F_PATTERN | DSI_F_TIMING | DSI_F_MEANS_ONLY | DSI_F_RNG_HALVES))
    return fail(nullptr, DSI_E_RANGE,
                "multi-drafter mode takes PER_TRIAL, PATTERN, TIMING, MEANS_ONLY and RNG_HALVES only");
  const bool means = opt->flags & DSI_F_MEANS_ONLY;
  if (means && (opt->flags & DSI_F_PER_TRIAL))
    return fail(nullptr, DSI_E_RANGE, "DSI_F_MEANS_ONLY excludes DSI_F_PER_TRIAL");
  if (opt->n_devices != 1 || opt->device < 0)
    return fail(nullptr, DSI_E_RANGE, "multi-drafter mode drives one device per process (n_devices = 1)");
  if (opt->world < 1 || opt->rank < 0 || opt->rank >= opt->world)
    return fail(nullptr, DSI_E_RANGE, "need 0 <= rank < world");
  if (opt->n_shards < 0 || opt->n_shards > 4096 || (opt->n_shards > 1 && opt->world > 1))
    return fail(nullptr, DSI_E_RANGE, "n_shards must be 0..4096 and > 1 only with world == 1");
  const bool host_coll = host_hook_set() && opt->world > 1;
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
  p.halves = (opt->flags & DSI_F_RNG_HALVES) ? 1 : 0;
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
    if (!host_hook_sum(hb.data(), hb.size()))
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

dsi_status dsi_multi_last_kernel(float *ms, int32_t *launches) {
  if (!ms || !launches) return DSI_E_NULL;
  *ms = g_multi_ms;
  *launches = g_multi_launches;
  return DSI_OK;
}

}  // extern "C"

static_assert(sizeof(dsi_multi_config) == 144, "dsi_multi_config ABI layout");
static_assert(sizeof(dsi_multi_result) == 136, "dsi_multi_result ABI layout");
