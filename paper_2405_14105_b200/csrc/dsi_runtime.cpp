// dsi_runtime.cpp -- the handle: create (validate, plan, shard, allocate, upload, NCCL
// communicator), update, run (kernel launches), reduce (all-reduce, partition check, FP64
// finalize), the device heatmap product, and the accessors / measurement hooks.
#include "dsi_host.h"

#include <atomic>

using namespace dsih;

namespace dsih {

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
  cudaFree(d.d_owned);
  cudaFree(d.d_raw);
  cudaFree(d.d_raw_next);
  cudaFree(d.d_cfg_next);
  cudaFree(d.d_stage);
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
  h->raw_pinned.release();
  h->stage_host.release();
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
dsi_status upload(dsi_sim *h, bool plan, bool cfg_table) {
  for (auto &d : h->dev) {
    CUDA_TRY(h, cudaSetDevice(d.ordinal));
    if (cfg_table)
      CUDA_TRY(h, cudaMemcpyAsync(d.d_cfg, h->dev_cfg.p, h->n_cfg * sizeof(DevCfg), cudaMemcpyHostToDevice,
                                  d.stream));
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

// Device buffers of the two-pass mode (sized by plan_two_pass; grown if an update needs more).
dsi_status alloc_two_pass(dsi_sim *h) {
  if (!h->two_pass) return DSI_OK;
  for (auto &d : h->dev) {
    CUDA_TRY(h, cudaSetDevice(d.ordinal));
    // capacities in bytes: an update that raises N grows every record (rec_bytes) even when
    // the record count stays the same
    const size_t rec_need = std::max<uint64_t>(1, h->total_records) * (size_t)h->rec_bytes;
    if (rec_need > d.records_cap || !d.d_records) {
      cudaFree(d.d_records);
      d.d_records = nullptr;
      d.records_cap = 0;
      CUDA_TRY(h, cudaMalloc((void **)&d.d_records, rec_need));
      d.records_cap = rec_need;
    }
    const size_t g_need = h->group_tile0.size() * sizeof(uint64_t);
    if (g_need > d.group_tile0_cap || !d.d_group_tile0) {
      cudaFree(d.d_group_tile0);
      d.d_group_tile0 = nullptr;
      d.group_tile0_cap = 0;
      CUDA_TRY(h, cudaMalloc((void **)&d.d_group_tile0, g_need));
      d.group_tile0_cap = g_need;
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

namespace {

constexpr dsi_status kHostPath = (dsi_status)-1;  // update_on_device: take the host path

bool device_update_eligible(const dsi_sim *h) {
  return h->dev.size() == 1 && !(h->opt.flags & (DSI_F_PER_TRIAL | DSI_F_HIST | DSI_F_PATTERN));
}

// The configurations as given into device memory `dst` on device 0's stream: straight from a
// caller's page-locked buffer, else through the pinned staging in slices (a parallel host copy of
// slice i while slice i-1 is in flight).  Asynchronous; the staging is reused by the next call
// only after a stream synchronization.
dsi_status copy_raw(dsi_sim *h, const dsi_config *cfg, dsi_config *dst) {
  DeviceState &d = h->dev[0];
  const size_t n = h->n_cfg;
  cudaPointerAttributes attr{};
  const bool pinned = cudaPointerGetAttributes(&attr, cfg) == cudaSuccess && attr.type == cudaMemoryTypeHost;
  cudaGetLastError();  // (a pageable pointer may leave an error behind on older drivers)
  if (pinned) {
    CUDA_TRY(h, cudaMemcpyAsync(dst, cfg, n * sizeof(dsi_config), cudaMemcpyHostToDevice, d.stream));
    return DSI_OK;
  }
  if (h->raw_pinned.n < n) CUDA_TRY(h, h->raw_pinned.alloc(n));
  constexpr size_t kSlices = 8;
  for (size_t sl = 0; sl < kSlices; ++sl) {
    const size_t b = n * sl / kSlices, e = n * (sl + 1) / kSlices;
    if (e <= b) continue;
    parallel_for(e - b, [&](size_t lo, size_t hi) {
      std::memcpy(h->raw_pinned.p + b + lo, cfg + b + lo, (hi - lo) * sizeof(dsi_config));
    }, 1u << 14);
    CUDA_TRY(h, cudaMemcpyAsync(dst + b, h->raw_pinned.p + b, (e - b) * sizeof(dsi_config), cudaMemcpyHostToDevice,
                                d.stream));
  }
  return DSI_OK;
}

dsi_status alloc_device_update(dsi_sim *h) {
  DeviceState &d = h->dev[0];
  CUDA_TRY(h, cudaSetDevice(d.ordinal));
  const size_t n = std::max<size_t>(1, h->n_cfg);
  if (!d.d_raw) CUDA_TRY(h, cudaMalloc((void **)&d.d_raw, n * sizeof(dsi_config)));
  if (!d.d_raw_next) CUDA_TRY(h, cudaMalloc((void **)&d.d_raw_next, n * sizeof(dsi_config)));
  if (!d.d_cfg_next) CUDA_TRY(h, cudaMalloc((void **)&d.d_cfg_next, n * sizeof(DevCfg)));
  if (!d.d_stage) CUDA_TRY(h, cudaMalloc((void **)&d.d_stage, sizeof(dsi::StageStatus)));
  if (!h->stage_host.p) CUDA_TRY(h, h->stage_host.alloc(1));
  return DSI_OK;
}

// The device path of dsi_sim_update: copy the configurations as given, validate and convert them on
// the GPU into the spare table (dsi_stage.cu), and commit -- swap the tables -- when every config
// is valid, n_trials unchanged, the launch limits unchanged and no plan needs rebuilding (the
// shared-stream plan or the means-only groups).  kHostPath otherwise: the host path then reports
// the error (with its message) or re-plans.  On commit the host tick table becomes stale; it is
// rebuilt from the device copy of the configurations when a host step needs it (ensure_ticks).
dsi_status update_on_device(dsi_sim *h, const dsi_config *cfg, Trace &tr) {
  if (!h->raw_valid) return kHostPath;
  dsi_status s = alloc_device_update(h);
  if (s != DSI_OK) return s;
  DeviceState &d = h->dev[0];
  s = copy_raw(h, cfg, d.d_raw_next);
  if (s != DSI_OK) return s;
  dsi::StageStatus init{};
  init.first_bad = ~0ull;
  init.max_n = init.max_keff = 1;
  *h->stage_host.p = init;
  CUDA_TRY(h, cudaMemcpyAsync(d.d_stage, h->stage_host.p, sizeof init, cudaMemcpyHostToDevice, d.stream));
  dsi::StageParams p{};
  p.raw = d.d_raw_next;
  p.prev = d.d_raw;
  p.out = d.d_cfg_next;
  p.n = h->n_cfg;
  p.tick = h->opt.tick;
  p.flags = h->opt.flags;
  p.st = d.d_stage;
  const int e = dsi::launch_stage_kernel(p, d.stream);
  if (e) return cuda_fail(h, (cudaError_t)e, "config staging launch");
  CUDA_TRY(h, cudaMemcpyAsync(h->stage_host.p, d.d_stage, sizeof init, cudaMemcpyDeviceToHost, d.stream));
  CUDA_TRY(h, cudaStreamSynchronize(d.stream));
  tr.mark("device-stage");
  const dsi::StageStatus st = *h->stage_host.p;
  const bool ttft = st.flags & dsi::STAGE_TTFT, fresh = st.flags & dsi::STAGE_FRESH;
  if (st.first_bad != ~0ull) return kHostPath;
  if (st.max_n != h->max_n || st.max_keff != h->max_keff || ttft != h->any_ttft || fresh != h->any_fresh)
    return kHostPath;
  if (h->shared && (st.flags & dsi::STAGE_PLAN_CHANGED)) return kHostPath;
  if (h->means_only && (st.flags & dsi::STAGE_GROUPS_CHANGED)) return kHostPath;
  // commit
  std::swap(d.d_cfg, d.d_cfg_next);
  std::swap(d.d_raw, d.d_raw_next);
  h->ticks_stale = true;
  h->k1_fast = !ttft && !fresh && st.work_k1 >= 0.25 * st.work;
  if (knobs().k1_fast >= 0) h->k1_fast = !ttft && !fresh && knobs().k1_fast != 0;
  h->ran = h->reduced = h->reduced_device = false;
  if (st.flags & dsi::STAGE_CELLS_CHANGED) h->heat_planned = h->heat_uploaded = false;
  return DSI_OK;
}

}  // namespace

// The host tick table after device updates: rebuilt from the device copy of the current
// configurations, which were validated when they were committed.
dsi_status ensure_ticks(dsi_sim *h) {
  if (!h->ticks_stale) return DSI_OK;
  DeviceState &d = h->dev[0];
  CUDA_TRY(h, cudaSetDevice(d.ordinal));
  if (h->raw_pinned.n < h->n_cfg) CUDA_TRY(h, h->raw_pinned.alloc(h->n_cfg));
  CUDA_TRY(h, cudaMemcpyAsync(h->raw_pinned.p, d.d_raw, h->n_cfg * sizeof(dsi_config), cudaMemcpyDeviceToHost,
                              d.stream));
  CUDA_TRY(h, cudaStreamSynchronize(d.stream));
  const dsi_status s = validate_all(h, h->raw_pinned.p, h->n_cfg, h->ticks);
  if (s != DSI_OK) return s;
  // (the pinned device-table staging is read only by the test modes' accessors, which never take
  // the device path, and rewritten by every host-path update)
  h->ticks_stale = false;
  return DSI_OK;
}

}  // namespace dsih

extern "C" {

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
                         DSI_F_REDUCE_TO_ROOT | DSI_F_RNG_HALVES;
  if (opt->flags & ~known) return fail(nullptr, DSI_E_RANGE, "unknown flag");
  if (opt->n_devices != 1)
    return fail(nullptr, DSI_E_RANGE, "n_devices must be 1: run one process per GPU (rank/world/nccl_id)");
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
  const bool host_coll = host_hook_set() && opt->world > 1;
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
  if (shared && (opt->flags & (DSI_F_PER_TRIAL | DSI_F_HIST | DSI_F_PATTERN)))
    return fail(nullptr, DSI_E_RANGE, "DSI_F_SHARED_STREAMS excludes PER_TRIAL, HIST and PATTERN");

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
    // dsi_sim_update validates into this spare table: allocated (and its pages touched by the
    // zero fill) here, so the first update does not pay ~0.1 s of page faults for 2.02e6 configs
    h->ticks_next.resize(n_cfg);
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
    // the TTFT configs' own (config, tile) units for the per-config kernel (zero units elsewhere)
    uint64_t ttft_trials = 0;
    for (const uint32_t c : h->shared_ttft) ttft_trials += h->ticks[c].trials;
    const uint64_t r = std::min<uint64_t>(
        128, std::max<uint64_t>(1, ttft_trials / ((uint64_t)kDefaultThreads * 148ull * 16 * 8 * total_devices)));
    h->tile_trials = (uint32_t)(kDefaultThreads * r);
    std::vector<char> is_ttft(n_cfg, 0);
    for (const uint32_t c : h->shared_ttft) is_ttft[c] = 1;
    h->prefix[0] = 0;
    for (size_t i = 0; i < n_cfg; ++i)
      h->prefix[i + 1] = h->prefix[i] + (is_ttft[i] ? (h->ticks[i].trials + h->tile_trials - 1) / h->tile_trials : 0);
    h->ttft_units = h->prefix[n_cfg];
  } else {
    const uint64_t threads = (uint64_t)h->block_threads;
    const uint64_t target_blocks = 148ull * 16 * 8 * (uint64_t)total_devices;
    uint64_t r = h->total_trials / (threads * target_blocks);
    // up to 128 x 128 trials per unit: whole configs of the paper's grids in one unit
    // (measured, profiles/r01_ab_tile.jsonl: cap 32 -> 128 is 0.65% faster on cfg3)
    r = std::min<uint64_t>(128, std::max<uint64_t>(1, r));
    if (knobs().tile_r >= 1 && knobs().tile_r <= 1024) r = (uint64_t)knobs().tile_r;
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
    std::vector<uint64_t> cand;  // unit indices a part may start at and still hold whole heatmap cells
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
    // SURVEY 8(e)'s cell-aligned option: parts snapped to heatmap-cell starts (per-config mode:
    // the first unit of each cell) or group starts (shared-stream mode, units in group order: a
    // cell's configs are all in one group) when that costs <= 4% balance; dsi_sim_heatmap then
    // exchanges the cells instead of every config's moments (means-only snaps its config ranges
    // below)
    if (parts > 1 && !means_only) {
      try {
        plan_heat_cells(h);
        h->heat_planned = true;
        if (shared) {
          bool ordered = true;
          for (size_t u = 1; u < h->crn_units.size() && ordered; ++u)
            ordered = h->crn_units[u].group >= h->crn_units[u - 1].group;
          for (size_t u = 0; ordered && u < h->crn_units.size(); ++u)
            if (u == 0 || h->crn_units[u].group != h->crn_units[u - 1].group) cand.push_back(u);
        } else {
          for (const dsi::HeatCell &c : h->heat_cells) cand.push_back(h->prefix[c.first]);
        }
        // the exchange a snapped partition saves: the 64-byte moments of every config through an
        // all-reduce at ~400 GB/s, 0.16 ns per config -- 160 cost units (1 unit ~ 1 ps of kernel
        // time, profiles/r02_cost_probe*.jsonl)
        snap_bounds(bounds, cost, cand, 160.0 * (double)n_cfg);
      } catch (...) {
        h->err = "host tables";
        return abort_create(DSI_E_NOMEM);
      }
    }
    h->part_bounds = bounds;
  }
  // shared-stream mode: the TTFT configs' per-config units, cost-balanced over the same parts
  std::vector<uint64_t> ttft_bounds(parts + 1, 0);
  if (shared && h->ttft_units) {
    try {
      std::vector<double> tc(h->ttft_units);
      for (const uint32_t c : h->shared_ttft)
        for (uint64_t u = h->prefix[c]; u < h->prefix[c + 1]; ++u) {
          const uint64_t first = (u - h->prefix[c]) * h->tile_trials;
          tc[u] = unit_cost(h->ticks[c], std::min<uint64_t>(h->tile_trials, h->ticks[c].trials - first));
        }
      dsi_shard_bounds(tc.data(), h->ttft_units, parts, ttft_bounds.data());
    } catch (...) {
      h->err = "host tables";
      return abort_create(DSI_E_NOMEM);
    }
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
      if (shared && h->ttft_units) d.ttft_ranges.emplace_back(ttft_bounds[part], ttft_bounds[part + 1]);
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
  if (h->heat_planned) {
    try {
      plan_cell_owners(h);
    } catch (...) {
      h->err = "host tables";
      return abort_create(DSI_E_NOMEM);
    }
  }
  if (shared) {
    s = plan_two_pass(h);
    if (s == DSI_OK) s = alloc_two_pass(h);
    if (s != DSI_OK) return abort_create(s);
  }
  s = upload(h);
  if (s != DSI_OK) return abort_create(s);
  if (device_update_eligible(h)) {  // the device copy a device update compares with (dsi_stage.cu)
    s = alloc_device_update(h);
    if (s == DSI_OK) s = copy_raw(h, cfg, h->dev[0].d_raw);
    if (s != DSI_OK) return abort_create(s);
    h->raw_valid = true;
  }
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
  if (device_update_eligible(h)) {
    const dsi_status sd = update_on_device(h, cfg, tr);
    if (sd != kHostPath) return sd;
  }
  {  // the host path compares with the current ticks
    const dsi_status se = ensure_ticks(h);
    if (se != DSI_OK) return se;
  }
  // validate into the spare table; h->ticks (and the whole handle) stay as they are on failure
  try {
    h->ticks_next.resize(n_cfg);
  } catch (...) {
    return fail(h, DSI_E_NOMEM, "host tables");
  }
  const int32_t old_n = h->max_n, old_keff = h->max_keff;
  const bool old_ttft = h->any_ttft, old_fresh = h->any_fresh;
  UpdateKeys keys;
  dsi_status s = validate_all(h, cfg, n_cfg, h->ticks_next, &h->ticks, &keys);
  tr.mark("validate");
  if (s == DSI_OK) s = derive_limits(h, h->ticks_next);  // the new configs may need a larger launch shape
  if (s != DSI_OK) return s;                              // derive_limits only commits on success
  if (h->means_only) {  // the histogram groups are fixed at create: their keys must not change
    const bool same = h->max_n <= kMeansMaxN && keys.groups_same;
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
  const bool replan = h->shared && !keys.plan_same;
  tr.mark("limits");
  if (replan) {
    // re-plan on the host first: the unit table's size is fixed at create
    const int32_t old_cpb = h->cfg_per_block, old_runs = h->max_runs;
    std::vector<uint32_t> old_perm;
    std::vector<dsi::CrnGroup> old_groups;
    std::vector<dsi::CrnUnit> old_units;
    std::vector<uint32_t> old_shared_ttft;
    h->ticks.swap(h->ticks_next);
    try {
      old_perm = h->perm;
      old_groups = h->groups;
      old_units = h->crn_units;
      old_shared_ttft = h->shared_ttft;
      std::vector<double> cost;
      s = plan_shared(h, cost);
    } catch (...) {
      s = fail(h, DSI_E_NOMEM, "host tables");
    }
    if (s == DSI_OK && (h->groups.size() != old_groups.size() || h->crn_units.size() != old_units.size() ||
                        h->shared_ttft != old_shared_ttft))
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
      if (!old_groups.empty() || !old_shared_ttft.empty()) {
        h->perm.swap(old_perm);
        h->groups.swap(old_groups);
        h->crn_units.swap(old_units);
        h->shared_ttft.swap(old_shared_ttft);
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
  // the staging table is filled in slices, each slice's DMA enqueued as soon as it is filled
  CUDA_TRY(h, fill_dev_cfg(h, /*upload_chunks=*/true));
  tr.mark("fill+upload");
  h->ran = h->reduced = h->reduced_device = false;
  if (!keys.cells_same || replan) h->heat_planned = h->heat_uploaded = false;  // else the cells stand
  dsi_status su = upload(h, replan, /*cfg_table=*/false);
  tr.mark("upload");
  if (su == DSI_OK && device_update_eligible(h)) {  // the device copy the next device update compares with
    su = alloc_device_update(h);
    if (su == DSI_OK) su = copy_raw(h, cfg, h->dev[0].d_raw);
    if (su == DSI_OK) CUDA_TRY(h, cudaStreamSynchronize(h->dev[0].stream));  // (the staging is reused)
    h->raw_valid = su == DSI_OK;
  }
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
  q.halves = (h->opt.flags & DSI_F_RNG_HALVES) ? 1 : 0;
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
    p.halves = (h->opt.flags & DSI_F_RNG_HALVES) ? 1 : 0;
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
      q.any_fresh = h->any_fresh ? 1 : 0;
      q.halves = p.halves;
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
      for (const auto &rg : d.ttft_ranges) {  // the TTFT configs: per-config kernel (TTFT variant)
        if (rg.second <= rg.first) continue;
        p.unit_begin = rg.first;
        const int e = dsi::launch_trial_kernel(p, rg.second - rg.first, kDefaultThreads, false, false, false, d.stream);
        if (e) return cuda_fail(h, (cudaError_t)e, "trial kernel launch (TTFT configs)");
        h->launches += 1;
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
  h->reduced = h->reduced_device = false;
  return DSI_OK;
}

namespace {

// The exchange step, enqueued: the cross-rank all-reduce of the moments, the partition check
// (every trial simulated exactly once) on the device and its flag copied back.  Asynchronous
// on device 0's stream; with DSI_F_REDUCE_TO_ROOT on a rank != 0 only the all-reduce.
dsi_status reduce_enqueue(dsi_sim *h, bool hist) {
  dsi_status st = sum_across(h, hist);
  if (st != DSI_OK) return st;
  if ((h->opt.flags & DSI_F_REDUCE_TO_ROOT) && h->opt.rank != 0) return DSI_OK;
  DeviceState &d0 = h->dev[0];
  CUDA_TRY(h, cudaSetDevice(d0.ordinal));
  const unsigned long long *src = h->use_nccl ? d0.d_red : d0.d_acc;
  if (!d0.d_heat_bad) CUDA_TRY(h, cudaMalloc((void **)&d0.d_heat_bad, sizeof(unsigned int)));
  if (!h->chunk_ev[0])
    for (auto &ev : h->chunk_ev) CUDA_TRY(h, cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
  CUDA_TRY(h, cudaMemsetAsync(d0.d_heat_bad, 0, sizeof(unsigned int), d0.stream));
  const int e = dsi::launch_check_trials(d0.d_cfg, src, h->n_cfg, d0.d_heat_bad, d0.stream);
  if (e) return cuda_fail(h, (cudaError_t)e, "partition check launch");
  h->launches += 1;
  CUDA_TRY(h, cudaMemcpyAsync(h->host_bad.p, d0.d_heat_bad, sizeof(unsigned int), cudaMemcpyDeviceToHost,
                              d0.stream));
  return DSI_OK;
}

// Wait for every device's stream (the all-reduce ran on each).
dsi_status sync_all(dsi_sim *h) {
  for (auto &d : h->dev) {
    CUDA_TRY(h, cudaSetDevice(d.ordinal));
    CUDA_TRY(h, cudaStreamSynchronize(d.stream));
  }
  return DSI_OK;
}

// Results [first, first + count) from the reduced moments on device 0: chunked D2H into the
// pinned mirror, the host finalizing chunk i while chunk i+1 is in flight.  The partition flag
// (reduce_enqueue) is checked before any result is written.
dsi_status finalize_range(dsi_sim *h, size_t first, size_t count, dsi_result *out, Trace &tr) {
  {
    const dsi_status se = ensure_ticks(h);  // (after device updates: the finalize reads the ticks)
    if (se != DSI_OK) return se;
  }
  DeviceState &d0 = h->dev[0];
  CUDA_TRY(h, cudaSetDevice(d0.ordinal));
  const unsigned long long *src = h->use_nccl ? d0.d_red : d0.d_acc;
  const size_t n_chunks = count < (1u << 16) ? 1 : kReduceChunks;
  for (size_t c = 0; c < n_chunks; ++c) {
    const size_t b = first + count * c / n_chunks, e = first + count * (c + 1) / n_chunks;
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
  const size_t cb = first + count * c / n_chunks, ce = first + count * (c + 1) / n_chunks;
  if (c) CUDA_TRY(h, cudaEventSynchronize(h->chunk_ev[c]));
  parallel_for(ce - cb, [&](size_t b, size_t e) {
  for (size_t i = cb + b; i < cb + e; ++i) {
    const unsigned long long *a = &h->host_acc.p[i * dsi::NF];
    const CfgTicks &t = h->ticks[i];
    dsi_result &r = out[i - first];
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
  return DSI_OK;
}

}  // namespace

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
  dsi_status st = reduce_enqueue(h, hist);
  if (st != DSI_OK) return st;
  tr.mark("allreduce-enqueue");
  if (root_only) {  // DSI_F_REDUCE_TO_ROOT: this rank contributed its sums; rank 0 checks and finalizes
    st = sync_all(h);
    if (st != DSI_OK) return st;
    h->reduced = h->reduced_device = true;
    return DSI_OK;
  }
  // every device now holds the global sums (or there is one device): read device 0
  DeviceState &d0 = h->dev[0];
  CUDA_TRY(h, cudaSetDevice(d0.ordinal));
  if (hist) {
    CUDA_TRY(h, cudaMemcpyAsync(h->host_seg.p, h->use_nccl ? d0.d_seg_red : d0.d_seg,
                                n_cfg * 64 * sizeof(unsigned long long), cudaMemcpyDeviceToHost, d0.stream));
    CUDA_TRY(h, cudaMemcpyAsync(h->host_si.p, h->use_nccl ? d0.d_si_red : d0.d_si,
                                h->si_bins_total * sizeof(unsigned long long), cudaMemcpyDeviceToHost,
                                d0.stream));
  }
  st = finalize_range(h, 0, n_cfg, out, tr);
  if (st != DSI_OK) return st;
  CUDA_TRY(h, cudaStreamSynchronize(d0.stream));  // the histogram copies (HIST), if any
  tr.mark("finalize");
  h->reduced = h->reduced_device = true;
  return DSI_OK;
}

dsi_status dsi_sim_reduce_device(dsi_sim *h) {
  if (!h) return DSI_E_NULL;
  Trace tr("dsi_sim_reduce_device");
  h->err.clear();
  if (!h->ran) return fail(h, DSI_E_STATE, "dsi_sim_reduce_device before dsi_sim_run");
  if (h->opt.flags & DSI_F_HIST) return fail(h, DSI_E_STATE, "DSI_F_HIST needs dsi_sim_reduce");
  const dsi_status st = reduce_enqueue(h, false);
  if (st != DSI_OK) return st;
  h->reduced_device = true;
  return DSI_OK;
}

dsi_status dsi_sim_fetch(dsi_sim *h, size_t first, size_t count, dsi_result *out) {
  if (!h) return DSI_E_NULL;
  Trace tr("dsi_sim_fetch");
  h->err.clear();
  if (!out && count) return fail(h, DSI_E_NULL, "out is NULL");
  if (first > h->n_cfg || count > h->n_cfg - first) return fail(h, DSI_E_RANGE, "[first, first + count) exceeds n_cfg");
  if (!h->reduced_device) return fail(h, DSI_E_STATE, "dsi_sim_fetch before dsi_sim_reduce_device");
  if ((h->opt.flags & DSI_F_REDUCE_TO_ROOT) && h->opt.rank != 0)
    return fail(h, DSI_E_STATE, "DSI_F_REDUCE_TO_ROOT: results are on rank 0");
  if (!count) return DSI_OK;
  return finalize_range(h, first, count, out, tr);
}

dsi_status dsi_sim_heatmap(dsi_sim *h, dsi_heatmap_cell *cells, size_t cap, size_t *n_cells) {
  if (!h) return DSI_E_NULL;
  Trace tr("dsi_sim_heatmap");
  h->err.clear();
  if (!n_cells) return fail(h, DSI_E_NULL, "n_cells is NULL");
  if (!h->heat_planned) {  // cells: maximal runs of equal (t_target, t_drafter, a, SP, N)
    const dsi_status se = ensure_ticks(h);
    if (se != DSI_OK) return se;
    try {
      plan_heat_cells(h);
      plan_cell_owners(h);
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
  if (!local && !h->reduced_device) {  // (dsi_sim_reduce_device already summed the moments)
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
    const size_t no = d0.owned_cells.size();
    if (no > d0.owned_cap) {
      cudaFree(d0.d_owned);
      d0.d_owned = nullptr;
      d0.owned_cap = 0;
      CUDA_TRY(h, cudaMalloc((void **)&d0.d_owned, no * sizeof(uint32_t)));
      d0.owned_cap = no;
    }
    if (no)
      CUDA_TRY(h, cudaMemcpyAsync(d0.d_owned, d0.owned_cells.data(), no * sizeof(uint32_t), cudaMemcpyHostToDevice,
                                  d0.stream));
    CUDA_TRY(h, cudaStreamSynchronize(d0.stream));  // the vectors are pageable
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
    p.idx = d0.d_owned;
    p.n_cells = (uint32_t)d0.owned_cells.size();
    if (p.n_cells) {
      const int e = dsi::launch_heatmap_kernel(p, d0.stream);
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
  // an update's upload: the configurations as given (device path) or the device table (host path)
  *h2d = (uint64_t)h->dev.size() * n * (device_update_eligible(h) ? sizeof(dsi_config) : sizeof(DevCfg));
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

}  // extern "C"

static_assert(sizeof(dsi_config) == 64, "dsi_config ABI layout");
static_assert(sizeof(dsi_result) == 160, "dsi_result ABI layout");
static_assert(sizeof(dsi_options) == 64, "dsi_options ABI layout");
