// dsi_plan.cpp -- work plans: the device config table, means-only histogram groups,
// shared-stream groups/slices/units (and the two-pass record plan), heatmap cells.
#include "dsi_host.h"

#include <algorithm>
#include <cmath>

using namespace dsih;

namespace dsih {

// Fill the pinned device-config staging table from h->ticks.  upload_chunks (dsi_sim_update,
// after validation succeeded and the streams are idle): the table is filled in kSlices slices and
// each slice's H2D copy is enqueued on every device's stream as soon as it is filled, so the DMA
// overlaps the filling of the rest.  Returns the first CUDA error of those copies.
cudaError_t fill_dev_cfg(dsi_sim *h, bool upload_chunks) {
  const bool pattern = h->opt.flags & DSI_F_PATTERN;
  const bool fresh = h->opt.flags & DSI_F_FRESH_VERIFIER;
  const size_t n = h->n_cfg;
  // prefix offsets (per-trial records, SI-histogram bins) in two passes over fixed chunks
  constexpr size_t K = 256, kSlices = 8;
  std::vector<uint64_t> rec(K + 1, 0), sib(K + 1, 0);
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
  for (size_t sl = 0; sl < kSlices; ++sl) {
    const size_t c0 = K * sl / kSlices, c1 = K * (sl + 1) / kSlices;
    parallel_for(c1 - c0, [&](size_t b, size_t e) {
      for (size_t c = c0 + b; c < c0 + e; ++c) {
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
    if (upload_chunks) {
      const size_t i0 = n * c0 / K, i1 = n * c1 / K;
      for (auto &d : h->dev) {
        if (i1 <= i0) continue;
        cudaError_t e = cudaSetDevice(d.ordinal);
        if (e == cudaSuccess)
          e = cudaMemcpyAsync(d.d_cfg + i0, h->dev_cfg.p + i0, (i1 - i0) * sizeof(DevCfg), cudaMemcpyHostToDevice,
                              d.stream);
        if (e != cudaSuccess) return e;
      }
    }
  }
  return cudaSuccess;
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

// The two-pass form needs 256-thread blocks, pass 2's two tile buffers within room for 3 blocks
// per SM (its register budget) and, with the fresh-verifier layout's 6-bit short-run counts, at
// most 63 stored runs per trial.
static bool two_pass_eligible(const dsi_sim *h, int th) {
  const bool ok = th == 256 && dsi::crn_eval_smem(h->max_runs, th, h->any_fresh) <= 64 * 1024 &&
                  (!h->any_fresh || h->max_runs <= 63);
  return knobs().crn_two_pass >= 0 ? ok && knobs().crn_two_pass != 0 : ok;
}

// Two-pass shared-stream mode (dsi_crn2.cu): records of (group, tile of TH trials), and
// for every device the tiles its units read (pass 1 writes exactly those).  Requires
// h->crn_units and the devices' unit ranges.
dsi_status plan_two_pass(dsi_sim *h) {
  const int th = h->cfg_per_block;
  h->two_pass = two_pass_eligible(h, th);
  if (!h->two_pass) return DSI_OK;
  try {
    h->rec_bytes = (uint32_t)dsi::crn_record_bytes(h->max_runs, th, h->any_fresh);
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

dsi_status plan_shared(dsi_sim *h, std::vector<double> &cost) {
  const size_t n = h->n_cfg;
  try {
    h->perm.resize(n);
    for (size_t i = 0; i < n; ++i) h->perm[i] = (uint32_t)i;
    const auto &t = h->ticks;
    // TTFT configs (first forwards cost more, R23) are not shared: their first segment has its own
    // cost table per config, so they run through the per-config kernel (create plans their units);
    // they sort to the end of the order and join no group
    auto ttft = [&](uint32_t i) { return t[i].t_t1 != t[i].t_t || t[i].t_d1 != t[i].t_d; };
    std::stable_sort(h->perm.begin(), h->perm.end(), [&](uint32_t a, uint32_t b) {
      const CfgTicks &x = t[a], &y = t[b];
      if (ttft(a) != ttft(b)) return !ttft(a);
      if (x.stream_id != y.stream_id) return x.stream_id < y.stream_id;
      if (x.thr != y.thr) return x.thr < y.thr;
      if (x.n != y.n) return x.n < y.n;
      if (x.trials != y.trials) return x.trials < y.trials;
      if (x.k != y.k) return x.k < y.k;
      if (x.t_t != y.t_t) return x.t_t < y.t_t;
      if (x.t_d != y.t_d) return x.t_d < y.t_d;
      return x.sp < y.sp;
    });
    size_t n_plain = 0;
    while (n_plain < n && !ttft(h->perm[n_plain])) ++n_plain;
    h->shared_ttft.assign(h->perm.begin() + n_plain, h->perm.end());
    std::sort(h->shared_ttft.begin(), h->shared_ttft.end());
    h->max_runs = h->max_n / 3 + 2;  // runs of >= 2 accepted drafts in one trial
    // groups first, then the block shape: configs per block follow the typical group size
    h->groups.clear();
    for (size_t i = 0; i < n_plain;) {
      const CfgTicks &k0 = t[h->perm[i]];
      size_t j = i + 1;
      while (j < n_plain) {
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
    const bool big_groups = n_plain >= 256 * h->groups.size();
    int th = (big_groups && dsi::crn_kernel_smem(h->max_n, 256, 256, h->max_runs, h->any_fresh) <= 48 * 1024) ? 256 : kCrnThreads;
    if (knobs().crn_threads == 128 || knobs().crn_threads == 256) th = knobs().crn_threads;
    h->cfg_per_block = th;
    h->block_threads = th;
    // units: (group, slice of cfg_per_block configs, range of trials); trials are split
    // until there are enough blocks to fill every SM of every device a few times.  With
    // 128-thread blocks a group's configs are first cut into maximal runs of "sums-only"
    // configs (k_eff = 1 and no queueing: every run of >= 2 accepted drafts is long and
    // the corrections are linear in per-trial sums, no run list needed) and the others;
    // sums-only units go first and run a kernel variant without run lists in shared memory
    // (so many more blocks fit an SM; large N, e.g. config 5, gains most).
    const bool split_sums = th == kCrnThreads && knobs().crn_sums_split != 0;
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
    // unit costs per trial (unit_cost's picoseconds): pass 2 sums its configs' shared_eval_cost;
    // the stream pass (Philox only when 0 < a < 1) runs once per group in the two-pass form
    // (~1.3 ps per token with the record writes: cfg3's pass 1, 0.134 ms for 10^8 trial-tokens;
    // each slice takes its share) and once per slice in the fused form (~0.62 ps per token)
    const bool two = two_pass_eligible(h, th);
    std::vector<double> eval_cost(slices, 0.0);
    for (size_t q = 0; q < slices; ++q)
      for (uint32_t p = slices_v[q].begin; p < slices_v[q].begin + slices_v[q].count; ++p)
        eval_cost[q] += shared_eval_cost(t[h->perm[p]], (h->opt.flags & DSI_F_FRESH_VERIFIER) != 0, two);
    auto stream_cost = [&](const Slice &sl) {
      const dsi::CrnGroup &g = h->groups[sl.group];
      const bool st = g.mode == dsi::MODE_STREAM;
      return two ? (double)g.n_tokens * (st ? 1.3 : 0.05) * sl.count / g.count
                 : (double)g.n_tokens * (st ? 0.62 : 0.05);
    };
    const int total_devices = h->opt.world * h->opt.n_devices;
    const uint64_t target = 148ull * 4 * 4 * (uint64_t)total_devices;
    const uint64_t split = slices ? std::max<uint64_t>(1, (target + slices - 1) / slices) : 1;  // (all TTFT: no slice)
    // a slice's trials are also cut until no unit costs more than 1/8 of a wave of blocks
    // (148 SMs x 3 resident blocks) on every device: one block is one unit, so the costliest
    // slices (a ~ 0.5-0.9 at small k: ~10x the cheapest) would otherwise run as a tail of long
    // blocks that no shard count shortens (profiles/r02_split_probe*: cfg3, half the blocks
    // took 80% of the time)
    double total_cost = 0.0;
    for (size_t q = 0; q < slices; ++q)
      total_cost += (double)h->groups[slices_v[q].group].n_trials * (stream_cost(slices_v[q]) + eval_cost[q]);
    const double cap = total_cost / (148.0 * 3 * 8 * total_devices);
    h->crn_units.clear();
    cost.clear();
    h->n_sums_units = 0;
    h->max_runs_normal = 1;
    for (int pass = 0; pass < 2; ++pass) {  // sums-only units first
      for (const Slice &sl : slices_v) {
        if (sl.sums != (pass == 0)) continue;
        const dsi::CrnGroup &g = h->groups[sl.group];
        const uint64_t tiles = (g.n_trials + th - 1) / th;
        const double sc = (double)g.n_trials * (stream_cost(sl) + eval_cost[&sl - slices_v.data()]);
        const uint64_t by_cost = cap > 0.0 ? (uint64_t)std::ceil(sc / cap) : 1;
        const uint64_t nchunks = std::min<uint64_t>(std::max(split, by_cost), tiles);
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
            // (a fresh-verifier config, k t_d > t_t, makes the block store every run of L >= 2)
            const bool fresh = h->opt.flags & DSI_F_FRESH_VERIFIER;
            for (uint32_t q = sl.begin; q < sl.begin + sl.count; ++q) {
              const CfgTicks &c = t[h->perm[q]];
              kmin = std::min(kmin, (fresh && c.kd > c.t_t) ? 1 : std::min(c.k, c.n));
            }
            h->max_runs_normal = std::max<int32_t>(h->max_runs_normal, (g.n_tokens - 1) / (kmin + 2) + 1);
          }
          cost.push_back((double)(u.t1 - u.t0) * (stream_cost(sl) + eval_cost[&sl - slices_v.data()]));
        }
      }
    }
  } catch (...) {
    return fail(h, DSI_E_NOMEM, "shared-stream plan");
  }
  h->total_units = h->crn_units.size();
  return DSI_OK;
}

// Heatmap cells: maximal runs of consecutive configs with equal (t_target, t_drafter, a, SP, N).
void plan_heat_cells(dsi_sim *h) {
  // a cell starts at config i when i = 0 or (t_target, t_drafter, a, SP, N) differ from config
  // i - 1's: the starts are found per chunk in parallel, then written at their prefix offsets
  const auto &t = h->ticks;
  const size_t n = h->n_cfg;
  auto starts = [&](size_t i) {
    return i == 0 || !(t[i].ut == t[i - 1].ut && t[i].ud == t[i - 1].ud && t[i].a == t[i - 1].a &&
                       t[i].sp == t[i - 1].sp && t[i].n == t[i - 1].n);
  };
  constexpr size_t K = 64;
  size_t cnt[K + 1] = {};
  parallel_for(K, [&](size_t b, size_t e) {
    for (size_t c = b; c < e; ++c) {
      size_t m = 0;
      for (size_t i = n * c / K; i < n * (c + 1) / K; ++i) m += starts(i);
      cnt[c + 1] = m;
    }
  }, 1);
  for (size_t c = 0; c < K; ++c) cnt[c + 1] += cnt[c];
  h->heat_cells.assign(cnt[K], dsi::HeatCell{0, 0, 0u});
  parallel_for(K, [&](size_t b, size_t e) {
    for (size_t c = b; c < e; ++c) {
      size_t w = cnt[c];
      for (size_t i = n * c / K; i < n * (c + 1) / K; ++i)
        if (starts(i)) h->heat_cells[w++].first = i;
    }
  }, 1);
  const size_t nc = h->heat_cells.size();
  for (size_t j = 0; j < nc; ++j)
    h->heat_cells[j].count = (uint32_t)((j + 1 < nc ? h->heat_cells[j + 1].first : n) - h->heat_cells[j].first);
}

// Snap the shard bounds to candidate unit indices (sorted): the partition whose bounds are all
// candidates and whose largest part costs least (bisection on that cost; a part is extended
// greedily to the furthest candidate within it), taken if its largest part costs at most 4% or
// `slack` (the exchange it saves, in cost units) more than the unsnapped one's.  The candidates
// are heatmap-cell starts (per-config mode) or group starts (shared-stream mode), so a snapped
// part holds whole cells (SURVEY 8(e)'s cell-aligned option).  Returns whether it snapped.
bool snap_bounds(std::vector<uint64_t> &bounds, const std::vector<double> &cost, const std::vector<uint64_t> &cand,
                 double slack) {
  const size_t parts = bounds.size() - 1, n = cost.size();
  if (parts < 2 || cand.empty()) return parts < 2;
  std::vector<double> pre(n + 1, 0.0);
  for (size_t u = 0; u < n; ++u) pre[u + 1] = pre[u] + cost[u];
  double cur = 0.0;
  for (size_t q = 0; q < parts; ++q) cur = std::max(cur, pre[bounds[q + 1]] - pre[bounds[q]]);
  std::vector<uint64_t> cuts;  // the candidates strictly inside (0, n), then n
  for (const uint64_t c : cand)
    if (c > 0 && c < n && (cuts.empty() || c > cuts.back())) cuts.push_back(c);
  cuts.push_back(n);
  // greedy partition with parts of cost <= T; false if it needs more than `parts` parts
  auto fit = [&](double T, std::vector<uint64_t> *out) {
    uint64_t s = 0;
    size_t q = 0;
    if (out) out->assign(parts + 1, n), (*out)[0] = 0;
    while (s < n) {
      if (q == parts) return false;
      // the furthest cut c > s with pre[c] - pre[s] <= T
      auto it = std::upper_bound(cuts.begin(), cuts.end(), s);
      auto lim = std::upper_bound(it, cuts.end(), pre[s] + T, [&](double v, uint64_t c) { return v < pre[c]; });
      if (lim == it) return false;
      s = *(lim - 1);
      if (out) (*out)[++q] = s;
      else ++q;
    }
    return true;
  };
  double lo = pre[n] / parts, hi = pre[n];
  if (!fit(hi, nullptr)) return false;
  for (int it = 0; it < 100 && hi - lo > 1e-9 * hi; ++it) {
    const double mid = 0.5 * (lo + hi);
    (fit(mid, nullptr) ? hi : lo) = mid;
  }
  if (hi > std::max(1.04 * cur, cur + slack)) return false;
  std::vector<uint64_t> nb;
  fit(hi, &nb);
  bounds.swap(nb);
  return true;
}

// Which part owns each heatmap cell: the cell-local heatmap (dsi_sim_heatmap evaluates a part's
// cells from that part's own moments and exchanges only the 64-byte cells) needs every config of
// a cell simulated by one part.  Sets h->cell_local and each device's owned_cells.
void plan_cell_owners(dsi_sim *h) {
  h->cell_local = false;
  for (auto &d : h->dev) d.owned_cells.clear();
  if (h->dev.size() != 1) return;
  const size_t n = h->n_cfg;
  const std::vector<uint64_t> &pb = h->means_only ? h->cfg_bounds : h->part_bounds;
  if (pb.size() < 2) return;
  const int parts = (int)pb.size() - 1;
  std::vector<int32_t> owner(n, -1);  // -2: split between parts
  auto mark = [&](size_t c, int32_t q) {
    int32_t &o = owner[c];
    o = (o == -1 || o == q) ? q : -2;
  };
  if (h->means_only) {  // parts evaluate config ranges
    for (int q = 0; q < parts; ++q)
      for (uint64_t c = pb[q]; c < pb[q + 1]; ++c) owner[c] = q;
  } else if (h->shared) {  // a unit touches every config of its slice
    if (!h->shared_ttft.empty()) return;  // (the TTFT configs' own units: the moments are exchanged)
    for (int q = 0; q < parts; ++q)
      for (uint64_t u = pb[q]; u < pb[q + 1]; ++u) {
        const dsi::CrnUnit &un = h->crn_units[u];
        for (uint32_t i = un.begin; i < un.begin + un.count; ++i) mark(h->perm[i], q);
      }
  } else {  // config c's units [prefix[c], prefix[c+1])
    for (size_t c = 0; c < n; ++c) {
      if (h->prefix[c + 1] == h->prefix[c]) continue;
      const int32_t q0 = (int32_t)(std::upper_bound(pb.begin(), pb.end(), h->prefix[c]) - pb.begin()) - 1;
      const int32_t q1 = (int32_t)(std::upper_bound(pb.begin(), pb.end(), h->prefix[c + 1] - 1) - pb.begin()) - 1;
      owner[c] = q0 == q1 ? q0 : -2;
    }
  }
  const int per_rank = parts / std::max(1, h->opt.world);
  const int lo = h->opt.rank * per_rank, hi = lo + per_rank;
  std::vector<uint32_t> mine;
  for (size_t j = 0; j < h->heat_cells.size(); ++j) {
    const dsi::HeatCell &c = h->heat_cells[j];
    const int32_t o = owner[c.first];
    if (o < 0) return;
    for (uint64_t i = c.first + 1; i < c.first + c.count; ++i)
      if (owner[i] != o) return;
    if (o >= lo && o < hi) mine.push_back((uint32_t)j);
  }
  h->dev[0].owned_cells.swap(mine);
  h->cell_local = true;
}

// One device per process and every cell owned by one part: dsi_sim_heatmap evaluates this
// process's cells from its own moments (no all-reduce of the moments).
bool cells_aligned(const dsi_sim *h) { return h->cell_local && h->dev.size() == 1; }

}  // namespace dsih
