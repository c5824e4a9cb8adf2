// dsi_heatmap.cpp -- the heatmap product over reduced per-config results
// (Fig. 3 and Fig. 5 of the paper: P:290-311).
//
// Host-only and O(n): a cell is a maximal run of consecutive configs sharing
// (t_target, t_drafter, accept_rate, sp_degree, n_tokens).  SI takes the minimal
// mean over the cell's lookaheads; DSI the minimal mean over the lookaheads that
// satisfy Eq. 1 at the cell's SP; ties go to the smallest lookahead.
#include <cmath>
#include <cstdio>
#include <limits>

#include "../../include/dsi_sim.h"

namespace {

bool same_cell(const dsi_config &a, const dsi_config &b) {
  return a.t_target == b.t_target && a.t_drafter == b.t_drafter && a.accept_rate == b.accept_rate &&
         a.sp_degree == b.sp_degree && a.n_tokens == b.n_tokens;
}

void fill_cell(const dsi_config *cfg, const dsi_result *res, size_t first, size_t count,
               dsi_heatmap_cell &c) {
  const double nan = std::numeric_limits<double>::quiet_NaN();
  const dsi_config &c0 = cfg[first];
  c.t_target = c0.t_target;
  c.t_drafter = c0.t_drafter;
  c.accept_rate = c0.accept_rate;
  c.sp_degree = c0.sp_degree;
  c.n_tokens = c0.n_tokens;
  c.first_cfg = first;
  c.n_cfg = count;
  c.nonsi = res[first].mean_nonsi;
  c.si_lookahead = -1;
  c.dsi_lookahead = -1;
  c.si = nan;
  c.dsi = nan;
  for (size_t i = first; i < first + count; ++i) {
    const int32_t k = cfg[i].lookahead;
    const double si = res[i].mean_si, dsi = res[i].mean_dsi;
    if (c.si_lookahead < 0 || si < c.si || (si == c.si && k < c.si_lookahead)) {
      c.si = si;
      c.si_lookahead = k;
    }
    if (res[i].eq1_feasible == 1 &&
        (c.dsi_lookahead < 0 || dsi < c.dsi || (dsi == c.dsi && k < c.dsi_lookahead))) {
      c.dsi = dsi;
      c.dsi_lookahead = k;
    }
  }
  // "X/Y plots the ratio between the run time of algorithm X and the run time of
  // algorithm Y"; panels (a) non-SI/SI ... (d) min(SI, non-SI)/DSI
  c.r_nonsi_si = c.nonsi / c.si;
  c.r_si_dsi = c.si / c.dsi;
  c.r_nonsi_dsi = c.nonsi / c.dsi;
  c.r_min_dsi = std::fmin(c.si, c.nonsi) / c.dsi;
}

}  // namespace

extern "C" {

dsi_status dsi_heatmap(const dsi_config *cfg, const dsi_result *res, size_t n, dsi_heatmap_cell *cells,
                       size_t cap, size_t *n_cells) {
  if (!cfg || !res || !n_cells) return DSI_E_NULL;
  size_t count = 0;
  for (size_t i = 0; i < n;) {
    size_t j = i + 1;
    while (j < n && same_cell(cfg[i], cfg[j])) ++j;
    if (cells) {
      if (count >= cap) return DSI_E_RANGE;
      fill_cell(cfg, res, i, j - i, cells[count]);
    }
    ++count;
    i = j;
  }
  *n_cells = count;
  return DSI_OK;
}

dsi_status dsi_heatmap_csv(const dsi_heatmap_cell *cells, size_t n, const char *path) {
  if (!cells || !path) return DSI_E_NULL;
  FILE *f = std::fopen(path, "w");
  if (!f) return DSI_E_RANGE;
  std::fprintf(f, "# dsi_heatmap v1\n");
  std::fprintf(f,
               "drafter_latency,acceptance_rate,nonsi,si,dsi,si_lookahead,dsi_lookahead,"
               "r_nonsi_si,r_si_dsi,r_nonsi_dsi,r_min_dsi\n");
  for (size_t i = 0; i < n; ++i) {
    const dsi_heatmap_cell &c = cells[i];
    std::fprintf(f, "%.6f,%.6f,%.6f,%.6f,%.6f,%d,%d,%.6f,%.6f,%.6f,%.6f\n", c.t_drafter, c.accept_rate,
                 c.nonsi, c.si, c.dsi, c.si_lookahead, c.dsi_lookahead, c.r_nonsi_si, c.r_si_dsi,
                 c.r_nonsi_dsi, c.r_min_dsi);
  }
  const bool ok = std::fclose(f) == 0;
  return ok ? DSI_OK : DSI_E_RANGE;
}

}  // extern "C"

static_assert(sizeof(dsi_heatmap_cell) == 112, "dsi_heatmap_cell ABI layout");
