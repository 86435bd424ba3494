// catsim/cat_engine.hpp -- drop-in for proj/include/catsim/cat_engine.hpp:
// CatConfig, CatStats, simulate_step and simulate with the reference's
// signatures, validation order and messages (src/cat_engine.cpp:83-90,
// :260-321).  The generations run on the B200 (ltl_run: one fused tcgen05
// step kernel per generation); the host Grid is uploaded once per call and
// the result downloaded once.  The unit-test entry points horizontal_step /
// vertical_step_* (the materialised H and R fields) are not provided: the
// device never materialises them.
#pragma once

#include <algorithm>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "catsim/device.hpp"
#include "catsim/grid.hpp"
#include "catsim/rule.hpp"

namespace catsim {

struct CatConfig {
  int f = kDefaultFragmentSide;
  int tile_w = 1;
  int tile_h = 14;
  NeighborhoodKind kind = NeighborhoodKind::Moore;
  int workers = 1;
  bool inject_band_fault = false;
};

struct CatStats {
  long long mma_count = 0;
  long long steps = 0;
  int32_t max_h = 0;
  int32_t max_r = 0;
  int fragments_per_row = 0;
  std::vector<uint32_t> mma_per_fragment;
};

namespace detail {

// cat_engine.cpp:83-90
inline void check_config(const CatConfig& cfg) {
  if (cfg.f != 4 && cfg.f != 8 && cfg.f != 16)
    throw std::invalid_argument("config error: fragment side must be 4, 8, or 16");
  if (cfg.tile_w < 1 || cfg.tile_h < 1)
    throw std::invalid_argument("config error: tile sides must be >= 1");
  if (cfg.workers < 1) throw std::invalid_argument("config error: workers must be >= 1");
}

inline ltl_rule_c to_c(const LtlRule& r) {
  ltl_rule_c c{};
  c.r = r.r;
  c.c = r.c;
  c.m = r.m;
  c.s1 = r.s1;
  c.s2 = r.s2;
  c.b1 = r.b1;
  c.b2 = r.b2;
  c.kind = r.kind == NeighborhoodKind::Moore ? LTL_KIND_MOORE : LTL_KIND_VON_NEUMANN;
  return c;
}

// CatStats of `steps` generations: the device reports the reference's MMA
// accounting (3 per fragment of the H pass over all fragment rows x interior
// columns, 3 per interior fragment of the R pass) and max-reduced H / R.
inline void add_stats(CatStats* stats, const ltl_stats_c& s, int fpr) {
  if (!stats) return;
  stats->mma_count += s.mma_count;
  stats->steps += s.steps;
  stats->max_h = std::max(stats->max_h, s.max_h);
  stats->max_r = std::max(stats->max_r, s.max_r);
  stats->fragments_per_row = fpr;
  stats->mma_per_fragment.assign(static_cast<std::size_t>(fpr) * fpr, 0u);
  for (int i = 0; i < fpr; ++i)
    for (int j = 1; j + 1 < fpr; ++j)
      stats->mma_per_fragment[static_cast<std::size_t>(i) * fpr + j] =
          (s.steps > 0 ? 3u : 0u) + (s.steps > 0 && i >= 1 && i + 1 < fpr ? 3u : 0u);
}

// the f check horizontal_step makes (check_engine_grid, cat_engine.cpp:98-102)
inline void check_grid_f(const Grid& grid, const CatConfig& cfg) {
  if (grid.f != cfg.f)
    throw std::invalid_argument("config error: grid fragment side " + std::to_string(grid.f) +
                                " disagrees with config f " + std::to_string(cfg.f));
}

// `steps` generations of `grid` (its layout) on the device into `out`'s
// interior (out may be grid); stats as the reference accumulates them.
inline void run_on_device(const Grid& grid, const LtlRule& rule, const CatConfig& cfg,
                          int steps, Grid& out, CatStats* stats) {
  if (grid.n == 0) {
    if (stats) stats->steps += steps;
    return;
  }
  DeviceGrid dev(grid.n, grid.f);
  const int32_t lay = c_layout(grid.layout);
  dev.check(ltl_upload(dev.get(), grid.cells.data(), lay));
  const ltl_rule_c rc = to_c(rule);
  uint32_t flags = stats ? LTL_FLAG_WANT_STATS : 0u;
  if (cfg.inject_band_fault) flags |= LTL_FLAG_INJECT_FAULT;
  ltl_stats_c s{};
  dev.check(ltl_run(dev.get(), &rc, steps, flags, stats ? &s : nullptr));
  // only the interior of `out` is written, as simulate_step does (:293-305)
  std::vector<uint8_t> next(grid.cells.size());
  dev.check(ltl_download(dev.get(), next.data(), c_layout(out.layout)));
  for (int y = 0; y < grid.n; ++y)
    for (int x = 0; x < grid.n; ++x) {
      const std::size_t k = out.index(y + grid.f, x + grid.f);
      out.cells[k] = next[k];
    }
  add_stats(stats, s, grid.fragments_per_row());
}

}  // namespace detail

// One generation: grid -> out (simulate_step, cat_engine.cpp:260-306).  Fills
// grid's periodic halo (as the reference does), writes out's interior and
// marks out's halo stale.
inline void simulate_step(Grid& grid, const LtlRule& rule, const CatConfig& cfg, Grid& out,
                          CatStats* stats = nullptr) {
  detail::check_config(cfg);
  if (&grid == &out) throw std::invalid_argument("config error: in-place step not supported");
  if (rule.kind != cfg.kind)
    throw std::invalid_argument("config error: rule kind disagrees with engine config");
  if (grid.layout != Layout::FragmentContiguous || out.layout != Layout::FragmentContiguous)
    throw std::invalid_argument("layout error: engine needs fragment-contiguous grids");
  if (out.n != grid.n || out.f != grid.f)
    throw std::invalid_argument("geometry error: output grid shape mismatch");
  fill_periodic_halo(grid);
  detail::check_grid_f(grid, cfg);
  detail::run_on_device(grid, rule, cfg, 1, out, stats);
  out.halo_valid = false;
}

// `steps` generations (simulate, cat_engine.cpp:308-321): one upload, all
// generations device-resident, one download.
inline Grid simulate(Grid grid, const LtlRule& rule, const CatConfig& cfg, int steps,
                     CatStats* stats = nullptr) {
  if (steps < 0) throw std::invalid_argument("config error: steps must be >= 0");
  if (steps == 0) return grid;
  detail::check_config(cfg);
  if (rule.kind != cfg.kind)
    throw std::invalid_argument("config error: rule kind disagrees with engine config");
  if (grid.layout != Layout::FragmentContiguous)
    throw std::invalid_argument("layout error: engine needs fragment-contiguous grids");
  detail::check_grid_f(grid, cfg);
  Grid out = grid;
  detail::run_on_device(grid, rule, cfg, steps, out, stats);
  out.halo_valid = false;
  return out;
}

}  // namespace catsim
