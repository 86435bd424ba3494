// catsim/cat_engine.hpp -- drop-in for proj/include/catsim/cat_engine.hpp:
// CatConfig, CatStats, simulate_step and simulate with the reference's
// signatures, validation order and messages (src/cat_engine.cpp:83-90,
// :260-321).  The generations run on the B200 (ltl_run: one fused tcgen05
// step kernel per generation); the host Grid is uploaded once per call and
// the result downloaded once.  The reference's fragment-level unit-test entry
// points horizontal_step / vertical_step_* (:123-258) materialise H and R
// through a debug kernel (ltl_fragment_pass); the step never does.
#pragma once

#include <algorithm>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "catsim/device.hpp"
#include "catsim/fragment.hpp"
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

// `steps` generations of `grid` (its layout) on the device with the engine
// `flags` select; the result lands in `out`'s interior only (out's halo is
// left as it was, as simulate_step leaves it, src/cat_engine.cpp:293-305):
// one pitched H2D of grid's interior, the generations, one pitched D2H.
inline void run_device_engine(const Grid& grid, const LtlRule& rule, int steps, uint32_t flags,
                              Grid& out, ltl_stats_c* s) {
  if (grid.n == 0) return;
  DeviceGrid dev(grid.n, grid.f);
  dev.check(ltl_upload(dev.get(), grid.cells.data(), c_layout(grid.layout)));
  const ltl_rule_c rc = to_c(rule);
  dev.check(ltl_run(dev.get(), &rc, steps, flags, s));
  dev.check(ltl_download_padded(dev.get(), out.cells.data(), c_layout(out.layout), 0));
}

// The CAT engine: `steps` generations into `out`'s interior (out may be grid);
// stats as the reference accumulates them.
inline void run_on_device(const Grid& grid, const LtlRule& rule, const CatConfig& cfg,
                          int steps, Grid& out, CatStats* stats) {
  if (grid.n == 0) {
    if (stats) stats->steps += steps;
    return;
  }
  uint32_t flags = stats ? LTL_FLAG_WANT_STATS : 0u;
  if (cfg.inject_band_fault) flags |= LTL_FLAG_INJECT_FAULT;
  ltl_stats_c s{};
  run_device_engine(grid, rule, steps, flags, out, stats ? &s : nullptr);
  add_stats(stats, s, grid.fragments_per_row());
}

}  // namespace detail

namespace detail {

inline std::vector<int32_t> band_words(const BandFragments& b) {
  std::vector<int32_t> w;
  w.reserve(3 * b.pi1.data.size());
  for (const Fragment* p : {&b.pi1, &b.pi2, &b.pi3}) w.insert(w.end(), p->data.begin(), p->data.end());
  return w;
}

// cat_engine.cpp:92-111
inline void check_engine_grid(const Grid& grid, const BandFragments& bands, const CatConfig& cfg) {
  check_config(cfg);
  if (grid.layout != Layout::FragmentContiguous)
    throw std::invalid_argument("layout error: engine needs a fragment-contiguous grid");
  check_grid_f(grid, cfg);
  if (bands.f != grid.f)
    throw std::invalid_argument("config error: band fragments built for f=" + std::to_string(bands.f));
  if (!grid.halo_valid) throw std::logic_error("sequencing error: periodic halo not filled");
}

inline int32_t field_max(const IntField& h) {
  int32_t m = 0;
  for (int32_t v : h.values) m = std::max(m, v);
  return m;
}

inline void add_pass_stats(CatStats* stats, int fpr, bool all_rows, int32_t max_h,
                           int32_t max_r) {
  if (!stats) return;
  long long mmas = 0;
  for (int i = all_rows ? 0 : 1; i < (all_rows ? fpr : fpr - 1); ++i)
    for (int j = 1; j + 1 < fpr; ++j) {
      stats->mma_per_fragment[static_cast<std::size_t>(i) * fpr + j] += 3;
      mmas += 3;
    }
  stats->mma_count += mmas;
  stats->max_h = std::max(stats->max_h, max_h);
  stats->max_r = std::max(stats->max_r, max_r);
}

}  // namespace detail

// Horizontal window sums of every fragment row, interior fragment columns
// (horizontal_step, cat_engine.cpp:123-161).
inline IntField horizontal_step(const Grid& grid, const BandFragments& bands, const CatConfig& cfg,
                                CatStats* stats = nullptr) {
  detail::check_engine_grid(grid, bands, cfg);
  IntField h = make_field(grid.n, grid.f, Layout::FragmentContiguous);
  const int fpr = grid.fragments_per_row();
  if (stats) {
    stats->fragments_per_row = fpr;
    stats->mma_per_fragment.assign(static_cast<std::size_t>(fpr) * fpr, 0u);
  }
  const std::vector<int32_t> bw = detail::band_words(bands);
  detail::check(ltl_fragment_pass(0, grid.n, grid.f, grid.cells.data(), bw.data(), nullptr,
                                  h.values.data()),
                nullptr);
  detail::add_pass_stats(stats, fpr, true, stats ? detail::field_max(h) : 0, 0);
  h.valid = true;
  return h;
}

// Full box sums, centre once (vertical_step_moore, cat_engine.cpp:163-208).
inline IntField vertical_step_moore(const IntField& h, const BandFragments& bands,
                                    const CatConfig& cfg, CatStats* stats = nullptr) {
  detail::check_config(cfg);
  if (h.layout != Layout::FragmentContiguous)
    throw std::invalid_argument("layout error: engine needs a fragment-contiguous field");
  if (!h.valid) throw std::logic_error("sequencing error: horizontal field not yet computed");
  if (bands.f != h.f || h.f != cfg.f)
    throw std::invalid_argument("config error: fragment side mismatch");
  IntField red = make_field(h.n, h.f, Layout::FragmentContiguous);
  const std::vector<int32_t> bw = detail::band_words(bands);
  const std::vector<uint8_t> no_cells(static_cast<std::size_t>(h.padded()) * h.padded(), 0);
  detail::check(ltl_fragment_pass(1, h.n, h.f, no_cells.data(), bw.data(), h.values.data(),
                                  red.values.data()),
                nullptr);
  detail::add_pass_stats(stats, h.fragments_per_row(), false, 0, stats ? detail::field_max(red) : 0);
  red.valid = true;
  return red;
}

// Cross sums, centre twice (vertical_step_von_neumann, cat_engine.cpp:210-258).
inline IntField vertical_step_von_neumann(const Grid& grid, const IntField& h,
                                          const BandFragments& bands, const CatConfig& cfg,
                                          CatStats* stats = nullptr) {
  detail::check_engine_grid(grid, bands, cfg);
  if (h.layout != Layout::FragmentContiguous || h.n != grid.n || h.f != grid.f)
    throw std::invalid_argument("layout error: horizontal field does not match the grid");
  if (!h.valid) throw std::logic_error("sequencing error: horizontal field not yet computed");
  IntField red = make_field(grid.n, grid.f, Layout::FragmentContiguous);
  const std::vector<int32_t> bw = detail::band_words(bands);
  detail::check(ltl_fragment_pass(2, grid.n, grid.f, grid.cells.data(), bw.data(),
                                  h.values.data(), red.values.data()),
                nullptr);
  detail::add_pass_stats(stats, grid.fragments_per_row(), false, 0,
                         stats ? detail::field_max(red) : 0);
  red.valid = true;
  return red;
}

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
  detail::run_on_device(grid, rule, cfg, steps, grid, stats);  // in place: upload, run, download
  grid.halo_valid = false;
  return grid;
}

}  // namespace catsim
