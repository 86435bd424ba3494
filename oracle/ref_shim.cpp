// ref_shim.cpp -- C entry points over the UNMODIFIED reference library.
//
// TEST INFRASTRUCTURE ONLY.  oracle/Makefile compiles this file together with
// /root/reference/proj/src/*.cpp (read in place, never copied) under
// -Dcatsim=catsim_ref into oracle/_ref/libcatsim_ref.so.  The macro renames the
// reference namespace so it can never collide with the product's own `catsim`
// symbols; quoted include paths are not macro-expanded, so the reference
// headers resolve unchanged.  Python (tests/, bench.py cpu_baseline and the
// --impl reference arm) reaches the reference through these functions only.
//
// Status codes: 0 ok, 1 std::invalid_argument, 2 std::logic_error,
// 3 std::out_of_range / runtime_error / anything else.
#include <chrono>
#include <cstdint>
#include <cstring>
#include <exception>
#include <stdexcept>
#include <string>
#include <thread>

#include "catsim/cat_engine.hpp"
#include "catsim/engines.hpp"
#include "catsim/fragment.hpp"
#include "catsim/grid.hpp"
#include "catsim/layout.hpp"
#include "catsim/rule.hpp"
#include "catsim/snapshot.hpp"
#include "tests/oracle.hpp"  // the reference's brute-force torus oracle (header, -I$(REF))

namespace {

thread_local std::string g_error;

template <typename Fn>
int guarded(Fn&& fn) {
  try {
    fn();
    g_error.clear();
    return 0;
  } catch (const std::invalid_argument& e) {
    g_error = e.what();
    return 1;
  } catch (const std::logic_error& e) {
    g_error = e.what();
    return 2;
  } catch (const std::exception& e) {
    g_error = e.what();
    return 3;
  }
}

catsim::Grid grid_from_interior(int n, int f, const uint8_t* interior) {
  catsim::Grid g = catsim::make_grid(n, f, catsim::Layout::RowMajor);
  for (int y = 0; y < n; ++y)
    for (int x = 0; x < n; ++x)
      g.interior(y, x) = interior[static_cast<std::size_t>(y) * n + x];
  return g;
}

void rule_to_ints(const catsim::LtlRule& r, int32_t* out) {
  out[0] = r.r;
  out[1] = r.c;
  out[2] = r.m;
  out[3] = r.s1;
  out[4] = r.s2;
  out[5] = r.b1;
  out[6] = r.b2;
  out[7] = r.kind == catsim::NeighborhoodKind::Moore ? 0 : 1;
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_error.c_str(); }

int ref_hardware_concurrency() {
  return static_cast<int>(std::thread::hardware_concurrency());
}

void ref_splitmix(uint64_t seed, int32_t count, uint64_t* out) {
  catsim::SplitMix64 rng(seed);
  for (int32_t i = 0; i < count; ++i) out[i] = rng.next();
}

int ref_alive_threshold(uint64_t z, double density) {
  return catsim::alive_threshold(z, density) ? 1 : 0;
}

int ref_init_random(int32_t n, double density, uint64_t seed, int32_t f,
                    int32_t fill_n, uint8_t* interior_out) {
  return guarded([&] {
    const catsim::Grid g = catsim::init_random(n, density, seed, f, fill_n);
    for (int y = 0; y < n; ++y)
      for (int x = 0; x < n; ++x)
        interior_out[static_cast<std::size_t>(y) * n + x] = g.interior(y, x);
  });
}

int ref_parse_rule(const char* text, int32_t* out8) {
  return guarded([&] { rule_to_ints(catsim::parse_ltl_rule(text), out8); });
}

int ref_preset_count() { return static_cast<int>(catsim::ltl_presets().size()); }

int ref_preset(int32_t index, const char** name, const char** rule,
               double* density) {
  const auto& all = catsim::ltl_presets();
  if (index < 0 || index >= static_cast<int32_t>(all.size())) return 1;
  *name = all[index].name;
  *rule = all[index].rule;
  *density = all[index].density;
  return 0;
}

void ref_von_neumann_probe_rule(int32_t r, int32_t* out8) {
  rule_to_ints(catsim::von_neumann_probe_rule(r), out8);
}

// run_engine(kind, ...) (src/engines.cpp:26-46) on an n x n interior.
// stats6 (optional): mma_count, steps, max_h, max_r, fragments_per_row,
// memory accesses (BASE).
int ref_run_engine(int32_t kind, int32_t n, int32_t f,
                   const uint8_t* interior_in, const char* rule_text,
                   int32_t steps, int32_t workers, int32_t tile_w,
                   int32_t tile_h, int32_t inject_fault,
                   uint8_t* interior_out, int64_t* stats6) {
  return guarded([&] {
    const catsim::LtlRule rule = catsim::parse_ltl_rule(rule_text);
    catsim::CatConfig cfg;
    cfg.f = f;
    cfg.kind = rule.kind;
    cfg.workers = workers;
    cfg.tile_w = tile_w;
    cfg.tile_h = tile_h;
    cfg.inject_band_fault = inject_fault != 0;
    const catsim::Grid initial = grid_from_interior(n, f, interior_in);
    catsim::RunStats stats;
    const catsim::Grid out = catsim::run_engine(
        static_cast<catsim::EngineKind>(kind), initial, rule, cfg, steps,
        stats6 ? &stats : nullptr);
    for (int y = 0; y < n; ++y)
      for (int x = 0; x < n; ++x)
        interior_out[static_cast<std::size_t>(y) * n + x] = out.interior(y, x);
    if (stats6) {
      stats6[0] = stats.cat.mma_count;
      stats6[1] = stats.cat.steps;
      stats6[2] = stats.cat.max_h;
      stats6[3] = stats.cat.max_r;
      stats6[4] = stats.cat.fragments_per_row;
      stats6[5] = stats.base.accesses();
    }
  });
}

// run_engine(Cat) (src/engines.cpp:30-35) split the way SURVEY.md §8d asks the
// CPU baseline to be reported: ms[0] = the whole call (layout conversion
// included, as catbench's time_run_ms, tools/catbench.cpp:123-130), ms[1] =
// simulate() alone (src/cat_engine.cpp:308-321, conversion excluded).
int ref_run_cat_timed(int32_t n, int32_t f, const uint8_t* interior_in,
                      const char* rule_text, int32_t steps, int32_t workers,
                      uint8_t* interior_out, double* ms2) {
  return guarded([&] {
    using clk = std::chrono::steady_clock;
    const catsim::LtlRule rule = catsim::parse_ltl_rule(rule_text);
    catsim::CatConfig cfg;
    cfg.f = f;
    cfg.kind = rule.kind;
    cfg.workers = workers;
    const catsim::Grid initial = grid_from_interior(n, f, interior_in);
    const auto t0 = clk::now();
    catsim::Grid frag = catsim::to_fragment_layout(initial);
    const auto t1 = clk::now();
    catsim::Grid done = catsim::simulate(std::move(frag), rule, cfg, steps);
    const auto t2 = clk::now();
    const catsim::Grid out = catsim::to_row_major(done);
    const auto t3 = clk::now();
    ms2[0] = std::chrono::duration<double, std::milli>(t3 - t0).count();
    ms2[1] = std::chrono::duration<double, std::milli>(t2 - t1).count();
    if (interior_out)
      for (int y = 0; y < n; ++y)
        for (int x = 0; x < n; ++x)
          interior_out[static_cast<std::size_t>(y) * n + x] = out.interior(y, x);
  });
}

// horizontal_step + vertical_step_{moore,von_neumann} (src/cat_engine.cpp:123-258)
// on a freshly halo-filled grid; outputs are the padded (n+2f)^2 fields in
// row-major order (halo rows/cols included, exactly as the reference leaves them).
int ref_reductions(int32_t n, int32_t f, const uint8_t* interior_in,
                   const char* rule_text, int32_t* h_out, int32_t* r_out) {
  return guarded([&] {
    const catsim::LtlRule rule = catsim::parse_ltl_rule(rule_text);
    catsim::CatConfig cfg;
    cfg.f = f;
    cfg.kind = rule.kind;
    catsim::Grid frag =
        catsim::to_fragment_layout(grid_from_interior(n, f, interior_in));
    catsim::fill_periodic_halo(frag);
    const catsim::BandFragments bands = catsim::gen_band_fragments(f, rule.r);
    const catsim::IntField h = catsim::horizontal_step(frag, bands, cfg);
    const catsim::IntField red =
        rule.kind == catsim::NeighborhoodKind::Moore
            ? catsim::vertical_step_moore(h, bands, cfg)
            : catsim::vertical_step_von_neumann(frag, h, bands, cfg);
    const int p = n + 2 * f;
    for (int y = 0; y < p; ++y)
      for (int x = 0; x < p; ++x) {
        h_out[static_cast<std::size_t>(y) * p + x] = h.at(y, x);
        r_out[static_cast<std::size_t>(y) * p + x] = red.at(y, x);
      }
  });
}

// The reference's own brute-force semantic oracle (tests/oracle.hpp:50-68,
// torus_rule_steps: explicit modular wrap, counts re-derived from the rule
// semantics).  It takes the LtlRule struct as given -- no parse_ltl_rule
// validation -- so it also defines the wide-radius extension (17 <= r <= 32)
// that the reference's engines reject.  rule8 = {r, c, m, s1, s2, b1, b2, kind}.
int ref_semantic_steps(int32_t n, const uint8_t* interior_in, const int32_t* rule8,
                       int32_t steps, uint8_t* interior_out) {
  return guarded([&] {
    catsim::LtlRule rule;
    rule.r = rule8[0];
    rule.c = rule8[1];
    rule.m = rule8[2];
    rule.s1 = rule8[3];
    rule.s2 = rule8[4];
    rule.b1 = rule8[5];
    rule.b2 = rule8[6];
    rule.kind = rule8[7] ? catsim::NeighborhoodKind::VonNeumannSimplified
                         : catsim::NeighborhoodKind::Moore;
    const catsim::Grid out = oracle::torus_rule_steps(grid_from_interior(n, 16, interior_in), rule, steps);
    for (int y = 0; y < n; ++y)
      for (int x = 0; x < n; ++x)
        interior_out[static_cast<std::size_t>(y) * n + x] = out.interior(y, x);
  });
}

// snapshot_write (src/snapshot.cpp:18-37) of an n x n interior in `layout`
// (0 row-major, 1 fragment-contiguous) to `path`.
int ref_snapshot_write(int32_t n, int32_t f, int32_t layout, const uint8_t* interior,
                       const char* path) {
  return guarded([&] {
    catsim::Grid g = grid_from_interior(n, f, interior);
    if (layout == 1) g = catsim::to_fragment_layout(g);
    catsim::snapshot_write(g, std::string(path));
  });
}

// snapshot_read (src/snapshot.cpp:39-91): geometry + layout first (interior
// may be NULL to probe), then the interior in row-major order.
int ref_snapshot_read(const char* path, int32_t* n, int32_t* f, int32_t* layout,
                      uint8_t* interior, int64_t capacity) {
  return guarded([&] {
    const catsim::Grid g = catsim::snapshot_read(std::string(path));
    *n = g.n;
    *f = g.f;
    *layout = g.layout == catsim::Layout::RowMajor ? 0 : 1;
    if (!interior) return;
    if (static_cast<int64_t>(g.n) * g.n > capacity)
      throw std::invalid_argument("capacity");
    for (int y = 0; y < g.n; ++y)
      for (int x = 0; x < g.n; ++x)
        interior[static_cast<std::size_t>(y) * g.n + x] = g.interior(y, x);
  });
}

}  // extern "C"
