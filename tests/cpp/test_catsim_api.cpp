// test_catsim_api.cpp -- the reference's own engine / grid / snapshot test
// cases (proj/tests/test_cat_engine.cpp, test_grid.cpp, test_snapshot.cpp),
// restated against this repo's header-only catsim API (include/catsim/),
// i.e. exactly what a reference user compiles after switching libraries.
// Built and run by tests/test_cpp_api.py; anchors (alive count + FNV-1a-64
// of reference runs, tests/golden/anchors.json) arrive on the command line.
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <fstream>
#include <iterator>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "catsim/catsim.hpp"

using namespace catsim;

static int g_fail = 0, g_checks = 0;
#define CHECK(cond)                                                            \
  do {                                                                         \
    ++g_checks;                                                                \
    if (!(cond)) {                                                             \
      ++g_fail;                                                                \
      std::fprintf(stderr, "%s:%d: CHECK failed: %s\n", __FILE__, __LINE__, #cond); \
    }                                                                          \
  } while (0)
#define CHECK_THROWS_AS(expr, exc, text)                                       \
  do {                                                                         \
    ++g_checks;                                                                \
    bool ok_ = false;                                                          \
    try {                                                                      \
      (void)(expr);                                                            \
    } catch (const exc& e_) {                                                  \
      ok_ = std::string(e_.what()).find(text) != std::string::npos;            \
      if (!ok_) std::fprintf(stderr, "  message was: %s\n", e_.what());        \
    } catch (const std::exception& e_) {                                       \
      std::fprintf(stderr, "  wrong exception: %s\n", e_.what());              \
    }                                                                          \
    if (!ok_) {                                                                \
      ++g_fail;                                                                \
      std::fprintf(stderr, "%s:%d: expected %s(%s) from %s\n", __FILE__, __LINE__, #exc, text, #expr); \
    }                                                                          \
  } while (0)

static CatConfig config_for(NeighborhoodKind kind) {
  CatConfig cfg;
  cfg.kind = kind;
  return cfg;
}
static Grid frag_grid(const Grid& g) { return to_fragment_layout(g); }

static std::string fnv(const Grid& g) {
  uint64_t h = 0xCBF29CE484222325ULL;
  for (int y = 0; y < g.n; ++y)
    for (int x = 0; x < g.n; ++x) {
      h ^= g.interior(y, x);
      h *= 0x100000001B3ULL;
    }
  char buf[17];
  std::snprintf(buf, sizeof buf, "%016llx", static_cast<unsigned long long>(h));
  return buf;
}

static void blinker_and_still_lifes() {  // test_cat_engine.cpp:153-190
  const LtlRule gol = parse_ltl_rule("R1,C2,M0,S2..3,B3..3,NM");
  const CatConfig cfg = config_for(NeighborhoodKind::Moore);
  Grid g = make_grid(16, 16);
  g.interior(7, 8) = g.interior(8, 8) = g.interior(9, 8) = 1;
  const Grid after1 = to_row_major(simulate(frag_grid(g), gol, cfg, 1));
  for (int y = 0; y < 16; ++y)
    for (int x = 0; x < 16; ++x)
      CHECK(after1.interior(y, x) == ((y == 8 && x >= 7 && x <= 9) ? 1 : 0));
  const Grid after2 = to_row_major(simulate(frag_grid(g), gol, cfg, 2));
  CHECK(!first_interior_difference(after2, g).has_value());

  Grid b = make_grid(16, 16);
  b.interior(4, 4) = b.interior(4, 5) = b.interior(5, 4) = b.interior(5, 5) = 1;
  CHECK(!first_interior_difference(to_row_major(simulate(frag_grid(b), gol, cfg, 4)), b));
  CHECK(count_alive(to_row_major(simulate(frag_grid(make_grid(16, 16)), gol, cfg, 3))) == 0);

  const LtlRule majority = parse_ltl_rule("R4,C2,M0,S40..80,B41..80,NM");
  const Grid all = init_random(32, 1.0, 0);
  CHECK(count_alive(to_row_major(simulate(frag_grid(all), majority, cfg, 2))) == 32 * 32);
}

static void step_loop_equals_simulate() {
  // simulate == repeated simulate_step (the reference's own definition,
  // cat_engine.cpp:308-321), Moore and VN, f = 4 / 8 / 16
  const char* texts[] = {"R1,C2,M0,S2..3,B3..3,NM", "R3,C2,M0,S15..23,B14..17,NM",
                         "R16,C2,M0,S170..296,B170..300,NM"};
  for (const char* text : texts) {
    const LtlRule rule = parse_ltl_rule(text);
    const CatConfig cfg = config_for(rule.kind);
    const Grid start = frag_grid(init_random(48, 0.3, 1000 + rule.r));
    Grid a = start, b = make_grid(48, 16, Layout::FragmentContiguous);
    for (int s = 0; s < 3; ++s) {
      simulate_step(a, rule, cfg, b, nullptr);
      std::swap(a, b);
    }
    CHECK(!first_interior_difference(simulate(start, rule, cfg, 3), a).has_value());
  }
  for (const int r : {1, 6, 16}) {
    const LtlRule rule = von_neumann_probe_rule(r);
    const CatConfig cfg = config_for(rule.kind);
    const Grid start = frag_grid(init_random(48, 0.25, 2000 + r));
    Grid a = start, b = make_grid(48, 16, Layout::FragmentContiguous);
    for (int s = 0; s < 3; ++s) {
      simulate_step(a, rule, cfg, b, nullptr);
      std::swap(a, b);
    }
    CHECK(!first_interior_difference(simulate(start, rule, cfg, 3), a).has_value());
  }
  // m=0 / m=1 formulations of life agree (:216-225)
  const Grid start = init_random(32, 0.35, 77);
  const CatConfig cfg = config_for(NeighborhoodKind::Moore);
  const Grid a = to_row_major(simulate(frag_grid(start), parse_ltl_rule("R1,C2,M0,S2..3,B3..3,NM"), cfg, 5));
  const Grid b = to_row_major(simulate(frag_grid(start), parse_ltl_rule("R1,C2,M1,S3..4,B3..3,NM"), cfg, 5));
  CHECK(!first_interior_difference(a, b).has_value());
  // smaller fragment sides end to end (:372-384)
  for (const int f : {4, 8}) {
    CatConfig c8 = cfg;
    c8.f = f;
    const Grid s0 = init_random(32, 0.35, 50 + f, f);
    const Grid got = to_row_major(simulate(to_fragment_layout(s0), parse_ltl_rule("R1,C2,M0,S2..3,B3..3,NM"), c8, 4));
    RunStats rs;
    const Grid via_engine = run_engine(EngineKind::Cat, s0, parse_ltl_rule("R1,C2,M0,S2..3,B3..3,NM"), c8, 4, &rs);
    CHECK(!first_interior_difference(got, via_engine).has_value());
    CHECK(rs.cat.steps == 4);
  }
}

static void errors_and_config() {  // :228-271
  const CatConfig cfg = config_for(NeighborhoodKind::Moore);
  const LtlRule gol = parse_ltl_rule("R1,C2,M0,S2..3,B3..3,NM");
  Grid ok = frag_grid(init_random(16, 0.5, 1));
  Grid out = make_grid(16, 16, Layout::FragmentContiguous);
  CHECK_THROWS_AS(simulate_step(ok, gol, cfg, ok), std::invalid_argument, "in-place step");
  CHECK_THROWS_AS(simulate_step(ok, von_neumann_probe_rule(1), cfg, out), std::invalid_argument,
                  "rule kind disagrees");
  Grid rm = init_random(16, 0.5, 1);
  CHECK_THROWS_AS(simulate_step(rm, gol, cfg, out), std::invalid_argument, "fragment-contiguous");
  Grid small = make_grid(32, 16, Layout::FragmentContiguous);
  CHECK_THROWS_AS(simulate_step(ok, gol, cfg, small), std::invalid_argument, "shape mismatch");
  CatConfig bad;
  bad.f = 5;
  CHECK_THROWS_AS(simulate_step(ok, gol, bad, out), std::invalid_argument, "fragment side must be");
  bad = CatConfig{};
  bad.tile_w = 0;
  CHECK_THROWS_AS(simulate_step(ok, gol, bad, out), std::invalid_argument, "tile sides");
  bad = CatConfig{};
  bad.workers = 0;
  CHECK_THROWS_AS(simulate_step(ok, gol, bad, out), std::invalid_argument, "workers");
  CHECK_THROWS_AS(simulate(ok, gol, CatConfig{}, -1), std::invalid_argument, "steps must be >= 0");
  const Grid start = frag_grid(init_random(32, 0.5, 3));
  CHECK(simulate(start, gol, cfg, 0).cells == start.cells);  // :273-279
  CHECK_THROWS_AS(parse_engine("gpu"), std::invalid_argument, "unknown engine 'gpu'");
  CHECK(parse_engine("cat") == EngineKind::Cat);
  CHECK_THROWS_AS(run_engine(EngineKind::Cat, start, gol, cfg, 1), std::invalid_argument,
                  "expected a row-major grid");
  CHECK_THROWS_AS(make_grid(17, 16), std::invalid_argument, "multiple of f");
  CHECK_THROWS_AS(init_random(16, 1.5, 1), std::invalid_argument, "density must be in [0, 1]");
  CHECK_THROWS_AS(init_random(16, 0.5, 1, 16, 32), std::invalid_argument, "fill_n exceeds n");
  CatConfig f8 = cfg;
  f8.f = 8;
  CHECK_THROWS_AS(simulate(frag_grid(init_random(32, 0.5, 1, 8)),
                           parse_ltl_rule("R16,C2,M0,S170..296,B170..300,NM"), f8, 1),
                  std::invalid_argument, "unsupported radius r=16 for fragment side f=8");
}

static void accounting_and_fault() {  // :281-305, :353-370
  for (const auto kind : {NeighborhoodKind::Moore, NeighborhoodKind::VonNeumannSimplified}) {
    const LtlRule rule = kind == NeighborhoodKind::Moore ? parse_ltl_rule("R1,C2,M0,S2..3,B3..3,NM")
                                                         : von_neumann_probe_rule(1);
    CatStats stats;
    Grid g = frag_grid(init_random(64, 0.4, 5));
    Grid out = make_grid(64, 16, Layout::FragmentContiguous);
    simulate_step(g, rule, config_for(kind), out, &stats);
    CHECK(stats.fragments_per_row == 6);
    long long total = 0;
    for (int i = 0; i < 6; ++i)
      for (int j = 0; j < 6; ++j) {
        const uint32_t count = stats.mma_per_fragment[i * 6 + j];
        total += count;
        const bool interior = i >= 1 && i <= 4 && j >= 1 && j <= 4;
        const bool halo_row = (i == 0 || i == 5) && j >= 1 && j <= 4;
        CHECK(count == (interior ? 6u : halo_row ? 3u : 0u));
      }
    CHECK(stats.mma_count == total);
    CHECK(stats.mma_count == 3 * (6 * 4) + 3 * 16);
    CHECK(stats.steps == 1);
    CHECK(g.halo_valid);  // simulate_step filled the input's halo (:275)
    CHECK(!out.halo_valid);
  }
  const LtlRule gol = parse_ltl_rule("R1,C2,M0,S2..3,B3..3,NM");
  const Grid start = init_random(64, 0.3, 7);
  CatConfig cfg = config_for(NeighborhoodKind::Moore);
  const Grid clean = to_row_major(simulate(frag_grid(start), gol, cfg, 2));
  cfg.inject_band_fault = true;
  bool detected = false;
  try {
    const Grid faulty = to_row_major(simulate(frag_grid(start), gol, cfg, 2));
    detected = first_interior_difference(clean, faulty).has_value();
  } catch (const std::logic_error&) {
    detected = true;
  }
  CHECK(detected);
}

static void grid_kats() {  // test_grid.cpp:50-63
  const Grid a = init_random(64, 0.37, 99), b = init_random(64, 0.37, 99);
  CHECK(a.cells == b.cells);
  CHECK(a.cells != init_random(64, 0.37, 100).cells);
  const Grid g = init_random(16, 0.5, 0);
  CHECK(g.interior(0, 0) == 0);
  CHECK(g.interior(0, 1) == 1);
  CHECK(g.interior(0, 2) == 1);
  CHECK(g.interior(0, 3) == 0);
  CHECK(count_alive(init_random(64, 0.0, 5)) == 0);
  CHECK(count_alive(init_random(64, 1.0, 5)) == 64 * 64);
  SplitMix64 rng(0);
  CHECK(rng.next() == 0xE220A8397B1DCDAFULL);
  Grid h = init_random(20, 0.5, 3, 4);
  fill_periodic_halo(h);
  CHECK(h.halo_valid);
  for (int y = 0; y < h.padded(); ++y)
    for (int x = 0; x < h.padded(); ++x)
      CHECK(h.at(y, x) == h.interior(((y - 4) % 20 + 20) % 20, ((x - 4) % 20 + 20) % 20));
}

static void snapshots(const std::string& golden_dir, const std::string& tmp) {
  Grid g = make_grid(16, 16);  // test_snapshot.cpp:34-46
  g.interior(2, 3) = 1;
  const std::string p = tmp + "/one.bin";
  snapshot_write(g, p);
  std::ifstream mine(p, std::ios::binary), gold(golden_dir + "/one_cell_16.bin", std::ios::binary);
  const std::string a((std::istreambuf_iterator<char>(mine)), {}),
      b((std::istreambuf_iterator<char>(gold)), {});
  CHECK(!a.empty() && a == b);
  const Grid frag = to_fragment_layout(init_random(32, 0.4, 2));  // :58-66
  snapshot_write(frag, tmp + "/frag.bin");
  const Grid back = snapshot_read(tmp + "/frag.bin");
  CHECK(back.layout == Layout::FragmentContiguous);
  CHECK(!back.halo_valid);
  CHECK(!first_interior_difference(frag, back).has_value());
  const Grid ref32 = snapshot_read(golden_dir + "/random_32_fragment.bin");
  CHECK(!first_interior_difference(ref32, back).has_value());
  snapshot_write(make_grid(0, 16), tmp + "/empty.bin");  // :68-74
  std::ifstream e(tmp + "/empty.bin", std::ios::binary);
  const std::string es((std::istreambuf_iterator<char>(e)), {});
  CHECK(es == "CATSNAP 1 0 16 rowmajor\n");
  CHECK(snapshot_read(tmp + "/empty.bin").n == 0);
  CHECK_THROWS_AS(snapshot_read("/no-such-dir/x.bin"), std::runtime_error, "cannot open");
}

static int wrapi(int v, int n) { return ((v % n) + n) % n; }

static void fragment_passes() {  // test_cat_engine.cpp:36-151, fragment.cpp
  const CatConfig moore = config_for(NeighborhoodKind::Moore);
  const CatConfig vn = config_for(NeighborhoodKind::VonNeumannSimplified);
  {  // single live cell spreads along its row
    Grid g = make_grid(16, 16);
    g.interior(8, 8) = 1;
    Grid frag = frag_grid(g);
    fill_periodic_halo(frag);
    const IntField h = horizontal_step(frag, gen_band_fragments(16, 1), moore);
    CHECK(h.valid);
    for (int y = 0; y < 16; ++y)
      for (int x = 0; x < 16; ++x)
        CHECK(h.at(y + 16, x + 16) == ((y == 8 && x >= 7 && x <= 9) ? 1 : 0));
    const BandFragments b1 = gen_band_fragments(16, 1);
    const IntField box = vertical_step_moore(horizontal_step(frag, b1, moore), b1, moore);
    for (int y = 0; y < 16; ++y)
      for (int x = 0; x < 16; ++x)
        CHECK(box.at(y + 16, x + 16) == ((std::abs(y - 8) <= 1 && std::abs(x - 8) <= 1) ? 1 : 0));
    const IntField hv = horizontal_step(frag, b1, vn);
    const IntField cross = vertical_step_von_neumann(frag, hv, b1, vn);
    for (int y = 0; y < 16; ++y)
      for (int x = 0; x < 16; ++x) {
        int expect = 0;
        if (y == 8 && x == 8) expect = 2;
        else if ((std::abs(y - 8) == 1 && x == 8) || (std::abs(x - 8) == 1 && y == 8)) expect = 1;
        CHECK(cross.at(y + 16, x + 16) == expect);
      }
  }
  {  // torus window / box / cross oracles at several radii
    const Grid base = init_random(48, 0.4, 7);
    for (const int r : {1, 3, 8, 16}) {
      Grid frag = frag_grid(base);
      fill_periodic_halo(frag);
      const BandFragments bands = gen_band_fragments(16, r);
      CatStats st;
      const IntField h = horizontal_step(frag, bands, moore, &st);
      const IntField box = vertical_step_moore(h, bands, moore, &st);
      const IntField hv = horizontal_step(frag, bands, vn);
      const IntField cross = vertical_step_von_neumann(frag, hv, bands, vn);
      int bad = 0;
      for (int y = 0; y < 48; ++y)
        for (int x = 0; x < 48; ++x) {
          int hs = 0, bs = 0, cs = 0;
          for (int dx = -r; dx <= r; ++dx) hs += base.interior(y, wrapi(x + dx, 48));
          for (int dy = -r; dy <= r; ++dy)
            for (int dx = -r; dx <= r; ++dx) bs += base.interior(wrapi(y + dy, 48), wrapi(x + dx, 48));
          for (int dy = -r; dy <= r; ++dy) cs += base.interior(wrapi(y + dy, 48), x);
          cs += hs;
          bad += h.at(y + 16, x + 16) != hs || box.at(y + 16, x + 16) != bs ||
                 cross.at(y + 16, x + 16) != cs;
        }
      CHECK(bad == 0);
      CHECK(st.max_h > 0 && st.max_h <= 2 * r + 1);
      CHECK(st.mma_count == 3 * (5 * 3) + 3 * 9);  // fpr = 5: H 5 rows x 3 cols, R 3 x 3
    }
  }
  {  // sequencing / layout errors (:228-242)
    const BandFragments bands = gen_band_fragments(16, 1);
    Grid stale = frag_grid(init_random(16, 0.5, 1));
    CHECK_THROWS_AS(horizontal_step(stale, bands, moore), std::logic_error, "periodic halo not filled");
    Grid row_major = init_random(16, 0.5, 1);
    fill_periodic_halo(row_major);
    CHECK_THROWS_AS(horizontal_step(row_major, bands, moore), std::invalid_argument, "fragment-contiguous");
    IntField unready = make_field(16, 16);
    CHECK_THROWS_AS(vertical_step_moore(unready, bands, moore), std::logic_error, "not yet computed");
    CHECK_THROWS_AS(gen_band_fragments(16, 17), std::invalid_argument, "unsupported radius r=17");
    CHECK(fp16_exactness_bound(16, NeighborhoodKind::Moore) == 1089);
    CHECK(fp16_exactness_bound(16, NeighborhoodKind::VonNeumannSimplified) == 66);
    const Fragment i4 = identity_fragment(4);
    Fragment a(4);
    for (int k = 0; k < 16; ++k) a.data[k] = k;
    CHECK(mma(a, i4, Fragment(4)).data == a.data);
  }
}

static void anchors(int argc, char** argv, int first) {
  // rule n density seed steps alive fnv (reference runs, anchors.json)
  for (int i = first; i + 6 < argc; i += 7) {
    const LtlRule rule = parse_ltl_rule(argv[i]);
    const int n = std::atoi(argv[i + 1]);
    const Grid start = init_random(n, std::atof(argv[i + 2]), std::strtoull(argv[i + 3], nullptr, 10));
    const int steps = std::atoi(argv[i + 4]);
    const Grid got = run_engine(EngineKind::Cat, start, rule, config_for(rule.kind), steps);
    CHECK(count_alive(got) == std::atoll(argv[i + 5]));
    CHECK(fnv(got) == argv[i + 6]);
  }
}

int main(int argc, char** argv) {
  if (argc < 3) {
    std::fprintf(stderr, "usage: %s GOLDEN_SNAPSHOT_DIR TMP_DIR [anchor...]\n", argv[0]);
    return 2;
  }
  try {
    blinker_and_still_lifes();
    step_loop_equals_simulate();
    errors_and_config();
    accounting_and_fault();
    grid_kats();
    fragment_passes();
    snapshots(argv[1], argv[2]);
    anchors(argc, argv, 3);
  } catch (const std::exception& e) {
    std::fprintf(stderr, "uncaught: %s\n", e.what());
    return 3;
  }
  std::printf("%d checks, %d failed\n", g_checks, g_fail);
  return g_fail ? 1 : 0;
}
