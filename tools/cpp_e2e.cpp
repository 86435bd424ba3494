// cpp_e2e.cpp -- where the time of the C++ drop-in path goes: catsim::run_engine
// (Cat) at n x n for `steps` generations with the reference's pageable Grid,
// split into context creation, upload, generations, download, destruction;
// against ltl_run_interior on the same grid.
//   g++ -std=c++20 -O2 -Iinclude tools/cpp_e2e.cpp -Lpaper_2406_17284_b200 -lltl_b200 \
//       -Wl,-rpath,$PWD/paper_2406_17284_b200 -o build/cpp_e2e && ./build/cpp_e2e 16384 20
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "catsim/catsim.hpp"

using clk = std::chrono::steady_clock;
static double ms(clk::time_point a, clk::time_point b) {
  return std::chrono::duration<double, std::milli>(b - a).count();
}

int main(int argc, char** argv) {
  const int n = argc > 1 ? std::atoi(argv[1]) : 16384;
  const int steps = argc > 2 ? std::atoi(argv[2]) : 20;
  const catsim::LtlRule rule = catsim::parse_ltl_rule("R5,C2,M1,S34..58,B34..45,NM");
  catsim::CatConfig cfg;
  const catsim::Grid g = catsim::init_random(n, 0.21, 1);
  for (int rep = 0; rep < 4; ++rep) {
    const auto t0 = clk::now();
    const catsim::Grid out = catsim::run_engine(catsim::EngineKind::Cat, g, rule, cfg, steps);
    const auto t1 = clk::now();
    // the same call, split
    ltl_ctx* ctx = nullptr;
    const auto a = clk::now();
    ltl_create_grid(&ctx, n, 16);
    const auto b = clk::now();
    ltl_upload(ctx, g.cells.data(), LTL_LAYOUT_ROW_MAJOR);
    const auto c = clk::now();
    const ltl_rule_c rc = catsim::detail::to_c(rule);
    ltl_run(ctx, &rc, steps, 0, nullptr);
    const auto d = clk::now();
    catsim::Grid o2 = g;
    const auto e = clk::now();
    ltl_download_padded(ctx, o2.cells.data(), LTL_LAYOUT_ROW_MAJOR, 0);
    const auto f = clk::now();
    std::vector<uint8_t> in(static_cast<size_t>(n) * n), res(in.size());
    for (int y = 0; y < n; ++y)
      for (int x = 0; x < n; ++x) in[static_cast<size_t>(y) * n + x] = g.interior(y, x);
    const auto h0 = clk::now();
    ltl_run_interior(ctx, in.data(), res.data(), &rc, steps, 0, nullptr);
    const auto h1 = clk::now();
    ltl_destroy(ctx);
    const auto h2 = clk::now();
    std::printf("rep %d: run_engine %.1f ms | create %.1f upload %.1f run %.1f copy-out-grid %.1f "
                "download %.1f destroy %.1f | ltl_run_interior (pageable dense) %.1f ms | same=%d\n",
                rep, ms(t0, t1), ms(a, b), ms(b, c), ms(c, d), ms(d, e), ms(e, f), ms(h1, h2),
                ms(h0, h1), out.cells == o2.cells);
  }
  return 0;
}
