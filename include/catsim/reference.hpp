// catsim/reference.hpp -- drop-in for proj/include/catsim/reference.hpp: the
// reference's two comparison engines, BASE (per-cell window sums) and PACK
// (eight byte lanes per 64-bit word), with their types, checks, messages and
// BASE's access accounting (src/reference.cpp).
//
// Here both run on the B200 as the CUDA-core ablations of this repo
// (csrc/ltl_stencil.cu): base_step / simulate_base -> the direct-sum stencil
// (LTL_FLAG_ENGINE_BASE, (2r+1)^2 adds per cell like the reference's BASE),
// pack_step / simulate_packed -> the packed-lane sliding-window stencil
// (LTL_FLAG_ENGINE_PACK).  PackedGrid and its pack / unpack / halo fill are the
// reference's host data format, kept on the host.  The device engines refill
// the periodic halo themselves (the reference requires it filled first and
// reads the same images).
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "catsim/cat_engine.hpp"
#include "catsim/grid.hpp"
#include "catsim/rule.hpp"

namespace catsim {

// Accesses BASE makes: every window read, the centre read and the write; a
// Moore cell costs (2r+1)^2 + 2 (reference.hpp:15-22).
struct BaseStats {
  long long window_reads = 0;
  long long cell_reads = 0;
  long long writes = 0;
  long long cells = 0;
  long long accesses() const { return window_reads + cell_reads + writes; }
};

namespace detail {

// reference.cpp:11-18
inline void check_base_inputs(const Grid& grid, const Grid& out) {
  if (grid.layout != Layout::RowMajor || out.layout != Layout::RowMajor)
    throw std::invalid_argument("layout error: expected row-major grids");
  if (!grid.halo_valid) throw std::logic_error("sequencing error: periodic halo not filled");
  if (out.n != grid.n || out.f != grid.f)
    throw std::invalid_argument("geometry error: output grid shape mismatch");
}

inline void count_base_accesses(BaseStats* st, const LtlRule& rule, int n, int steps) {
  if (!st) return;
  const long long cells = static_cast<long long>(n) * n * steps;
  const long long w = 2LL * rule.r + 1;
  st->window_reads += cells * (rule.kind == NeighborhoodKind::Moore ? w * w : 2 * w);
  st->cell_reads += cells;
  st->writes += cells;
  st->cells += cells;
}

inline void check_pack_width(int padded) {
  if (padded % 8 != 0)
    throw std::invalid_argument("geometry error: padded width " + std::to_string(padded) +
                                " must be a multiple of 8 to pack");
}

inline void check_pack_halo(int f, int r) {
  const int need = 8 * ((r + 7) / 8);  // whole neighbour words per side
  if (f < need)
    throw std::invalid_argument("geometry error: halo " + std::to_string(f) +
                                " too small for radius " + std::to_string(r) +
                                " word gathers (needs >= " + std::to_string(need) + ")");
}

}  // namespace detail

// One generation of the per-cell engine: row-major grids, grid's halo filled.
inline void base_step(const Grid& grid, const LtlRule& rule, Grid& out, BaseStats* stats = nullptr) {
  detail::check_base_inputs(grid, out);
  detail::run_device_engine(grid, rule, 1, LTL_FLAG_ENGINE_BASE, out, nullptr);
  detail::count_base_accesses(stats, rule, grid.n, 1);
  out.halo_valid = false;
}

// `steps` generations, the halo refreshed before each (reference.cpp:78-92).
inline Grid simulate_base(Grid grid, const LtlRule& rule, int steps, BaseStats* stats = nullptr) {
  if (steps < 0) throw std::invalid_argument("config error: steps must be >= 0");
  if (steps == 0) return grid;
  if (grid.layout != Layout::RowMajor)
    throw std::invalid_argument("layout error: expected row-major grids");
  detail::run_device_engine(grid, rule, steps, LTL_FLAG_ENGINE_BASE, grid, nullptr);
  detail::count_base_accesses(stats, rule, grid.n, steps);
  grid.halo_valid = false;
  return grid;
}

// Eight cells per 64-bit word, lane 0 in the least-significant byte.
struct PackedGrid {
  int n = 0;
  int f = kDefaultFragmentSide;
  bool halo_valid = false;
  std::vector<uint64_t> words;

  int padded() const { return n + 2 * f; }
  int words_per_row() const { return padded() / 8; }
  uint8_t cell(int y, int x) const {
    const uint64_t w = words[static_cast<std::size_t>(y) * words_per_row() + x / 8];
    return static_cast<uint8_t>(w >> (8 * (x % 8)));
  }
  void set_cell(int y, int x, uint8_t v) {
    uint64_t& w = words[static_cast<std::size_t>(y) * words_per_row() + x / 8];
    const int shift = 8 * (x % 8);
    w = (w & ~(uint64_t{0xFF} << shift)) | (uint64_t{v} << shift);
  }
};

inline PackedGrid pack(const Grid& grid) {
  detail::check_pack_width(grid.padded());
  PackedGrid out;
  out.n = grid.n;
  out.f = grid.f;
  out.halo_valid = grid.halo_valid;
  const int p = grid.padded();
  out.words.assign(static_cast<std::size_t>(p) * (p / 8), 0);
  for (int y = 0; y < p; ++y)
    for (int x = 0; x < p; ++x)
      out.words[static_cast<std::size_t>(y) * (p / 8) + x / 8] |= uint64_t{grid.at(y, x)}
                                                                  << (8 * (x % 8));
  return out;
}

inline Grid unpack(const PackedGrid& packed) {
  Grid out = make_grid(packed.n, packed.f, Layout::RowMajor);
  const int p = packed.padded();
  for (int y = 0; y < p; ++y)
    for (int x = 0; x < p; ++x) out.at(y, x) = packed.cell(y, x);
  out.halo_valid = packed.halo_valid;
  return out;
}

inline void fill_periodic_halo(PackedGrid& packed) {
  if (packed.n > 0) {
    Grid g = unpack(packed);
    fill_periodic_halo(g);
    packed.words = pack(g).words;
  }
  packed.halo_valid = true;
}

// One generation on packed words (the interior words of `out` are written).
inline void pack_step(const PackedGrid& packed, const LtlRule& rule, PackedGrid& out) {
  if (!packed.halo_valid) throw std::logic_error("sequencing error: periodic halo not filled");
  if (out.n != packed.n || out.f != packed.f)
    throw std::invalid_argument("geometry error: output grid shape mismatch");
  detail::check_pack_halo(packed.f, rule.r);
  const Grid in = unpack(packed);
  Grid next = unpack(out);
  detail::run_device_engine(in, rule, 1, LTL_FLAG_ENGINE_PACK, next, nullptr);
  out.words = pack(next).words;
  out.halo_valid = false;
}

inline PackedGrid simulate_packed(PackedGrid packed, const LtlRule& rule, int steps) {
  if (steps < 0) throw std::invalid_argument("config error: steps must be >= 0");
  if (steps == 0) return packed;
  detail::check_pack_halo(packed.f, rule.r);
  Grid g = unpack(packed);
  detail::run_device_engine(g, rule, steps, LTL_FLAG_ENGINE_PACK, g, nullptr);
  PackedGrid out = pack(g);
  out.halo_valid = false;
  return out;
}

}  // namespace catsim
