// catsim/grid.hpp -- drop-in for the reference's proj/include/catsim/grid.hpp:
// the same Grid / IntField value types, make_grid, init_random,
// fill_periodic_halo, count_alive and first_interior_difference, with the
// same error messages.  init_random and fill_periodic_halo run on the device
// (ltl_init_random, ltl_fill_halo); the grid itself stays a host value type.
#pragma once

#include <cmath>
#include <cstddef>
#include <cstdint>
#include <cstring>
#include <optional>
#include <stdexcept>
#include <string>
#include <vector>

#include "catsim/device.hpp"

namespace catsim {

inline constexpr int kDefaultFragmentSide = 16;

// In-memory cell order of the padded buffer (grid.hpp:14).
enum class Layout { RowMajor, FragmentContiguous };

namespace detail {

inline std::size_t fragment_offset(int f, int fragments_per_row, int y, int x) {
  const int fy = y / f, fx = x / f;
  return (static_cast<std::size_t>(fy) * fragments_per_row + fx) *
             (static_cast<std::size_t>(f) * f) +
         static_cast<std::size_t>(y % f) * f + (x % f);
}

inline int32_t c_layout(Layout l) {
  return l == Layout::RowMajor ? LTL_LAYOUT_ROW_MAJOR : LTL_LAYOUT_FRAGMENT;
}

// grid.cpp:11-17
inline void check_geometry(int n, int f) {
  if (f <= 0) throw std::invalid_argument("geometry error: f must be positive");
  if (n < 0 || n % f != 0)
    throw std::invalid_argument("geometry error: n (" + std::to_string(n) +
                                ") must be a non-negative multiple of f (" +
                                std::to_string(f) + ")");
}

}  // namespace detail

// splitmix64 (grid.hpp:31-43), the stream pinned by the reference's KATs.
struct SplitMix64 {
  uint64_t state;
  explicit SplitMix64(uint64_t seed) : state(seed) {}
  uint64_t next() {
    state += 0x9E3779B97F4A7C15ULL;
    uint64_t z = state;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
  }
};

// Exact "z / 2^64 < density" (grid.cpp:21-39): compared in integers on the
// scaled mantissa.
inline bool alive_threshold(uint64_t z, double density) {
  if (std::isnan(density) || density <= 0.0) return false;
  if (density >= 1.0) return true;
  int e = 0;
  const double frac = std::frexp(density, &e);
  const uint64_t m = static_cast<uint64_t>(std::ldexp(frac, 53));
  const int sh = e + 11;
  if (sh >= 0) return z < (m << sh);
  if (-sh >= 64) return z == 0;
  const int right = -sh;  // z * 2^right < m  <=>  z < ceil(m / 2^right)
  const uint64_t t = (m >> right) + (((m & ((1ULL << right) - 1)) != 0) ? 1 : 0);
  return z < t;
}

struct Grid {
  int n = 0;
  int f = kDefaultFragmentSide;
  Layout layout = Layout::RowMajor;
  bool halo_valid = false;
  std::vector<uint8_t> cells;  // (n + 2f)^2 values in {0, 1}

  int halo() const { return f; }
  int padded() const { return n + 2 * f; }
  int fragments_per_row() const { return padded() / f; }
  std::size_t index(int y, int x) const {
    if (layout == Layout::RowMajor) return static_cast<std::size_t>(y) * padded() + x;
    return detail::fragment_offset(f, fragments_per_row(), y, x);
  }
  uint8_t at(int y, int x) const { return cells[index(y, x)]; }
  uint8_t& at(int y, int x) { return cells[index(y, x)]; }
  uint8_t interior(int iy, int ix) const { return at(iy + f, ix + f); }
  uint8_t& interior(int iy, int ix) { return at(iy + f, ix + f); }
};

struct IntField {
  int n = 0;
  int f = kDefaultFragmentSide;
  Layout layout = Layout::FragmentContiguous;
  bool valid = false;
  std::vector<int32_t> values;

  int padded() const { return n + 2 * f; }
  int fragments_per_row() const { return padded() / f; }
  std::size_t index(int y, int x) const {
    if (layout == Layout::RowMajor) return static_cast<std::size_t>(y) * padded() + x;
    return detail::fragment_offset(f, fragments_per_row(), y, x);
  }
  int32_t at(int y, int x) const { return values[index(y, x)]; }
  int32_t& at(int y, int x) { return values[index(y, x)]; }
};

// All-dead grid (grid.cpp:41-49).
inline Grid make_grid(int n, int f = kDefaultFragmentSide, Layout layout = Layout::RowMajor) {
  detail::check_geometry(n, f);
  Grid g;
  g.n = n;
  g.f = f;
  g.layout = layout;
  detail::fresh_cells(g.cells, static_cast<std::size_t>(g.padded()) * g.padded());
  return g;
}

namespace detail {

// A grid of `like`'s geometry and layout whose halo bytes are `like`'s and
// whose interior is left zero for a device result to land in -- the output
// of run_engine without copying a whole grid it is about to overwrite.
inline Grid grid_like(const Grid& like) {
  Grid g;
  g.n = like.n;
  g.f = like.f;
  g.layout = like.layout;
  g.halo_valid = like.halo_valid;
  const std::size_t p = static_cast<std::size_t>(like.padded());
  fresh_cells(g.cells, p * p);
  if (like.layout == Layout::RowMajor) {
    const std::size_t f = static_cast<std::size_t>(like.f), n = static_cast<std::size_t>(like.n);
    for (std::size_t y = 0; y < p; ++y) {
      const uint8_t* src = like.cells.data() + y * p;
      uint8_t* dst = g.cells.data() + y * p;
      if (y < f || y >= f + n) {
        std::memcpy(dst, src, p);
      } else {
        std::memcpy(dst, src, f);
        std::memcpy(dst + f + n, src + f + n, f);
      }
    }
  } else {
    g.cells = like.cells;
  }
  return g;
}

}  // namespace detail

inline IntField make_field(int n, int f = kDefaultFragmentSide,
                           Layout layout = Layout::FragmentContiguous) {
  detail::check_geometry(n, f);
  IntField h;
  h.n = n;
  h.f = f;
  h.layout = layout;
  h.values.assign(static_cast<std::size_t>(h.padded()) * h.padded(), 0);
  return h;
}

// init_random (grid.cpp:61-73): generated on the device (counter-form
// splitmix64, bit-identical, ltl_init_random) and landed in the row-major
// grid's interior by one pitched copy; the halo stays dead and stale.
inline Grid init_random(int n, double density, uint64_t seed, int f = kDefaultFragmentSide,
                        int fill_n = -1) {
  if (!(density >= 0.0 && density <= 1.0) || std::isnan(density))
    throw std::invalid_argument("init_random: density must be in [0, 1]");
  if (fill_n < 0) fill_n = n;
  if (fill_n > n) throw std::invalid_argument("init_random: fill_n exceeds n");
  Grid g = make_grid(n, f, Layout::RowMajor);
  if (n == 0 || fill_n == 0) return g;
  detail::DeviceGrid dev(n, f);
  dev.check(ltl_init_random(dev.get(), density, seed, fill_n));
  dev.check(ltl_download_padded(dev.get(), g.cells.data(), LTL_LAYOUT_ROW_MAJOR, 0));
  return g;
}

// fill_periodic_halo (grid.cpp:75-94): the halo cells' periodic images, on the
// host (ltl_host_fill_halo: 4fn + 4f^2 cells, the interior is not touched).
inline void fill_periodic_halo(Grid& grid) {
  if (grid.n > 0)
    detail::check(ltl_host_fill_halo(grid.cells.data(), grid.n, grid.f, detail::c_layout(grid.layout)),
                  nullptr);
  grid.halo_valid = true;
}

inline long long count_alive(const Grid& grid) {
  long long n = 0;
  for (int y = 0; y < grid.n; ++y)
    for (int x = 0; x < grid.n; ++x) n += grid.interior(y, x);
  return n;
}

struct CellCoord {
  int y = 0, x = 0;
};

inline std::optional<CellCoord> first_interior_difference(const Grid& a, const Grid& b) {
  if (a.n != b.n) throw std::invalid_argument("geometry error: grids differ in n");
  for (int y = 0; y < a.n; ++y)
    for (int x = 0; x < a.n; ++x)
      if (a.interior(y, x) != b.interior(y, x)) return CellCoord{y, x};
  return std::nullopt;
}

}  // namespace catsim
