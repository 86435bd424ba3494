// catsim/snapshot.hpp -- drop-in for proj/include/catsim/snapshot.hpp:
// CATSNAP v1 ("CATSNAP 1 <n> <f> <rowmajor|fragment>\n" + the n x n interior
// bytes, row-major), byte-identical to the reference's files, stream and
// path overloads (src/snapshot.cpp:18-91).
//
// A host Grid is written / read on the host (rows of the interior, no device
// round trip); the header checks are the library's (ltl_snapshot_parse_header,
// the same code the device-streamed ltl_snapshot_read uses), so every
// malformed-file message is the reference's.  Device-resident grids stream
// straight from HBM with ltl_snapshot_write / ltl_snapshot_read instead.
#pragma once

#include <cstring>
#include <fstream>
#include <istream>
#include <ostream>
#include <stdexcept>
#include <string>
#include <vector>

#include "catsim/device.hpp"
#include "catsim/grid.hpp"

namespace catsim {

namespace detail {

[[noreturn]] inline void snapshot_fail(const std::string& why) {
  throw std::runtime_error("snapshot format error: " + why);
}

}  // namespace detail

inline void snapshot_write(const Grid& grid, std::ostream& out) {
  out << "CATSNAP 1 " << grid.n << ' ' << grid.f << ' '
      << (grid.layout == Layout::RowMajor ? "rowmajor" : "fragment") << '\n';
  std::vector<char> row(static_cast<std::size_t>(grid.n));
  for (int y = 0; y < grid.n; ++y) {
    if (grid.layout == Layout::RowMajor) {
      std::memcpy(row.data(), &grid.cells[grid.index(y + grid.f, grid.f)], row.size());
    } else {  // f-byte runs of the fragment rows
      for (int x0 = 0; x0 < grid.n; x0 += grid.f)
        std::memcpy(row.data() + x0, &grid.cells[grid.index(y + grid.f, x0 + grid.f)],
                    static_cast<std::size_t>(grid.f));
    }
    out.write(row.data(), static_cast<std::streamsize>(row.size()));
  }
  if (!out) detail::snapshot_fail("write failed");
}

inline void snapshot_write(const Grid& grid, const std::string& path) {
  std::ofstream out(path, std::ios::binary);
  if (!out) detail::snapshot_fail("cannot open '" + path + "' for writing");
  snapshot_write(grid, out);
}

inline Grid snapshot_read(std::istream& in) {
  std::string header;
  const bool any = static_cast<bool>(std::getline(in, header));
  int32_t n = 0, f = 0, lay = 0;
  detail::check(ltl_snapshot_parse_header(header.c_str(), any ? 1 : 0, &n, &f, &lay), nullptr);
  Grid g = make_grid(n, f, lay == LTL_LAYOUT_ROW_MAJOR ? Layout::RowMajor
                                                       : Layout::FragmentContiguous);
  std::vector<char> row(static_cast<std::size_t>(n));
  for (int y = 0; y < n; ++y) {
    in.read(row.data(), static_cast<std::streamsize>(row.size()));
    if (in.gcount() != static_cast<std::streamsize>(row.size()))
      detail::snapshot_fail("truncated payload (expected " + std::to_string(n) + "x" +
                            std::to_string(n) + " cells)");
    for (int x = 0; x < n; ++x) {
      const auto v = static_cast<uint8_t>(row[static_cast<std::size_t>(x)]);
      if (v > 1) detail::snapshot_fail("cell byte out of {0,1}");
      g.interior(y, x) = v;
    }
  }
  g.halo_valid = false;  // a read-back grid has a stale halo
  return g;
}

inline Grid snapshot_read(const std::string& path) {
  std::ifstream in(path, std::ios::binary);
  if (!in) detail::snapshot_fail("cannot open '" + path + "' for reading");
  return snapshot_read(in);
}

}  // namespace catsim
