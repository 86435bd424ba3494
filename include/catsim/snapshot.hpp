// catsim/snapshot.hpp -- drop-in for proj/include/catsim/snapshot.hpp (path
// overloads): CATSNAP v1 files, byte-identical to the reference's, streamed
// through the device (ltl_snapshot_write / ltl_snapshot_read).
#pragma once

#include <cstdio>
#include <stdexcept>
#include <string>
#include <vector>

#include "catsim/device.hpp"
#include "catsim/grid.hpp"

namespace catsim {

inline void snapshot_write(const Grid& grid, const std::string& path) {
  if (grid.n == 0) {  // header only; no device grid needed
    std::FILE* fh = std::fopen(path.c_str(), "wb");
    if (!fh)
      throw std::runtime_error("snapshot format error: cannot open '" + path + "' for writing");
    const std::string header = "CATSNAP 1 0 " + std::to_string(grid.f) + " " +
                               (grid.layout == Layout::RowMajor ? "rowmajor" : "fragment") + "\n";
    const bool ok = std::fwrite(header.data(), 1, header.size(), fh) == header.size();
    if (std::fclose(fh) != 0 || !ok) throw std::runtime_error("snapshot format error: write failed");
    return;
  }
  detail::DeviceGrid dev(grid.n, grid.f);
  const int32_t lay = detail::c_layout(grid.layout);
  dev.check(ltl_upload(dev.get(), grid.cells.data(), lay));
  dev.check(ltl_snapshot_write(dev.get(), path.c_str(), lay));
}

inline Grid snapshot_read(const std::string& path) {
  int32_t n = 0, f = 0, lay = 0;
  detail::check(ltl_snapshot_probe(path.c_str(), &n, &f, &lay), nullptr);
  const Layout layout = lay == LTL_LAYOUT_ROW_MAJOR ? Layout::RowMajor : Layout::FragmentContiguous;
  Grid g = make_grid(n, f, layout);
  if (n > 0) {
    detail::DeviceGrid dev(n, f);
    dev.check(ltl_snapshot_read(dev.get(), path.c_str(), &lay));
    std::vector<uint8_t> padded(g.cells.size());
    dev.check(ltl_download(dev.get(), padded.data(), lay));
    for (int y = 0; y < n; ++y)  // the halo of a read-back grid stays dead and stale
      for (int x = 0; x < n; ++x) g.interior(y, x) = padded[g.index(y + f, x + f)];
  }
  g.halo_valid = false;
  return g;
}

}  // namespace catsim
