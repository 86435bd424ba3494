// ltl_halo.cu -- periodic ghost-cell refresh of one device slab.
//
// Device counterpart of fill_periodic_halo (src/grid.cpp:75-94): every halo
// cell receives its modular interior image.  Column wrap is local to the slab;
// the rows above / below the slab come from the interiors of the neighbouring
// slabs (`above`, `below`), which may live on peer GPUs -- the reads then go
// over NVLink straight out of the peer's HBM (peer access / IPC mappings).
// With one slab all three views are the same buffer and this is exactly the
// reference's single-grid fill, including n < 16 where images wrap repeatedly.
#include <cuda_runtime.h>

#include <cstdint>

#include "ltl_kernels.cuh"

namespace ltl {
namespace {

__device__ __forceinline__ int wrap(int v, int n) {
  const int m = v % n;
  return m < 0 ? m + n : m;
}

__global__ void ltl_halo_kernel(SlabView self, SlabView above, SlabView below) {
  const int rows = self.rows, cols = self.cols;
  const int64_t band = static_cast<int64_t>(kHalo) * (cols + 2 * kHalo);  // cells per row band
  const int64_t side = static_cast<int64_t>(rows) * 2 * kHalo;            // left+right columns
  // rows < 0 on the neighbour views: row bands come from an external transport
  const bool rows_too = above.rows >= 0 && below.rows >= 0;
  const int64_t total = 2 * band + side;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    if (!rows_too && i < 2 * band) continue;
    int py, px;
    if (i < 2 * band) {
      const int64_t b = i % band;
      py = static_cast<int>(b / (cols + 2 * kHalo)) + (i < band ? 0 : rows + kHalo);
      px = static_cast<int>(b % (cols + 2 * kHalo));
    } else {
      const int64_t s = i - 2 * band;
      py = static_cast<int>(s / (2 * kHalo)) + kHalo;
      const int c = static_cast<int>(s % (2 * kHalo));
      px = c < kHalo ? c : cols + c;  // left: 0..15, right: cols+16..cols+31
    }
    const int sx = wrap(px - kHalo, cols);
    const SlabView* src;
    int sy;
    if (py < kHalo) {
      src = &above;
      sy = wrap(py - kHalo, above.rows);
    } else if (py >= rows + kHalo) {
      src = &below;
      sy = wrap(py - kHalo - rows, below.rows);
    } else {
      src = &self;
      sy = py - kHalo;
    }
    self.buf[py * self.pitch + px] = src->buf[(sy + kHalo) * src->pitch + (sx + kHalo)];
  }
}

}  // namespace

cudaError_t launch_halo_fill(const SlabView& self, const SlabView& above, const SlabView& below,
                             cudaStream_t stream) {
  if (self.rows <= 0 || self.cols <= 0) return cudaSuccess;
  const int64_t total = 2LL * kHalo * (self.cols + 2 * kHalo) + 2LL * kHalo * self.rows;
  int blocks = static_cast<int>((total + 255) / 256);
  if (blocks > 148 * 16) blocks = 148 * 16;
  ltl_halo_kernel<<<blocks, 256, 0, stream>>>(self, above, below);
  return cudaGetLastError();
}

}  // namespace ltl
