// ltl_halo.cu -- periodic ghost-cell refresh of one device slab.
//
// Device counterpart of fill_periodic_halo (src/grid.cpp:75-94): every halo
// cell receives its modular interior image.  Column wrap is local to the slab;
// the rows above / below the slab come from the interiors of the neighbouring
// slabs (`above`, `below`), which may live on peer GPUs -- the reads then go
// over NVLink straight out of the peer's HBM (peer access).  With one slab all
// three views are the same buffer and this is exactly the reference's
// single-grid fill, including n < 16 where images wrap repeatedly.
//
// All sources are interior cells (never other halo cells), so the parts below
// run concurrently without ordering (`parts` selects them; the step kernel
// fuses them for tile-aligned slabs, ltl_tc.cu):
//   blockIdx.y == 0  side columns of the interior rows (32 cells per row)
//   blockIdx.y == 1  the 16 rows above, all logical columns [-16, cols + 16)
//   blockIdx.y == 2  the 16 rows below
// In the strip layout (ltl_kernels.cuh) a 16-row halo band of one strip is a
// contiguous 2 KB block; interior columns move 16 bytes at a time.
#include <cuda_runtime.h>

#include <cstdint>

#include "ltl_kernels.cuh"

namespace ltl {
namespace {

__device__ __forceinline__ int wrap(int v, int n) {
  const int m = v % n;
  return m < 0 ? m + n : m;
}

__global__ void ltl_halo_kernel(SlabView self, SlabView above, SlabView below, int parts) {
  // PDL: start early, but read the interiors only once the step is complete
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  asm volatile("griddepcontrol.wait;" ::: "memory");
  const int rows = self.rows, cols = self.cols;
  const int tid = blockIdx.x * blockDim.x + threadIdx.x;
  const int nthreads = gridDim.x * blockDim.x;
  if (blockIdx.y == 0) {
    if (!(parts & kHaloCols)) return;
    for (int i = tid; i < rows * 2 * kHalo; i += nthreads) {
      const int y = i / (2 * kHalo), c = i % (2 * kHalo);
      const int px = c < kHalo ? c - kHalo : cols + (c - kHalo);  // [-16, 0) or [cols, cols+16)
      const int py = y + kHalo;
      self.buf[self.offset(py, px)] = self.buf[self.offset(py, wrap(px, cols))];
    }
    return;
  }
  if (!(parts & kHaloRows)) return;
  const bool top = blockIdx.y == 1;
  const SlabView& src = top ? above : below;
  // interior columns in 16-byte groups (cols % 16 == 0), edge cells one by one
  const bool vec = (cols % 16) == 0;
  const int groups = vec ? cols / 16 : 0;
  const int edge = vec ? 2 * kHalo : cols + 2 * kHalo;
  const int per_row = groups + edge;
  for (int i = tid; i < kHalo * per_row; i += nthreads) {
    const int t = i / per_row, e = i % per_row;
    const int py = top ? t : rows + kHalo + t;
    const int sy = (top ? wrap(t - kHalo, src.rows) : wrap(t, src.rows)) + kHalo;
    if (e < groups) {
      const int px = 16 * e;
      *reinterpret_cast<uint4*>(self.buf + self.offset(py, px)) =
          *reinterpret_cast<const uint4*>(src.buf + src.offset(sy, px));
    } else {
      const int b = e - groups;
      const int px = vec ? (b < kHalo ? b - kHalo : cols + b - kHalo) : b - kHalo;
      self.buf[self.offset(py, px)] = src.buf[src.offset(sy, wrap(px, cols))];
    }
  }
}

}  // namespace

cudaError_t launch_halo_fill(const SlabView& self, const SlabView& above, const SlabView& below,
                             int parts, cudaStream_t stream) {
  if (self.rows <= 0 || self.cols <= 0 || parts == 0) return cudaSuccess;
  const int64_t side = 2LL * kHalo * self.rows;
  const int64_t band = kHalo * (self.cols / 4 + 2LL * kHalo);
  int64_t work = side > band ? side : band;
  int blocks = static_cast<int>((work + 255) / 256);
  if (blocks > 148 * 4) blocks = 148 * 4;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(blocks, 3);
  cfg.blockDim = dim3(256);
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, ltl_halo_kernel, self, above, below, parts);
}

}  // namespace ltl
