// ltl_stencil.cu -- the classical CUDA-core ablation: shared-memory out-halo
// stencil that sums the whole (2r+1)^2 box (Moore) or the 2(2r+1) cross (VN)
// per cell, i.e. the paper's SHARED baseline, on the same
// device slab layout (column strips) as the tensor-core path.  It is also the engine the
// parity tests run next to the tcgen05 kernel: same inputs, same bytes out.
//
// Work per cell grows as (2r+1)^2 -- that radius dependence is exactly what
// the banded-MMA formulation removes (src/cat_engine.cpp).
#include <cuda_runtime.h>

#include <cstdint>

#include "ltl_kernels.cuh"

namespace ltl {
namespace {

constexpr int kTX = 64;   // output columns per block
constexpr int kTY = 32;   // output rows per block
constexpr int kBX = 32, kBY = 8;
constexpr int kSX = kTX + 2 * kHalo;  // 96
constexpr int kSY = kTY + 2 * kHalo;  // 64

__global__ void __launch_bounds__(kBX* kBY)
    ltl_stencil_kernel(const SlabView in, const SlabView out, RuleConsts rc, int inject_fault,
                       DeviceStats* stats) {
  __shared__ uint8_t tile[kSY][kSX];
  const int x0 = blockIdx.x * kTX, y0 = blockIdx.y * kTY;
  const int tid = threadIdx.y * kBX + threadIdx.x;
  const int rows = in.rows, cols = in.cols;
  const int rows_pad = rows + 2 * kHalo;
  // out-halo load: padded rows [y0, y0+kSY), logical cols [x0-16, x0-16+kSX)
  for (int i = tid; i < kSY * kSX; i += kBX * kBY) {
    const int ty = i / kSX, tx = i % kSX;
    const int py = y0 + ty, px = x0 - kHalo + tx;
    tile[ty][tx] = (py < rows_pad && px < cols + kHalo) ? in.buf[in.offset(py, px)] : 0;
  }
  __syncthreads();
  const int r = rc.r;
  int32_t max_h = 0, max_r = 0, bad = 0;
#pragma unroll 1
  for (int j = 0; j < kTX / kBX; ++j) {
#pragma unroll 1
    for (int i = 0; i < kTY / kBY; ++i) {
      const int ly = threadIdx.y + kBY * i, lx = threadIdx.x + kBX * j;
      const int cy = ly + kHalo, cx = lx + kHalo;
      int32_t h = 0;
      for (int dx = -r; dx <= r; ++dx) h += tile[cy][cx + dx];
      int32_t red;
      if (rc.kind == 0) {
        red = 0;
        for (int dy = -r; dy <= r; ++dy)
          for (int dx = -r; dx <= r; ++dx) red += tile[cy + dy][cx + dx];
      } else {
        red = h;
        for (int dy = -r; dy <= r; ++dy) red += tile[cy + dy][cx];
      }
      const uint32_t st = tile[cy][cx];
      if (inject_fault && ((x0 + lx) & 127) == 0) red -= st;  // mirror of the TC fault hook
      const int y = y0 + ly, x = x0 + lx;
      if (y < rows && x < cols) {
        max_h = max(max_h, h);
        max_r = max(max_r, red);
        bad |= (st && red < rc.neg_live);
        const int32_t lo = st ? rc.lo_live : rc.lo_dead;
        const uint32_t w = static_cast<uint32_t>(st ? rc.w_live : rc.w_dead);
        out.buf[out.offset(y + kHalo, x)] = (static_cast<uint32_t>(red - lo) <= w) ? 1 : 0;
      }
    }
  }
  if (stats) {
    for (int off = 16; off > 0; off >>= 1) {
      max_h = max(max_h, __shfl_xor_sync(0xffffffffu, max_h, off));
      max_r = max(max_r, __shfl_xor_sync(0xffffffffu, max_r, off));
    }
    if (threadIdx.x == 0) {
      atomicMax(&stats->max_h, max_h);
      atomicMax(&stats->max_r, max_r);
    }
    if (__any_sync(0xffffffffu, bad) && threadIdx.x == 0) atomicOr(&stats->error, 1);
  }
}

}  // namespace

cudaError_t launch_stencil_step(const SlabView& in, const SlabView& out, const RuleConsts& rule,
                                int32_t inject_fault, DeviceStats* stats, cudaStream_t stream) {
  if (in.rows <= 0 || in.cols <= 0) return cudaSuccess;
  dim3 grid((in.cols + kTX - 1) / kTX, (in.rows + kTY - 1) / kTY);
  ltl_stencil_kernel<<<grid, dim3(kBX, kBY), 0, stream>>>(in, out, rule, inject_fault, stats);
  return cudaGetLastError();
}

}  // namespace ltl
