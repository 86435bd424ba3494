// ltl_init.cu -- deterministic random fill, generated on the device.
//
// init_random (src/grid.cpp:61-73) draws one splitmix64 value per interior
// cell of the top-left fill_n x fill_n block in row-major order.  splitmix64
// (include/catsim/grid.hpp:31-43) is a counter-based generator -- the k-th
// draw is mix(seed + (k+1) * 0x9E3779B97F4A7C15) -- so cell (y, x) can be
// drawn independently with k = y * fill_n + x.  alive_threshold
// (src/grid.cpp:21-39) is an exact comparison against density * 2^64; the
// host reduces it to "z < T" (or "always") once, so the device predicate is
// a single 64-bit compare and the grid is bit-identical to the reference's.
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>

#include "ltl_kernels.cuh"

namespace ltl {
namespace {

__device__ __forceinline__ uint64_t splitmix_at(uint64_t seed, uint64_t k) {
  uint64_t z = seed + (k + 1) * 0x9E3779B97F4A7C15ULL;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

__global__ void ltl_init_kernel(SlabView s, int32_t row0, int32_t fill_rows, int32_t fill_cols,
                                uint64_t seed, uint64_t threshold, int32_t mode) {
  // mode 0: never alive, 1: always alive, 2: z < threshold
  const int64_t total = static_cast<int64_t>(s.rows) * s.cols;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int32_t y = static_cast<int32_t>(i / s.cols), x = static_cast<int32_t>(i % s.cols);
    const int32_t gy = row0 + y;
    uint8_t v = 0;
    if (gy < fill_rows && x < fill_cols) {
      if (mode == 1) v = 1;
      else if (mode == 2)
        v = splitmix_at(seed, static_cast<uint64_t>(gy) * fill_cols + x) < threshold ? 1 : 0;
    }
    s.buf[(y + kHalo) * s.pitch + (x + kHalo)] = v;
  }
}

}  // namespace

// Exact reduction of alive_threshold(z, density) to {never, always, z < T}.
void density_threshold(double density, int32_t* mode, uint64_t* threshold) {
  *threshold = 0;
  if (std::isnan(density) || density <= 0.0) {
    *mode = 0;
    return;
  }
  if (density >= 1.0) {
    *mode = 1;
    return;
  }
  int e = 0;
  const double frac = std::frexp(density, &e);
  const uint64_t m = static_cast<uint64_t>(std::ldexp(frac, 53));
  const int sh = e + 11;  // <= 11 because density < 1
  *mode = 2;
  if (sh >= 0) {
    *threshold = m << sh;  // m < 2^53, sh <= 11: fits in 64 bits
  } else if (-sh >= 64) {
    *threshold = 1;  // only z = 0 sits below a bound in (0, 1)
  } else {
    // z * 2^right < m  <=>  z < ceil(m / 2^right)
    const int right = -sh;
    *threshold = (m >> right) + (((m & ((1ULL << right) - 1)) != 0) ? 1 : 0);
  }
}

cudaError_t launch_init_random(const SlabView& s, int32_t row0, int32_t fill_rows,
                               int32_t fill_cols, double density, uint64_t seed,
                               cudaStream_t stream) {
  if (s.rows <= 0 || s.cols <= 0) return cudaSuccess;
  int32_t mode;
  uint64_t thr;
  density_threshold(density, &mode, &thr);
  const int64_t total = static_cast<int64_t>(s.rows) * s.cols;
  int blocks = static_cast<int>((total + 255) / 256);
  if (blocks > 148 * 32) blocks = 148 * 32;
  ltl_init_kernel<<<blocks, 256, 0, stream>>>(s, row0, fill_rows, fill_cols, seed, thr, mode);
  return cudaGetLastError();
}

}  // namespace ltl
