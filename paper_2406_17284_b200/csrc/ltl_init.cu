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
  // mode 0: never alive, 1: always alive, 2: z < threshold.  Rows over
  // blockIdx.y (grid-stride), four consecutive cells per thread (one 32-bit
  // store; four aligned cells never straddle a 128-column strip).
  for (int32_t y = blockIdx.y; y < s.rows; y += gridDim.y) {
    const int32_t gy = row0 + y;
    for (int32_t x0 = 4 * (blockIdx.x * blockDim.x + threadIdx.x); x0 < s.cols;
         x0 += 4 * gridDim.x * blockDim.x) {
      uint32_t word = 0;
#pragma unroll
      for (int b = 0; b < 4; ++b) {
        const int32_t x = x0 + b;
        uint32_t v = 0;
        if (gy < fill_rows && x < fill_cols) {
          if (mode == 1) v = 1;
          else if (mode == 2)
            v = splitmix_at(seed, static_cast<uint64_t>(gy) * fill_cols + x) < threshold ? 1 : 0;
        }
        word |= v << (8 * b);
      }
      uint8_t* cell = s.buf + s.offset(y + kHalo, x0);
      if (x0 + 4 <= s.cols) {
        *reinterpret_cast<uint32_t*>(cell) = word;
      } else {
        for (int b = 0; x0 + b < s.cols; ++b) cell[b] = static_cast<uint8_t>(word >> (8 * b));
      }
    }
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
  const int bx = (s.cols + 4 * 256 - 1) / (4 * 256);
  const int by = s.rows < 4096 ? s.rows : 4096;
  ltl_init_kernel<<<dim3(bx, by), 256, 0, stream>>>(s, row0, fill_rows, fill_cols, seed, thr,
                                                     mode);
  return cudaGetLastError();
}

}  // namespace ltl
