// ubench_stream3.cu -- strip-contiguous vs row-major streaming for the LTL step
// (no compute).  The slab is stored as column strips of 128 cells, each strip
// a contiguous [rows + 32][128] byte block, so one 64-row chunk of a strip is
// one contiguous 8 KB block (one SWIZZLE_128B TMA box).  The 16-column halos
// come from the neighbouring strips as 32-column side boxes (SWIZZLE_32B).
//   mode 0: row-major, whole strips per CTA (the current kernel's pattern)
//   mode 1: strip-contiguous, own box only
//   mode 2: strip-contiguous, own box + 2 side boxes
//   mode 3: strip-contiguous, horizontal walk: a CTA owns bands of B rows and
//           walks the strips left to right; per step ONE contiguous box of
//           B + 32 rows x 128 B (the vertical halo rows come along), the
//           horizontal halo is the previous / next step's box (SMEM reuse).
// Work split for modes 1/2: the S*chunks (strip, chunk) pairs in strip-major
// order, CTA b takes the contiguous range [b*T/G, (b+1)*T/G).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o build/ubench_stream3 tools/ubench_stream3.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

#include "../paper_2406_17284_b200/csrc/ptx_sm100.cuh"

using namespace ltl::ptx;

constexpr int kStages = 6;
constexpr uint32_t kStageBytes = 256 * 128;  // 32 KB

struct Cfg {
  int mode, n, strips, chunks, rows_pad, band;
};

__global__ void __launch_bounds__(128, 1)
    kern(const __grid_constant__ CUtensorMap own, const __grid_constant__ CUtensorMap side,
         const __grid_constant__ CUtensorMap out, Cfg c) {
  extern __shared__ uint8_t raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + kStages * kStageBytes);
  uint64_t* empty = full + kStages;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (threadIdx.x == 0) {
    for (int i = 0; i < kStages; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    fence_barrier_init();
  }
  __syncthreads();
  const long long T = static_cast<long long>(c.strips) * c.chunks;
  long long t0, t1;
  if (c.mode == 0) {
    t0 = 0;
    t1 = 0;
  } else if (c.mode == 3) {
    const long long TB = static_cast<long long>(c.n / c.band) * c.strips;
    t0 = TB * blockIdx.x / gridDim.x;
    t1 = TB * (blockIdx.x + 1) / gridDim.x;
  } else {
    t0 = T * blockIdx.x / gridDim.x;
    t1 = T * (blockIdx.x + 1) / gridDim.x;
  }
  auto for_each = [&](auto&& f) {
    uint32_t g = 0;
    if (c.mode == 0) {
      for (int s = blockIdx.x; s < c.strips; s += gridDim.x)
        for (int k = 0; k < c.chunks; ++k, ++g) f(g, s, k);
    } else if (c.mode == 3) {
      // (band, strip) pairs in band-major order: k = band, s = strip
      for (long long t = t0; t < t1; ++t, ++g) f(g, static_cast<int>(t % c.strips), static_cast<int>(t / c.strips));
    } else {
      for (long long t = t0; t < t1; ++t, ++g) f(g, static_cast<int>(t / c.chunks), static_cast<int>(t % c.chunks));
    }
  };
  if (warp == 0 && lane == 0) {
    for_each([&](uint32_t g, int s, int k) {
      const uint32_t st = g % kStages;
      mbar_wait(&empty[st], ((g / kStages) & 1) ^ 1);
      uint8_t* dst = smem + st * kStageBytes;
      if (c.mode == 3) {
        mbar_arrive_expect_tx(&full[st], (c.band + 32) * 128);
        tma_load_2d(dst, &own, &full[st], 0, (s + 1) * c.rows_pad + k * c.band);
      } else if (c.mode == 0) {
        mbar_arrive_expect_tx(&full[st], 5 * 64 * 32);
        for (int q = 0; q < 5; ++q) tma_load_2d(dst + q * 2048, &side, &full[st], s * 128 + 32 * q, k * 64);
      } else {
        const int base = (s + 1) * c.rows_pad + k * 64;  // storage row of strip s+1 (pad strip 0)
        mbar_arrive_expect_tx(&full[st], c.mode == 2 ? kStageBytes : 64 * 128);
        tma_load_2d(dst, &own, &full[st], 0, base);
        if (c.mode == 2) {
          tma_load_2d(dst + 8192, &side, &full[st], 96, base - c.rows_pad);
          tma_load_2d(dst + 8192 + 2048, &side, &full[st], 0, base + c.rows_pad);
        }
      }
    });
  } else if (warp == 1 && lane == 0) {
    for_each([&](uint32_t g, int s, int k) {
      const uint32_t st = g % kStages;
      mbar_wait(&full[st], (g / kStages) & 1);
      uint8_t* src = smem + st * kStageBytes;
      if (c.mode == 3) {
        tma_store_2d(&out, src, 0, (s + 1) * c.rows_pad + 16 + k * c.band);
      } else if (c.mode == 0) {
        for (int q = 0; q < 4; ++q) tma_store_2d(&out, src + q * 2048, s * 128 + 32 * q, k * 64);
      } else {
        tma_store_2d(&out, src, 0, (s + 1) * c.rows_pad + 16 + k * 64);
      }
      tma_store_commit();
      tma_store_wait_read<0>();
      mbar_arrive(&empty[st]);
    });
    tma_store_wait_all<0>();
  }
}

using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*,
                              CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion,
                              CUtensorMapFloatOOBfill);
static EncodeFn enc;

static void map2d(CUtensorMap* m, void* base, uint64_t w, uint64_t h, uint64_t pitch, uint32_t bw,
                  uint32_t bh, CUtensorMapSwizzle sw) {
  cuuint64_t dims[2] = {w, h}, str[1] = {pitch};
  cuuint32_t box[2] = {bw, bh}, es[2] = {1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, base, dims, str, box, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) std::printf("encode failed %d\n", (int)r);
}

void run(int n, int mode, int grid, const char* name, int band = 64) {
  const int S = n / 128, rows_pad = n + 32, chunks = n / 64;
  size_t bytes;
  if (mode == 0) {
    const int pitch = (n + 32 + 127) / 128 * 128;
    bytes = static_cast<size_t>(rows_pad) * pitch;
  } else {
    bytes = static_cast<size_t>(S + 2) * rows_pad * 128;
  }
  uint8_t *a, *b;
  cudaMalloc(&a, bytes);
  cudaMalloc(&b, bytes);
  cudaMemset(a, 1, bytes);
  CUtensorMap own, side, out;
  if (mode == 0) {
    const int pitch = (n + 32 + 127) / 128 * 128;
    map2d(&side, a, n + 32, rows_pad, pitch, 32, 64, CU_TENSOR_MAP_SWIZZLE_32B);
    map2d(&own, a, n + 32, rows_pad, pitch, 32, 64, CU_TENSOR_MAP_SWIZZLE_32B);
    map2d(&out, b + 16 * pitch + 16, n, n, pitch, 32, 64, CU_TENSOR_MAP_SWIZZLE_32B);
  } else {
    const uint64_t h = static_cast<uint64_t>(S + 2) * rows_pad;
    const uint32_t lrows = mode == 3 ? band + 32 : 64, srows = mode == 3 ? band : 64;
    map2d(&own, a, 128, h, 128, 128, lrows, CU_TENSOR_MAP_SWIZZLE_128B);
    map2d(&side, a, 128, h, 128, 32, 64, CU_TENSOR_MAP_SWIZZLE_32B);
    map2d(&out, b, 128, h, 128, 128, srows, CU_TENSOR_MAP_SWIZZLE_128B);
  }
  Cfg c{mode, n, S, chunks, rows_pad, band};
  const size_t smem = kStages * kStageBytes + 2 * kStages * 8 + 1024;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int w = 0; w < 3; ++w) kern<<<grid, 128, smem>>>(own, side, out, c);
  cudaEventRecord(e0);
  const int it = 20;
  for (int w = 0; w < it; ++w) kern<<<grid, 128, smem>>>(own, side, out, c);
  cudaEventRecord(e1);
  cudaError_t err = cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  const double us = ms * 1000 / it;
  std::printf("n=%5d B=%3d %-36s grid=%3d %8.1f us  %6.0f GB/s (2 B/cell)  %s\n", n, band, name, grid, us,
              2.0 * (mode == 3 ? n / band * band : n) * n / (us * 1e3), cudaGetErrorString(err));
  cudaFree(a);
  cudaFree(b);
}

int main() {
  void* fp = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &q);
  enc = reinterpret_cast<EncodeFn>(fp);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int n : {16384, 32768, 65536}) {
    run(n, 1, sms, "strip-contig own box");
    for (int b : {64, 96, 128, 224}) run(n, 3, sms, "strip-contig horizontal band walk", b);
    for (int b : {64, 128, 224}) run(n, 3, 2 * sms, "horizontal band walk 2/SM", b);
  }
  return 0;
}
