// ubench_stream2.cu -- streaming-pattern study for the LTL step (no compute).
// Mode V: vertical streaming (CTA walks a 128-col strip down in 64-row chunks;
//         loads 160 cols x 64 rows, stores 128 x 64)       -- the current kernel
// Mode H: horizontal streaming (CTA owns a band of 64 output rows, loads 96
//         rows x 160 cols per 128-col step walking along x) -- candidate
// Mode T: vertical, but each CTA streams `W` adjacent strips as one unit
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o build/ubench_stream2 tools/ubench_stream2.cu
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

#include "../paper_2406_17284_b200/csrc/ptx_sm100.cuh"

using namespace ltl::ptx;

constexpr int kStages = 8;
constexpr uint32_t kStageMax = 96 * 288;

struct Cfg {
  int sync_every;  // >0: CTAs keep within one window of `sync_every` steps of each other
  unsigned int* progress;
  int mode;        // 0 = V, 1 = H
  int n;           // interior side
  int units;       // strips (V) or bands (H)
  int steps;       // chunks per unit (V: row chunks, H: column steps)
  int in_rows;     // rows per load (64 for V, 96 for H)
  int in_cols;     // columns per load (160 or 128*W+32)
  int out_cols;    // columns stored per step
};

__global__ void __launch_bounds__(128, 1) kern(const __grid_constant__ CUtensorMap lmap,
                                              const __grid_constant__ CUtensorMap smap, Cfg c) {
  extern __shared__ uint8_t raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + kStages * kStageMax);
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
  const int nbox = c.in_cols / 32;
  const uint32_t box_bytes = 32 * c.in_rows;
  if (warp == 0 && lane == 0) {
    uint32_t g = 0;
    for (int u = blockIdx.x; u < c.units; u += gridDim.x)
      for (int k = 0; k < c.steps; ++k, ++g) {
        const uint32_t s = g % kStages;
        mbar_wait(&empty[s], ((g / kStages) & 1) ^ 1);
        if (c.sync_every > 0 && g % c.sync_every == 0) {
          // publish my progress, then wait until every CTA reached g - window
          const unsigned int epoch = g / c.sync_every;
          atomicAdd(c.progress + epoch % 64, 1u);
          if (epoch >= 2) {
            volatile unsigned int* slot = c.progress + (epoch - 2) % 64;
            while (*slot < gridDim.x) __nanosleep(200);
          }
        }
        mbar_arrive_expect_tx(&full[s], nbox * box_bytes);
        const int x0 = c.mode == 0 ? u * (c.in_cols - 32) : k * 128;
        const int y0 = c.mode == 0 ? k * 64 : u * 64;
        for (int b = 0; b < nbox; ++b)
          tma_load_2d(smem + s * kStageMax + b * box_bytes, &lmap, &full[s], x0 + 32 * b, y0);
      }
  } else if (warp == 1 && lane == 0) {
    uint32_t g = 0;
    for (int u = blockIdx.x; u < c.units; u += gridDim.x)
      for (int k = 0; k < c.steps; ++k, ++g) {
        const uint32_t s = g % kStages;
        mbar_wait(&full[s], (g / kStages) & 1);
        const int x0 = c.mode == 0 ? u * (c.in_cols - 32) : k * 128;
        const int y0 = c.mode == 0 ? k * 64 : u * 64;
        for (int b = 0; b < c.out_cols / 32; ++b)
          tma_store_2d(&smap, smem + s * kStageMax + b * box_bytes, x0 + 32 * b, y0);
        tma_store_commit();
        tma_store_wait_read<2>();
        mbar_arrive(&empty[s]);  // (approximate: the slot may still be read by a store)
      }
    tma_store_wait_all<0>();
  }
}

using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*,
                              CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion,
                              CUtensorMapFloatOOBfill);

static EncodeFn enc;

void run(int n, int mode, int wide, int grid, const char* name, int sync_every = 0) {
  const int pad = n + 32, pitch = (pad + 127) / 128 * 128;
  uint8_t *a, *b;
  cudaMalloc(&a, (size_t)pad * pitch);
  cudaMalloc(&b, (size_t)pad * pitch);
  cudaMemset(a, 1, (size_t)pad * pitch);
  const int in_rows = mode == 0 ? 64 : 96;
  CUtensorMap lmap, smap;
  cuuint64_t dims[2] = {(cuuint64_t)pad, (cuuint64_t)pad}, str[1] = {(cuuint64_t)pitch};
  cuuint32_t box[2] = {32, (cuuint32_t)in_rows}, es[2] = {1, 1};
  enc(&lmap, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, a, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
      CU_TENSOR_MAP_SWIZZLE_32B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  cuuint64_t sd[2] = {(cuuint64_t)n, (cuuint64_t)n};
  cuuint32_t sbox[2] = {32, 64};
  enc(&smap, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, b + 16 * pitch + 16, sd, str, sbox, es,
      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_32B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
      CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  Cfg c;
  c.sync_every = sync_every;
  cudaMalloc(&c.progress, 64 * sizeof(unsigned int));
  c.mode = mode;
  c.n = n;
  c.in_rows = in_rows;
  c.in_cols = 128 * wide + 32;
  c.out_cols = 128 * wide;
  c.units = mode == 0 ? n / (128 * wide) : n / 64;
  c.steps = mode == 0 ? n / 64 : n / 128;
  const size_t smem = kStages * kStageMax + 2 * kStages * 8 + 1024;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int w = 0; w < 2; ++w) {
    cudaMemset(c.progress, 0, 64 * sizeof(unsigned int));
    kern<<<grid, 128, smem>>>(lmap, smap, c);
  }
  cudaEventRecord(e0);
  const int it = 10;
  for (int w = 0; w < it; ++w) {
    cudaMemsetAsync(c.progress, 0, 64 * sizeof(unsigned int));
    kern<<<grid, 128, smem>>>(lmap, smap, c);
  }
  cudaEventRecord(e1);
  cudaError_t err = cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  const double us = ms * 1000 / it;
  std::printf("n=%5d %-32s grid=%3d units=%5d %8.1f us  %6.0f GB/s  %s\n", n, name, grid, c.units, us,
              2.0 * n * n / (us * 1e3), cudaGetErrorString(err));
  cudaFree(a);
  cudaFree(b);
}

int main() {
  void* fp = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &q);
  enc = reinterpret_cast<EncodeFn>(fp);
  for (int n : {16384, 32768}) {
    run(n, 0, 1, n / 128 < 148 ? n / 128 : 128, "V strip128 (<=128 CTAs)");
    run(n, 0, 1, n / 128 < 148 ? n / 128 : 128, "V strip128 synced/8", 8);
    run(n, 0, 1, n / 128 < 148 ? n / 128 : 128, "V strip128 synced/32", 32);
  }
  run(32768, 0, 1, 148, "V strip128 148 CTAs");
  run(32768, 0, 1, 148, "V strip128 148 CTAs synced/8", 8);
  return 0;
}
