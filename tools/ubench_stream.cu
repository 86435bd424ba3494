// ubench_stream.cu -- what HBM bandwidth does the LTL kernel's access pattern
// allow?  Persistent CTAs stream 128-column strips of a padded 16384^2 u8 grid
// down in 64-row chunks exactly like ltl_tc.cu (TMA boxes of `box_w` bytes x
// 64 rows covering 160 input columns, a `stages`-deep ring), and TMA-store the
// 128 interior columns of every chunk to a second grid.  No compute.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o build/ubench_stream tools/ubench_stream.cu
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

#include "../paper_2406_17284_b200/csrc/ptx_sm100.cuh"

using namespace ltl::ptx;

constexpr int kStages = 8;
constexpr int kRows = 64;

struct Cfg {
  int strips, chunks, segs, box_w, nbox, wide;  // wide: strips (128 cols) per unit
};

__global__ void __launch_bounds__(128, 1) stream_kernel(const __grid_constant__ CUtensorMap lmap,
                                                        const __grid_constant__ CUtensorMap smap,
                                                        Cfg c) {
  extern __shared__ uint8_t raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  const uint32_t stage_bytes = 288 * kRows;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + kStages * stage_bytes);
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
  const int units = c.strips * c.segs;
  if (warp == 0 && lane == 0) {
    uint32_t g = 0;
    for (int u = blockIdx.x; u < units; u += gridDim.x) {
      const int strip = u % c.strips, seg = u / c.strips;
      const int c0 = c.chunks * seg / c.segs, c1 = c.chunks * (seg + 1) / c.segs;
      for (int k = c0; k <= c1; ++k, ++g) {
        const uint32_t s = g % kStages;
        mbar_wait(&empty[s], ((g / kStages) & 1) ^ 1);
        mbar_arrive_expect_tx(&full[s], c.nbox * c.box_w * kRows);
        for (int b = 0; b < c.nbox; ++b)
          tma_load_2d(smem + s * stage_bytes + b * c.box_w * kRows, &lmap, &full[s],
                      strip * 128 * c.wide + b * c.box_w, k * kRows);
      }
    }
  } else if (warp == 1 && lane == 0) {
    uint32_t g = 0;
    for (int u = blockIdx.x; u < units; u += gridDim.x) {
      const int strip = u % c.strips, seg = u / c.strips;
      const int c0 = c.chunks * seg / c.segs, c1 = c.chunks * (seg + 1) / c.segs;
      for (int k = c0; k <= c1; ++k, ++g) {
        const uint32_t s = g % kStages;
        mbar_wait(&full[s], (g / kStages) & 1);
        if (k < c1) {
          for (int b = 0; b < 4 * c.wide; ++b)
            tma_store_2d(&smap, smem + s * stage_bytes + b * 32 * kRows,
                         strip * 128 * c.wide + 32 * b, k * kRows);
          tma_store_commit();
          tma_store_wait_read<0>();
        }
        mbar_arrive(&empty[s]);
      }
    }
    tma_store_wait_all<0>();
  }
}

using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*,
                              CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion,
                              CUtensorMapFloatOOBfill);

int run(int n);
int main() {
  run(16384);
  run(32768);
  return 0;
}
int run(int n) {
  const int pad = n + 32, pitch = (pad + 127) / 128 * 128;
  uint8_t *a, *b;
  cudaMalloc(&a, (size_t)pad * pitch);
  cudaMalloc(&b, (size_t)pad * pitch);
  cudaMemset(a, 1, (size_t)pad * pitch);
  void* fp = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &q);
  EncodeFn enc = reinterpret_cast<EncodeFn>(fp);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const size_t smem = kStages * 288 * kRows + 2 * kStages * 8 + 1024;
  cudaFuncSetAttribute(stream_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  struct V { int box_w; CUtensorMapSwizzle swz; CUtensorMapL2promotion promo; int wide; const char* name; };
  V vars[] = {
      {32, CU_TENSOR_MAP_SWIZZLE_32B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, 1, "box32 x5, 1 strip/unit"},
      {32, CU_TENSOR_MAP_SWIZZLE_32B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, 2, "box32 x9, 2 strips/unit"},
      {32, CU_TENSOR_MAP_SWIZZLE_32B, CU_TENSOR_MAP_L2_PROMOTION_NONE, 1, "box32 x5 nopromo"},
      {96, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, 2, "box96 x3, 2 strips/unit"},
  };
  for (const V& v : vars) {
    CUtensorMap lmap, smap;
    cuuint64_t dims[2] = {(cuuint64_t)pad, (cuuint64_t)pad}, str[1] = {(cuuint64_t)pitch};
    cuuint32_t box[2] = {(cuuint32_t)v.box_w, 64}, es[2] = {1, 1};
    enc(&lmap, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, a, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        v.swz, v.promo, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    cuuint64_t sd[2] = {(cuuint64_t)n, (cuuint64_t)n};
    cuuint32_t sbox[2] = {32, 64};
    enc(&smap, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, b + 16 * pitch + 16, sd, str, sbox, es,
        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_32B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    const int strips = n / 128 / v.wide;
    int segs = 1;
    while ((strips * segs) % sms != 0 && segs < 200) ++segs;
    if (segs >= 200) segs = 1;
    const int grid = strips * segs < sms ? strips * segs : sms;
    Cfg c{strips, n / 64, segs, v.box_w, (128 * v.wide + 32) / v.box_w, v.wide};
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int w = 0; w < 3; ++w) stream_kernel<<<grid, 128, smem>>>(lmap, smap, c);
    cudaEventRecord(e0);
    const int it = 20;
    for (int w = 0; w < it; ++w) stream_kernel<<<grid, 128, smem>>>(lmap, smap, c);
    cudaEventRecord(e1);
    cudaError_t err = cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double us = ms * 1000 / it;
    std::printf("n=%d %-34s segs=%d grid=%d %8.1f us/pass  %7.0f GB/s (2 B/cell)  %s\n", n, v.name, segs, grid, us,
                2.0 * n * n / (us * 1e3), cudaGetErrorString(err));
  }
  cudaFree(a);
  cudaFree(b);
  return 0;
}
