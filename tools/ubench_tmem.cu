// ubench_tmem.cu -- microbenchmark: TMEM load/store throughput per SM on B200.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o build/ubench_tmem tools/ubench_tmem.cu
// Each CTA (1 per SM) allocates 256 TMEM columns; W warps (W%4 = lane quarter)
// repeatedly load / store 32 columns and wait; reports bytes per SM-cycle.
#include <cstdio>
#include <cstdint>
#include "../paper_2406_17284_b200/csrc/ptx_sm100.cuh"

using namespace ltl::ptx;

template <int MODE>
__global__ void bench(int iters, long long* cycles, uint32_t* sink) {
  __shared__ uint32_t slot;
  const uint32_t warp = threadIdx.x / 32;
  if (warp == 0) tmem_alloc(&slot, 256);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  const uint32_t q = warp & 3;
  const uint32_t base = tmem + ((q * 32) << 16) + 32 * ((warp / 4) % 4);
  uint32_t acc = 0;
  __syncthreads();
  const long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    if (MODE == 0) {  // 32x32b.x32 load (4 KB per warp)
      uint32_t v[32];
      tmem_ld_32x32b_x32(base, v);
      tmem_ld_wait();
#pragma unroll
      for (int j = 0; j < 32; ++j) acc += v[j];
    } else if (MODE == 1) {  // 32x32b.x16.pack16 (reads 32 columns)
      uint32_t v[16];
      tmem_ld_32x32b_x16_pack16(base, v);
      tmem_ld_wait();
#pragma unroll
      for (int j = 0; j < 16; ++j) acc += v[j];
    } else if (MODE == 2) {  // 16x256b.x2.pack16 on both lane halves (32 columns)
      uint32_t v[8], w[8];
      tmem_ld_16x256b_x2_pack16(base, v);
      tmem_ld_16x256b_x2_pack16(base + (16u << 16), w);
      tmem_ld_wait();
#pragma unroll
      for (int j = 0; j < 8; ++j) acc += v[j] + w[j];
    } else {  // 32x32b.x8 store (1 KB per warp)
      uint32_t v[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) v[j] = acc + j + i;
      tmem_st_32x32b_x8(base, v);
      tmem_st_wait();
    }
  }
  __syncthreads();
  const long long t1 = clock64();
  if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
  if (acc == 0x12345678) sink[0] = acc;
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tmem, 256);
}

template <int MODE>
void run(const char* name, int warps, double bytes_per_warp_iter) {
  const int iters = 4096, sms = 148;
  long long* d;
  uint32_t* sink;
  cudaMalloc(&d, sms * sizeof(long long));
  cudaMalloc(&sink, 4);
  bench<MODE><<<sms, 32 * warps>>>(iters, d, sink);
  cudaError_t e = cudaDeviceSynchronize();
  long long h[148];
  cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
  double avg = 0;
  for (int i = 0; i < sms; ++i) avg += h[i];
  avg /= sms;
  std::printf("%-28s warps=%2d  %8.1f cycles/iter  %7.1f B/cycle/SM  (%s)\n", name, warps,
              avg / iters, bytes_per_warp_iter * warps * iters / avg, cudaGetErrorString(e));
  cudaFree(d);
  cudaFree(sink);
}

int main() {
  for (int w : {4, 8, 16}) {
    run<0>("ld 32x32b.x32", w, 4096);
    run<1>("ld 32x32b.x16.pack16", w, 4096);
    run<2>("ld 16x256b.x2.pack16 x2", w, 4096);
    run<3>("st 32x32b.x8", w, 1024);
  }
  return 0;
}
