// ubench_mma.cu -- tcgen05.mma kind::i8 issue/execute rate on B200 for the
// shapes the LTL step uses: SS (A and B from SMEM descriptors) vs TS (A from
// TMEM), N = 32 / 64 / 128, one accumulator vs rotating accumulators.
// One CTA per SM, one elected thread issues `reps` MMAs back to back, commits,
// waits; reports cycles per MMA (median over CTAs).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o build/ubench_mma tools/ubench_mma.cu
#include <cstdint>
#include <cstdio>
#include <vector>
#include <algorithm>
#include <string>

#include "../paper_2406_17284_b200/csrc/ptx_sm100.cuh"

using namespace ltl::ptx;

template <int KIND>
__device__ __forceinline__ void mma_any_ss(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  if (KIND == 0) mma_i8_ss(d, a, b, idesc, acc);
  else if (KIND == 1)
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                 "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d), "l"(a), "l"(b), "r"(idesc), "r"(acc) : "memory");
  else if (KIND == 2)
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                 "tcgen05.mma.cta_group::1.kind::f8f6f4 [%0], %1, %2, %3, p;\n\t}" ::"r"(d), "l"(a), "l"(b), "r"(idesc), "r"(acc) : "memory");
  else
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                 "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(d), "l"(a), "l"(b), "r"(idesc), "r"(acc) : "memory");
}
template <int KIND>
__device__ __forceinline__ void mma_any_ts(uint32_t d, uint32_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  if (KIND == 0) mma_i8_ts(d, a, b, idesc, acc);
  else if (KIND == 1)
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                 "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d), "r"(a), "l"(b), "r"(idesc), "r"(acc) : "memory");
  else if (KIND == 2)
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                 "tcgen05.mma.cta_group::1.kind::f8f6f4 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d), "r"(a), "l"(b), "r"(idesc), "r"(acc) : "memory");
  else
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                 "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d), "r"(a), "l"(b), "r"(idesc), "r"(acc) : "memory");
}

__host__ __device__ constexpr uint32_t idesc_kind(int kind, int m, int n) {
  // c_format [4,6): F32 = 1, S32 = 2; a/b format [7,10)/[10,13): i8 U8 = 0,
  // f16 F16 = 0, f8f6f4 E4M3 = 0, tf32 TF32 = 2
  return ((kind == 0 ? 2u : 1u) << 4) | ((kind == 3 ? 2u : 0u) << 7) | ((kind == 3 ? 2u : 0u) << 10) |
         (static_cast<uint32_t>(n >> 3) << 17) | (static_cast<uint32_t>(m >> 4) << 24);
}

struct Cfg {
  int ts;     // A from TMEM
  int n;      // N
  int accs;   // rotating accumulators
  int reps;
};

template <int KIND>
__global__ void __launch_bounds__(128, 1) kern(Cfg c, long long* out) {
  extern __shared__ uint8_t raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint32_t slot;
  __shared__ uint64_t bar;
  const int warp = threadIdx.x / 32;
  for (int i = threadIdx.x; i < 65536 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0x01010101u;
  fence_proxy_async_smem();
  if (warp == 0) tmem_alloc(&slot, 512);
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_barrier_init();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  if (warp == 1 && elect_one()) {
    const uint64_t adesc = smem_desc_sw32_kmajor(smem_u32(smem));
    const uint64_t bdesc = smem_desc_sw128_kmajor(smem_u32(smem + 32768));
    const uint32_t idesc = idesc_kind(KIND, 128, c.n);
    // warm
    mma_any_ss<KIND>(tmem, adesc, bdesc, idesc, 0);
    mma_commit(&bar);
    mbar_wait(&bar, 0);
    const long long t0 = clock64();
    for (int i = 0; i < c.reps; ++i) {
      const uint32_t d = tmem + 256 + (i % c.accs) * c.n;  // accumulators from column 256
      if (c.ts)
        mma_any_ts<KIND>(d, tmem + 8 * (i % 8), bdesc + ((32 * (i % 4)) >> 4), idesc, i >= c.accs);
      else
        mma_any_ss<KIND>(d, adesc + ((4096 * (i % 4)) >> 4), bdesc + ((32 * (i % 4)) >> 4), idesc,
                  i >= c.accs);
    }
    mma_commit(&bar);
    mbar_wait(&bar, 1);
    const long long t1 = clock64();
    out[blockIdx.x] = t1 - t0;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tmem, 512);
}

__global__ void __launch_bounds__(128, 1) kern_unit(int units, long long* out) {
  extern __shared__ uint8_t raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint32_t slot;
  __shared__ uint64_t bar;
  const int warp = threadIdx.x / 32;
  for (int i = threadIdx.x; i < 65536 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0x01010101u;
  fence_proxy_async_smem();
  if (warp == 0) tmem_alloc(&slot, 512);
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_barrier_init();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  if (warp == 1 && elect_one()) {
    const uint64_t adesc = smem_desc_sw32_kmajor(smem_u32(smem));
    const uint64_t bdesc = smem_desc_sw128_kmajor(smem_u32(smem + 32768));
    const long long t0 = clock64();
    for (int u = 0; u < units; ++u) {
      for (int q = 0; q < 6; ++q)
        mma_i8_ss(tmem, adesc + ((4096 * (q % 4)) >> 4), bdesc + ((32 * (q % 4)) >> 4),
                  idesc_i8_u8u8_s32(128, 160), q > 0);
      for (int k = 0; k < 10; ++k)
        mma_i8_ts(tmem + 320 + 64 * (k / 5), tmem + 160 + 8 * (k % 5), bdesc + ((32 * (k % 4)) >> 4),
                  idesc_i8_u8u8_s32(128, 64), (k % 5) > 0);
    }
    mma_commit(&bar);
    mbar_wait(&bar, 0);
    out[blockIdx.x] = clock64() - t0;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tmem, 512);
}

template <int KIND>
void run_kind(const char* kname, int sms, long long* d) {
  const size_t smem = 96 * 1024;
  cudaFuncSetAttribute(kern<KIND>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  for (int ts : {0, 1})
    for (int n : {32, 64, 96, 128, 160, 192, 256}) {
      Cfg c{ts, n, 1, 512};
      kern<KIND><<<sms, 128, smem>>>(c, d);
      cudaError_t e = cudaDeviceSynchronize();
      std::vector<long long> h(sms);
      cudaMemcpy(h.data(), d, sms * sizeof(long long), cudaMemcpyDeviceToHost);
      std::sort(h.begin(), h.end());
      const double cyc = static_cast<double>(h[sms / 2]) / c.reps;
      const int kbytes = 32;
      const double macs = 128.0 * n * (KIND == 1 ? kbytes / 2 : KIND == 3 ? kbytes / 4 : kbytes);
      std::printf("%-7s %s N=%3d  %7.1f cyc/MMA  %7.0f MAC/cyc/SM  %s\n", kname, ts ? "TS" : "SS", n,
                  cyc, macs / cyc, cudaGetErrorString(e));
    }
}

// Dense kind::i8 peak of the whole GPU: every SM issues `reps` M128 N256 K32
// MMAs (SS and TS) back to back into two rotating accumulators; ops =
// 2*M*N*K per MMA, wall time from CUDA events around the launch.
void peak_i8(int sms, long long* d, const char* json_path) {
  const size_t smem = 96 * 1024;
  cudaFuncSetAttribute(kern<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  double best[2] = {0, 0};
  int clk_khz = 0;
  cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
  for (int ts : {0, 1}) {
    for (int it = 0; it < 5; ++it) {
      Cfg c{ts, 256, 1, 1 << 15};
      cudaEventRecord(e0);
      kern<0><<<sms, 128, smem>>>(c, d);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms = 0;
      cudaEventElapsedTime(&ms, e0, e1);
      const double ops = 2.0 * 128 * 256 * 32 * c.reps * sms;
      best[ts] = std::max(best[ts], ops / (ms * 1e-3) / 1e12);
    }
  }
  std::printf("i8 dense peak (M128 N256 K32, %d SMs, best of 5): SS %.1f TOPS, TS %.1f TOPS\n", sms,
              best[0], best[1]);
  if (json_path) {
    if (FILE* fh = std::fopen(json_path, "w")) {
      std::fprintf(fh,
                   "{\"i8_peak_tops\": %.1f, \"i8_peak_tops_ss\": %.1f, \"i8_peak_tops_ts\": %.1f, "
                   "\"sms\": %d, \"sm_clock_khz_attr\": %d, \"how\": \"tools/ubench_mma.cu --peak: "
                   "%d MMAs of M128 N256 K32 kind::i8 per SM back to back, 2*M*N*K ops each, CUDA "
                   "events around the launch, best of 5\"}\n",
                   std::max(best[0], best[1]), best[0], best[1], sms, clk_khz, 1 << 15);
      std::fclose(fh);
    }
  }
}

int main(int argc, char** argv) {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  long long* d;
  cudaMalloc(&d, sms * sizeof(long long));
  if (argc > 1 && std::string(argv[1]) == "--peak") {
    peak_i8(sms, d, argc > 2 ? argv[2] : nullptr);
    return 0;
  }
  run_kind<0>("i8", sms, d);
  {
    const size_t smem = 96 * 1024;
    cudaFuncSetAttribute(kern_unit, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    const int units = 200;
    kern_unit<<<sms, 128, smem>>>(units, d);
    cudaError_t e = cudaDeviceSynchronize();
    std::vector<long long> h(sms);
    cudaMemcpy(h.data(), d, sms * sizeof(long long), cudaMemcpyDeviceToHost);
    std::sort(h.begin(), h.end());
    std::printf("LTL unit (6 x SS N160 + 10 x TS N64): %.1f cyc/unit  %s\n",
                static_cast<double>(h[sms / 2]) / units, cudaGetErrorString(e));
  }
  return 0;
}
