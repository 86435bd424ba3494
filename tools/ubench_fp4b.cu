// ubench_fp4b.cu -- second 4-bit-cell probe: the pieces the
// packed-cell step needs beyond tools/ubench_fp4.cu.
//   1. kind::f8f6f4, A e4m3 in TMEM x B e2m1 (nibble 1 = 0.5) from a
//      16U4_ALIGN16B SW128 TMA box, with D = f16: where the f16 results sit in
//      TMEM (one per 32-bit column, low half?) and what .pack::16b loads give;
//   2. back-to-back issue cost (cycles per MMA, M128 K32 TS) at N = 64 / 160
//      of kind::i8 (s32) vs kind::f8f6f4 e4m3 x e2m1 (f16 D and f32 D).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 -o build/ubench_fp4b tools/ubench_fp4b.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cuda_fp16.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "../paper_2406_17284_b200/csrc/ptx_sm100.cuh"

using namespace ltl::ptx;

constexpr int kRows = 160;
constexpr int kCols = 128;
constexpr int kM = 128;

__host__ __device__ constexpr uint8_t e4m3(int v) {  // 0, 2, 4, 6
  return v == 0 ? 0x00 : v == 2 ? 0x40 : v == 4 ? 0x48 : 0x4C;
}
__host__ __device__ constexpr uint32_t idesc_fp4(int m, int n, bool f32) {
  return ((f32 ? 1u : 0u) << 4) | (0u << 7) | (5u << 10) | (static_cast<uint32_t>(n >> 3) << 17) |
         (static_cast<uint32_t>(m >> 4) << 24);
}
__device__ __forceinline__ void mma_fp4_ts(uint32_t d, uint32_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
               "tcgen05.mma.cta_group::1.kind::f8f6f4 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d), "r"(a), "l"(b),
               "r"(idesc), "r"(acc)
               : "memory");
}

__global__ void __launch_bounds__(128, 1)
    probe(const __grid_constant__ CUtensorMap load_map, const uint8_t* a_vals, uint32_t* raw_out,
          uint32_t* pk_out, long long* cyc, int* status) {
  extern __shared__ uint8_t rawsm[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(rawsm) + 1023) & ~uintptr_t(1023));
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + kRows * 128);
  uint32_t* tslot = reinterpret_cast<uint32_t*>(bar + 4);
  const int t = threadIdx.x, warp = t / 32;
  if (t == 0) {
    for (int i = 0; i < 4; ++i) mbar_init(&bar[i], 1);
    fence_barrier_init();
  }
  if (warp == 0) tmem_alloc(tslot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tslot;
  if (t == 0) {
    mbar_arrive_expect_tx(&bar[0], kRows * kCols / 2);
    tma_load_2d(smem, &load_map, &bar[0], 0, 0);
  }
  {  // A: 128 lanes x 128 e4m3 bytes = 32 columns at 448..479
    uint32_t w[8];
    for (int c = 0; c < 4; ++c) {
      for (int i = 0; i < 8; ++i) {
        uint32_t word = 0;
        for (int b = 0; b < 4; ++b) word |= static_cast<uint32_t>(a_vals[t * kCols + 32 * c + 4 * i + b]) << (8 * b);
        w[i] = word;
      }
      tmem_st_32x32b_x8(tmem + ((32u * warp) << 16) + 448 + 8 * c, w);
    }
    tmem_st_wait();
  }
  bool landed = false;
  for (long i = 0; i < 2000000 && !landed; ++i) landed = mbar_try_wait(smem_u32(&bar[0]), 0);
  if (t == 0) status[0] = landed ? 1 : 0;
  __syncthreads();
  if (!landed) {
    if (warp == 0) tmem_dealloc(tmem, 512);
    return;
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint64_t bdesc = smem_desc_sw128_kmajor(smem_u32(smem));
  // 1. f16 D at column 0
  if (t == 0) {
    for (int q = 0; q < 4; ++q) mma_fp4_ts(tmem, tmem + 448 + 8 * q, bdesc + ((32 * q) >> 4), idesc_fp4(kM, kRows, false), q);
    mma_commit(&bar[1]);
  }
  mbar_wait(&bar[1], 0);
  tc_fence_after();
  for (int c0 = 0; c0 < kRows; c0 += 32) {
    uint32_t v[32];
    tmem_ld_32x32b_x32(tmem + ((32u * warp) << 16) + c0, v);
    tmem_ld_wait();
    for (int i = 0; i < 32; ++i) raw_out[t * kRows + c0 + i] = v[i];
  }
  {
    uint32_t v[32];
    tmem_ld_32x32b_x32_pack16(tmem + ((32u * warp) << 16), v);
    tmem_ld_wait();
    for (int i = 0; i < 32; ++i) pk_out[t * 32 + i] = v[i];
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  // 2. issue cost: 64 MMAs back to back per configuration
  if (t == 0) {
    int k = 0;
    for (int n : {64, 160}) {
      for (int kind = 0; kind < 3; ++kind) {
        const uint32_t idesc = kind == 0 ? idesc_i8_u8u8_s32(kM, n) : idesc_fp4(kM, n, kind == 2);
        const long long c0 = clock64();
        for (int i = 0; i < 64; ++i) {
          const uint32_t d = tmem + (i & 1) * 160;
          if (kind == 0) mma_i8_ts(d, tmem + 448 + 8 * (i & 3), bdesc, idesc, i > 1);
          else mma_fp4_ts(d, tmem + 448 + 8 * (i & 3), bdesc, idesc, i > 1);
        }
        mma_commit(&bar[2]);
        mbar_wait(&bar[2], k & 1);
        cyc[k++] = clock64() - c0;
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tmem, 512);
}

using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*,
                              CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion,
                              CUtensorMapFloatOOBfill);

int main() {
  void* fp = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &q);
  EncodeFn enc = reinterpret_cast<EncodeFn>(fp);
  std::vector<uint8_t> cells(kRows * kCols), packed(kRows * kCols / 2, 0);
  srand(11);
  for (int i = 0; i < kRows * kCols; ++i) cells[i] = rand() % 3 == 0;
  for (int y = 0; y < kRows; ++y)
    for (int x = 0; x < kCols; ++x)
      packed[y * (kCols / 2) + x / 2] |= static_cast<uint8_t>(cells[y * kCols + x] << (4 * (x & 1)));
  std::vector<int> aint(kM * kCols);
  std::vector<uint8_t> a8(kM * kCols);
  for (int i = 0; i < kM * kCols; ++i) {
    const int v = 2 * (rand() % 4);  // 0, 2, 4, 6
    aint[i] = v;
    a8[i] = e4m3(v);
  }
  uint8_t *d_x, *d_a;
  uint32_t *d_raw, *d_pk;
  long long* d_cyc;
  int* d_status;
  cudaMalloc(&d_x, packed.size());
  cudaMalloc(&d_a, a8.size());
  cudaMalloc(&d_raw, kM * kRows * 4);
  cudaMalloc(&d_pk, kM * 32 * 4);
  cudaMalloc(&d_cyc, 16 * 8);
  cudaMalloc(&d_status, 16);
  cudaMemcpy(d_x, packed.data(), packed.size(), cudaMemcpyHostToDevice);
  cudaMemcpy(d_a, a8.data(), a8.size(), cudaMemcpyHostToDevice);
  CUtensorMap lm;
  const cuuint64_t dims[2] = {kCols, kRows};
  const cuuint64_t strides[1] = {kCols / 2};
  const cuuint32_t box[2] = {kCols, kRows};
  const cuuint32_t es[2] = {1, 1};
  CUresult r = enc(&lm, CU_TENSOR_MAP_DATA_TYPE_16U4_ALIGN16B, 2, d_x, dims, strides, box, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("encode: %d\n", static_cast<int>(r));
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  probe<<<1, 128, 64 * 1024>>>(lm, d_a, d_raw, d_pk, d_cyc, d_status);
  cudaError_t e = cudaDeviceSynchronize();
  int st = 0;
  cudaMemcpy(&st, d_status, 4, cudaMemcpyDeviceToHost);
  printf("launch %s, landed %d\n", cudaGetErrorString(e), st);
  if (e != cudaSuccess || !st) return 1;
  std::vector<uint32_t> raw(kM * kRows), pk(kM * 32);
  cudaMemcpy(raw.data(), d_raw, raw.size() * 4, cudaMemcpyDeviceToHost);
  cudaMemcpy(pk.data(), d_pk, pk.size() * 4, cudaMemcpyDeviceToHost);
  auto ref = [&](int x, int y) {
    int s = 0;
    for (int k = 0; k < kCols; ++k) s += aint[x * kCols + k] * cells[y * kCols + k];
    return s / 2.0;  // cells are 0.5
  };
  printf("lane 0 raw cols 0..5:");
  for (int i = 0; i < 6; ++i) printf(" %08x", raw[i]);
  printf("\nexpected D[0][0..5]:");
  for (int i = 0; i < 6; ++i) printf(" %g", ref(0, i));
  printf("\n");
  // hypothesis A: column y holds f16 of D[x][y] in its low 16 bits
  int badA = 0, badB = 0, badP = 0;
  for (int x = 0; x < kM; ++x)
    for (int y = 0; y < kRows; ++y) {
      __half_raw h;
      h.x = static_cast<uint16_t>(raw[x * kRows + y] & 0xFFFF);
      if (__half2float(__half(h)) != ref(x, y)) ++badA;
    }
  // hypothesis B: column c holds D[x][2c] (low) and D[x][2c+1] (high)
  for (int x = 0; x < kM; ++x)
    for (int y = 0; y < kRows; ++y) {
      __half_raw h;
      h.x = static_cast<uint16_t>((raw[x * kRows + y / 2] >> (16 * (y & 1))) & 0xFFFF);
      if (__half2float(__half(h)) != ref(x, y)) ++badB;
    }
  // pack16 load of columns 0..63: register i = rows 2i (low), 2i+1 (high) under A
  for (int x = 0; x < kM; ++x)
    for (int i = 0; i < 32; ++i)
      for (int hh = 0; hh < 2; ++hh) {
        __half_raw h;
        h.x = static_cast<uint16_t>((pk[x * 32 + i] >> (16 * hh)) & 0xFFFF);
        if (__half2float(__half(h)) != ref(x, 2 * i + hh)) ++badP;
      }
  printf("f16 D one per column (low half): %s (%d bad)\n", badA ? "FAIL" : "PASS", badA);
  printf("f16 D two per column:            %s (%d bad)\n", badB ? "FAIL" : "PASS", badB);
  printf("pack16 load -> f16x2 rows (2i, 2i+1): %s (%d bad)\n", badP ? "FAIL" : "PASS", badP);
  std::vector<long long> cyc(6);
  cudaMemcpy(cyc.data(), d_cyc, 6 * 8, cudaMemcpyDeviceToHost);
  const char* kn[3] = {"i8 s32", "f8f6f4 e4m3xe2m1 f16", "f8f6f4 e4m3xe2m1 f32"};
  for (int k = 0; k < 6; ++k)
    printf("N=%3d %-22s %.1f cycles/MMA\n", k < 3 ? 64 : 160, kn[k % 3], cyc[k] / 64.0);
  return 0;
}
