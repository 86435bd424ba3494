// ubench_fp4.cu -- feasibility probe for 4-bit cells:
//   1. a TMA load of nibble-packed rows (CU_TENSOR_MAP_DATA_TYPE_16U4_ALIGN16B,
//      SWIZZLE_128B) lands in SMEM in the padded fp4 operand layout, and the
//      transaction byte count it reports;
//   2. tcgen05.mma.kind::f8f6f4 with A (e4m3 bytes) in TMEM and that SMEM box
//      as the e2m1 B operand computes D[x][y] = sum_k A[x][k] * X[y][k] in f32;
//   3. a TMA store of nibble-packed rows (16U4_ALIGN8B) from SMEM.
// Checked against the CPU; prints PASS / FAIL per item.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 -o build/ubench_fp4 tools/ubench_fp4.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "../paper_2406_17284_b200/csrc/ptx_sm100.cuh"

using namespace ltl::ptx;

constexpr int kRows = 160;   // box rows (N of the MMA)
constexpr int kCols = 128;   // elements per row (K = 4 chunks of 32)
constexpr int kM = 128;

// e4m3 encodings of the A values used: 0, 1, 2, 128
__host__ __device__ constexpr uint8_t e4m3(int v) {
  return v == 0 ? 0x00 : v == 1 ? 0x38 : v == 2 ? 0x40 : 0x70;
}
__host__ __device__ constexpr uint32_t idesc_f8f6f4(int m, int n) {
  return (1u << 4)        // D f32
         | (0u << 7)      // A e4m3
         | (5u << 10)     // B e2m1
         | (static_cast<uint32_t>(n >> 3) << 17) | (static_cast<uint32_t>(m >> 4) << 24);
}

__global__ void __launch_bounds__(128, 1)
    probe(const __grid_constant__ CUtensorMap load_map, const __grid_constant__ CUtensorMap store_map,
          const uint8_t* a_vals, float* d_out, uint8_t* smem_dump, uint32_t tx_bytes, int* status) {
  extern __shared__ uint8_t raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + kRows * 128 + 8192);
  uint32_t* tslot = reinterpret_cast<uint32_t*>(bar + 2);
  const int t = threadIdx.x, warp = t / 32;
  if (t == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    fence_barrier_init();
  }
  if (warp == 0) tmem_alloc(tslot, 256);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tslot;
  if (t == 0) {
    mbar_arrive_expect_tx(&bar[0], tx_bytes);
    tma_load_2d(smem, &load_map, &bar[0], 0, 0);
  }
  // A (M = 128 lanes, K = 128 e4m3 bytes = 32 columns) into TMEM columns 192..223
  {
    uint32_t w[8];
    for (int c = 0; c < 4; ++c) {
      for (int i = 0; i < 8; ++i) {
        uint32_t word = 0;
        for (int b = 0; b < 4; ++b) word |= static_cast<uint32_t>(a_vals[t * kCols + 32 * c + 4 * i + b]) << (8 * b);
        w[i] = word;
      }
      tmem_st_32x32b_x8(tmem + ((32u * warp) << 16) + 192 + 8 * c, w);
    }
    tmem_st_wait();
  }
  // bounded wait for the TMA (a wrong byte count must not hang the GPU)
  bool landed = false;
  for (long i = 0; i < 2000000 && !landed; ++i) landed = mbar_try_wait(smem_u32(&bar[0]), 0);
  if (t == 0) status[0] = landed ? 1 : 0;
  __syncthreads();
  if (!landed) {
    if (warp == 0) tmem_dealloc(tmem, 256);
    return;
  }
  for (int i = t; i < kRows * 128; i += 128) smem_dump[i] = smem[i];
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (t == 0) {
    const uint64_t bdesc = smem_desc_sw128_kmajor(smem_u32(smem));
    for (int q = 0; q < 4; ++q)
      asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                   "tcgen05.mma.cta_group::1.kind::f8f6f4 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tmem),
                   "r"(tmem + 192 + 8 * q), "l"(bdesc + ((32 * q) >> 4)), "r"(idesc_f8f6f4(kM, kRows)),
                   "r"(q)
                   : "memory");
    mma_commit(&bar[1]);
  }
  mbar_wait(&bar[1], 0);
  tc_fence_after();
  for (int c0 = 0; c0 < kRows; c0 += 32) {
    uint32_t v[32];
    tmem_ld_32x32b_x32(tmem + ((32u * warp) << 16) + c0, v);
    tmem_ld_wait();
    for (int i = 0; i < 32; ++i) d_out[t * kRows + c0 + i] = __uint_as_float(v[i]);
  }
  // 3. store probe: 64 rows of packed nibbles written by threads, TMA-stored
  uint8_t* st = smem + kRows * 128;  // 64 rows x 64 B
  for (int i = t; i < 64 * 64; i += 128) st[i] = static_cast<uint8_t>(i * 7 + 3);
  fence_proxy_async_smem();
  __syncthreads();
  if (t == 0) {
    tma_store_2d(&store_map, st, 0, 0);
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tmem, 256);
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
  // X: kRows x kCols cells in {0, 1}, stored as e2m1 nibbles (1.0 = 0x2), two per byte
  std::vector<uint8_t> cells(kRows * kCols), packed(kRows * kCols / 2, 0);
  srand(7);
  for (int i = 0; i < kRows * kCols; ++i) cells[i] = rand() % 3 == 0;
  for (int y = 0; y < kRows; ++y)
    for (int x = 0; x < kCols; ++x)
      packed[y * (kCols / 2) + x / 2] |= static_cast<uint8_t>((cells[y * kCols + x] ? 0x2 : 0x0) << (4 * (x & 1)));
  std::vector<int> aint(kM * kCols);
  std::vector<uint8_t> a8(kM * kCols);
  for (int i = 0; i < kM * kCols; ++i) {
    const int v = (rand() % 5 == 0) ? 128 : rand() % 3;  // 0, 1, 2, 128
    aint[i] = v;
    a8[i] = e4m3(v);
  }
  uint8_t *d_x, *d_a, *d_dump, *d_st;
  float* d_d;
  int* d_status;
  cudaMalloc(&d_x, packed.size());
  cudaMalloc(&d_a, a8.size());
  cudaMalloc(&d_d, kM * kRows * sizeof(float));
  cudaMalloc(&d_dump, kRows * 128);
  cudaMalloc(&d_st, 64 * 64);
  cudaMalloc(&d_status, 4 * sizeof(int));
  cudaMemcpy(d_x, packed.data(), packed.size(), cudaMemcpyHostToDevice);
  cudaMemcpy(d_a, a8.data(), a8.size(), cudaMemcpyHostToDevice);
  CUtensorMap lm, sm;
  {
    const cuuint64_t dims[2] = {kCols, kRows};
    const cuuint64_t strides[1] = {kCols / 2};
    const cuuint32_t box[2] = {kCols, kRows};
    const cuuint32_t es[2] = {1, 1};
    CUresult r = enc(&lm, CU_TENSOR_MAP_DATA_TYPE_16U4_ALIGN16B, 2, d_x, dims, strides, box, es,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                     CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("encode load map (16U4_ALIGN16B, SW128): %d\n", static_cast<int>(r));
    const cuuint64_t sd[2] = {128, 64};
    const cuuint64_t ss[1] = {64};
    const cuuint32_t sb[2] = {128, 64};
    r = enc(&sm, CU_TENSOR_MAP_DATA_TYPE_16U4_ALIGN8B, 2, d_st, sd, ss, sb, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("encode store map (16U4_ALIGN8B): %d\n", static_cast<int>(r));
  }
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  for (uint32_t tx : {static_cast<uint32_t>(kRows * kCols / 2), static_cast<uint32_t>(kRows * 128)}) {
    cudaMemset(d_status, 0, 4 * sizeof(int));
    cudaMemset(d_d, 0, kM * kRows * sizeof(float));
    probe<<<1, 128, 64 * 1024>>>(lm, sm, d_a, d_d, d_dump, tx, d_status);
    cudaError_t e = cudaDeviceSynchronize();
    int st = 0;
    cudaMemcpy(&st, d_status, sizeof st, cudaMemcpyDeviceToHost);
    printf("tx_bytes %u: launch %s, TMA landed %d\n", tx, cudaGetErrorString(e), st);
    if (e != cudaSuccess) return 1;
    if (!st) continue;
    std::vector<uint8_t> dump(kRows * 128);
    cudaMemcpy(dump.data(), d_dump, dump.size(), cudaMemcpyDeviceToHost);
    // expected padded layout: row y, 16-element group g -> 16-byte chunk (g ^ (y & 7)),
    // first 8 bytes = the packed nibbles, last 8 = gap
    int layout_ok = 1;
    for (int y = 0; y < kRows && layout_ok; ++y)
      for (int g = 0; g < 8; ++g)
        for (int b = 0; b < 8; ++b)
          if (dump[y * 128 + ((g ^ (y & 7)) << 4) + b] != packed[y * 64 + 8 * g + b]) layout_ok = 0;
    printf("  smem layout = packed 8 B + 8 B gap per 16 elements, SW128: %s\n", layout_ok ? "PASS" : "FAIL");
    if (!layout_ok) {
      printf("  row 0 bytes:");
      for (int i = 0; i < 32; ++i) printf(" %02x", dump[i]);
      printf("\n  packed row 0:");
      for (int i = 0; i < 16; ++i) printf(" %02x", packed[i]);
      printf("\n");
    }
    std::vector<float> d(kM * kRows);
    cudaMemcpy(d.data(), d_d, d.size() * sizeof(float), cudaMemcpyDeviceToHost);
    int bad = 0;
    for (int x = 0; x < kM; ++x)
      for (int y = 0; y < kRows; ++y) {
        long ref = 0;
        for (int k = 0; k < kCols; ++k) ref += static_cast<long>(aint[x * kCols + k]) * cells[y * kCols + k];
        if (d[x * kRows + y] != static_cast<float>(ref)) {
          if (bad < 4) printf("  D[%d][%d] = %g, expected %ld\n", x, y, d[x * kRows + y], ref);
          ++bad;
        }
      }
    printf("  kind::f8f6f4 e4m3(TMEM) x e2m1(SMEM) -> f32: %s (%d mismatches)\n", bad ? "FAIL" : "PASS", bad);
    std::vector<uint8_t> stv(64 * 64);
    cudaMemcpy(stv.data(), d_st, stv.size(), cudaMemcpyDeviceToHost);
    int st_ok = 1;
    for (int i = 0; i < 64 * 64; ++i) st_ok &= stv[i] == static_cast<uint8_t>(i * 7 + 3);
    printf("  TMA store 16U4_ALIGN8B (packed smem -> packed global): %s\n", st_ok ? "PASS" : "FAIL");
  }
  return 0;
}
