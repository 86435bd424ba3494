// host_pack_bench.cpp -- can the host bit-pack a u8 cell grid faster than PCIe
// moves it?  Times, on the GPU box: pinned H2D / D2H of 1 GiB, and packing
// 1 GiB of {0,1} bytes into 128 MiB of bits (AVX2 movemask) / unpacking it,
// with 1..64 threads.
// Build: g++ -O3 -mavx2 -std=c++17 -pthread tools/host_pack_bench.cpp -I/usr/local/cuda/include \
//          -L/usr/local/cuda/lib64 -lcudart -o build/host_pack_bench
#include <cuda_runtime.h>
#include <immintrin.h>

#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <thread>
#include <vector>

static double now() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

static void pack_range(const uint8_t* in, uint8_t* out, size_t n32_0, size_t n32_1) {
  for (size_t i = n32_0; i < n32_1; ++i) {
    __m256i v = _mm256_loadu_si256(reinterpret_cast<const __m256i*>(in + 32 * i));
    v = _mm256_slli_epi16(v, 7);
    const uint32_t m = static_cast<uint32_t>(_mm256_movemask_epi8(v));
    std::memcpy(out + 4 * i, &m, 4);
  }
}

static void unpack_range(const uint8_t* in, uint8_t* out, size_t n32_0, size_t n32_1) {
  const __m256i shuf = _mm256_setr_epi8(0, 0, 0, 0, 0, 0, 0, 0, 1, 1, 1, 1, 1, 1, 1, 1, 2, 2, 2, 2, 2, 2,
                                        2, 2, 3, 3, 3, 3, 3, 3, 3, 3);
  const __m256i bits = _mm256_set1_epi64x(static_cast<long long>(0x8040201008040201ULL));
  const __m256i one = _mm256_set1_epi8(1);
  for (size_t i = n32_0; i < n32_1; ++i) {
    uint32_t m;
    std::memcpy(&m, in + 4 * i, 4);
    __m256i v = _mm256_shuffle_epi8(_mm256_set1_epi32(static_cast<int>(m)), shuf);
    v = _mm256_min_epu8(_mm256_and_si256(v, bits), one);
    _mm256_storeu_si256(reinterpret_cast<__m256i*>(out + 32 * i), v);
  }
}

template <class F>
static double par(int t, size_t n32, F f) {
  const double t0 = now();
  std::vector<std::thread> th;
  for (int k = 0; k < t; ++k) th.emplace_back([&, k] { f(n32 * k / t, n32 * (k + 1) / t); });
  for (auto& x : th) x.join();
  return now() - t0;
}

int main() {
  const size_t n = size_t(1) << 30;
  uint8_t *h, *hp, *d;
  cudaMallocHost(&h, n);
  cudaMallocHost(&hp, n / 8);
  cudaMalloc(&d, n);
  for (size_t i = 0; i < n; ++i) h[i] = (i * 2654435761u >> 13) & 1;
  std::vector<uint8_t> pageable(n);
  std::memcpy(pageable.data(), h, n);
  printf("hardware_concurrency %u\n", std::thread::hardware_concurrency());
  for (int rep = 0; rep < 2; ++rep) {
    double t0 = now();
    cudaMemcpy(d, h, n, cudaMemcpyHostToDevice);
    double t1 = now();
    cudaMemcpy(h, d, n, cudaMemcpyDeviceToHost);
    double t2 = now();
    cudaMemcpy(d, hp, n / 8, cudaMemcpyHostToDevice);
    double t3 = now();
    printf("pinned H2D 1 GiB %.2f ms (%.1f GB/s), D2H %.2f ms, H2D 128 MiB %.2f ms\n", (t1 - t0) * 1e3,
           n / (t1 - t0) / 1e9, (t2 - t1) * 1e3, (t3 - t2) * 1e3);
  }
  const size_t n32 = n / 32;
  for (int t : {1, 4, 8, 16, 32, 64}) {
    if (t > 2 * static_cast<int>(std::thread::hardware_concurrency())) break;
    double best_p = 1e9, best_u = 1e9, best_pp = 1e9;
    for (int rep = 0; rep < 3; ++rep) {
      best_p = std::min(best_p, par(t, n32, [&](size_t a, size_t b) { pack_range(h, hp, a, b); }));
      best_pp = std::min(best_pp, par(t, n32, [&](size_t a, size_t b) { pack_range(pageable.data(), hp, a, b); }));
      best_u = std::min(best_u, par(t, n32, [&](size_t a, size_t b) { unpack_range(hp, h, a, b); }));
    }
    printf("threads %2d: pack %.2f ms (%.0f GB/s of cells), pack pageable %.2f ms, unpack %.2f ms (%.0f GB/s)\n", t,
           best_p * 1e3, n / best_p / 1e9, best_pp * 1e3, best_u * 1e3, n / best_u / 1e9);
  }
  // check
  std::vector<uint8_t> chk(n / 8);
  pack_range(pageable.data(), chk.data(), 0, n32);
  unpack_range(chk.data(), h, 0, n32);
  printf("roundtrip %s\n", std::memcmp(h, pageable.data(), n) == 0 ? "ok" : "BAD");
  return 0;
}
