// xfer_bits.cpp -- host side of the bit-packed host <-> device transfers.
//
// A grid crosses PCIe as one bit per cell instead of the reference's byte per
// cell (Grid::cells, include/catsim/grid.hpp:60): the host packs rows of {0, 1}
// bytes into bits on all its cores while the previous chunk is in flight, the
// device expands them (ltl_layout.cu); downloads mirror that.  On the B200
// box's 16 host cores packing runs at ~130 GB/s of cells and unpacking at
// ~80 GB/s against PCIe's 55 GB/s (tools/host_pack_bench.cpp), so a 1 GiB grid
// moves in ~9 / ~14 ms instead of 19.4 ms each way.  AVX-512BW when the CPU
// has it, else AVX2 (function-level target attributes + a runtime check: the
// library itself is built without -m flags); without either the callers keep
// the byte-per-cell copies.
#include <immintrin.h>

#include <algorithm>
#include <atomic>
#include <condition_variable>
#include <cstdint>
#include <cstring>
#include <functional>
#include <mutex>
#include <thread>
#include <vector>

#include "internal.hpp"

namespace ltl_host {
namespace {

// one row: row_bytes % 32 == 0; returns the OR of (byte & 0xFE) (0: all cells valid)
__attribute__((target("avx512f,avx512bw"))) uint32_t pack_row_512(const uint8_t* src, uint8_t* dst,
                                                                  size_t row_bytes) {
  const __m512i one = _mm512_set1_epi8(1);
  __m512i bad = _mm512_setzero_si512();
  size_t i = 0;
  for (; i + 64 <= row_bytes; i += 64) {
    const __m512i v = _mm512_loadu_si512(src + i);
    bad = _mm512_or_si512(bad, _mm512_andnot_si512(one, v));
    const uint64_t m = _mm512_test_epi8_mask(v, one);
    std::memcpy(dst + i / 8, &m, 8);
  }
  uint32_t b = _mm512_test_epi8_mask(bad, bad) ? 1u : 0u;
  for (; i < row_bytes; i += 8) {  // 32-byte tail
    uint8_t m = 0;
    for (int k = 0; k < 8; ++k) {
      m |= static_cast<uint8_t>((src[i + k] & 1u) << k);
      b |= src[i + k] & 0xFEu;
    }
    dst[i / 8] = m;
  }
  return b;
}

__attribute__((target("avx512f,avx512bw"))) void unpack_row_512(const uint8_t* src, uint8_t* dst,
                                                                size_t row_bytes) {
  const __m512i one = _mm512_set1_epi8(1);
  size_t i = 0;
  if (reinterpret_cast<uintptr_t>(dst) % 64 == 0) {
    // non-temporal: the destination is not read first (no read-for-ownership)
    for (; i + 64 <= row_bytes; i += 64) {
      uint64_t m;
      std::memcpy(&m, src + i / 8, 8);
      _mm512_stream_si512(reinterpret_cast<__m512i*>(dst + i), _mm512_maskz_mov_epi8(m, one));
    }
  }
  for (; i + 64 <= row_bytes; i += 64) {
    uint64_t m;
    std::memcpy(&m, src + i / 8, 8);
    _mm512_storeu_si512(dst + i, _mm512_maskz_mov_epi8(m, one));
  }
  for (; i < row_bytes; ++i) dst[i] = (src[i / 8] >> (i % 8)) & 1u;
}

__attribute__((target("avx2"))) uint32_t pack_row_256(const uint8_t* src, uint8_t* dst,
                                                      size_t row_bytes) {
  const __m256i hi = _mm256_set1_epi8(static_cast<char>(0xFE));
  __m256i bad = _mm256_setzero_si256();
  size_t i = 0;
  for (; i + 32 <= row_bytes; i += 32) {
    const __m256i v = _mm256_loadu_si256(reinterpret_cast<const __m256i*>(src + i));
    bad = _mm256_or_si256(bad, _mm256_and_si256(v, hi));
    const uint32_t m = static_cast<uint32_t>(_mm256_movemask_epi8(_mm256_slli_epi16(v, 7)));
    std::memcpy(dst + i / 8, &m, 4);
  }
  uint32_t b = _mm256_testz_si256(bad, bad) ? 0u : 1u;
  for (; i < row_bytes; ++i) {
    if (i % 8 == 0) dst[i / 8] = 0;
    dst[i / 8] |= static_cast<uint8_t>((src[i] & 1u) << (i % 8));
    b |= src[i] & 0xFEu;
  }
  return b;
}

__attribute__((target("avx2"))) void unpack_row_256(const uint8_t* src, uint8_t* dst,
                                                    size_t row_bytes) {
  const __m256i shuf = _mm256_setr_epi8(0, 0, 0, 0, 0, 0, 0, 0, 1, 1, 1, 1, 1, 1, 1, 1, 2, 2, 2, 2, 2,
                                        2, 2, 2, 3, 3, 3, 3, 3, 3, 3, 3);
  const __m256i bits = _mm256_set1_epi64x(static_cast<long long>(0x8040201008040201ULL));
  const __m256i one = _mm256_set1_epi8(1);
  size_t i = 0;
  for (; i + 32 <= row_bytes; i += 32) {
    uint32_t m;
    std::memcpy(&m, src + i / 8, 4);
    __m256i v = _mm256_shuffle_epi8(_mm256_set1_epi32(static_cast<int>(m)), shuf);
    v = _mm256_min_epu8(_mm256_and_si256(v, bits), one);
    _mm256_storeu_si256(reinterpret_cast<__m256i*>(dst + i), v);
  }
  for (; i < row_bytes; ++i) dst[i] = (src[i / 8] >> (i % 8)) & 1u;
}

int isa() {  // 2: AVX-512BW, 1: AVX2, 0: neither
  static const int v = __builtin_cpu_supports("avx512bw") && __builtin_cpu_supports("avx512f") ? 2
                       : __builtin_cpu_supports("avx2")                                          ? 1
                                                                                                 : 0;
  return v;
}

// A fixed pool of worker threads (created on first use, parked on a condition
// variable between jobs): a transfer is cut into chunks of 32 MB of bits and
// every chunk is one job, so spawning threads per chunk would cost ~ms.  One
// job at a time (jobs from several host threads queue on the mutex).
class Pool {
 public:
  explicit Pool(int n) : n_(n) {
    for (int t = 1; t < n_; ++t) std::thread([this, t] { worker(t); }).detach();  // parked for good
  }
  int size() const { return n_; }
  // fn(t) for t in [0, n_): the caller runs part 0
  void run(const std::function<void(int)>& fn) {
    std::lock_guard<std::mutex> job(job_mu_);
    {
      std::lock_guard<std::mutex> lk(mu_);
      fn_ = &fn;
      pending_ = n_ - 1;
      ++epoch_;
    }
    cv_.notify_all();
    fn(0);
    std::unique_lock<std::mutex> lk(mu_);
    done_.wait(lk, [this] { return pending_ == 0; });
    fn_ = nullptr;
  }

 private:
  void worker(int t) {
    uint64_t seen = 0;
    for (;;) {
      const std::function<void(int)>* fn;
      {
        std::unique_lock<std::mutex> lk(mu_);
        cv_.wait(lk, [&] { return epoch_ != seen; });
        seen = epoch_;
        fn = fn_;
      }
      (*fn)(t);
      std::lock_guard<std::mutex> lk(mu_);
      if (--pending_ == 0) done_.notify_one();
    }
  }
  int n_;
  std::mutex job_mu_, mu_;
  std::condition_variable cv_, done_;
  const std::function<void(int)>* fn_ = nullptr;
  int pending_ = 0;
  uint64_t epoch_ = 0;
};

Pool& pool() {
  static Pool* p = new Pool(static_cast<int>(std::min(16u, std::max(1u, std::thread::hardware_concurrency()))));
  return *p;  // never destroyed: the parked workers outlive static destruction
}

template <typename Fn>
void over_threads(int64_t nrows, int threads, Fn&& fn) {
  const int T = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>({threads, nrows, pool().size()})));
  if (T == 1) {
    fn(0, nrows);
    return;
  }
  const std::function<void(int)> part = [&](int t) {
    if (t < T) fn(nrows * t / T, nrows * (t + 1) / T);
  };
  pool().run(part);
}

}  // namespace

bool bits_available() { return isa() > 0; }

int xfer_threads() {
  return static_cast<int>(std::min(16u, std::max(1u, std::thread::hardware_concurrency())));
}

bool cells_to_bits(const uint8_t* src, size_t pitch, size_t row_bytes, int64_t nrows, uint8_t* dst,
                   int threads) {
  std::atomic<uint32_t> bad{0};
  const bool wide = isa() == 2;
  over_threads(nrows, threads, [&](int64_t r0, int64_t r1) {
    uint32_t b = 0;
    for (int64_t r = r0; r < r1; ++r) {
      const uint8_t* s = src + static_cast<size_t>(r) * pitch;
      uint8_t* d = dst + static_cast<size_t>(r) * (row_bytes / 8);
      b |= wide ? pack_row_512(s, d, row_bytes) : pack_row_256(s, d, row_bytes);
    }
    if (b) bad.fetch_or(1u);
  });
  return bad.load() == 0;
}

void bits_to_cells(const uint8_t* src, uint8_t* dst, size_t pitch, size_t row_bytes, int64_t nrows,
                   int threads) {
  const bool wide = isa() == 2;
  over_threads(nrows, threads, [&](int64_t r0, int64_t r1) {
    for (int64_t r = r0; r < r1; ++r) {
      const uint8_t* s = src + static_cast<size_t>(r) * (row_bytes / 8);
      uint8_t* d = dst + static_cast<size_t>(r) * pitch;
      if (wide) unpack_row_512(s, d, row_bytes);
      else unpack_row_256(s, d, row_bytes);
    }
    _mm_sfence();  // order the non-temporal stores before the caller returns
  });
}

}  // namespace ltl_host
