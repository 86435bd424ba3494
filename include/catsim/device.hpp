// catsim/device.hpp -- the glue between the catsim C++ API of this repo and
// the C-ABI of libltl_b200.so (include/ltl_b200.h): status codes back to the
// reference's exception classes, and an owning device-context handle.
//
// Header-only: a program that used the reference's `catsim` library switches
// by compiling against include/ (these headers keep the reference's names and
// signatures, proj/include/catsim/*.hpp) and linking -lltl_b200.
#pragma once

#include <cstddef>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#if defined(__linux__)
#include <sys/mman.h>
#endif

#include "ltl_b200.h"

namespace catsim {
namespace detail {

// LTL_ERR_* -> the exception class the reference throws for the same error.
[[noreturn]] inline void throw_status(int status, const std::string& msg) {
  switch (status) {
    case LTL_ERR_INVALID_ARGUMENT: throw std::invalid_argument(msg);
    case LTL_ERR_LOGIC: throw std::logic_error(msg);
    default: throw std::runtime_error(msg);  // runtime / device failures
  }
}

inline void check(int status, const ltl_ctx* ctx) {
  if (status != LTL_OK) throw_status(status, ltl_last_error(ctx));
}

// The device torus of a call.  One slab (the API's calls): borrowed from a
// per-thread cache keyed by (n, f) -- the device buffers, streams and tensor
// maps of the previous call of the same geometry are reused, so repeated
// run_engine / simulate calls pay no cudaMalloc / cudaFree (a 2 x 273 MB free
// measured up to 0.8 s, profiles/cpp_e2e_r02.txt).  The cached context is
// released when the geometry changes; at thread exit it is left to the
// process teardown.  Several slabs: a fresh ltl_create, destroyed with the object.
class DeviceGrid {
 public:
  DeviceGrid(int n, int f, int slabs = 1) {
    if (slabs == 1) {
      Cache& c = cache();
      if (!c.ctx || c.n != n || c.f != f) {
        if (c.ctx) ltl_destroy(c.ctx);
        c.ctx = nullptr;
        const int st = ltl_create_grid(&c.ctx, n, f);
        if (st != LTL_OK) throw_status(st, ltl_last_error(nullptr));
        c.n = n;
        c.f = f;
      }
      ctx_ = c.ctx;
      owned_ = false;
      return;
    }
    const int st = ltl_create(&ctx_, n, f, slabs, nullptr);
    if (st != LTL_OK) throw_status(st, ltl_last_error(nullptr));
  }
  ~DeviceGrid() {
    if (owned_) ltl_destroy(ctx_);
  }
  DeviceGrid(const DeviceGrid&) = delete;
  DeviceGrid& operator=(const DeviceGrid&) = delete;
  ltl_ctx* get() const { return ctx_; }
  void check(int status) const { detail::check(status, ctx_); }

 private:
  struct Cache {
    ltl_ctx* ctx = nullptr;
    int n = -1, f = -1;
  };
  static Cache& cache() {
    thread_local Cache c;
    return c;
  }
  ltl_ctx* ctx_ = nullptr;
  bool owned_ = true;
};

// A fresh cells vector of `bytes` zeros.  Large ones are advised onto
// transparent huge pages before their first touch: a fresh 270 MB grid
// otherwise costs ~120 ms of 4 KB page faults (profiles/cpp_e2e_r02.txt).
inline void fresh_cells(std::vector<uint8_t>& v, std::size_t bytes) {
  std::vector<uint8_t>().swap(v);
  v.reserve(bytes);
#if defined(__linux__) && defined(MADV_HUGEPAGE)
  constexpr std::uintptr_t kHuge = std::uintptr_t{2} << 20;
  if (bytes >= 4 * kHuge) {
    const std::uintptr_t lo = (reinterpret_cast<std::uintptr_t>(v.data()) + kHuge - 1) & ~(kHuge - 1);
    const std::uintptr_t hi = (reinterpret_cast<std::uintptr_t>(v.data()) + bytes) & ~(kHuge - 1);
    if (hi > lo) madvise(reinterpret_cast<void*>(lo), hi - lo, MADV_HUGEPAGE);
  }
#endif
  v.resize(bytes);
}

}  // namespace detail
}  // namespace catsim
