// catsim/device.hpp -- the glue between the catsim C++ API of this repo and
// the C-ABI of libltl_b200.so (include/ltl_b200.h): status codes back to the
// reference's exception classes, and an owning device-context handle.
//
// Header-only: a program that used the reference's `catsim` library switches
// by compiling against include/ (these headers keep the reference's names and
// signatures, proj/include/catsim/*.hpp) and linking -lltl_b200.
#pragma once

#include <stdexcept>
#include <string>

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

// One device torus: owns the device buffers of a simulation.  One slab:
// ltl_create_grid (any f > 0 of a host Grid); several: ltl_create.
class DeviceGrid {
 public:
  DeviceGrid(int n, int f, int slabs = 1) {
    const int st = slabs == 1 ? ltl_create_grid(&ctx_, n, f) : ltl_create(&ctx_, n, f, slabs, nullptr);
    if (st != LTL_OK) throw_status(st, ltl_last_error(nullptr));
  }
  ~DeviceGrid() { ltl_destroy(ctx_); }
  DeviceGrid(const DeviceGrid&) = delete;
  DeviceGrid& operator=(const DeviceGrid&) = delete;
  ltl_ctx* get() const { return ctx_; }
  void check(int status) const { detail::check(status, ctx_); }

 private:
  ltl_ctx* ctx_ = nullptr;
};

}  // namespace detail
}  // namespace catsim
