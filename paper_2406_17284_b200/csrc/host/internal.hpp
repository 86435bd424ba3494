// internal.hpp -- declarations shared between the host-side translation units
// of libltl_b200.so (not part of the public API).
#pragma once

#include <cstddef>
#include <cstdint>

#include "catsim/rule.hpp"
#include "ltl_b200.h"

namespace catsim {

// The reference's rule validation (src/rule.cpp:32-57), throwing the same
// std::invalid_argument messages; max_radius > 16 is the wide-radius extension.
void validate_rule(const LtlRule& rule, int max_radius = kMaxRadius);

inline LtlRule from_c(const ltl_rule_c& c) {
  LtlRule r;
  r.r = c.r;
  r.c = c.c;
  r.m = c.m;
  r.s1 = c.s1;
  r.s2 = c.s2;
  r.b1 = c.b1;
  r.b2 = c.b2;
  r.kind = c.kind == LTL_KIND_MOORE ? NeighborhoodKind::Moore : NeighborhoodKind::VonNeumannSimplified;
  return r;
}

inline ltl_rule_c to_c(const LtlRule& r) {
  ltl_rule_c c;
  c.r = r.r;
  c.c = r.c;
  c.m = r.m;
  c.s1 = r.s1;
  c.s2 = r.s2;
  c.b1 = r.b1;
  c.b2 = r.b2;
  c.kind = r.kind == NeighborhoodKind::Moore ? LTL_KIND_MOORE : LTL_KIND_VON_NEUMANN;
  return c;
}

}  // namespace catsim

// Bit-packed host <-> device transfers (host/xfer_bits.cpp): rows of
// row_bytes (% 32 == 0) cells at host `pitch` <-> contiguous rows of
// row_bytes / 8 bytes of bits (cell x of a row = bit x % 8 of byte x / 8).
namespace ltl_host {
bool bits_available();  // AVX-512BW or AVX2 on this CPU
int xfer_threads();     // host threads for the packing (<= 16)
// false if a byte is neither 0 nor 1 (the caller then copies bytes)
bool cells_to_bits(const uint8_t* src, size_t pitch, size_t row_bytes, int64_t nrows, uint8_t* dst,
                   int threads);
void bits_to_cells(const uint8_t* src, uint8_t* dst, size_t pitch, size_t row_bytes, int64_t nrows,
                   int threads);
}  // namespace ltl_host
