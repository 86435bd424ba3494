// ltl_kernels.cuh -- device-side interfaces shared by the LTL kernels and the
// C-ABI runtime (ltl_runtime.cu).
#pragma once

#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>

namespace ltl {

// Halo width of every device slab, rows and columns.  The reference keeps a
// halo of f (<= 16) cells (include/catsim/grid.hpp:62); the device keeps 16
// whatever f is, because r <= 16 always and the halo only has to hold r.
constexpr int kHalo = 16;

// Rule constants the epilogues need, pre-reduced on the host from LtlRule
// (include/catsim/rule.hpp:17-32) and apply_transition (src/rule.cpp:99-111):
//   dead cell:  next = (unsigned)(R - lo_dead) <= w_dead       (count = R)
//   live cell:  next = (unsigned)(R - lo_live) <= w_live       (count = R - (mult - m))
//   live cell with R < neg_live  -> the reference's negative-count guard.
struct RuleConsts {
  int32_t r;
  int32_t kind;  // 0 Moore (center once), 1 simplified von Neumann (center twice)
  int32_t lo_dead, w_dead;
  int32_t lo_live, w_live;
  int32_t neg_live;  // mult - m
};

// One device slab: rows [row0, row0 + rows) of the global torus, all cols.
// Buffer geometry: (rows + 2*kHalo) x pitch bytes, interior at (kHalo, kHalo).
struct SlabView {
  uint8_t* buf;
  int32_t rows;
  int32_t cols;
  int64_t pitch;
};

struct DeviceStats {
  int32_t max_h;
  int32_t max_r;
  int32_t error;  // negative-count guard tripped
  int32_t pad;
};

// ---- tcgen05 banded-MMA step (ltl_tc.cu)
struct TcLaunch {
  const CUtensorMap* load_map;   // padded slab, box {32, 32}, SWIZZLE_32B
  const CUtensorMap* store_map;  // interior of the destination slab, box {128, 32}
  int32_t rows, cols;
  RuleConsts rule;
  int32_t inject_fault;
  DeviceStats* stats;  // nullptr -> no stats reduction
  int32_t grid;        // CTAs (0 = auto)
  int32_t seg_chunks;  // unused (kept for ABI of the launch struct)
  long long* trace;    // debug timeline (LTL_TC_TRACE), nullptr = off
  uint32_t* pace;      // 65 zeroed words for CTA pacing (nullptr = off); the
                       // kernel leaves them zeroed again when it exits
};
cudaError_t launch_tc_step(const TcLaunch& a, cudaStream_t stream);
size_t tc_smem_bytes();

// Host-side tensor-map builders (driver entry point fetched at runtime).
cudaError_t make_load_map(CUtensorMap* map, const SlabView& s);
cudaError_t make_store_map(CUtensorMap* map, const SlabView& s);

// ---- CUDA-core shared-memory stencil ablation (ltl_stencil.cu)
cudaError_t launch_stencil_step(const SlabView& in, const SlabView& out, const RuleConsts& rule,
                                int32_t inject_fault, DeviceStats* stats, cudaStream_t stream);

// ---- device init_random (ltl_init.cu): cell (gy, x) of the global torus gets
// splitmix64 draw number gy * fill_cols + x when gy < fill_rows and x < fill_cols.
void density_threshold(double density, int32_t* mode, uint64_t* threshold);
cudaError_t launch_init_random(const SlabView& s, int32_t row0, int32_t fill_rows,
                               int32_t fill_cols, double density, uint64_t seed,
                               cudaStream_t stream);

// ---- periodic halo refresh (ltl_halo.cu)
// Fills the halo of `self` from the interiors of `above` (rows over the top
// edge), `below` (rows under the bottom edge) and `self` (column wrap).  For a
// single slab all three are the same buffer.
cudaError_t launch_halo_fill(const SlabView& self, const SlabView& above, const SlabView& below,
                             cudaStream_t stream);

}  // namespace ltl
