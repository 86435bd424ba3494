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

// Column-strip width of the device layout (= the M of the tcgen05 MMAs).
constexpr int kStrip = 128;

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

// One device slab: rows [row0, row0 + rows) of the global torus, all cols,
// stored as column STRIPS (the reference's Grid::cells is one row-major
// vector, grid.hpp:60; on the device the layout is chosen for HBM streaming).
//
//   logical column px in [-128, 128 * (strips - 1)) lives in storage strip
//   (px + 128) / 128 at byte (px + 128) % 128 of its row; strip 0 and the
//   strip after the last interior one are padding that hold the 16 halo
//   columns.  Each strip is a contiguous block of (rows + 32) rows x 128 B:
//   padded row py in [0, rows + 32), interior rows at [16, 16 + rows).
//
// A 64..256-row piece of one strip is therefore ONE contiguous HBM block,
// which is what lets the step kernel stream at copy bandwidth
// (tools/ubench_stream3.cu; profiles/).
struct SlabView {
  uint8_t* buf;
  int32_t rows;
  int32_t cols;
  int32_t strips;       // storage strips = interior strips + 2
  int64_t strip_bytes;  // (rows + 2 * kHalo) * kStrip

  __host__ __device__ __forceinline__ int64_t offset(int32_t py, int32_t px) const {
    const int32_t sx = px + kStrip;
    return static_cast<int64_t>(sx >> 7) * strip_bytes + static_cast<int64_t>(py) * kStrip +
           (sx & (kStrip - 1));
  }
  __host__ __device__ __forceinline__ int64_t bytes() const { return strips * strip_bytes; }
};

// 4-bit copy of a slab for the packed tcgen05 step: the same strips and padded
// rows, 64 bytes per strip row, cell x of a row in the low (x even) or high
// nibble of byte x / 2 (nibble value 1 = alive: e2m1 0.5, the pass-1 B operand
// as it is).  B_alg = 1 byte per cell update.
constexpr int kPkRow = kStrip / 2;
struct PackedView {
  uint8_t* buf;
  int32_t rows;
  int32_t cols;
  int32_t strips;       // storage strips (as SlabView)
  int64_t strip_bytes;  // (rows + 2 * kHalo) * kPkRow
  __host__ __device__ __forceinline__ int64_t bytes() const { return strips * strip_bytes; }
};

__host__ __device__ inline int32_t interior_strips(int32_t cols) {
  return (cols + kStrip - 1) / kStrip;
}
__host__ __device__ inline int32_t storage_strips(int32_t cols) {
  return interior_strips(cols) + 2;
}

struct DeviceStats {
  int32_t max_h;
  int32_t max_r;
  int32_t error;  // negative-count guard tripped
  int32_t pad;
  // The reference throws at the FIRST negative count in its serial traversal
  // (simulate_step's rule loop, src/cat_engine.cpp:291-303: generation, then
  // tiles of tile_h x tile_w fragments row-major, fragments, cells) with the
  // count in the message (src/rule.cpp:104-107).  Min over
  // (generation << 40 | traversal position << 3 | -count); all-ones = none.
  unsigned long long first_negative;
};

// Traversal position of interior cell (y, x) in the reference's rule loop
// with its default tiles (CatConfig tile_w = 1, tile_h = 14,
// include/catsim/cat_engine.hpp:18-19) and one worker.
__host__ __device__ inline unsigned long long negative_key(int gen, int y, int x, int f, int n_cols,
                                                           int neg) {
  constexpr int kTileH = 14;
  const long long fi = y / f, fj = x / f;              // interior fragment coordinates
  const long long tiles_per_row = n_cols / f;          // tile_w = 1: one fragment column each
  const long long tile = (fi / kTileH) * tiles_per_row + fj;
  const long long pos = ((tile * kTileH + fi % kTileH) * f + (y % f)) * f + (x % f);
  return (static_cast<unsigned long long>(gen) << 40) | (static_cast<unsigned long long>(pos) << 3) |
         static_cast<unsigned long long>(neg & 7);
}

// ---- tcgen05 banded-MMA step (ltl_tc.cu)
constexpr int kTcBand = 128;                  // output rows per unit
constexpr int kTcBox = kTcBand + 2 * kHalo;   // rows per TMA box (160)
// Periodic wrap done by the LOADS instead of a halo refresh (fill_periodic_halo,
// src/grid.cpp:75-94): with cols % 128 == 0 the 16 side columns of strip 0 /
// S-1 are simply the boxes of strip S-1 / 0; with one whole-torus slab and
// rows % 32 == 0 the 16 rows above band 0 / below the last band are loaded
// from the other end of the same strip.  The halo cells in HBM are then never
// read by the step, so it writes none (no halo kernel between generations).
__host__ __device__ inline bool tc_wrap_cols(int32_t cols) {
  return cols >= kStrip && cols % kStrip == 0;
}
__host__ __device__ inline bool tc_wrap_rows(int32_t rows) {
  return rows >= 32 && rows % 32 == 0;
}
// load maps for boxes carrying kH = 16 (r <= 16) or 32 (17 <= r <= 32) halo
// rows: [0] whole (128 + 2 kH)-row boxes, [1] kH-row wrap pieces, [2] band-0
// bodies (128 + kH rows), [3] last-band bodies (rows of the last band + kH)
constexpr int kTcLoadMaps = 4;
constexpr int kTcMaxRadius = 32;  // the kH = 32 boxes (PAPER.md:561's "+16 expansion")
struct TcLaunch {
  const CUtensorMap* load_maps;  // kTcLoadMaps maps over the source slab, SWIZZLE_128B
  const CUtensorMap* store_map;  // destination interior rows, {128, 64, 1} boxes, SWIZZLE_128B
  // Multi-generation (persistent) launch: `gens` generations ping-ponging
  // between the two buffers, units released to the next generation through
  // per-unit completion counters (flags, bands x strips u32, all equal to
  // flag_base on entry; +2 per generation).  gens <= 1: one generation.
  const CUtensorMap* load_maps_b;  // maps of the destination buffer (as a source)
  const CUtensorMap* store_map_b;  // store map of the source buffer
  int32_t gens;
  uint32_t* flags;
  uint32_t flag_base;

  // Ring of slabs (multi-GPU, one generation per launch), pull model: the
  // first / last band's 16 rows above / below are loaded from the
  // neighbours' slabs (ring_up / ring_down: piece maps over their buffers
  // holding generation G, peer memory), gated by their done counters
  // (ltl_tc.cu Params::ring).  Needs wrap_cols and rows % 32 == 0.
  int32_t ring;
  uint32_t ring_gen;
  int32_t up_rows;
  const CUtensorMap* ring_up;
  const CUtensorMap* ring_down;
  const uint32_t* up_done;
  const uint32_t* down_done;
  uint32_t* my_done;
  uint32_t* my_ticket;
  // multi-generation ring launches (gens > 1): ring_up / ring_down point at
  // TWO maps each (the neighbour's buffer of generation 0, then of 1), and
  // the neighbours' per-unit counters (NULL: this slab's own, a self-ring)
  const uint32_t* up_flags;
  const uint32_t* down_flags;
  int32_t wrap_cols, wrap_rows;
  int32_t rows, cols;
  RuleConsts rule;
  int32_t inject_fault;     // CatConfig.inject_band_fault (src/cat_engine.cpp:277)
  int32_t fault_f;          // fragment side f of the faulted band fragments
  int32_t fault_row_phase;  // global row of local row 0, mod f
  int32_t gen_base;         // generation number of this launch's first generation
  int32_t row0;             // global row of local row 0 (reference traversal order)
  DeviceStats* stats;  // nullptr -> no stats reduction
  int32_t halo;        // box halo rows kH: 16 (0 = default) or 32 (r > 16; every wrap by
                       // the loads: wrap_cols and wrap_rows or ring; maps built for 32)
  int32_t grid;        // CTAs (0 = auto)
  long long* trace;    // debug timeline (LTL_TC_TRACE), nullptr = off
  int32_t packed;      // 4-bit cells: maps over PackedSlab buffers (halo 16, whole-torus
                       // slab, every wrap by the loads)
  uint32_t* dyn;       // one launch per generation: 2 zeroed words (remainder cursor,
                       // exit ticket) for the dynamic schedule; nullptr = static
};
cudaError_t launch_tc_step(const TcLaunch& a, cudaStream_t stream);
int tc_persistent_ctas(int32_t rows, int32_t cols, int num_sms);  // 0: no multi-generation launch
int tc_sweep_chunks(int32_t strips, int32_t bands, int ctas);  // chunks per band of a multi-generation launch
size_t tc_smem_bytes(int halo, bool packed = false);

// Host-side tensor-map builders (driver entry point fetched at runtime).
cudaError_t make_load_maps(CUtensorMap* maps, const SlabView& s, int halo = kHalo);
cudaError_t make_store_map(CUtensorMap* map, const SlabView& s);
// The same over the 4-bit copy of a slab (PackedView: 64-byte strip rows):
// loads as 16U4_ALIGN16B boxes (the padded e2m1 operand layout, SWIZZLE_128B),
// stores of 64 x 64-byte staging tiles (SWIZZLE_64B).
struct PackedView;
cudaError_t make_load_maps_packed(CUtensorMap* maps, const PackedView& s);
cudaError_t make_store_map_packed(CUtensorMap* map, const PackedView& s);
// halo-row (16 / 32) SWIZZLE_128B pieces over a slab (the ring's rows from a neighbour).
cudaError_t make_piece_map(CUtensorMap* map, const SlabView& s, int halo = kHalo);

// ---- CUDA-core stencil ablations (ltl_stencil.cu): kEngineBase sums the
// (2r+1)^2 box / 2(2r+1) cross per cell (the paper's SHARED baseline),
// kEnginePack keeps packed 16-bit-lane sliding-window sums (O(1) per cell).
constexpr int kEngineBase = 0, kEnginePack = 1;
cudaError_t launch_stencil_step(const SlabView& in, const SlabView& out, const RuleConsts& rule,
                                int engine, DeviceStats* stats, cudaStream_t stream);

// ---- the reference's fragment-level passes, materialised (ltl_fragment.cu)
// stage 0 horizontal, 1 vertical Moore, 2 vertical von Neumann; padded
// (n + 2f)^2 fragment-contiguous fields, bands = pi1 | pi2 | pi3 (f x f each).
cudaError_t launch_fragment_pass(int stage, int n, int f, const uint8_t* cells,
                                 const int32_t* bands, const int32_t* h, int32_t* out,
                                 cudaStream_t stream);

// ---- device init_random (ltl_init.cu): cell (gy, x) of the global torus gets
// splitmix64 draw number gy * fill_cols + x when gy < fill_rows and x < fill_cols.
void density_threshold(double density, int32_t* mode, uint64_t* threshold);
cudaError_t launch_init_random(const SlabView& s, int32_t row0, int32_t fill_rows,
                               int32_t fill_cols, double density, uint64_t seed,
                               cudaStream_t stream);

// ---- periodic halo refresh (ltl_halo.cu)
// Fills the halo of `self` from the interiors of `above` (rows over the top
// edge), `below` (rows under the bottom edge) and `self` (column wrap).  For a
// single slab all three are the same buffer.  `parts`: kHaloCols | kHaloRows.
constexpr int kHaloCols = 1, kHaloRows = 2;
cudaError_t launch_halo_fill(const SlabView& self, const SlabView& above, const SlabView& below,
                             int parts, cudaStream_t stream);

// ---- layout conversion and edge exchange (ltl_layout.cu)
// Dense row-major rows x cols interior <-> strip slab interior.
cudaError_t launch_to_strips(const uint8_t* dense, const SlabView& s, cudaStream_t stream);
cudaError_t launch_from_strips(const SlabView& s, uint8_t* dense, cudaStream_t stream);
// Dense interior in fragment-contiguous order (f in {4, 8, 16}; rows and
// cols multiples of f) <-> strip slab interior.
cudaError_t launch_frag_relayout(uint8_t* dense, const SlabView& s, int f, bool to_strips,
                                 cudaStream_t stream);
// dense {0, 1} bytes <-> bits (bit k % 8 of byte k / 8 = byte k), n % 32 == 0:
// the device side of the bit-packed host transfers.
cudaError_t launch_bits_to_cells(const uint8_t* bits, uint8_t* cells, int64_t n, cudaStream_t stream);
// (*bad |= 1 if a byte is neither 0 nor 1)
cudaError_t launch_cells_to_bits(const uint8_t* cells, uint8_t* bits, int64_t n, int32_t* bad,
                                 cudaStream_t stream);
// bits (row-major, cols % 32 == 0) <-> the interior of a slab's strips.
cudaError_t launch_bits_to_strips(const uint8_t* bits, const SlabView& s, cudaStream_t stream);
cudaError_t launch_strips_to_bits(const SlabView& s, uint8_t* bits, int32_t* bad, cudaStream_t stream);
// u8 slab <-> its 4-bit copy (every padded row of every strip).
cudaError_t launch_pack_cells(const SlabView& s, const PackedView& pk, cudaStream_t stream);
cudaError_t launch_unpack_cells(const PackedView& pk, const SlabView& s, cudaStream_t stream);
// *bad |= 1 if any of dense[0, n) is not 0 / 1 (snapshot payloads).
cudaError_t launch_check_cells(const uint8_t* dense, int64_t n, int32_t* bad,
                               cudaStream_t stream);
// top[16][cols] <- interior rows [0, 16); bot[16][cols] <- rows [rows-16, rows).
cudaError_t launch_pack_edges(const SlabView& s, uint8_t* top, uint8_t* bot, cudaStream_t stream);
// halo rows above <- top_halo[16][cols], below <- bot_halo[16][cols] (with the
// column wrap of those rows, i.e. the corners).
cudaError_t launch_unpack_halo(const SlabView& s, const uint8_t* top_halo,
                               const uint8_t* bot_halo, cudaStream_t stream);

}  // namespace ltl
