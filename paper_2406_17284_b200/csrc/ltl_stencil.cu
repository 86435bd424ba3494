// ltl_stencil.cu -- the classical CUDA-core ablations, on the same device
// slab layout (column strips, ltl_kernels.cuh) as the tensor-core path and
// bit-identical to it (tests/test_gpu_parity.py).  They are the GPU
// counterparts of the reference's comparison engines (EngineKind::Base /
// Pack, proj/include/catsim/engines.hpp:11) and of the paper's CUDA-core
// baselines:
//
//   base  the paper's SHARED stencil: every cell sums its whole (2r+1)^2 box
//         (Moore) / 2(2r+1) cross (VN) out of a shared-memory tile, four cells
//         per thread in byte lanes -- (2r+1)^2 adds per cell, the radius
//         dependence the banded-MMA formulation removes.
//   pack  the strongest CUDA-core formulation we know: separable sums with
//         O(1) work per cell at any radius -- horizontal window sums from
//         16-bit-lane prefix sums of each tile row (direct sums for r <= 2),
//         then vertical sliding sums down the columns (one add of a biased
//         byte difference per row), packed four cells per 32-bit register
//         end to end, with the rule folded into 16-bit SIMD range tests.
//
// Both: one CTA per (128-column strip, TY-row chunk); the tile -- padded rows
// [y0, y0 + TY + 32) of the strip (ONE contiguous block in the strip layout)
// plus the 16 columns on either side -- is staged in SMEM with 16-byte loads;
// outputs leave as coalesced 4-byte stores (a warp writes a strip row).
// Templated on the radius so every window offset is a compile-time constant.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <utility>

#include "ltl_kernels.cuh"

namespace ltl {
namespace {

constexpr int kThreads = 256;
// Tile rows hold logical columns [-16, 144) of the strip (160 bytes) at a
// 176-byte pitch: 11 16-byte chunks, odd, so the 16-byte loads of 8
// consecutive rows (the pack engine's row pass, one row per thread) fall in
// 8 different bank groups, and every row is 16-byte aligned for 128-bit
// shared loads / stores.
constexpr int kTileCols = kStrip + 2 * kHalo;  // 160
constexpr int kTileW = kTileCols + 16;         // row pitch in bytes

__device__ __forceinline__ uint32_t prmt(uint32_t a, uint32_t b, uint32_t sel) {
  uint32_t d;
  asm("prmt.b32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(sel));
  return d;
}
template <uint32_t kLut>
__device__ __forceinline__ uint32_t lop3(uint32_t a, uint32_t b, uint32_t c) {
  uint32_t d;
  asm("lop3.b32 %0, %1, %2, %3, %4;" : "=r"(d) : "r"(a), "r"(b), "r"(c), "n"(kLut));
  return d;
}
// four byte lanes -> two words of 16-bit lanes (lanes 0,1 / 2,3)
__device__ __forceinline__ uint32_t widen_lo(uint32_t w) { return prmt(w, 0u, 0x4140u); }
__device__ __forceinline__ uint32_t widen_hi(uint32_t w) { return prmt(w, 0u, 0x4342u); }
// bytes k .. k+3 of a row held in registers as 32-bit words (k folds to a
// constant once the caller's loops are unrolled)
__device__ __forceinline__ uint32_t bytes_at(const uint32_t* w, int k) {
  return (k & 3) ? __funnelshift_r(w[k >> 2], w[(k >> 2) + 1], 8 * (k & 3)) : w[k >> 2];
}

// The birth/survival rule on two cells per register (16-bit lanes hold
// Z = R + K*state, < 4096): bit 15 / 31 of the result = next state
// (apply_transition, src/rule.cpp:99-111; same constants as ltl_tc.cu).
struct SimdRule {
  uint32_t ca, cb, cc, cd, g_live, g_neg, r_mask;
  __device__ SimdRule(const RuleConsts& rc, uint32_t K) {
    ca = (0x8000u - rc.lo_dead) * 0x10001u;
    cb = (0x7FFFu - (rc.lo_dead + rc.w_dead)) * 0x10001u;
    cc = (0x8000u - (K + rc.lo_live)) * 0x10001u;
    cd = (0x7FFFu - (K + rc.lo_live + rc.w_live)) * 0x10001u;
    g_live = (0x8000u - K) * 0x10001u;
    g_neg = (0x8000u - (K + rc.neg_live)) * 0x10001u;
    r_mask = (K - 1) * 0x10001u;
  }
  __device__ __forceinline__ uint32_t pair(uint32_t z) const {
    const uint32_t a = z + ca, b = z + cb, c = z + cc, d = z + cd;
    return lop3<0x70>(lop3<0xBA>(a, b, c), c, d);  // ((a & ~b) | c) & ~(c & d)
  }
  // live cell whose count R - (mult - m) is negative (the reference's guard)
  __device__ __forceinline__ uint32_t negative(uint32_t z) const {
    return (z + g_live) & ~(z + g_neg) & 0x80008000u;
  }
};

// The same rule on FOUR cells per register (8-bit lanes hold Z = R + 64 state,
// < 128): usable while R < 64 -- Moore r <= 3 (R <= 49), VN r <= 15
// (R <= 62).  Bit 7 of each byte of the result = next state.  Half the
// instructions of two 16-bit pairs, and no widening of the sums.
constexpr uint32_t kByteK = 64;
template <int R, int KIND>
__host__ __device__ constexpr bool byte_rule() { return KIND == 0 ? R <= 3 : R <= 15; }

struct ByteRule {
  uint32_t ca, cb, cc, cd, g_live, g_neg;
  __device__ ByteRule(const RuleConsts& rc) {
    ca = (0x80u - rc.lo_dead) * 0x01010101u;
    cb = (0x7Fu - (rc.lo_dead + rc.w_dead)) * 0x01010101u;
    cc = (0x80u - (kByteK + rc.lo_live)) * 0x01010101u;
    cd = (0x7Fu - (kByteK + rc.lo_live + rc.w_live)) * 0x01010101u;
    g_live = (0x80u - kByteK) * 0x01010101u;
    g_neg = (0x80u - (kByteK + rc.neg_live)) * 0x01010101u;
  }
  // four next states as 0/1 bytes
  __device__ __forceinline__ uint32_t next4(uint32_t z) const {
    const uint32_t a = z + ca, b = z + cb, c = z + cc, d = z + cd;
    return (lop3<0x70>(lop3<0xBA>(a, b, c), c, d) >> 7) & 0x01010101u;
  }
  __device__ __forceinline__ uint32_t negative(uint32_t z) const {
    return (z + g_live) & ~(z + g_neg) & 0x80808080u;
  }
};

// four next states (0/1 bytes) from the rule results of lanes (x, x+1), (x+2, x+3)
__device__ __forceinline__ uint32_t next_word(uint32_t a, uint32_t b) {
  return prmt(a, b, 0xFDB9u) & 0x01010101u;
}

// stage padded rows [y0, y0 + TY + 32) x logical columns [x0 - 16, x0 + 144)
// of the slab into tile[TY + 32][kTileW] (rows past the slab read as 0).
// The strip's own 128 columns are ONE contiguous block of the strip layout
// (16-byte chunk i at byte 16 i); the 16 side columns are one chunk per row
// of the neighbour strips.  16-byte cp.async copies (LDGSTS): the data goes
// global -> SMEM without a register round trip or an SMEM store instruction
// (ncu of the register-staged version: the tile stores waited on their loads
// and crowded the shared-memory instruction queue of the compute phase).
__device__ __forceinline__ void cp_async16(uint8_t* dst, const void* src, bool valid) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;"
               ::"r"(static_cast<uint32_t>(__cvta_generic_to_shared(dst))), "l"(src),
               "r"(valid ? 16 : 0)
               : "memory");
}

template <int TY>
__device__ __forceinline__ void load_tile(const SlabView& in, int strip, int y0, uint8_t* tile) {
  constexpr int kRows = TY + 2 * kHalo;
  constexpr int kMain = kRows * 8, kSide = kRows * 2;
  const int valid_rows = min(kRows, in.rows + 2 * kHalo - y0);
  const uint8_t* mid = in.buf + static_cast<int64_t>(strip + 1) * in.strip_bytes +
                       static_cast<int64_t>(y0) * kStrip;
  const uint8_t* left = mid - in.strip_bytes + (kStrip - kHalo);
  const uint8_t* right = mid + in.strip_bytes;
  for (int i = static_cast<int>(threadIdx.x); i < kMain; i += kThreads) {
    const bool v = (i >> 3) < valid_rows;  // zero-filled past the slab
    cp_async16(tile + (i >> 3) * kTileW + kHalo + 16 * (i & 7),
               v ? mid + 16 * i : in.buf, v);
  }
  for (int i = static_cast<int>(threadIdx.x); i < kSide; i += kThreads) {
    const int row = i >> 1;
    const bool v = row < valid_rows;
    cp_async16(tile + row * kTileW + ((i & 1) ? kHalo + kStrip : 0),
               v ? (i & 1 ? right : left) + row * kStrip : in.buf, v);
  }
  asm volatile("cp.async.commit_group;\n\tcp.async.wait_group 0;" ::: "memory");
}

// store four next states at interior row y, columns x .. x+3 (clipped to cols)
__device__ __forceinline__ void store_word(const SlabView& out, int y, int x, uint32_t w) {
  if (x + 3 < out.cols) {
    *reinterpret_cast<uint32_t*>(out.buf + out.offset(y + kHalo, x)) = w;
  } else {
    for (int b = 0; b < 4 && x + b < out.cols; ++b) out.buf[out.offset(y + kHalo, x + b)] = (w >> (8 * b)) & 1u;
  }
}

__device__ __forceinline__ void flush_stats(DeviceStats* stats, uint32_t max_h4, uint32_t max_r2,
                                            uint32_t bad) {
  int32_t mh = static_cast<int32_t>(max(max(max_h4 & 0xFF, (max_h4 >> 8) & 0xFF),
                                        max((max_h4 >> 16) & 0xFF, max_h4 >> 24)));
  int32_t mr = static_cast<int32_t>(max(max_r2 & 0xFFFF, max_r2 >> 16));
  for (int off = 16; off > 0; off >>= 1) {
    mh = max(mh, __shfl_xor_sync(0xffffffffu, mh, off));
    mr = max(mr, __shfl_xor_sync(0xffffffffu, mr, off));
  }
  if ((threadIdx.x & 31) == 0) {
    atomicMax(&stats->max_h, mh);
    atomicMax(&stats->max_r, mr);
  }
  if (__any_sync(0xffffffffu, bad != 0) && (threadIdx.x & 31) == 0) atomicOr(&stats->error, 1);
}

// ============================ base: direct (2r+1)^2 sums ======================
constexpr int kBaseTY = 128;

template <int R, int KIND, bool kChecked>
__global__ void __launch_bounds__(kThreads)
    base_kernel(const SlabView in, const SlabView out, const RuleConsts rc, DeviceStats* stats) {
  __shared__ __align__(16) uint8_t tile[(kBaseTY + 2 * kHalo) * kTileW];
  const int strip = blockIdx.x, y0 = blockIdx.y * kBaseTY;
  load_tile<kBaseTY>(in, strip, y0, tile);
  __syncthreads();
  const int j = threadIdx.x & 31;                  // output word: columns 4j .. 4j+3
  const int seg = threadIdx.x >> 5;                // 16-row segment
  const int x = strip * kStrip + 4 * j;
  const uint32_t K = KIND == 0 ? 2048u : 128u;
  const SimdRule sr(rc, K);
  const uint32_t hmask = x + 3 < in.cols ? 0xFFFFFFFFu : (x >= in.cols ? 0u : (1u << (8 * (in.cols - x))) - 1u);
  const uint32_t rmask_lo = (x < in.cols ? 0xFFFFu : 0u) | (x + 1 < in.cols ? 0xFFFF0000u : 0u);
  const uint32_t rmask_hi = (x + 2 < in.cols ? 0xFFFFu : 0u) | (x + 3 < in.cols ? 0xFFFF0000u : 0u);
  uint32_t max_h = 0, max_r = 0, bad = 0;
  constexpr int kW0 = (16 - R) >> 2;                     // first word a row window touches
  constexpr int kNW = ((16 + 3 + R) >> 2) - kW0 + 1;     // words per row window
  const int ys = seg * (kBaseTY / 8);
  const int nrows = max(0, min(kBaseTY / 8, in.rows - (y0 + ys)));
  const bool full_word = x + 3 < in.cols;
  uint8_t* optr = out.buf + out.offset(y0 + ys + kHalo, min(x, in.cols - 1));
  constexpr bool kByte = byte_rule<R, KIND>();  // R < 64: sums and rule in byte lanes
  const ByteRule br(rc);
  for (int yy = 0; yy < nrows; ++yy, optr += kStrip) {
    const int y = ys + yy;  // output row within the chunk
    uint32_t acc_lo = 0, acc_hi = 0, acc_b = 0, h_centre = 0, v_cross = 0;
#pragma unroll
    for (int dy = -R; dy <= R; ++dy) {
      const uint32_t* trow =
          reinterpret_cast<const uint32_t*>(tile + (kHalo + y + dy) * kTileW) + j + kW0;
      uint32_t w[kNW];
#pragma unroll
      for (int k = 0; k < kNW; ++k) w[k] = trow[k];
      if (KIND == 0 || dy == 0) {
        uint32_t h = 0;  // row window sums of the four cells, byte lanes (<= 33)
#pragma unroll
        for (int dx = -R; dx <= R; ++dx) h += bytes_at(w, 16 + dx - 4 * kW0);
        if (dy == 0) h_centre = h;
        if (KIND == 0 && kByte) {
          acc_b += h;  // <= 49
        } else if (KIND == 0) {
          acc_lo += widen_lo(h);
          acc_hi += widen_hi(h);
        }
      }
      if (KIND == 1) v_cross += bytes_at(w, 16 - 4 * kW0);  // column sum, byte lanes
    }
    const uint32_t st = *reinterpret_cast<const uint32_t*>(tile + (kHalo + y) * kTileW + 16 + 4 * j);
    uint32_t nw;
    if constexpr (kByte) {  // Z = R + 64 state in byte lanes
      const uint32_t zb = (KIND == 0 ? acc_b : h_centre + v_cross) + st * kByteK;
      nw = br.next4(zb);
      if constexpr (kChecked) {
        max_h = __vmaxu4(max_h, h_centre & hmask);
        max_r = __vmaxu4(max_r, zb & ((kByteK - 1) * 0x01010101u) & hmask);
        bad |= br.negative(zb) & hmask;
      }
    } else {
      if (KIND == 1) {  // R = H + V (centre twice), plus 128 * state: all < 256
        const uint32_t zb = h_centre + v_cross + (st << 7);
        acc_lo = widen_lo(zb);
        acc_hi = widen_hi(zb);
      } else {
        acc_lo += widen_lo(st) << 11;
        acc_hi += widen_hi(st) << 11;
      }
      nw = next_word(sr.pair(acc_lo), sr.pair(acc_hi));
      if constexpr (kChecked) {
        max_h = __vmaxu4(max_h, h_centre & hmask);
        max_r = __vmaxu2(max_r, acc_lo & sr.r_mask & rmask_lo);
        max_r = __vmaxu2(max_r, acc_hi & sr.r_mask & rmask_hi);
        bad |= (sr.negative(acc_lo) & rmask_lo) | (sr.negative(acc_hi) & rmask_hi);
      }
    }
    if (full_word) *reinterpret_cast<uint32_t*>(optr) = nw;
    else if (x < in.cols) store_word(out, y0 + y, x, nw);
  }
  if constexpr (kChecked && kByte)  // byte-lane R maxima -> the 16-bit layout flush_stats reduces
    max_r = max(max(max_r & 0xFF, (max_r >> 8) & 0xFF), max((max_r >> 16) & 0xFF, max_r >> 24));
  if constexpr (kChecked) flush_stats(stats, max_h, max_r, bad);
}

// ====================== pack: separable, O(1) per cell ========================
constexpr int kPackTY = 128;
constexpr int kHW = kStrip;         // H tile row: the 128 output columns
constexpr int kHStride = kHW / 4 + 1;  // 33 words: the row pass's stores hit 32 banks

// kN words from a 16-byte aligned shared address, as 128-bit loads.
template <int kN>
__device__ __forceinline__ void load_words(const uint32_t* src, uint32_t (&w)[kN]) {
  static_assert(kN % 4 == 0, "whole 16-byte loads");
#pragma unroll
  for (int k = 0; k < kN; k += 4) {
    const uint4 v = reinterpret_cast<const uint4*>(src)[k / 4];
    w[k] = v.x;
    w[k + 1] = v.y;
    w[k + 2] = v.z;
    w[k + 3] = v.w;
  }
}

// Horizontal window sums of one 32-column quarter of a tile row (output
// columns 32q .. 32q+31 = tile columns 16 + 32q ..), written as bytes to
// hrow[8q .. 8q+7]; returns their byte-lane max over valid columns.
template <int R>
__device__ __forceinline__ uint32_t row_window_sums(const uint32_t* trow, int q, uint32_t* hrow,
                                                    uint32_t valid_words) {
  uint32_t max_h = 0;
  if constexpr (R <= 2) {
    // direct: 2r+1 funnel-shifted words per four columns
    constexpr int kW0 = ((16 - R) >> 2) & ~3;             // first word, 16-byte aligned
    constexpr int kNW = (((16 + 31 + R) >> 2) + 2 - kW0 + 3) & ~3;
    uint32_t w[kNW];
    load_words<kNW>(trow + 8 * q + kW0, w);
#pragma unroll
    for (int o = 0; o < 8; ++o) {
      uint32_t h = 0;
#pragma unroll
      for (int dx = -R; dx <= R; ++dx) {
        h += bytes_at(w, 16 + 4 * o + dx - 4 * kW0);
      }
      hrow[8 * q + o] = h;
      if (o < static_cast<int>(valid_words)) max_h = __vmaxu4(max_h, h);
    }
  } else {
    // prefix sums in 16-bit lanes: P(k) = sum of tile columns [32q + kA, k];
    // H(x) = P(16 + x + r) - P(16 + x - r - 1)
    constexpr int kA = (16 - R - 1) & ~15;            // first column (16-byte aligned)
    constexpr int kEnd = 16 + 31 + R;                 // last column needed
    constexpr int kNW = ((((kEnd - kA) >> 2) + 1) + 3) & ~3;  // words of cells, whole uint4s
    uint32_t cw[kNW];
    load_words<kNW>(trow + 8 * q + (kA >> 2), cw);
    uint32_t pl[2 * kNW];                             // (P(2m), P(2m+1)), relative to kA
    uint32_t c = 0;
#pragma unroll
    for (int k = 0; k < kNW; ++k) {
      const uint32_t p = cw[k] * 0x01010101u;        // byte-lane prefix (<= 4)
      const uint32_t cc = c * 0x10001u;
      pl[2 * k] = widen_lo(p) + cc;
      pl[2 * k + 1] = widen_hi(p) + cc;
      c += p >> 24;
    }
#pragma unroll
    for (int o = 0; o < 8; ++o) {
      uint32_t hp[2];
#pragma unroll
      for (int s = 0; s < 2; ++s) {
        const int X = 4 * o + 2 * s;
        const int a = 16 + X + R - kA, b = 16 + X - R - 1 - kA;  // offsets of the two pairs
        const uint32_t pa = (a & 1) ? __funnelshift_r(pl[a >> 1], pl[(a >> 1) + 1], 16) : pl[a >> 1];
        const uint32_t pb = (b & 1) ? __funnelshift_r(pl[b >> 1], pl[(b >> 1) + 1], 16) : pl[b >> 1];
        hp[s] = pa - pb;  // lanes (H(x), H(x+1)) <= 33, no borrow (P is non-decreasing)
      }
      const uint32_t h = prmt(hp[0], hp[1], 0x6420u);  // four byte lanes
      hrow[8 * q + o] = h;
      if (o < static_cast<int>(valid_words)) max_h = __vmaxu4(max_h, h);
    }
  }
  return max_h;
}

template <int R, int KIND, bool kChecked>
__global__ void __launch_bounds__(kThreads)
    pack_kernel(const SlabView in, const SlabView out, const RuleConsts rc, DeviceStats* stats) {
  constexpr int kRows = kPackTY + 2 * kHalo;
  // dynamic: 16 bytes of front padding (at r = 16 the row pass of the first
  // quarter starts its prefix one 16-byte chunk before column -16 of the row:
  // garbage that cancels in every prefix difference, but it must be inside
  // the allocation), the tile, the H rows y0-r .. y0+TY+r
  extern __shared__ __align__(16) uint8_t pack_smem[];
  uint8_t* const tile = pack_smem + 16;
  uint32_t* const htile = reinterpret_cast<uint32_t*>(tile + kRows * kTileW);
  const int strip = blockIdx.x, y0 = blockIdx.y * kPackTY;
  load_tile<kPackTY>(in, strip, y0, tile);
  __syncthreads();
  const int x_strip = strip * kStrip;
  uint32_t max_h = 0, max_r = 0, bad = 0;
  // ---- phase 1: horizontal window sums H of tile rows 16-r .. 16+TY+r-1
  constexpr int kHRows = kPackTY + 2 * R;
  for (int item = threadIdx.x; item < kHRows * 4; item += kThreads) {
    const int q = item / kHRows, hr = item % kHRows;  // a warp: consecutive rows, one quarter
    const int trow = kHalo - R + hr;  // tile row
    const int y = y0 + trow - kHalo;  // interior row
    int vw = 0;                       // valid words of this quarter (checked stats)
    if (kChecked && hr >= R && hr < R + kPackTY && y < in.rows) {
      const int vc = in.cols - (x_strip + 32 * q);
      vw = vc <= 0 ? 0 : vc >= 32 ? 8 : vc / 4;  // whole words only (cols % 4 tail below)
    }
    const uint32_t mh = row_window_sums<R>(reinterpret_cast<const uint32_t*>(tile + trow * kTileW),
                                           q, htile + hr * kHStride, static_cast<uint32_t>(vw));
    if (kChecked) max_h = __vmaxu4(max_h, mh);
  }
  __syncthreads();
  if (kChecked) {  // a partial last word of the torus (cols % 4 != 0)
    const int vc = in.cols - x_strip;
    if (vc > 0 && vc < kStrip && (vc & 3) && threadIdx.x < kPackTY && y0 + threadIdx.x < in.rows) {
      const uint32_t h = htile[(R + threadIdx.x) * kHStride + (vc >> 2)];
      max_h = __vmaxu4(max_h, h & ((1u << (8 * (vc & 3))) - 1u));
    }
  }
  // ---- phase 2: vertical sliding sums down each 4-column word, 16-row segments
  const int j = threadIdx.x & 31;
  const int seg = threadIdx.x >> 5;
  const int x = x_strip + 4 * j;
  constexpr uint32_t K = KIND == 0 ? 2048u : 128u;
  constexpr bool kByte = byte_rule<R, KIND>();  // R < 64: sums and rule in byte lanes
  const SimdRule sr(rc, K);
  const ByteRule br(rc);
  const uint32_t rmask_lo = (x < in.cols ? 0xFFFFu : 0u) | (x + 1 < in.cols ? 0xFFFF0000u : 0u);
  const uint32_t rmask_hi = (x + 2 < in.cols ? 0xFFFFu : 0u) | (x + 3 < in.cols ? 0xFFFF0000u : 0u);
  const uint32_t rmask_b = x + 3 < in.cols ? 0xFFFFFFFFu
                           : (x >= in.cols ? 0u : (1u << (8 * (in.cols - x))) - 1u);
  constexpr int kSeg = kPackTY / 8;
  const int ys = seg * kSeg;
  const uint32_t* hcol = htile + j;  // H word of H row k: hcol[k * kHStride]
  const uint8_t* ccol = tile + 16 + 4 * j;
  // Moore: R lanes (byte lanes when kByte, else 16-bit lo / hi); VN: V (vertical
  // cell sums) bytes in lo
  uint32_t lo = 0, hi = 0;
  if (KIND == 0) {
    // R(ys) = sum of H rows ys .. ys + 2r (H row k = interior row y0 - r + k);
    // byte lanes for up to 7 rows (<= 231), then widened
    uint32_t g = 0;
#pragma unroll
    for (int k = 0; k <= 2 * R; ++k) {
      g += hcol[(ys + k) * kHStride];
      if (!kByte && (k % 7 == 6 || k == 2 * R)) {
        lo += widen_lo(g);
        hi += widen_hi(g);
        g = 0;
      }
    }
    if (kByte) lo = g;  // <= 49
  } else {
#pragma unroll
    for (int k = -R; k <= R; ++k) lo += *reinterpret_cast<const uint32_t*>(ccol + (kHalo + ys + k) * kTileW);
  }
  const int nrows = max(0, min(kSeg, in.rows - (y0 + ys)));
  const bool full_word = x + 3 < in.cols;
  uint8_t* const optr = out.buf + out.offset(y0 + ys + kHalo, min(x, in.cols - 1));
  // row yy of the segment: the H rows entering / leaving the window (Moore),
  // the cell rows entering / leaving (VN), the centre -- fixed offsets from
  // these bases, so the unrolled full-segment loop addresses with immediates
  const uint32_t* const h_in = hcol + (ys + 2 * R) * kHStride;
  const uint32_t* const h_mid = hcol + (ys + R) * kHStride;
  const uint8_t* const c_mid = ccol + (kHalo + ys) * kTileW;
  auto row = [&](int yy) {
    if (yy > 0) {
      if (KIND == 0 && kByte) {
        // R += H(y + r) - H(y - r - 1), byte lanes: the sum before the
        // subtraction is >= the subtrahend in every lane (no borrow)
        lo = lo + h_in[yy * kHStride] - h_in[(yy - 2 * R - 1) * kHStride];
      } else if (KIND == 0) {
        // R += H(y + r) - H(y - r - 1): a biased byte difference (31..97), widened
        const uint32_t d = h_in[yy * kHStride] + 0x40404040u - h_in[(yy - 2 * R - 1) * kHStride];
        lo += widen_lo(d) - 0x00400040u;
        hi += widen_hi(d) - 0x00400040u;
      } else {
        lo += *reinterpret_cast<const uint32_t*>(c_mid + (yy + R) * kTileW) -
              *reinterpret_cast<const uint32_t*>(c_mid + (yy - R - 1) * kTileW);
      }
    }
    const uint32_t st = *reinterpret_cast<const uint32_t*>(c_mid + yy * kTileW);
    uint32_t nw;
    if constexpr (kByte) {
      // Z = R + 64 state in byte lanes (R < 64): Moore R = lo, VN R = H + V
      const uint32_t zb = (KIND == 0 ? lo : h_mid[yy * kHStride] + lo) + st * kByteK;
      nw = br.next4(zb);
      if constexpr (kChecked) {
        max_r = __vmaxu4(max_r, zb & ((kByteK - 1) * 0x01010101u) & rmask_b);
        bad |= br.negative(zb) & rmask_b;
      }
    } else {
      uint32_t zl, zh;
      if (KIND == 0) {
        zl = lo + (widen_lo(st) << 11);
        zh = hi + (widen_hi(st) << 11);
      } else {  // R = H + V (centre twice), + 128 * state: all < 256 in byte lanes
        const uint32_t zb = h_mid[yy * kHStride] + lo + (st << 7);
        zl = widen_lo(zb);
        zh = widen_hi(zb);
      }
      nw = next_word(sr.pair(zl), sr.pair(zh));
      if constexpr (kChecked) {
        max_r = __vmaxu2(max_r, zl & sr.r_mask & rmask_lo);
        max_r = __vmaxu2(max_r, zh & sr.r_mask & rmask_hi);
        bad |= (sr.negative(zl) & rmask_lo) | (sr.negative(zh) & rmask_hi);
      }
    }
    if (full_word) *reinterpret_cast<uint32_t*>(optr + yy * kStrip) = nw;
    else if (x < in.cols) store_word(out, y0 + ys + yy, x, nw);
  };
  if (nrows == kSeg && full_word) {  // the common case: a whole segment, whole words
#pragma unroll
    for (int yy = 0; yy < kSeg; ++yy) row(yy);
  } else {
    for (int yy = 0; yy < nrows; ++yy) row(yy);
  }
  if constexpr (kChecked) {
    // byte-lane R maxima -> the 16-bit layout flush_stats reduces
    if (kByte) max_r = max(max(max_r & 0xFF, (max_r >> 8) & 0xFF), max((max_r >> 16) & 0xFF, max_r >> 24));
    flush_stats(stats, max_h, max_r, bad);
  }
}

template <int R>
constexpr size_t pack_smem_bytes() {
  return 16 + static_cast<size_t>(kPackTY + 2 * kHalo) * kTileW +
         static_cast<size_t>(kPackTY + 2 * R) * kHStride * sizeof(uint32_t);
}

template <int R>
cudaError_t launch_r(const SlabView& in, const SlabView& out, const RuleConsts& rc, int engine,
                     DeviceStats* stats, cudaStream_t stream) {
  const int strips = interior_strips(in.cols);
  const int ty = engine == kEnginePack ? kPackTY : kBaseTY;
  const dim3 grid(strips, (in.rows + ty - 1) / ty);
  // CTAs per SM: with the cp.async tile loads as many as the SMEM allows
  // (same-box A/B at 32768^2, tools/gpu_r02ao.sh: pack r = 1 with five CTAs
  // 2.84e12 vs four 2.73e12 vs three 2.45e12; base r = 1 with seven 2.24e12
  // vs five 2.12e12).  The register-staged loads of round 1 wanted caps (the
  // fifth pack CTA's tile stores flooded the shared-memory instruction queue);
  // the A/B knobs stay.
  size_t smem = engine == kEnginePack ? pack_smem_bytes<R>() : 0;
  if (engine == kEnginePack)
    if (const char* e = std::getenv("LTL_PACK_MIN_SMEM"))  // A/B: CTAs per SM
      smem = std::max<size_t>(pack_smem_bytes<R>(), static_cast<size_t>(std::atol(e)));
  if (engine == kEngineBase)
    if (const char* e = std::getenv("LTL_BASE_PAD_SMEM"))  // A/B: CTAs per SM
      smem = static_cast<size_t>(std::atol(e));
  if (smem > 48 * 1024) {
    // the attribute is per device: set on each when a launch needs more than
    // it was set to (a per-launch call serialises launches measurably)
    static size_t set_to[64] = {};
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    if (dev < 0 || dev >= 64) return cudaErrorInvalidDevice;
    if (set_to[dev] < smem) {
      for (auto fn : {pack_kernel<R, 0, true>, pack_kernel<R, 0, false>, pack_kernel<R, 1, true>,
                      pack_kernel<R, 1, false>}) {
        e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 static_cast<int>(smem));
        if (e != cudaSuccess) return e;
      }
      set_to[dev] = smem;
    }
  }
#define LTL_STENCIL_LAUNCH(KERNEL, KIND)                                                   \
  (stats ? KERNEL<R, KIND, true><<<grid, kThreads, smem, stream>>>(in, out, rc, stats)     \
         : KERNEL<R, KIND, false><<<grid, kThreads, smem, stream>>>(in, out, rc, nullptr))
  if (engine == kEnginePack) {
    if (rc.kind == 0) LTL_STENCIL_LAUNCH(pack_kernel, 0);
    else LTL_STENCIL_LAUNCH(pack_kernel, 1);
  } else {
    if (rc.kind == 0) LTL_STENCIL_LAUNCH(base_kernel, 0);
    else LTL_STENCIL_LAUNCH(base_kernel, 1);
  }
#undef LTL_STENCIL_LAUNCH
  return cudaGetLastError();
}

template <int... Rs>
cudaError_t dispatch(std::integer_sequence<int, Rs...>, int r, const SlabView& in,
                     const SlabView& out, const RuleConsts& rc, int engine, DeviceStats* stats,
                     cudaStream_t stream) {
  cudaError_t e = cudaErrorInvalidValue;
  ((r == Rs + 1 ? (e = launch_r<Rs + 1>(in, out, rc, engine, stats, stream), 0) : 0), ...);
  return e;
}

}  // namespace

cudaError_t launch_stencil_step(const SlabView& in, const SlabView& out, const RuleConsts& rule,
                                int engine, DeviceStats* stats, cudaStream_t stream) {
  if (in.rows <= 0 || in.cols <= 0) return cudaSuccess;
  if (engine != kEngineBase && engine != kEnginePack) return cudaErrorInvalidValue;
  return dispatch(std::make_integer_sequence<int, kHalo>{}, rule.r, in, out, rule, engine, stats,
                  stream);
}

}  // namespace ltl
