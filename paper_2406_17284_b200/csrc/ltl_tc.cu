// ltl_tc.cu -- one Larger-than-Life generation as two banded tcgen05 MMAs.
//
// Replaces the reference hot path src/cat_engine.cpp:260-306 (simulate_step:
// horizontal_step :123-161, vertical_step_moore :163-208,
// vertical_step_von_neumann :210-258, rule loop :293-303).  The reference
// restates the paper's method with 16x16 int32 fragments and three band
// fragments pi1/pi2/pi3 (src/fragment.cpp:23-41).  Here the same banded
// products run on the 5th-generation tensor cores in their native shapes:
//
//   tile     a 128-column strip of the slab, streamed down in 64-row chunks
//   pass 1   D1[x][y] = sum_k A1[x][k] * X[y][k]            tcgen05.mma kind::i8
//            A1 = 128 x 160 band, resident in SMEM; X = TMA-loaded 64 x 160
//            chunk (K-major, SWIZZLE_32B); M = 128 (x), N = 64 (y), K = 5 x 32.
//            A1[x][k] = [|k-16-x| <= r] + 128*[k == x+16]: the extra 128 on
//            the centre carries the cell state out in bit 7 (H <= 33 < 128).
//   convert  epilogue: D1 (s32 in TMEM) -> two byte planes written back into
//            TMEM as K-major A operands of pass 2 (no SMEM round trip):
//              Moore: H = D1 & 0x7F and S = D1 & 0x80 (state * 128)
//              VN   : H' = D1 (= H + 128*state) and s = state
//   pass 2   D2[x][j] = sum over the 96 H rows around output chunk c
//              Moore: H*Bv + S*(16*Iv)  = R_box   + 2048*state
//              VN   : H'*Iv + s*Bv      = R_cross + 128*state
//            6 MMAs (A from TMEM, band B from SMEM).  Folding the state into
//            the accumulator makes the birth/survival rule (apply_transition,
//            src/rule.cpp:99-111) a pure function of one 12-bit number Z.
//   rule     Z is read back two cells per register (16-bit lanes); the two
//            range tests (dead: b1..b2, live: K+s1'..K+s2') are four biased
//            adds and two LOP3s per register (bit 15 of each lane = result).
//   store    the D2 columns are permuted (out_row_of_col) so that
//            stmatrix.trans writes each 16x256b TMEM fragment straight into a
//            row-major SWIZZLE_32B 32x32 staging tile per warp -> TMA store of
//            the next generation (no CTA-wide barrier on the output path).
//
// Every quantity is an exact small integer (H <= 33, R <= 1089, Z < 4096), so
// the result is bit-identical to the reference's int32 loops.
//
// One persistent CTA per SM (all 512 TMEM columns), 15 warps:
//   warp 0        TMA producer            warp 1   pass-1 MMA issuer, TMEM owner
//   warps 2..5    convert D1 (warp w: TMEM lane quarter w%4 = 32 strip columns)
//   warps 6..13   rule + store D2 (quarter w%4, 32 of the 64 chunk rows each)
//   warp 14       pass-2 MMA issuer
// Every stage hands over through mbarrier rings, so TMA, both MMA passes and
// both epilogue groups overlap across chunks.
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>

#include "ltl_kernels.cuh"
#include "ptx_sm100.cuh"

namespace ltl {
namespace {

using namespace ptx;

constexpr int kStripCols = 128;  // M of both MMAs = output columns per strip
constexpr int kRows = 64;        // N of both MMAs = rows per chunk
constexpr int kKTile = 160;      // 128 + 2*16 input columns per strip
constexpr int kKChunks = kKTile / 32;
constexpr int kXStages = 10;  // 10 KB each: ~100 KB of loads in flight per SM
constexpr int kA2Slots = 4;
constexpr int kD1Slots = 2;
constexpr int kD2Slots = 2;
constexpr int kConvWarps = 4;
constexpr int kOutWarps = 8;
constexpr int kThreads = 32 * (3 + kConvWarps + kOutWarps);  // 480
constexpr int kConvThreads = 32 * kConvWarps;
constexpr int kOutThreads = 32 * kOutWarps;
constexpr int kWarpP2 = 2 + kConvWarps + kOutWarps;  // 14
constexpr int kNumBands = 9;  // Bv_j, Iv_j, 16*Iv_j for the 3 K chunks of pass 2

// Shared-memory carve-up (offsets from a 1024-aligned base).
constexpr uint32_t kSmemA1 = 0;                                    // 5 x 128 x 32 B
constexpr uint32_t kBandBytes = kRows * 32;                        // 2 KB: [64 n][32 k]
constexpr uint32_t kSmemBand = kSmemA1 + kKChunks * 128 * 32;      // 9 x 2 KB
constexpr uint32_t kSmemX = kSmemBand + kNumBands * kBandBytes;    // kXStages x 10 KB
constexpr uint32_t kXChunkBytes = kRows * 32;                      // one 32-column box
constexpr uint32_t kXStageBytes = kKChunks * kXChunkBytes;         // 10240
constexpr uint32_t kSmemStage = kSmemX + kXStages * kXStageBytes;  // 8 warps x 2 x 1 KB
constexpr uint32_t kSmemBars = kSmemStage + kOutWarps * 2 * 1024;
constexpr uint32_t kNumBars = 2 * (kXStages + kD1Slots + kA2Slots + kD2Slots);
constexpr uint32_t kSmemTotal = kSmemBars + kNumBars * 8 + 16;
constexpr uint32_t kSmemAlloc = kSmemTotal + 1024;  // alignment slack
static_assert(kSmemAlloc <= 227 * 1024, "shared memory budget");

// TMEM columns: the whole 512 of the SM.
constexpr uint32_t kTmemCols = 512;
constexpr uint32_t kTmemD1 = 0;    // kD1Slots x 64
constexpr uint32_t kTmemD2 = 128;  // kD2Slots x 64
constexpr uint32_t kTmemA2 = 256;  // kA2Slots x 32 (plane 0 at +0, plane 1 at +16)

constexpr uint32_t kIdesc = idesc_i8_u8u8_s32(128, kRows);

struct Params {
  int32_t rows, cols;
  int32_t num_strips, chunks;  // strips of 128 columns, 64-row chunks per strip
  int32_t segs;                // row segments per strip (units = num_strips * segs)
  RuleConsts rule;
  int32_t inject_fault;
  DeviceStats* stats;
  long long* trace;  // debug timeline of CTA 0 (only with -DLTL_TC_TRACE_BUILD)
  uint32_t* pace;    // 65 words of zeroed global memory, or nullptr (pacing off)
};

// Soft pacing of the CTAs' TMA producers.  Streaming strips runs near the HBM
// copy rate only while every CTA reads the same rows at the same time (DRAM
// page / TLB locality, tools/ubench_stream2.cu); small per-SM speed
// differences otherwise accumulate into drift over hundreds of chunks.  Every
// kPaceEvery H chunks a producer publishes its epoch and waits (bounded) until
// all CTAs have reached epoch - kPaceWindow.  It is only a hint: a wait that
// exceeds kPaceTimeout cycles disables pacing for that CTA, so co-residency is
// never required for correctness.
constexpr int kPaceEvery = 8;
constexpr int kPaceWindow = 2;
constexpr long long kPaceTimeout = 400000;  // ~200 us

__device__ __forceinline__ bool pace(uint32_t* pace_buf, uint32_t g) {
  const uint32_t epoch = g / kPaceEvery;
  atomicAdd(pace_buf + epoch % 64, 1u);
  if (epoch < kPaceWindow) return true;
  const uint32_t e = epoch - kPaceWindow;
  const uint32_t need = gridDim.x * (e / 64 + 1);
  volatile uint32_t* slot = pace_buf + e % 64;
  const long long t0 = clock64();
  while (*slot < need) {
    if (clock64() - t0 > kPaceTimeout) return false;
    __nanosleep(256);
  }
  return true;
}

__device__ __forceinline__ void pace_reset(uint32_t* pace_buf) {
  // last CTA out zeroes the slots for the next launch (stream-ordered)
  __threadfence();
  if (atomicAdd(pace_buf + 64, 1u) == gridDim.x - 1) {
    for (int i = 0; i < 65; ++i) pace_buf[i] = 0;
    __threadfence();
  }
}

#ifdef LTL_TC_TRACE_BUILD
#define LTL_TRACE(ev, idx) \
  do { if (p.trace && blockIdx.x == 0 && (idx) < 64) p.trace[(ev) * 64 + (idx)] = clock64(); } while (0)
#else
#define LTL_TRACE(ev, idx) do { } while (0)
#endif

// Static schedule.  A unit is (strip, row segment); unit u is strip u % S,
// segment u / S, and CTA b walks units b, b + G, b + 2G, ...  The host picks
// segs and G so that every CTA gets the same work (G = S * segs, or several
// whole strips each when S exceeds the CTA slots).  Consecutive CTAs then
// stream neighbouring strips down the same rows at the same time, so the
// 32 overlapping halo columns and the 256-byte L2 promotion of each strip's
// loads are shared through L2 instead of being fetched twice from HBM.
// Every role of the CTA iterates the same units in the same order.
struct UnitIter {
  int32_t u;
  const Params& p;
  __device__ explicit UnitIter(const Params& pp) : u(blockIdx.x), p(pp) {}
  __device__ bool next(int& strip, int& c0, int& nc) {
    if (u >= p.num_strips * p.segs) return false;
    strip = u % p.num_strips;
    const int seg = u / p.num_strips;
    c0 = static_cast<int>(static_cast<int64_t>(p.chunks) * seg / p.segs);
    nc = static_cast<int>(static_cast<int64_t>(p.chunks) * (seg + 1) / p.segs) - c0;
    u += gridDim.x;
    return true;
  }
};

// D2 column j holds chunk row out_row_of_col(j).  Within each 32-column half,
// with j = [e, m, a0, a1, v] (bit 0 first) the row is [e, a0, a1, m, v]: the
// stmatrix fragment of column group (m, v) of a 16x256b load then covers the 8
// consecutive rows 8*(m + 2v) .. +7 of that half.
__host__ __device__ constexpr int out_row_of_col(int j) {
  return (j & 32) | (j & 1) | (((j >> 2) & 3) << 1) | (((j >> 1) & 1) << 3) | (j & 16);
}

__device__ __forceinline__ uint32_t pack_pairs(uint32_t p0, uint32_t p1) {
  return __byte_perm(p0, p1, 0x6420);  // low bytes of four 16-bit lanes
}

// Two cells per register: lanes hold Z = R + K*state (< 4096).  Bit 15 (31)
// of the result is the next state of the low (high) cell.
struct SimdRule {
  uint32_t ca, cb, cc, cd;
};

__device__ __forceinline__ uint32_t rule_pair(uint32_t z, const SimdRule& k) {
  const uint32_t a = z + k.ca;  // Z >= b1
  const uint32_t b = z + k.cb;  // Z >  b2
  const uint32_t c = z + k.cc;  // Z >= K + s1'
  const uint32_t d = z + k.cd;  // Z >  K + s2'
  const uint32_t e = lop3<0xBA>(a, b, c);  // (a & ~b) | c
  return lop3<0x70>(e, c, d);             // e & ~(c & d)
}

template <bool kChecked>
__global__ void __launch_bounds__(kThreads, 1)
    ltl_tc_step_kernel(const __grid_constant__ CUtensorMap load_map,
                       const __grid_constant__ CUtensorMap store_map, const Params p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + kSmemBars);
  uint64_t* x_full = bars;
  uint64_t* x_empty = x_full + kXStages;
  uint64_t* d1_full = x_empty + kXStages;
  uint64_t* d1_empty = d1_full + kD1Slots;
  uint64_t* a2_full = d1_empty + kD1Slots;
  uint64_t* a2_empty = a2_full + kA2Slots;
  uint64_t* d2_full = a2_empty + kA2Slots;
  uint64_t* d2_empty = d2_full + kD2Slots;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(d2_empty + kD2Slots);

  const uint32_t warp = warp_id();
  const uint32_t lane = threadIdx.x & 31;
  const int r = p.rule.r;
  const bool vn = p.rule.kind != 0;

  // ---- one-time setup: resident bands (generic-proxy writes), barriers, TMEM
  // (built a 32-bit word -- 4 consecutive k -- at a time; the swizzle moves
  // whole 16-byte chunks, so a word stays contiguous)
  for (uint32_t w = threadIdx.x; w < 128u * kKTile / 4; w += kThreads) {
    const int m = static_cast<int>(w / (kKTile / 4)), k0 = 4 * static_cast<int>(w % (kKTile / 4));
    uint32_t word = 0;
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      const int d = k0 + b - 16 - m;
      uint32_t v = (d >= -r && d <= r) ? 1u : 0u;
      if (d == 0) {
        v += 128u;  // state marker
        if (p.inject_fault && m == 0) v = 128u;  // test hook: drop one centre entry
      }
      word |= v << (8 * b);
    }
    *reinterpret_cast<uint32_t*>(smem + kSmemA1 + (k0 / 32) * 4096 + sw32_offset(m, k0 % 32)) =
        word;
  }
  // pass-2 B tiles [64 n][32 k]: tile t = kind * 3 + j, K chunk j covers rows
  // 32j .. 32j+31 of the 96-row H window; output row rho sits at window row 16 + rho
  for (uint32_t w = threadIdx.x; w < kNumBands * kRows * 8u; w += kThreads) {
    const int t = static_cast<int>(w / (kRows * 8)), j = static_cast<int>((w / 8) % kRows),
              k0 = 4 * static_cast<int>(w % 8);
    const int kind = t / 3, kc = t % 3;
    const int rho = out_row_of_col(j);
    uint32_t word = 0;
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      const int d = 32 * kc + k0 + b - 16 - rho;  // window row - centre row
      int v;
      if (kind == 0) v = (d >= -r && d <= r);      // band
      else if (kind == 1) v = (d == 0);            // centre
      else v = 16 * (d == 0);                      // 16 * centre (state * 2048)
      word |= static_cast<uint32_t>(v) << (8 * b);
    }
    *reinterpret_cast<uint32_t*>(smem + kSmemBand + t * kBandBytes + sw32_offset(j, k0)) = word;
  }
  fence_proxy_async_smem();
  if (warp == 0 && lane == 0) {
    prefetch_tmap(&load_map);
    prefetch_tmap(&store_map);
    for (int i = 0; i < kXStages; ++i) {
      mbar_init(&x_full[i], 1);
      mbar_init(&x_empty[i], 1);
    }
    for (int i = 0; i < kD1Slots; ++i) {
      mbar_init(&d1_full[i], 1);
      mbar_init(&d1_empty[i], kConvThreads);
    }
    for (int i = 0; i < kA2Slots; ++i) {
      mbar_init(&a2_full[i], kConvThreads);
      mbar_init(&a2_empty[i], 1);
    }
    for (int i = 0; i < kD2Slots; ++i) {
      mbar_init(&d2_full[i], 1);
      mbar_init(&d2_empty[i], kOutThreads);
    }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc(tmem_slot, kTmemCols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  // Everything above only touched this CTA's SMEM/TMEM, so it overlapped the
  // previous kernel's tail (PDL).  The grid is read from here on.
  pdl_launch_dependents();
  pdl_wait_prerequisites();

  if (warp == 0) {
    // ================= TMA producer =================
    if (elect_one()) {
      uint32_t g = 0;
      bool pacing = p.pace != nullptr;
      UnitIter it(p);
      int strip, c0, nc;
      while (it.next(strip, c0, nc)) {
        for (int k = 0; k <= nc; ++k, ++g) {
          const uint32_t s = g % kXStages;
          mbar_wait(&x_empty[s], ((g / kXStages) & 1) ^ 1);
          if (pacing && g % kPaceEvery == 0) pacing = pace(p.pace, g);
          LTL_TRACE(0, g);
          uint8_t* dst = smem + kSmemX + s * kXStageBytes;
          mbar_arrive_expect_tx(&x_full[s], kXStageBytes);
#pragma unroll
          for (int q = 0; q < kKChunks; ++q)
            tma_load_2d(dst + q * kXChunkBytes, &load_map, &x_full[s],
                        strip * kStripCols + 32 * q, (c0 + k) * kRows);
        }
      }
      if (p.pace) pace_reset(p.pace);
    }
  } else if (warp == 1) {
    // ================= pass-1 MMA issuer =================
    const uint64_t a1_desc = smem_desc_sw32_kmajor(smem_u32(smem + kSmemA1));
    const uint64_t x_desc = smem_desc_sw32_kmajor(smem_u32(smem + kSmemX));
    uint32_t g = 0;
    UnitIter it(p);
    int strip, c0, nc;
    while (it.next(strip, c0, nc)) {
      for (int k = 0; k <= nc; ++k, ++g) {
        const uint32_t s = g % kXStages, d1 = g % kD1Slots;
        mbar_wait(&x_full[s], (g / kXStages) & 1);
        mbar_wait(&d1_empty[d1], ((g / kD1Slots) & 1) ^ 1);
        LTL_TRACE(1, g);
        tc_fence_after();
        if (elect_one()) {
          const uint64_t xd = x_desc + ((s * kXStageBytes) >> 4);
#pragma unroll
          for (int q = 0; q < kKChunks; ++q)
            mma_i8_ss(tmem + kTmemD1 + kRows * d1, a1_desc + ((q * 4096) >> 4),
                      xd + ((q * kXChunkBytes) >> 4), kIdesc, q > 0);
          mma_commit(&x_empty[s]);
          mma_commit(&d1_full[d1]);
        }
        __syncwarp();
      }
    }
  } else if (warp < 2 + kConvWarps) {
    // ================= convert warps (D1 -> pass-2 A planes) =================
    const uint32_t q = warp & 3;  // TMEM lane quarter = 32 strip columns
    const uint32_t trow = tmem + ((q * 32) << 16);
    uint32_t max_h = 0, g = 0;
    UnitIter it(p);
    int strip, c0, nc;
    while (it.next(strip, c0, nc)) {
      for (int k = 0; k <= nc; ++k, ++g) {
        const uint32_t d1 = g % kD1Slots, s = g % kA2Slots;
        mbar_wait(&d1_full[d1], (g / kD1Slots) & 1);
        tc_fence_after();
        uint32_t v[32];
        tmem_ld_32x32b_x32_pack16(trow + kTmemD1 + kRows * d1, v);
        tmem_ld_wait();
        tc_fence_before();
        mbar_arrive(&d1_empty[d1]);
        uint32_t plane0[16], plane1[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          const uint32_t raw = pack_pairs(v[2 * j], v[2 * j + 1]);  // 4 rows of H + 128*state
          if (vn) {
            plane0[j] = raw;
            plane1[j] = (raw >> 7) & 0x01010101u;
          } else {
            plane0[j] = raw & 0x7F7F7F7Fu;
            plane1[j] = raw & 0x80808080u;
          }
          if constexpr (kChecked) max_h = __vmaxu4(max_h, raw & 0x7F7F7F7Fu);
        }
        mbar_wait(&a2_empty[s], ((g / kA2Slots) & 1) ^ 1);
        tc_fence_after();
        tmem_st_32x32b_x16(trow + kTmemA2 + 32 * s, plane0);
        tmem_st_32x32b_x16(trow + kTmemA2 + 32 * s + 16, plane1);
        tmem_st_wait();
        tc_fence_before();
        mbar_arrive(&a2_full[s]);
      }
    }
    if constexpr (kChecked) {
      int32_t mh = static_cast<int32_t>(max(max(max_h & 0xFF, (max_h >> 8) & 0xFF),
                                            max((max_h >> 16) & 0xFF, max_h >> 24)));
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) mh = max(mh, __shfl_xor_sync(0xffffffffu, mh, off));
      if (lane == 0) atomicMax(&p.stats->max_h, mh);
    }
  } else if (warp == kWarpP2) {
    // ================= pass-2 MMA issuer =================
    // K chunk j of the 96-row window: H chunk c rows 0..31 (j=0), 32..63 (j=1),
    // H chunk c+1 rows 0..31 (j=2) = TMEM column offsets +0, +8, next slot +0.
    const uint64_t band_desc = smem_desc_sw32_kmajor(smem_u32(smem + kSmemBand));
    auto tile = [&](int t) { return band_desc + ((t * kBandBytes) >> 4); };
    // plane 0 pairs with band (Moore) / centre (VN); plane 1 with 16*centre / band
    const int t_p0 = vn ? 3 : 0, t_p1 = vn ? 0 : 6;
    uint32_t g = 0, o = 0;
    UnitIter it(p);
    int strip, c0, nc;
    while (it.next(strip, c0, nc)) {
      for (int c = 0; c < nc; ++c, ++o) {
        const uint32_t gg = g + c;
        const uint32_t s0 = gg % kA2Slots, s1 = (gg + 1) % kA2Slots, d2 = o % kD2Slots;
        mbar_wait(&a2_full[s0], (gg / kA2Slots) & 1);
        mbar_wait(&a2_full[s1], ((gg + 1) / kA2Slots) & 1);
        mbar_wait(&d2_empty[d2], ((o / kD2Slots) & 1) ^ 1);
        LTL_TRACE(4, o);
        tc_fence_after();
        if (elect_one()) {
          const uint32_t dcol = tmem + kTmemD2 + kRows * d2;
          const uint32_t a0 = tmem + kTmemA2 + 32 * s0, a1 = tmem + kTmemA2 + 32 * s1;
          mma_i8_ts(dcol, a0, tile(t_p0 + 0), kIdesc, 0);
          mma_i8_ts(dcol, a0 + 8, tile(t_p0 + 1), kIdesc, 1);
          mma_i8_ts(dcol, a1, tile(t_p0 + 2), kIdesc, 1);
          mma_i8_ts(dcol, a0 + 16, tile(t_p1 + 0), kIdesc, 1);
          mma_i8_ts(dcol, a0 + 24, tile(t_p1 + 1), kIdesc, 1);
          mma_i8_ts(dcol, a1 + 16, tile(t_p1 + 2), kIdesc, 1);
          mma_commit(&d2_full[d2]);
          mma_commit(&a2_empty[s0]);
          // the unit's final H chunk is only ever the second operand: free it too
          if (c == nc - 1) mma_commit(&a2_empty[s1]);
        }
        __syncwarp();
      }
      g += nc + 1;
    }
  } else {
    // ================= output warps (D2 -> rule -> next generation) ==========
    // Warp w owns strip columns 32*(w%4)..+32 and chunk rows 32*half..+32 (its
    // own staging slots and TMA stores: no CTA-wide barrier on this path).
    const uint32_t q = warp & 3;
    const uint32_t half = (warp - (2 + kConvWarps)) >> 2;
    const uint32_t trow = tmem + ((q * 32) << 16) + 32 * half;
    const RuleConsts rc = p.rule;
    const uint32_t K = vn ? 128u : 2048u;
    SimdRule sr;
    sr.ca = (0x8000u - rc.lo_dead) * 0x10001u;
    sr.cb = (0x7FFFu - (rc.lo_dead + rc.w_dead)) * 0x10001u;
    sr.cc = (0x8000u - (K + rc.lo_live)) * 0x10001u;
    sr.cd = (0x7FFFu - (K + rc.lo_live + rc.w_live)) * 0x10001u;
    const uint32_t g_live = (0x8000u - K) * 0x10001u;
    const uint32_t g_neg = (0x8000u - (K + rc.neg_live)) * 0x10001u;
    const uint32_t r_mask = (K - 1) * 0x10001u;
    uint32_t max_r = 0, bad = 0;
    // staging: per warp 2 slots of [32 rows][32 B], SWIZZLE_32B (16-byte
    // chunk ^= (row >> 2) & 1); this thread addresses row `lane`.
    const uint32_t wslot = warp - (2 + kConvWarps);
    uint8_t* my_stage = smem + kSmemStage + wslot * 2048;
    const uint32_t stage_u32 = smem_u32(my_stage);
    const uint32_t addr_h0 = lane * 32 + ((0u ^ ((lane >> 2) & 1)) << 4);
    const uint32_t addr_h1 = lane * 32 + ((1u ^ ((lane >> 2) & 1)) << 4);
    uint32_t o = 0;
    UnitIter it(p);
    int strip, c0, nc;
    while (it.next(strip, c0, nc)) {
      for (int c = 0; c < nc; ++c, ++o) {
        const uint32_t d2 = o % kD2Slots, slot = o & 1;
        mbar_wait(&d2_full[d2], (o / kD2Slots) & 1);
        tc_fence_after();
        uint32_t z0[8], z1[8];
        tmem_ld_16x256b_x2_pack16(trow + kTmemD2 + kRows * d2, z0);
        tmem_ld_16x256b_x2_pack16(trow + (16u << 16) + kTmemD2 + kRows * d2, z1);
        tmem_ld_wait();
        tc_fence_before();
        mbar_arrive(&d2_empty[d2]);
        uint32_t w0[4], w1[4];
#pragma unroll
        for (int v = 0; v < 2; ++v) {
          const uint32_t a0 = rule_pair(z0[4 * v + 0], sr), b0 = rule_pair(z0[4 * v + 1], sr);
          const uint32_t a2 = rule_pair(z0[4 * v + 2], sr), b2 = rule_pair(z0[4 * v + 3], sr);
          w0[2 * v + 0] = prmt(a0, a2, 0xFDB9) & 0x01010101u;
          w0[2 * v + 1] = prmt(b0, b2, 0xFDB9) & 0x01010101u;
          const uint32_t c0r = rule_pair(z1[4 * v + 0], sr), d0r = rule_pair(z1[4 * v + 1], sr);
          const uint32_t c2r = rule_pair(z1[4 * v + 2], sr), d2r = rule_pair(z1[4 * v + 3], sr);
          w1[2 * v + 0] = prmt(c0r, c2r, 0xFDB9) & 0x01010101u;
          w1[2 * v + 1] = prmt(d0r, d2r, 0xFDB9) & 0x01010101u;
        }
        if constexpr (kChecked) {
#pragma unroll
          for (int i = 0; i < 8; ++i) {
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              const uint32_t z = h ? z1[i] : z0[i];
              max_r = __vmaxu2(max_r, z & r_mask);
              bad |= (z + g_live) & ~(z + g_neg) & 0x80008000u;  // live and count < 0
            }
          }
        }
        // this warp's staging slot was last read by its TMA store of chunk o-2
        if (lane == 0) tma_store_wait_read<1>();
        __syncwarp();
        const uint32_t sa = stage_u32 + slot * 1024;
        stmatrix_x4_trans_b8(sa + addr_h0, w0[0], w0[1], w0[2], w0[3]);
        stmatrix_x4_trans_b8(sa + addr_h1, w1[0], w1[1], w1[2], w1[3]);
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) {
          tma_store_2d(&store_map, my_stage + slot * 1024, strip * kStripCols + 32 * q,
                       (c0 + c) * kRows + 32 * half);
          tma_store_commit();
          if (warp == 2 + kConvWarps) LTL_TRACE(11, o);
        }
      }
    }
    if (lane == 0) tma_store_wait_all<0>();
    if constexpr (kChecked) {
      int32_t mr = static_cast<int32_t>(max(max_r & 0xFFFF, max_r >> 16));
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) mr = max(mr, __shfl_xor_sync(0xffffffffu, mr, off));
      if (lane == 0) atomicMax(&p.stats->max_r, mr);
      if (__any_sync(0xffffffffu, bad != 0) && lane == 0) atomicOr(&p.stats->error, 1);
    }
  }

  __syncwarp();
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc(tmem, kTmemCols);
}

}  // namespace

size_t tc_smem_bytes() { return kSmemAlloc; }

cudaError_t launch_tc_step(const TcLaunch& a, cudaStream_t stream) {
  static int num_sms = 0;
  if (num_sms == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&num_sms, cudaDevAttrMultiProcessorCount, dev);
    for (auto fn : {ltl_tc_step_kernel<false>, ltl_tc_step_kernel<true>}) {
      cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           static_cast<int>(kSmemAlloc));
      if (e != cudaSuccess) return e;
    }
  }
  if (a.rows <= 0 || a.cols <= 0) return cudaSuccess;
  Params p{};
  p.rows = a.rows;
  p.cols = a.cols;
  p.num_strips = (a.cols + kStripCols - 1) / kStripCols;
  p.chunks = (a.rows + kRows - 1) / kRows;
  p.rule = a.rule;
  p.inject_fault = a.inject_fault;
  p.stats = a.stats;
  p.trace = a.trace;
  p.pace = a.pace;
  if (std::getenv("LTL_TC_NO_PACE")) p.pace = nullptr;
  // Balanced units (UnitIter).  Measured on B200 (tools/ubench_stream2.cu,
  // profiles/): streaming whole strips with every CTA on the same rows and the
  // in-flight strips covering an aligned power-of-two span of each row runs
  // at ~4.7-5 TB/s, while 148 concurrent strips (an unaligned 148/256 of the
  // row) or many short segments drop to ~2.6-3.1 TB/s.  So for wide grids
  // (S >= 64 strips) use the largest divisor G of S with G <= SMs, one whole
  // strip per unit (CTA b streams strips b, b + G, ...).  Small grids split
  // strips into row segments to fill the GPU.
  const int slots = num_sms;
  const int S = p.num_strips;
  int64_t grid;
  int wide_grid = 0;
  if (S >= 64)
    for (int g = slots; g >= 1; --g)
      if (S % g == 0) {
        wide_grid = g;
        break;
      }
  if (wide_grid >= slots / 2) {
    p.segs = 1;
    grid = wide_grid;
  } else if (S <= slots) {
    int segs = slots / S;
    const int max_segs = p.chunks / 2 > 1 ? p.chunks / 2 : 1;
    if (segs > max_segs) segs = max_segs;
    p.segs = segs;
    grid = static_cast<int64_t>(S) * segs;
  } else {
    p.segs = 1;
    const int per_cta = (S + slots - 1) / slots;
    grid = (S + per_cta - 1) / per_cta;
  }
  if (a.grid > 0 && a.grid < grid) grid = a.grid;
  // tuning knobs (benchmark sweeps only): LTL_TC_SEGS=<segments per strip>,
  // LTL_TC_GRID=<CTAs>
  if (const char* e = std::getenv("LTL_TC_SEGS")) {
    const int v = std::atoi(e);
    if (v >= 1 && v <= p.chunks) {
      p.segs = v;
      grid = static_cast<int64_t>(S) * v;
      if (grid > slots) grid = slots;
    }
  }
  if (const char* e = std::getenv("LTL_TC_GRID")) {
    const int v = std::atoi(e);
    if (v >= 1 && v <= slots) grid = v;
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(static_cast<unsigned>(grid));
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = kSmemAlloc;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  if (a.stats)
    return cudaLaunchKernelEx(&cfg, ltl_tc_step_kernel<true>, *a.load_map, *a.store_map, p);
  return cudaLaunchKernelEx(&cfg, ltl_tc_step_kernel<false>, *a.load_map, *a.store_map, p);
}

}  // namespace ltl
