// ltl_tc.cu -- one Larger-than-Life generation as two banded tcgen05 MMAs.
//
// Replaces the reference hot path src/cat_engine.cpp:260-306 (simulate_step:
// horizontal_step :123-161, vertical_step_moore :163-208,
// vertical_step_von_neumann :210-258, rule loop :293-303).  The reference
// restates the paper's method with 16x16 int32 fragments and three band
// fragments pi1/pi2/pi3 (src/fragment.cpp:23-41).  Here the same banded
// products run on the 5th-generation tensor cores in their native shapes, over
// the strip-contiguous slab layout of ltl_kernels.cuh.
//
// Design rule (measured, tools/ubench_mma.cu, profiles/): every tcgen05.mma
// costs >= ~85 SM cycles whatever its N up to 128 (any kind); only N = 256
// reaches the tensor peak.  So the step is organised to issue as FEW, as WIDE
// MMAs as TMEM allows -- 16 per 128 x 128 output tile:
//
//   unit     (band, strip): output rows [128 b, 128 b + 128) x the 128
//            columns of strip t.  A CTA walks runs of consecutive strips of
//            one band (SegIter: per-launch segments, or the multi-generation
//            sweep).
//   box      one TMA load per unit: padded rows [128 b, 128 b + 160) of
//            strip t = ONE contiguous 20 KB block (SWIZZLE_128B).  The 16 halo
//            rows above and below come with it; the 16 halo columns on each
//            side are the previous / next box, still resident in SMEM.
//   pass 1   D1[x][y] = sum_k A1[x][k] * X[y][k]        6 x tcgen05.mma kind::i8
//            M = 128 (x), N = 160 (all box rows), K = 6 x 32 = columns
//            [-32, 160) of the strip (box t-1 chunk 3, box t chunks 0..3,
//            box t+1 chunk 0).  A1[x][k] = [|k-32-x| <= r] + 128*[k == x+32],
//            resident in TMEM: the row window sums (the reference's H) with
//            the cell state in bit 7 (H <= 33 < 128).
//   convert  D1 (s32 in TMEM) -> two byte planes written back into TMEM as
//            K-major A operands of pass 2 (no SMEM round trip):
//              Moore: Pb = H            Pi = 128 * state
//              VN   : Pb = state        Pi = H + 128 * state
//            Pi is stored 16 rows up (row y at byte y - 16), so the centre
//            rows of every 64-row output sub-block are two aligned K chunks.
//   pass 2   per 64-row output sub-block s (window = box rows [64s, 64s+96)):
//            D2[x][j] = Pb . Bv (3 chunks) + Pi . c*Iv (2 chunks), N = 64,
//            A in TMEM:  Moore: R_box + 2048*state   VN: R_cross + 128*state
//            Folding the state into the accumulator makes the birth/survival
//            rule (apply_transition, src/rule.cpp:99-111) a pure function of
//            one 12-bit number Z.
//   rule     Z is read back two cells per register (16-bit lanes); the two
//            range tests (dead: b1..b2, live: K+s1'..K+s2') are four biased
//            adds and two LOP3s per register (bit 15 of each lane = result).
//   store    the D2 columns are permuted (out_row_of_col) so that
//            stmatrix.trans writes each 16x256b TMEM fragment straight into
//            the group's row-major SWIZZLE_128B 64x128 staging tile; the store
//            warp writes it with one 8 KB TMA store of the next generation
//            (no CTA-wide barrier on the output path).
//
// Every quantity is an exact small integer (H <= 33, R <= 1089, Z < 4096), so
// the result is bit-identical to the reference's int32 loops.
//
// One CTA per SM (all 512 TMEM columns), 16 warps:
//   warp 0        TMA producer (+ unit flags of multi-generation launches,
//                 ring counters of slabs, the run-time remainder schedule of
//                 the kDyn instantiations: it takes unit ranges from a global
//                 cursor and hands them to the other warps, SegIter)
//   warp 1        pass-1 MMA issuer, TMEM owner
//   warps 2..5    convert D1 (warp w: TMEM lane quarter w%4 = 32 strip columns)
//   warps 6..13   rule + stage D2: group g = 0 / 1 takes sub-block g of every unit
//   warp 14       pass-2 MMA issuer
//   warp 15       TMA stores, unit publication (multi-generation launches)
// Every stage hands over through mbarrier rings, so TMA, both MMA passes and
// both epilogue groups overlap across sub-blocks and units.  Measured limit
// (DESIGN.md §3.1): ~1450 cycles per unit, where the kernel's instruction
// issue (~4000 warp instructions per unit at IPC ~2.6) and its HBM share at
// 2 B/cell coincide.  kPk: the same step on 4-bit cells (pass 1 on
// kind::f8f6f4).
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdlib>

#include "ltl_kernels.cuh"
#include "ptx_sm100.cuh"

namespace ltl {
namespace {

using namespace ptx;

constexpr int kBand = kTcBand;            // 128 output rows per unit
constexpr int kSub = 64;                  // pass-2 N: output rows per sub-block
constexpr int kSubs = kBand / kSub;       // 2
constexpr int kKChunks = 6;               // pass-1 K = 192 columns [-32, 160): r <= 32
constexpr int kSlots = 2;                 // D1 / plane slots (units in flight)
constexpr int kConvWarps = 4;
constexpr int kOutWarps = 8;
constexpr int kThreads = 32 * (4 + kConvWarps + kOutWarps);  // 512
constexpr int kConvThreads = 32 * kConvWarps;
constexpr int kGroupThreads = 128;  // one output group
constexpr int kWarpOut0 = 2 + kConvWarps;
constexpr int kWarpP2 = kWarpOut0 + kOutWarps;  // 14
constexpr int kWarpStore = kWarpP2 + 1;           // 15
constexpr uint32_t kTileBytes = kSub * 32;        // 2 KB pass-2 B tile [64 n][32 k]
constexpr uint32_t kTmemCols = 512;               // all of the SM's TMEM
constexpr uint32_t kSegSlots = 8;                 // dynamic-schedule segment ring
constexpr uint32_t kSegReaders = 15;              // warps that read it: all but the producer
static_assert(kSubs == 2 && kSlots == kSubs, "one output group per sub-block; barrier arrays sized kSubs");

// Geometry of one kernel variant, by the halo rows kH its boxes carry:
//   kH = 16  r <= 16 (the reference's range, src/rule.cpp:33-35): 160-row
//            boxes, the product configuration;
//   kH = 32  17 <= r <= 32, the paper's "+16 expansion" (a
//            radius range the reference rejects): 192-row boxes, four pass-2
//            band chunks, one D2 buffer shared by the two output groups
//            (TMEM), 7 box stages and 2 staging slots per group (SMEM).
// The pass-1 K range [-32, 160) already covers a horizontal radius of 32.
// 4-bit cells: the f16 D1 is moved into the binade [1024, 2048) (bit pattern
// 0x6400 + D1) by a 7th pass-1 MMA (1, default) or by an add.f16x2 per
// register in the convert (0, A/B).
#ifndef LTL_PK_BIAS_MMA
#define LTL_PK_BIAS_MMA 1
#endif
__device__ __forceinline__ uint32_t hadd2_u32(uint32_t a, uint32_t b) {
  uint32_t d;
  asm("add.rn.f16x2 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b));
  return d;
}

template <int kH, bool kPk = false>
struct Geo {
  static_assert(kH == 16 || kH == 32, "halo rows");
  static_assert(!kPk || kH == 16, "4-bit cells: r <= 16 boxes only");
  static constexpr int kBox = kBand + 2 * kH;              // 160 / 192 box rows (one TMA box)
  static constexpr int kRowOff = kHalo - kH;               // padded row of box row 0, minus 128 b
  static constexpr int kBandChunks = (kSub + 2 * kH) / 32;  // pass-2 band K chunks: 3 / 4
  static constexpr int kNumTiles = kBandChunks + 4;         // + Iv0..1, W*Iv0..1
#ifndef LTL_PK_XSTAGES
#define LTL_PK_XSTAGES 9
#endif
  static constexpr int kXStages = kPk ? LTL_PK_XSTAGES : kH == 16 ? 8 : 7;  // 3 in use + prefetched
#ifndef LTL_PK_STAGE_SLOTS
#define LTL_PK_STAGE_SLOTS 3
#endif
  static constexpr int kStageSlots = kPk ? LTL_PK_STAGE_SLOTS : kH == 16 ? 3 : 2;  // per output group
  // 4-bit cells (kPk): HBM rows of a strip are 64 B (two cells per byte, cell
  // 2i in the low nibble); a TMA box lands in the padded 16U4_ALIGN16B SMEM
  // layout (8 bytes of nibbles + 8 unused per 16 cells: the same 128-byte SMEM
  // rows as u8 cells), the output staging tile is 64 rows x 64 B.
  static constexpr uint32_t kRowBytes = kPk ? kStrip / 2 : kStrip;   // HBM bytes per strip row
  static constexpr uint32_t kStageBytes = kSub * kRowBytes;           // 8 / 4 KB staging tile
  // D2 buffers (64 columns each).  kH = 32: sub-block 1's only; sub-block 0's
  // D2 goes into the free columns [kD2InSlot, +64) of the unit's D1 slot
  // (the planes use [0, 80)), so the slot is free once pass 2 is done AND
  // output group 0 has read it (slot_empty counts both).
#ifdef LTL_D2_SLOT16  // A/B: the same for the kH = 16 boxes (planes [0, 72), D2 [96, 160))
  static constexpr int kD2Bufs = 1;
#else
  static constexpr int kD2Bufs = kH == 16 ? 2 : 1;
#endif
  static constexpr uint32_t kD2InSlot = kBox - kSub;       // 128 (kH = 32)
  // centre weight W of pass 2 (Moore: Z = R + 128 W state must clear R <= (2r+1)^2)
  // (4-bit cells, Moore: pass 2 sums 2 H, Z = 2 R + 4096 state, R <= 1089)
  static constexpr uint32_t kCentreW = kPk ? 32u : kH == 16 ? 16u : 64u;   // K = 2048 / 8192 / 4096
  static constexpr uint32_t kVnK = kH == 16 ? 128u : 256u;     // VN: R <= 2(2r+1)
  static constexpr uint32_t kBoxBytes = kBox * kStrip;      // 20 / 24 KB of SMEM
  static constexpr uint32_t kBoxTx = kBox * kRowBytes;      // HBM bytes of one box
  static_assert(kBox % 32 == 0 && kBox <= 256, "box rows: whole K chunks, one TMA box");

  // Shared-memory carve-up (offsets from a 1024-aligned base).
  static constexpr uint32_t kSmemX = 0;
  static constexpr uint32_t kSmemBand = kSmemX + kXStages * kBoxBytes;
  // 4-bit cells: a resident B tile of e2m1 1.0 (160 rows x 32 cells, SW32,
  // 5 KB) for pass 1's bias MMA, D1 += 1024 (A = e4m3 32.0 x 32 k)
  static constexpr uint32_t kOnesBytes = kPk ? kBox * 32 : 0;
  static constexpr uint32_t kSmemOnes = kSmemBand + kNumTiles * kTileBytes;
  static constexpr uint32_t kSmemStage = kSmemOnes + kOnesBytes;
  static constexpr uint32_t kSmemBars = kSmemStage + kSubs * kStageSlots * kStageBytes;
  static constexpr uint32_t kNumBars =
      2 * kXStages + 4 * kSlots + 2 * kSubs + 2 * kSubs * kStageSlots;
  // dynamic remainder schedule (SegIter): a ring of segment descriptors
  // handed from the producer warp to the other roles
  static constexpr uint32_t kSmemSeg = (kSmemBars + kNumBars * 8 + 16 + 15) & ~15u;
  static constexpr uint32_t kSmemTotal = kSmemSeg + kSegSlots * (16 + 2 * 8);
  static constexpr uint32_t kSmemAlloc = kSmemTotal + 1024;  // alignment slack
  static_assert(kSmemAlloc <= 227 * 1024, "shared memory budget");

  // TMEM columns.  A slot first holds D1 (kBox s32 columns); once the convert
  // warps have read it into registers they write the two byte planes over its
  // first columns, which pass 2 reads.  Two slots: pass 1 of unit h+1 runs
  // while unit h is converted and reduced.
  static constexpr uint32_t kPbCols = kBox / 4;    // one byte per box row
  static constexpr uint32_t kPiCols = kBand / 4;   // 32: one byte per centre row
  static constexpr uint32_t kSlotCols = kBox;
  static constexpr uint32_t kTmemSlot = 0;
  static constexpr uint32_t kPbOff = 0;
  static constexpr uint32_t kPiOff = kPbCols;
  static constexpr uint32_t kTmemD2 = kTmemSlot + kSlots * kSlotCols;
  static constexpr uint32_t kTmemA1 = kTmemD2 + kD2Bufs * kSub;  // pass-1 A: 192 k / 4 = 48
  static constexpr uint32_t kTmemBias = kTmemA1 + kKChunks * 8;  // 4-bit cells: bias A chunk (8)
  static_assert(kPiOff + kPiCols <= kSlotCols, "planes fit in the D1 slot");
  static_assert(kD2Bufs == kSubs || kPiOff + kPiCols <= kD2InSlot, "slot D2 clear of the planes");
  static_assert(kTmemBias + (kPk ? 8 : 0) <= kTmemCols, "TMEM budget");
  static_assert(kSmemStage % 1024 == 0, "staging tiles: swizzle-atom aligned");
  static_assert(kSlotCols % 8 == 0 && kPiOff % 8 == 0 && kTmemD2 % 8 == 0, "A operand alignment");

  // pass 1: u8 cells -> kind::i8 (s32 D1); 4-bit cells -> kind::f8f6f4 with
  // e4m3 band weights x e2m1 cells (nibble 1 = 0.5), f16 D1 (exact: <= 67)
  static constexpr uint32_t kIdesc1 =
      kPk ? idesc_f8f6f4_e4m3_e2m1_f16(128, kBox) : idesc_i8_u8u8_s32(128, kBox);
  static constexpr uint32_t kIdesc2 = idesc_i8_u8u8_s32(128, kSub);
};

// Tensor maps of both generation buffers: set 0 = {loads of the launch's
// current buffer, stores into the other}, set 1 = the reverse (generation g
// of a multi-generation launch uses set g % 2).
struct TcMaps {
  CUtensorMap load[2][kTcLoadMaps];
  CUtensorMap store[2];
  CUtensorMap ring_up[2];    // ring: 16-row pieces of the upper neighbour's slab (peer
  CUtensorMap ring_down[2];  // memory), [its buffer of generation gg % 2 of the launch]
};

struct Params {
  int32_t rows, cols;
  int32_t strips;  // interior strips
  int32_t bands;
  RuleConsts rule;
  // CatConfig.inject_band_fault: the reference flips pi2(0,0) of every f x f
  // band fragment (src/cat_engine.cpp:277), i.e. the centre term of the
  // horizontal sums of columns == 0 mod f and of the vertical sums of rows
  // == 0 mod f (global coordinates) drops out.  Same here: pass-1 A1 entry
  // (x, x) for strip columns x == 0 mod f, pass-2 band entry (rho, rho) for
  // output rows rho with (row0 + rho) == 0 mod f.
  int32_t inject_fault;
  int32_t fault_f, fault_row_phase;
  int32_t gen_base, row0;  // generation / global row of this launch's first (negative_key)
  int32_t wrap_cols, wrap_rows;  // periodic wrap done by the loads (tc_wrap_*)
  int32_t gens;                  // generations in this launch (persistent when > 1)
  int32_t sweep_chunks;          // chunks per band of a persistent launch (SegIter)
  // Ring of row slabs (multi-GPU), pull model: the first / last band's 16
  // rows above / below are TMA-loaded straight out of the neighbours' slabs
  // (peer memory over NVLink, P2P or CUDA IPC) -- the halo exchange is part
  // of the step's own loads.  Every slab counts its finished step kernels in
  // *my_done (the launch's last CTA publishes G + 1); a CTA waits once for a
  // neighbour's counter to reach G before its first piece from that slab.
  // That wait also orders our next stores to rows the neighbour reads after
  // its previous step: only first / last band units write those rows.
  int32_t ring;
  uint32_t ring_gen;             // G: this launch turns generation G into G + 1
  int32_t up_rows;               // the upper neighbour's slab height
  const uint32_t* up_done;       // the neighbours' counters (peer memory)
  const uint32_t* down_done;
  uint32_t* my_done;             // this slab's counter and its CTA ticket
  uint32_t* my_ticket;
  // Multi-generation ring launches: the neighbours' per-unit counters (same
  // geometry, same flag_base: every slab of the ring runs the same launches)
  // stand for the bands above band 0 / below the last band, read at system
  // scope; edge units are published at system scope.
  const uint32_t* up_flags;
  const uint32_t* down_flags;
  uint32_t* flags;               // per-unit completion counters (bands x strips)
  uint32_t flag_base;            // their common value when the launch starts
  DeviceStats* stats;
  long long* trace;  // debug timeline of CTA 0 (only with -DLTL_TC_TRACE_BUILD)
  // one launch per generation: the remainder after the whole-band rounds is
  // handed out at run time ([0] unit cursor, [1] CTA exit ticket; zero
  // between launches), nullptr = the static remainder runs
  uint32_t* dyn;
};

#ifdef LTL_TC_TRACE_BUILD
#define LTL_TRACE(ev, idx) \
  do { if (p.trace && blockIdx.x == 0 && (idx) < 256) p.trace[(ev) * 256 + (idx)] = clock64(); } while (0)
__device__ __forceinline__ long long global_ns() {
  long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define LTL_TRACE_CTA(ev) \
  do { if (p.trace && threadIdx.x == 0) p.trace[(ev) * 256 + blockIdx.x] = global_ns(); } while (0)
// cycles spent in each wait site, summed over the launch by CTA 0 (row 13)
#define LTL_WAIT(site, bar, par)                                                   \
  do {                                                                             \
    const long long w0_ = clock64();                                               \
    mbar_wait(bar, par);                                                           \
    if (p.trace && blockIdx.x == 0 && (threadIdx.x & 31) == 0)                     \
      atomicAdd(reinterpret_cast<unsigned long long*>(&p.trace[13 * 256 + (site)]), \
                static_cast<unsigned long long>(clock64() - w0_));                 \
  } while (0)
#else
#define LTL_TRACE(ev, idx) do { } while (0)
#define LTL_TRACE_CTA(ev) do { } while (0)
#define LTL_WAIT(site, bar, par) mbar_wait(bar, par)
#endif

// Static schedule over the bands x strips units.  A CTA walks runs of
// consecutive strips of one band (a segment [t0, t1) streams boxes t0-1 ..
// t1, its 16-column side halos included); every role of the CTA iterates the
// same segments in the same order.  The point of the order is that units of
// vertically adjacent bands are processed at about the same time by different
// CTAs, so the 32 box rows they share come from HBM once and from L2 the
// second time (otherwise ~20 % of all reads are that overlap again):
//   * full rounds: while at least G bands remain for every CTA, CTA b walks
//     whole bands b + rG, all CTAs in step (65536^2: three rounds);
//   * the remaining bands' units are cut into G contiguous runs in band-major
//     order, and with the column wrap done by the loads (cols % 128 == 0) band
//     k's strips start at the rotation rot_k = round(k (S - U'/G)) mod S, a run
//     crossing the torus seam (strip t is t mod S): CTA b + 1 then meets band
//     k + 1 at the strip where CTA b meets band k.
// Multi-generation (persistent) launches sweep instead: generation g is cut
// into chunks of C per band (band position k, chunk j: strips
// [jS/C, (j+1)S/C) of band (k + g) mod B), numbered g*B*C + k*C + j and dealt
// round-robin to the CTAs, so all CTAs advance through the bands together as
// one wavefront across generation boundaries.  Rotating the band order by one
// per generation puts every input of a unit (bands k-1 .. k+1 of generation
// g-1 = its sweep positions k .. k+2) (B - 2) bands behind it in the global
// order: no unit waits in steady state, whatever the CTA count, and no CTA
// holds units of a generation before all of its units of the previous one
// (deadlock-free with all CTAs resident).
// Segment descriptors of the dynamic remainder (one launch per generation):
// the producer warp takes unit ranges from a global cursor (guided: about
// half of the remainder's fair share per CTA, at least 8 units, never past a
// band's end) and hands each to the 15 other warps through this SMEM ring.
// CTAs on slower SMs (measured: a few % longer per unit on some of them)
// then take fewer units instead of finishing last.
struct SegRing {
  int4* e;
  uint64_t* full;
  uint64_t* empty;
};

#ifndef LTL_DYN_MIN  // dynamic remainder: smallest grab (units), fair-share divisor
#define LTL_DYN_MIN 8
#endif
#ifndef LTL_DYN_DIV
#define LTL_DYN_DIV 2
#endif
template <bool kDyn>
struct SegIter {
  int64_t u, u_end, U;  // remainder part: linear unit range of this CTA
  int32_t S, G, B0, round, rounds;
  bool rotate;
  // sweep (multi-generation) mode: global chunk index, this generation's end
  int64_t ci, c_base, c_end;
  int32_t C, B, gen;
  // dynamic remainder
  uint32_t* dyn;
  SegRing ring;
  uint32_t seq;
  bool producer;
  uint32_t pend_u, pend_e;  // producer: the part of its last grab past a band's end
  __device__ SegIter(const Params& p, int gen_, const SegRing& ring_ = SegRing{}, bool producer_ = false)
      : S(p.strips), G(static_cast<int32_t>(gridDim.x)), round(0), rotate(p.wrap_cols != 0),
        C(p.gens > 1 ? p.sweep_chunks : 0), B(p.bands), gen(gen_),
        // (only after whole-band rounds: with none -- 8192^2, 16384^2 per launch --
        // the all-dynamic order loses the rotated remainder's L2 locality:
        // 34.0 -> 35.7 us; at 32768^2 345 -> 338 us, tools/gpu_r02au.sh)
        dyn(!kDyn || p.gens > 1 || p.bands < static_cast<int32_t>(gridDim.x) ? nullptr : p.dyn),
        ring(ring_), seq(0), producer(producer_),
        pend_u(0), pend_e(0) {
    if (C > 0) {
      c_base = static_cast<int64_t>(gen) * B * C;
      c_end = c_base + static_cast<int64_t>(B) * C;
      ci = c_base + ((static_cast<int64_t>(blockIdx.x) - c_base) % G + G) % G;
      rounds = 0;
      u = u_end = 0;
      return;
    }
    rounds = p.bands / G;  // whole bands per CTA in step
    B0 = rounds * G;       // first band of the remainder
    U = static_cast<int64_t>(p.bands - B0) * S;
    u = U * blockIdx.x / G;
    u_end = U * (blockIdx.x + 1) / G;
  }
  __device__ bool next(int& band, int& t0, int& t1) {
    if (C > 0) {
      if (ci >= c_end) return false;
      const int m = static_cast<int>(ci - c_base);
      const int k = m / C, j = m % C;
      band = (k + gen) % B;
      t0 = S * j / C;
      t1 = S * (j + 1) / C;
      ci += G;
      return true;
    }
    if (round < rounds) {
      band = static_cast<int>(blockIdx.x) + round * G;
      ++round;
      t0 = 0;
      t1 = S;
      return true;
    }
    if constexpr (kDyn) {
      if (dyn) return dyn_next(band, t0, t1);
    }
    if (u >= u_end) return false;
    const int k = static_cast<int>(u / S);  // band within the remainder
    band = B0 + k;
    t0 = static_cast<int>(u % S);
    const int64_t e = min(u_end, static_cast<int64_t>(k + 1) * S);
    t1 = t0 + static_cast<int>(e - u);
    u = e;
    if (rotate) {
      // rot = round(k * (S - U / G)) mod S, in exact integers
      const int64_t SG = static_cast<int64_t>(S) * G;
      const int64_t num = (static_cast<int64_t>(k) * (((SG - U) % SG + SG) % SG)) % SG;
      const int r = static_cast<int>(((num + G / 2) / G) % S);
      t0 += r;
      t1 += r;
    }
    return true;
  }
  __device__ bool dyn_next(int& band, int& t0, int& t1) {
    const uint32_t lane = threadIdx.x & 31;
    const uint32_t slot = seq % kSegSlots, par = (seq / kSegSlots) & 1;
    ++seq;
    int4 sg = make_int4(-1, 0, 0, 0);
    if (producer) {
      if (lane == 0) {
        // one atomicAdd per grab (a CAS loop over 148 producers serialises),
        // taken when the previous one is used up -- not earlier: a CTA that
        // reserves its next range ahead of time keeps it while it is slow
        // (measured: 347 vs 339 us at 32768^2).  A grab past a band's end is
        // published as two segments.
        const uint32_t total = static_cast<uint32_t>(U), su = static_cast<uint32_t>(S);
        if (pend_u >= pend_e) {
          const uint32_t c = *reinterpret_cast<volatile uint32_t*>(dyn);
          const uint32_t rem = c < total ? total - c : 0u;
          const uint32_t want =
              min(su, max(static_cast<uint32_t>(LTL_DYN_MIN),
                          rem / (static_cast<uint32_t>(LTL_DYN_DIV) * static_cast<uint32_t>(G))));
          const uint32_t u0 = atomicAdd(dyn, want);
          pend_u = min(u0, total);
          pend_e = min(u0 + want, total);
        }
        if (pend_u < pend_e) {
          const uint32_t e = min(pend_e, (pend_u / su + 1) * su);  // this band's part
          sg = make_int4(B0 + static_cast<int>(pend_u / su), static_cast<int>(pend_u % su),
                         static_cast<int>(pend_u % su + (e - pend_u)), 0);
          pend_u = e;
        }
        mbar_wait(&ring.empty[slot], par ^ 1);
        ring.e[slot] = sg;
        mbar_arrive(&ring.full[slot]);
      }
      sg.x = __shfl_sync(0xffffffffu, sg.x, 0);
      sg.y = __shfl_sync(0xffffffffu, sg.y, 0);
      sg.z = __shfl_sync(0xffffffffu, sg.z, 0);
    } else {
      mbar_wait(&ring.full[slot], par);
      const volatile int* ve = reinterpret_cast<const volatile int*>(&ring.e[slot]);
      sg = make_int4(ve[0], ve[1], ve[2], 0);
      __syncwarp(__activemask());
      if (lane == 0) mbar_arrive(&ring.empty[slot]);
    }
    if (sg.x < 0) return false;
    band = sg.x;
    t0 = sg.y;
    t1 = sg.z;
    return true;
  }
};

// D2 column j holds sub-block row out_row_of_col(j).  Within each 32-column
// half, with j = [e, m, a0, a1, v] (bit 0 first) the row is [e, a0, a1, m, v]:
// the stmatrix fragment of column group (m, v) of a 16x256b load then covers
// the 8 consecutive rows 8*(m + 2v) .. +7 of that half.
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

// TMEM lane (= pass-1 A row = D1 / D2 lane) of strip column x: the identity
// for u8 cells; for 4-bit cells lanes 16j + i and 16j + 8 + i hold columns
// 16j + 2i and 16j + 2i + 1, so the 16x256b loads of the output warps hand
// every thread the two cells of one output byte.
template <bool kPk>
__host__ __device__ constexpr int lane_x(int lane) {
  return kPk ? (lane & ~15) | ((lane & 7) << 1) | ((lane >> 3) & 1) : lane;
}

template <int kH, bool kChecked, bool kRing, bool kPk, bool kDyn>
__global__ void __launch_bounds__(kThreads, 1)
    ltl_tc_step_kernel(const __grid_constant__ TcMaps maps, const Params p) {
  using G = Geo<kH, kPk>;
  constexpr uint32_t kStageBytes = G::kStageBytes;
  constexpr int kBox = G::kBox;
  constexpr int kXStages = G::kXStages;
  constexpr int kStageSlots = G::kStageSlots;
  constexpr uint32_t kBoxBytes = G::kBoxBytes;
  constexpr uint32_t kSmemX = G::kSmemX, kSmemBand = G::kSmemBand, kSmemStage = G::kSmemStage,
                     kSmemBars = G::kSmemBars;
  constexpr uint32_t kSlotCols = G::kSlotCols, kTmemSlot = G::kTmemSlot, kTmemD2 = G::kTmemD2,
                     kTmemA1 = G::kTmemA1, kPbOff = G::kPbOff, kPiOff = G::kPiOff;
  LTL_TRACE_CTA(10);  // kernel entry (trace build)
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + kSmemBars);
  uint64_t* x_full = bars;
  uint64_t* x_empty = x_full + kXStages;
  uint64_t* d1_full = x_empty + kXStages;     // pass 1 -> convert
  uint64_t* a2_full = d1_full + kSlots;       // convert -> pass 2 (planes written)
  uint64_t* slot_empty = a2_full + kSlots;    // pass 2 -> pass 1 (slot reusable)
  uint64_t* d2_full = slot_empty + kSlots;
  // staging tile handshake with the store warp: [group][slot]
  uint64_t* d2_empty = d2_full + kSubs;
  uint64_t* st_full = d2_empty + kSubs;              // output group -> store warp
  uint64_t* st_empty = st_full + kSubs * kStageSlots; // store warp -> output group
  // kH = 32: sub-block 0's D2 sits in the unit's slot, so pass 2 may run up to
  // two units ahead of output group 0 -- one "D2 written" barrier per slot
  uint64_t* d2_slot_full = st_empty + kSubs * kStageSlots;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(d2_slot_full + kSlots);
  SegRing seg;
  seg.e = reinterpret_cast<int4*>(smem + G::kSmemSeg);
  seg.full = reinterpret_cast<uint64_t*>(smem + G::kSmemSeg + kSegSlots * 16);
  seg.empty = seg.full + kSegSlots;

  const uint32_t warp = warp_id();
  const uint32_t lane = threadIdx.x & 31;
  const int r = p.rule.r;
  const bool vn = p.rule.kind != 0;

  // ---- one-time setup: resident bands (generic-proxy writes), barriers, TMEM
  // pass-2 B tiles [64 n][32 k]: n = D2 column j (output row rho = out_row_of_col(j)),
  //   t < nb          band, K chunk t = window rows 32t .. 32t+31 (centre at kH + rho)
  //   t = nb, nb+1    centre, K chunk of the shifted plane (centre at rho)
  //   t = nb+2, nb+3  W * centre (Moore: state * 128 W)
  // (nb = G::kBandChunks).  kH = 32, VN: the band's centre entry also carries
  // 128 (Pb = state there), so Z = R + 256 state clears R <= 2 (2r + 1).
  constexpr int nb = G::kBandChunks;
  // The twelve warps outside 2..5 build the band tiles while warps 2..5
  // compute the pass-1 A table in registers (the prologue sits on the
  // critical path of the last SM at every generation boundary).
  constexpr uint32_t kTileThreads = kThreads - 32 * kConvWarps;
  const bool a_warp = warp >= 2 && warp < 2 + kConvWarps;
  uint32_t a1[kKChunks * 8];
  if (a_warp) {
    const int m = lane_x<kPk>(32 * static_cast<int>(warp & 3) + static_cast<int>(lane));
    // pi2(0,0) flipped in this column's fragment (one modulo per thread: the
    // table below is fully unrolled, and this prologue sits on the critical
    // path of the last SM at every generation boundary)
    const bool fault_col = p.inject_fault && m % p.fault_f == 0;
#pragma unroll
    for (int c = 0; c < kKChunks * 8; ++c) {
      uint32_t word = 0;
#pragma unroll
      for (int b = 0; b < 4; ++b) {
        const int d = 4 * c + b - 32 - m;
        const bool in = d >= -r && d <= r;
        const bool drop = d == 0 && fault_col;
        uint32_t v;
        if constexpr (kPk) {
          // e4m3 weights on cells of 0.5: window 4.0 (0x48) -> 2 per live
          // cell, centre 6.0 (0x4C) -> 3: D1 = 2 H + state; faulted centre
          // 2.0 (0x40) -> the state marker only
          v = d == 0 ? (drop ? 0x40u : 0x4Cu) : in ? 0x48u : 0u;
        } else {
          // D1 = H + 128 state (the state marker in bit 7)
          v = d == 0 ? (drop ? 128u : 129u) : in ? 1u : 0u;
        }
        word |= v << (8 * b);
      }
      a1[c] = word;
    }
  } else {
    const uint32_t tid_t = threadIdx.x < 64 ? threadIdx.x : threadIdx.x - 32 * kConvWarps;
    for (uint32_t w = tid_t; w < G::kNumTiles * kSub * 8u; w += kTileThreads) {
      const int t = static_cast<int>(w / (kSub * 8)), j = static_cast<int>((w / 8) % kSub),
                k0 = 4 * static_cast<int>(w % 8);
      const int rho = out_row_of_col(j);
      uint32_t word = 0;
#pragma unroll
      for (int b = 0; b < 4; ++b) {
        int v;
        if (t < nb) {
          const int d = 32 * t + k0 + b - kH - rho;
          v = (d >= -r && d <= r);
          if (p.inject_fault && d == 0 && (rho + p.fault_row_phase) % p.fault_f == 0) v = 0;
          if (kH == 32 && vn && d == 0) v += 128;
        } else {
          const int c = (t - nb) % 2;
          v = (32 * c + k0 + b == rho) ? (t >= nb + 2 ? static_cast<int>(G::kCentreW) : 1) : 0;
        }
        word |= static_cast<uint32_t>(v) << (8 * b);
      }
      *reinterpret_cast<uint32_t*>(smem + kSmemBand + t * kTileBytes + sw32_offset(j, k0)) = word;
    }
  }
  if constexpr (kPk) {  // e2m1 1.0 = nibble 2 everywhere (data and padding: layout-free)
    for (uint32_t w = threadIdx.x; w < G::kOnesBytes / 4; w += kThreads)
      reinterpret_cast<uint32_t*>(smem + G::kSmemOnes)[w] = 0x22222222u;
  }
  fence_proxy_async_smem();
  if (warp == 0 && lane == 0) {
    // Prefetch every load / store map of the grid (all four load maps even
    // when the first / last band ones are used by few CTAs: 16384^2 98.4 ->
    // 95.6 us); the ring maps are fetched on first use.
    for (int set = 0; set < (p.gens > 1 ? 2 : 1); ++set) {
      for (int i = 0; i < kTcLoadMaps; ++i) prefetch_tmap(&maps.load[set][i]);
      prefetch_tmap(&maps.store[set]);
    }
    for (int i = 0; i < kXStages; ++i) {
      mbar_init(&x_full[i], 1);
      mbar_init(&x_empty[i], 1);
    }
    for (int i = 0; i < kSlots; ++i) {
      mbar_init(&d1_full[i], 1);
      mbar_init(&a2_full[i], kConvThreads);
      mbar_init(&slot_empty[i], G::kD2Bufs == kSubs ? 1 : 1 + kGroupThreads);
    }
    for (int i = 0; i < kSubs; ++i) {
      mbar_init(&d2_full[i], 1);
      mbar_init(&d2_slot_full[i], 1);  // (kSlots == kSubs == 2)
      mbar_init(&d2_empty[i], kGroupThreads);
    }
    for (int i = 0; i < kSubs * kStageSlots; ++i) {
      mbar_init(&st_full[i], 1);
      mbar_init(&st_empty[i], 1);
    }
    if constexpr (kDyn) {
      for (uint32_t i = 0; i < kSegSlots; ++i) {
        mbar_init(&seg.full[i], 1);
        mbar_init(&seg.empty[i], kSegReaders);
      }
    }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc(tmem_slot, kTmemCols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  // pass-1 A1 [128 x][192 k] resident in TMEM (the A operand of a .ts MMA is
  // cheaper than an SMEM descriptor one, tools/ubench_mma.cu): lane x holds
  // A1[x][k] = [|k-32-x| <= r] + 128*[k == x+32], four k per column; warps
  // 2..5 write their lane quarter.
  if (a_warp) {
    const uint32_t trow = tmem + ((32u * (warp & 3)) << 16) + kTmemA1;
#pragma unroll
    for (int c = 0; c < kKChunks; ++c) {
      uint32_t v8[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) v8[i] = a1[8 * c + i];
      tmem_st_32x32b_x8(trow + 8 * c, v8);
    }
    if constexpr (kPk) {  // e4m3 32.0 (0x60) x 32 k: the bias MMA adds 1024
      const uint32_t v8[8] = {0x60606060u, 0x60606060u, 0x60606060u, 0x60606060u,
                              0x60606060u, 0x60606060u, 0x60606060u, 0x60606060u};
      tmem_st_32x32b_x8(trow + (G::kTmemBias - kTmemA1), v8);
    }
    tmem_st_wait();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  // Everything above only touched this CTA's SMEM/TMEM, so it overlapped the
  // previous kernel's tail (PDL).  The grid is read from here on.
  LTL_TRACE_CTA(12);  // prologue done
  pdl_launch_dependents();
  pdl_wait_prerequisites();
  LTL_TRACE_CTA(14);

  if (warp == 0) {
    // ================= TMA producer: boxes t0-1 .. t1 of every segment =======
    // The whole warp walks the schedule; lane 0 issues.  In a multi-generation
    // launch generation gg reads what gg-1 wrote: box (band, strip) holds rows
    // of units (band-1 .. band+1, strip) of gg-1 (periodic in band), whose
    // flags must have reached flag_base + 2 gg.  The lanes read the flags of
    // 32 boxes at once (one L2 round trip per 32 boxes, not three per box).
    uint32_t g = 0;
    bool up_ready = false, down_ready = false;  // ring: neighbours' generation G seen
    for (int gg = 0; gg < p.gens; ++gg) {
      const CUtensorMap* lm = maps.load[gg & 1];
      const uint32_t target = p.flag_base + 2u * static_cast<uint32_t>(gg);
      SegIter<kDyn> it(p, gg, seg, true);
      int band, t0, t1;
      while (it.next(band, t0, t1)) {
        const bool edge_rows = p.wrap_rows || kRing;  // rows beyond the slab by piece loads
        const bool first = edge_rows && band == 0;
        const bool last = edge_rows && band == p.bands - 1;
        const int last_rows = p.rows - kBand * band;  // interior rows of the last band
        const int nbox = t1 - t0 + 2;
        auto storage_strip = [&](int k) {  // logical strip t0-1+k (or its image)
          return p.wrap_cols ? (t0 - 1 + k + p.strips) % p.strips + 1 : t0 + k;
        };
        const bool peer_up = kRing && band == 0;  // band -1 is the upper slab's last
        const bool peer_down = kRing && band == p.bands - 1;
        auto flag_ptr = [&](int db, int k) -> const uint32_t* {
          const int b = band + db;
          const int64_t col = storage_strip(k) - 1;
          if (kRing && b < 0) return p.up_flags + static_cast<int64_t>(p.bands - 1) * p.strips + col;
          if (kRing && b >= p.bands) return p.down_flags + col;
          return p.flags + static_cast<int64_t>((b + p.bands) % p.bands) * p.strips + col;
        };
        auto flag_ld = [&](int db, int k) {
          const bool peer = (db < 0 && peer_up) || (db > 0 && peer_down);
          return peer ? ld_acquire_sys(flag_ptr(db, k)) : ld_acquire(flag_ptr(db, k));
        };
        for (int k0 = 0; k0 < nbox; k0 += 32) {
          uint32_t ready = ~0u;
          if (gg > 0) {
            const int k = k0 + static_cast<int>(lane);
            bool ok = true;
            if (k < nbox) {
              const uint32_t f0 = flag_ld(-1, k);
              const uint32_t f1 = flag_ld(0, k);
              const uint32_t f2 = flag_ld(1, k);
              ok = static_cast<int32_t>(f0 - target) >= 0 && static_cast<int32_t>(f1 - target) >= 0 &&
                   static_cast<int32_t>(f2 - target) >= 0;
            }
            ready = __ballot_sync(0xffffffffu, ok);
            __syncwarp();  // order the lanes' acquires before lane 0's loads
            // acquired generic-proxy flags -> async-proxy (TMA) reads; once
            // per window: the proxy fence is not free
            if (lane == 0) fence_proxy_async_global();
          }
          for (int k = k0; k < min(nbox, k0 + 32); ++k, ++g) {
            if (gg > 0 && !((ready >> (k - k0)) & 1u)) {
              if (static_cast<int>(lane) == k - k0) {
#ifdef LTL_TC_TRACE_BUILD
                const long long w0_ = clock64();
#endif
                for (int db = -1; db <= 1; ++db) {
                  if ((db < 0 && peer_up) || (db > 0 && peer_down))
                    wait_flag_geq_sys(flag_ptr(db, k), target);
                  else
                    wait_flag_geq(flag_ptr(db, k), target);
                }
#ifdef LTL_TC_TRACE_BUILD
                if (p.trace && blockIdx.x == 0) {
                  atomicAdd(reinterpret_cast<unsigned long long*>(&p.trace[13 * 256 + 17]),
                            static_cast<unsigned long long>(clock64() - w0_));
                  if (g < 256) {
                    p.trace[8 * 256 + g] = clock64() - w0_;
                    p.trace[9 * 256 + g] = gg * 100000 + band * 1000 + storage_strip(k);
                  }
                }
#endif
              }
              __syncwarp();
              if (lane == 0) fence_proxy_async_global();
            }
            if (lane == 0) {
              const uint32_t s = g % kXStages;
              LTL_WAIT(0, &x_empty[s], ((g / kXStages) & 1) ^ 1);
              LTL_TRACE(0, g);
              const int strip = storage_strip(k);
              uint8_t* dst = smem + kSmemX + s * kBoxBytes;
              if (!first && !last) {
                mbar_arrive_expect_tx(&x_full[s], G::kBoxTx);
#ifdef LTL_DIAG_L2_READS  // timing probe only (wrong results): every box from band 1 (L2-resident)
                tma_load_3d(dst, &lm[0], &x_full[s], 0, kBand + G::kRowOff, strip);
#else
                tma_load_3d(dst, &lm[0], &x_full[s], 0, band * kBand + G::kRowOff, strip);
#endif
              } else {
                // first / last band of a whole torus: the kH rows beyond the
                // edge are loaded from the other end of the strip (padded row 16 + y)
                const int body = last ? last_rows : kBand;  // interior rows in the box body
                mbar_arrive_expect_tx(&x_full[s], (last ? last_rows + 2 * kH : kBox) * G::kRowBytes);
                int row = 0;  // box row being filled
                if (kRing && first && !up_ready) {
                  wait_flag_geq_sys(p.up_done, p.ring_gen);
                  fence_proxy_async_global();  // acquired -> TMA reads
                  up_ready = true;
                }
                if (kRing && last && !down_ready) {
                  wait_flag_geq_sys(p.down_done, p.ring_gen);
                  fence_proxy_async_global();
                  down_ready = true;
                }
                if (first) {  // rows -kH .. -1: the torus' other end / the upper slab's last rows
                  if (kRing)
                    tma_load_3d(dst, &maps.ring_up[gg & 1], &x_full[s], 0, p.up_rows + G::kRowOff,
                                strip);
                  else
                    tma_load_3d(dst, &lm[1], &x_full[s], 0, p.rows + G::kRowOff, strip);
                  row = kH;
                }
                if (first && !last) {  // rows 0 .. 128 + kH - 1
                  tma_load_3d(dst + row * kStrip, &lm[2], &x_full[s], 0, kHalo, strip);
                } else {  // last band body: padded rows from 128 * band - kH (its top
                          // halo included unless it is also the first band)
                  tma_load_3d(dst + row * kStrip, &lm[3], &x_full[s], 0,
                              first ? kHalo : band * kBand + G::kRowOff, strip);
                  // rows rows .. rows + kH - 1: the torus' rows 0 .. kH-1 / the lower slab's first rows
                  uint8_t* bot = dst + (row + body + (first ? 0 : kH)) * kStrip;
                  tma_load_3d(bot, kRing ? &maps.ring_down[gg & 1] : &lm[1], &x_full[s], 0, kHalo,
                              strip);
                }
              }
            }
            __syncwarp();
          }
        }
      }
    }
  } else if (warp == 1) {
    // ================= pass-1 MMA issuer: one N = 160 block per unit =========
    const uint32_t a1 = tmem + kTmemA1;  // K chunk q at column a1 + 8q
    const uint64_t x_desc = smem_desc_sw128_kmajor(smem_u32(smem + kSmemX));
    auto box = [&](uint32_t idx) { return x_desc + (((idx % kXStages) * kBoxBytes) >> 4); };
    uint32_t g = 0, h = 0;
    for (int gg = 0; gg < p.gens; ++gg) {
    SegIter<kDyn> it(p, gg, seg);
    int band, t0, t1;
    while (it.next(band, t0, t1)) {
      for (int t = t0; t < t1; ++t, ++h) {
        const uint32_t gl = g + (t - t0), go = gl + 1, gr = gl + 2;
        LTL_WAIT(1, &x_full[gl % kXStages], (gl / kXStages) & 1);
        LTL_WAIT(1, &x_full[go % kXStages], (go / kXStages) & 1);
        LTL_WAIT(1, &x_full[gr % kXStages], (gr / kXStages) & 1);
        const uint32_t sl = h % kSlots;
        LTL_WAIT(2, &slot_empty[sl], ((h / kSlots) & 1) ^ 1);
        LTL_TRACE(1, h);
        tc_fence_after();
        if (elect_one()) {
          const uint32_t dcol = tmem + kTmemSlot + kSlotCols * sl;
          auto mma1 = [&](uint32_t a, uint64_t b, uint32_t acc) {
            if constexpr (kPk) mma_f8f6f4_ts(dcol, a, b, G::kIdesc1, acc);
            else mma_i8_ts(dcol, a, b, G::kIdesc1, acc);
          };
          // (the padded 4-bit SMEM layout keeps 32 cells per 32 bytes: the
          // same K-chunk offsets as u8 cells)
          if constexpr (kPk && LTL_PK_BIAS_MMA) {
            // D1 = 1024 + 2 H + state (f16): each f16's low byte is 2 H + state
            mma1(tmem + G::kTmemBias, smem_desc_sw32_kmajor(smem_u32(smem + G::kSmemOnes)), 0);
            mma1(a1, box(gl) + (96 >> 4), 1);
          } else {
            mma1(a1, box(gl) + (96 >> 4), 0);
          }
#pragma unroll
          for (int q = 1; q <= 4; ++q) mma1(a1 + 8 * q, box(go) + ((32 * (q - 1)) >> 4), 1);
          mma1(a1 + 40, box(gr), 1);
          mma_commit(&d1_full[sl]);
          mma_commit(&x_empty[gl % kXStages]);  // box t-1 is done
          if (t == t1 - 1) {
            mma_commit(&x_empty[go % kXStages]);
            mma_commit(&x_empty[gr % kXStages]);
          }
        }
        __syncwarp();
      }
      g += (t1 - t0) + 2;
    }
    }
  } else if (warp < kWarpOut0) {
    // ================= convert warps (D1 -> pass-2 A planes) =================
    const uint32_t q = warp & 3;  // TMEM lane quarter = 32 strip columns
    const uint32_t trow = tmem + ((q * 32) << 16);
    uint32_t max_h = 0, h = 0;
    for (int gg = 0; gg < p.gens; ++gg) {
    SegIter<kDyn> it(p, gg, seg);
    int band, t0, t1;
    while (it.next(band, t0, t1)) {
      for (int t = t0; t < t1; ++t, ++h) {
        const uint32_t sl = h % kSlots;
        const uint32_t slot_col = trow + kTmemSlot + kSlotCols * sl;
        LTL_WAIT(3 + (warp & 3), &d1_full[sl], (h / kSlots) & 1);
        if (warp == 2 && lane == 0) LTL_TRACE(2, h);
        tc_fence_after();
        // all kBox box rows, two rows (16-bit lanes) per register
        uint32_t va[32], vb[32], vc[kBox / 2 - 64];
        tmem_ld_32x32b_x32_pack16(slot_col, va);
        tmem_ld_32x32b_x32_pack16(slot_col + 64, vb);
        if constexpr (kBox == 192)
          tmem_ld_32x32b_x32_pack16(slot_col + 128, *reinterpret_cast<uint32_t(*)[32]>(vc));
        else
          tmem_ld_32x32b_x16_pack16(slot_col + 128, *reinterpret_cast<uint32_t(*)[16]>(vc));
        tmem_ld_wait();
        if constexpr (kPk && !LTL_PK_BIAS_MMA) {
#pragma unroll
          for (int k = 0; k < 32; ++k) va[k] = hadd2_u32(va[k], 0x64006400u);
#pragma unroll
          for (int k = 0; k < 32; ++k) vb[k] = hadd2_u32(vb[k], 0x64006400u);
#pragma unroll
          for (int k = 0; k < kBox / 2 - 64; ++k) vc[k] = hadd2_u32(vc[k], 0x64006400u);
        }
        auto reg = [&](int k) -> uint32_t { return k < 32 ? va[k] : k < 64 ? vb[k - 32] : vc[k - 64]; };
        auto raw_word = [&](int i) -> uint32_t {  // box rows 4i .. 4i+3 as bytes
          return pack_pairs(reg(2 * i), reg(2 * i + 1));
        };
        if constexpr (kChecked) {
          const bool x_ok = (t % p.strips) * kStrip +
                                lane_x<kPk>(32 * static_cast<int>(q) + static_cast<int>(lane)) < p.cols;
          const int prow0 = band * kBand + G::kRowOff;  // padded row of box row 0
#pragma unroll
          for (int i = 0; i < kBox / 2; ++i) {
            const uint32_t pr = reg(i);
#pragma unroll
            for (int hh = 0; hh < 2; ++hh) {
              const int prow = prow0 + 2 * i + hh;
              const uint32_t hv = kPk ? ((pr >> (16 * hh)) & 0xFFu) >> 1 : (pr >> (16 * hh)) & 0x7Fu;
              if (x_ok && prow >= kHalo && prow < p.rows + kHalo) max_h = max(max_h, hv);
            }
          }
        }
        if (warp == 2 && lane == 0) LTL_TRACE(3, h);
        // the planes overwrite the D1 columns this thread has just read
        const uint32_t pb_col = slot_col + kPbOff;
        const uint32_t pi_col = slot_col + kPiOff;
#pragma unroll
        for (int c = 0; c < kBox / 32; ++c) {  // 32-row chunk c = words 8c .. 8c+7
          uint32_t pb[8], pi[8];
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const uint32_t raw = raw_word(8 * c + i);
            if constexpr (kPk) {  // bytes 2 H + state (the f16 D1 + 1024's low bytes)
              // Moore: Pb = 2 H (pass 2 sums 2 R), Pi = 128 state;
              // VN: Pb = state, Pi = H + 128 state
              const uint32_t sb = (raw << 7) & 0x80808080u;
              pb[i] = vn ? raw & 0x01010101u : raw & 0xFEFEFEFEu;
              pi[i] = vn ? ((raw >> 1) & 0x7F7F7F7Fu) | sb : sb;
            } else {  // bytes H + 128 state
              pb[i] = vn ? (raw >> 7) & 0x01010101u : raw & 0x7F7F7F7Fu;
              pi[i] = vn ? raw : raw & 0x80808080u;
            }
          }
          tmem_st_32x32b_x8(pb_col + 8 * c, pb);
          if constexpr (kH == 16) {
            // Pi holds row y at byte y - 16: words 0..3 of chunk c -> Pi words
            // 8c-4 .. 8c-1, words 4..7 -> 8c .. 8c+3 (rows 0..15, 144..159 unused)
            if (c > 0) tmem_st_32x32b_x4(pi_col + 8 * c - 4, pi[0], pi[1], pi[2], pi[3]);
            if (c < kBox / 32 - 1) tmem_st_32x32b_x4(pi_col + 8 * c, pi[4], pi[5], pi[6], pi[7]);
          } else {
            // Pi holds row y at byte y - 32: chunk c -> Pi chunk c - 1 (rows
            // 0..31, 160..191 unused)
            if (c > 0 && c < kBox / 32 - 1) tmem_st_32x32b_x8(pi_col + 8 * (c - 1), pi);
          }
        }
        tmem_st_wait();
        tc_fence_before();
        mbar_arrive(&a2_full[sl]);
        if (warp == 2 && lane == 0) LTL_TRACE(8, h);  // convert done (per-launch traces)
      }
    }
    }
    if constexpr (kChecked) {
      int32_t mh = static_cast<int32_t>(max_h);
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) mh = max(mh, __shfl_xor_sync(0xffffffffu, mh, off));
      if (lane == 0) atomicMax(&p.stats->max_h, mh);
    }
  } else if (warp == kWarpP2) {
    // ================= pass-2 MMA issuer =================
    // sub-block s: band over Pb chunks 2s .. 2s+nb-1 (box rows 64s ..
    // 64s+64+2kH-1), centre over Pi chunks 2s, 2s+1 (centre rows 64s .. 64s+63,
    // shifted)
    const uint64_t band_desc = smem_desc_sw32_kmajor(smem_u32(smem + kSmemBand));
    auto tile = [&](int t) { return band_desc + ((t * kTileBytes) >> 4); };
    const int ti = vn ? nb : nb + 2;
    uint32_t h = 0;
    for (int gg = 0; gg < p.gens; ++gg) {
    SegIter<kDyn> it(p, gg, seg);
    int band, t0, t1;
    while (it.next(band, t0, t1)) {
      for (int t = t0; t < t1; ++t, ++h) {
        const uint32_t sl = h % kSlots;
        LTL_WAIT(7, &a2_full[sl], (h / kSlots) & 1);
        for (int s = 0; s < kSubs; ++s) {
          if constexpr (G::kD2Bufs == kSubs) {
            LTL_WAIT(8, &d2_empty[s], (h & 1) ^ 1);
          } else if (s == 1) {  // sub-block 0's D2 lives in the slot (gated by slot_empty)
            LTL_WAIT(8, &d2_empty[1], (h & 1) ^ 1);
          }
          LTL_TRACE(4, 2 * h + s);
          tc_fence_after();
          if (elect_one()) {
            const uint32_t dcol = G::kD2Bufs == kSubs ? tmem + kTmemD2 + kSub * s
                                  : s == 0 ? tmem + kTmemSlot + kSlotCols * sl + G::kD2InSlot
                                           : tmem + kTmemD2;
            const uint32_t pb = tmem + kTmemSlot + kSlotCols * sl + kPbOff + 16 * s;
            const uint32_t pi = tmem + kTmemSlot + kSlotCols * sl + kPiOff + 16 * s;
#pragma unroll
            for (int c = 0; c < nb; ++c) mma_i8_ts(dcol, pb + 8 * c, tile(c), G::kIdesc2, c > 0);
#ifndef LTL_DIAG_NO_CENTRE  // timing probe only (wrong results): pass 2 without the centre chunks
            mma_i8_ts(dcol, pi, tile(ti), G::kIdesc2, 1);
            mma_i8_ts(dcol, pi + 8, tile(ti + 1), G::kIdesc2, 1);
#endif
            if (G::kD2Bufs != kSubs && s == 0) mma_commit(&d2_slot_full[sl]);
            else mma_commit(&d2_full[s]);
            if (s == kSubs - 1) mma_commit(&slot_empty[sl]);
          }
          __syncwarp();
        }
      }
    }
    }
  } else if (warp == kWarpStore) {
    // ================= store warp: staging tiles -> HBM, unit flags ==========
    // Issues every output TMA store (one 8 KB box per sub-block), frees the
    // staging slots once read, and in a multi-generation launch publishes
    // each unit to the next generation once both its stores have landed.
    // The gpu-scope release that needs costs ~1.4 us per batch (measured):
    // it must stay off the output groups' critical path.
    if (lane == 0) {
      constexpr int kPubLag = 8;          // units per publication batch
      uint32_t pend[2 * kPubLag];         // units stored, not yet published
      uint32_t npend = 0, h = 0, n_open = 0;  // n_open: committed, slot not yet freed
      int open_slot[2] = {0, 0};
      for (int gg = 0; gg < p.gens; ++gg) {
        SegIter<kDyn> it(p, gg, seg);
        int band, t0, t1;
        while (it.next(band, t0, t1)) {
          for (int t = t0; t < t1; ++t, ++h) {
            const uint32_t slot = h % kStageSlots;
            for (int grp = 0; grp < kSubs; ++grp) {
              mbar_wait(&st_full[grp * kStageSlots + slot], (h / kStageSlots) & 1);
              const uint8_t* src = smem + kSmemStage + (grp * kStageSlots + slot) * kStageBytes;
              tma_store_3d(&maps.store[gg & 1], src, 0, band * kBand + kSub * grp,
                           t % p.strips + 1);
              tma_store_commit();
              // the previous group's store has read its slot: free it
              tma_store_wait_read<1>();
              if (n_open) mbar_arrive(&st_empty[open_slot[0]]);
              open_slot[0] = grp * kStageSlots + slot;
              n_open = 1;
            }
            if (p.gens > 1) {
              pend[h % (2 * kPubLag)] = static_cast<uint32_t>(band * p.strips + t % p.strips);
              if (++npend == 2 * kPubLag) {
                tma_store_wait_all<2 * kPubLag>();  // 2 groups per unit
                fence_proxy_async_global();
                bool edge = false;  // ring: neighbours read edge-band units' counters
                if (kRing) {
                  const uint32_t lo = static_cast<uint32_t>(p.strips);  // band 0: [0, S)
                  const uint32_t hi = static_cast<uint32_t>(p.bands - 1) * lo;  // last band
                  for (int k = 0; k < kPubLag; ++k) {
                    const uint32_t u = pend[(h + 1 + k) % (2 * kPubLag)];
                    edge |= u < lo || u >= hi;
                  }
                }
                if (edge) fence_acq_rel_sys();
                else fence_acq_rel_gpu();           // one release for the batch
                for (int k = 0; k < kPubLag; ++k)
                  red_relaxed_add(p.flags + pend[(h + 1 + k) % (2 * kPubLag)], 2);
                npend -= kPubLag;
              }
            }
          }
        }
        if (p.gens > 1) {  // the generation's last units: publish them too
          tma_store_wait_all<0>();
          fence_proxy_async_global();
          if (kRing) fence_acq_rel_sys();
          else fence_acq_rel_gpu();
          for (uint32_t k = 0; k < npend; ++k)
            red_relaxed_add(p.flags + pend[(h - npend + k) % (2 * kPubLag)], 2);
          npend = 0;
        }
      }
      tma_store_wait_all<0>();
      (void)open_slot[1];
    }
  } else {
    // ================= output warps (D2 -> rule -> next generation) ==========
    // Group grp takes sub-block grp (64 rows) of every unit; warp w owns strip
    // columns 32*(w%4)..+32 of it as two 32 x 32 tiles (its own staging slots
    // and TMA stores: no CTA-wide barrier on this path).
    const uint32_t q = warp & 3;
    const uint32_t grp = (warp - kWarpOut0) >> 2;
    // D2 of this group's sub-block: its own buffer, or (kH = 32, group 0) the
    // free columns of unit h's D1 slot
    const bool d2_in_slot = G::kD2Bufs != kSubs && grp == 0;
    const uint32_t trow_base = tmem + ((q * 32) << 16);
    const uint32_t trow_fixed = trow_base + kTmemD2 + (G::kD2Bufs == kSubs ? kSub * grp : 0);
    const RuleConsts rc = p.rule;
    const uint32_t K = vn ? G::kVnK : 128u * G::kCentreW;  // Z = zs R + K state
    const uint32_t zs = kPk && !vn ? 2u : 1u;                  // 4-bit cells, Moore: 2 R
    SimdRule sr;
    sr.ca = (0x8000u - zs * rc.lo_dead) * 0x10001u;
    sr.cb = (0x7FFFu - zs * (rc.lo_dead + rc.w_dead)) * 0x10001u;
    sr.cc = (0x8000u - (K + zs * rc.lo_live)) * 0x10001u;
    sr.cd = (0x7FFFu - (K + zs * (rc.lo_live + rc.w_live))) * 0x10001u;
    const uint32_t g_live = (0x8000u - K) * 0x10001u;
    const uint32_t g_neg = (0x8000u - (K + zs * rc.neg_live)) * 0x10001u;
    const uint32_t r_mask = (K - 1) * 0x10001u;
    uint32_t max_r = 0, bad = 0;
    // staging: the group's whole 64-row x 128-column sub-block in one
    // SWIZZLE_128B tile (16-byte chunk c of row y at chunk c ^ (y & 7)), three
    // slots per group; each warp writes its 32 columns (chunks 2q, 2q+1) with
    // stmatrix.trans, thread `lane` addressing row 32 tt + lane; the store
    // warp then writes it with ONE TMA store (8 KB of contiguous strip rows).
    const uint8_t* grp_stage = smem + kSmemStage + grp * kStageSlots * kStageBytes;
    const uint32_t grp_stage_u32 = smem_u32(grp_stage);
    const bool leader = (warp & 3) == 0 && lane == 0;  // signals the store warp
    uint32_t st_off[2][2];  // [tile][16-byte half] byte offset within a slot
#pragma unroll
    for (int tt = 0; tt < 2; ++tt)
#pragma unroll
      for (int hh = 0; hh < 2; ++hh) {
        const uint32_t y = 32 * tt + lane, c = 2 * q + hh;
        // 4-bit cells: 64-byte rows, SWIZZLE_64B (chunk q ^ ((y >> 1) & 3)),
        // one 16-byte chunk (32 cells) per warp
        st_off[tt][hh] = kPk ? y * G::kRowBytes + ((q ^ ((y >> 1) & 3)) << 4)
                             : y * kStrip + ((c ^ (y & 7)) << 4);
      }
    uint32_t h = 0;
    for (int gg = 0; gg < p.gens; ++gg) {
    SegIter<kDyn> it(p, gg, seg);
    int band, t0, t1;
    while (it.next(band, t0, t1)) {
      for (int t = t0; t < t1; ++t, ++h) {
        if (d2_in_slot) LTL_WAIT(9 + (warp - kWarpOut0), &d2_slot_full[h % kSlots], (h / kSlots) & 1);
        else LTL_WAIT(9 + (warp - kWarpOut0), &d2_full[grp], h & 1);
        if (lane == 0 && warp == kWarpOut0) LTL_TRACE(5, h);
        if (lane == 0 && warp == kWarpOut0 + 4) LTL_TRACE(7, h);
        tc_fence_after();
        const uint32_t trow =
            d2_in_slot ? trow_base + kTmemSlot + kSlotCols * (h % kSlots) + G::kD2InSlot : trow_fixed;
        uint32_t z[2][2][8];  // [tile (rows 32*tt ..)][lane half][register]
#pragma unroll
        for (int tt = 0; tt < 2; ++tt) {
          tmem_ld_16x256b_x2_pack16(trow + 32 * tt, z[tt][0]);
          tmem_ld_16x256b_x2_pack16(trow + (16u << 16) + 32 * tt, z[tt][1]);
        }
        tmem_ld_wait();
        tc_fence_before();
        if (d2_in_slot) mbar_arrive(&slot_empty[h % kSlots]);
        else mbar_arrive(&d2_empty[grp]);
        if (lane == 0 && warp == kWarpOut0) LTL_TRACE(6, h);
        uint32_t w[2][2][4];  // [tile][lane half][stmatrix register]
#pragma unroll
        for (int tt = 0; tt < 2; ++tt) {
          if constexpr (kPk) {
            // registers jj (even column 2i) and jj + 2 (odd column 2i + 1)
            // of lane half hh make output byte 8 hh + i of the warp's 16:
            // register 2v + e = [rows (c, c+1) of half 0, of half 1]
#pragma unroll
            for (int v = 0; v < 2; ++v)
#pragma unroll
              for (int e = 0; e < 2; ++e) {
                const uint32_t ra0 = rule_pair(z[tt][0][4 * v + e], sr);
                const uint32_t ra1 = rule_pair(z[tt][1][4 * v + e], sr);
                const uint32_t rb0 = rule_pair(z[tt][0][4 * v + e + 2], sr);
                const uint32_t rb1 = rule_pair(z[tt][1][4 * v + e + 2], sr);
                // bytes [row c, row c+1] x [half 0, half 1]: even column 0x01, odd 0x10
                const uint32_t even = prmt(ra0, ra1, 0xFDB9) & 0x01010101u;
                const uint32_t odd = prmt(rb0, rb1, 0xFDB9);  // 0x00 / 0xFF bytes
                w[tt][0][2 * v + e] = lop3<0xF8>(even, odd, 0x10101010u);  // even | (odd & C)
              }
          } else {
#pragma unroll
            for (int hh = 0; hh < 2; ++hh) {
              const uint32_t* zz = z[tt][hh];
#pragma unroll
              for (int v = 0; v < 2; ++v) {
                const uint32_t a0 = rule_pair(zz[4 * v + 0], sr), b0 = rule_pair(zz[4 * v + 1], sr);
                const uint32_t a2 = rule_pair(zz[4 * v + 2], sr), b2 = rule_pair(zz[4 * v + 3], sr);
                w[tt][hh][2 * v + 0] = prmt(a0, a2, 0xFDB9) & 0x01010101u;
                w[tt][hh][2 * v + 1] = prmt(b0, b2, 0xFDB9) & 0x01010101u;
              }
            }
          }
        }
        const int ybase = band * kBand + kSub * static_cast<int>(grp);  // rows of tile 0
        if constexpr (kChecked) {
#pragma unroll
          for (int tt = 0; tt < 2; ++tt) {
            // register jj of lane half hh: strip column 16hh + lane/4 + 8((jj>>1)&1)
            // of this quarter, D2 columns c, c+1 with c = 4(lane%4) + 2(jj&1) + 16(jj>>2)
#pragma unroll
            for (int hh = 0; hh < 2; ++hh) {
#pragma unroll
              for (int jj = 0; jj < 8; ++jj) {
                const int xl = lane_x<kPk>(32 * static_cast<int>(q) + 16 * hh +
                                           static_cast<int>(lane >> 2) + 8 * ((jj >> 1) & 1)) -
                               32 * static_cast<int>(q);
                const int c = 4 * static_cast<int>(lane & 3) + 2 * (jj & 1) + 16 * (jj >> 2);
                const int y0 = ybase + 32 * tt;
                const bool xv = (t % p.strips) * kStrip + 32 * static_cast<int>(q) + xl < p.cols;
                const bool v0 = xv && y0 + out_row_of_col(c) < p.rows;
                const bool v1 = xv && y0 + out_row_of_col(c + 1) < p.rows;
                const uint32_t mask = (v0 ? 0xFFFFu : 0u) | (v1 ? 0xFFFF0000u : 0u);
                const uint32_t zz = z[tt][hh][jj];
                max_r = __vmaxu2(max_r, zz & r_mask & mask);
                const uint32_t neg = (zz + g_live) & ~(zz + g_neg) & 0x80008000u & mask;  // live, count < 0
                bad |= neg;
                if (neg) {  // rare (band faults only): where the reference would throw
#pragma unroll
                  for (int e = 0; e < 2; ++e) {
                    if (!((neg >> (16 * e)) & 0x8000u)) continue;
                    const int zl = static_cast<int>((zz >> (16 * e)) & 0xFFFFu);
                    const int cnt = (zl - static_cast<int>(K)) / static_cast<int>(zs) - rc.neg_live;  // < 0
                    const int y = p.row0 + y0 + out_row_of_col(c + e);
                    const int x = (t % p.strips) * kStrip + 32 * static_cast<int>(q) + xl;
                    atomicMin(&p.stats->first_negative,
                              negative_key(p.gen_base + gg, y, x, p.fault_f, p.cols, -cnt));
                  }
                }
              }
            }
          }
        }
        // hand the sub-block to the store warp through staging slot h % 3
        const uint32_t slot = h % kStageSlots;
        const uint32_t sa = grp_stage_u32 + slot * kStageBytes;
        mbar_wait(&st_empty[grp * kStageSlots + slot], ((h / kStageSlots) & 1) ^ 1);
#pragma unroll
        for (int tt = 0; tt < 2; ++tt) {
          stmatrix_x4_trans_b8(sa + st_off[tt][0], w[tt][0][0], w[tt][0][1], w[tt][0][2], w[tt][0][3]);
          if constexpr (!kPk)
            stmatrix_x4_trans_b8(sa + st_off[tt][1], w[tt][1][0], w[tt][1][1], w[tt][1][2], w[tt][1][3]);
        }
        fence_proxy_async_smem();
        named_barrier(1 + grp, kGroupThreads);
        if (leader) mbar_arrive(&st_full[grp * kStageSlots + slot]);
        if (lane == 0 && warp == kWarpOut0) LTL_TRACE(11, h);
      }
    }
    }
    if constexpr (kChecked) {
      int32_t mr = static_cast<int32_t>(max(max_r & 0xFFFF, max_r >> 16) / zs);
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) mr = max(mr, __shfl_xor_sync(0xffffffffu, mr, off));
      if (lane == 0) atomicMax(&p.stats->max_r, mr);
      if (__any_sync(0xffffffffu, bad != 0) && lane == 0) atomicOr(&p.stats->error, 1);
    }
  }

  __syncwarp();
  tc_fence_before();
  __syncthreads();
  LTL_TRACE_CTA(15);
  if (kRing && threadIdx.x == 0) {
    // Every store of this CTA has completed (the store warp waited for them
    // before the barrier).  One ticket per CTA; the launch's last CTA
    // publishes generation G + 1 to the neighbours.
    fence_proxy_async_global();
    fence_acq_rel_sys();
    if (atomicAdd(p.my_ticket, 1u) + 1u == gridDim.x) {
      *p.my_ticket = 0u;  // the next launch (after this grid completes) counts anew
      fence_acq_rel_sys();
      red_relaxed_add_sys(p.my_done, static_cast<uint32_t>(p.gens));  // generations completed
    }
  }
  if (kDyn && p.dyn && p.gens == 1 && p.bands >= static_cast<int32_t>(gridDim.x) &&
      threadIdx.x == 0) {
    // every segment of this CTA has been taken: the launch's last CTA rearms
    // the cursor for the next launch (which reads it after griddepcontrol.wait)
    __threadfence();
    if (atomicAdd(p.dyn + 1, 1u) + 1u == gridDim.x) {
      p.dyn[0] = 0u;
      p.dyn[1] = 0u;
      __threadfence();
    }
  }
  if (warp == 1) tmem_dealloc(tmem, kTmemCols);
}

}  // namespace

size_t tc_smem_bytes(int halo, bool packed) {
  return packed ? Geo<16, true>::kSmemAlloc : halo == 32 ? Geo<32>::kSmemAlloc : Geo<16>::kSmemAlloc;
}

// Multi-generation launches (SegIter's sweep): one CTA per SM, all resident.
// A generation boundary of one-launch-per-generation costs ~12.7 us (grid
// drain + refill: per-launch time = 12.7 us + 5.09 ns x units at 16384^2 ..
// 65536^2), the sweep ~5.5 ns per unit (its chunk edges re-read ~20 % more
// box bytes from L2) and no boundary: it wins below ~190 units per SM and
// generation (16384^2: 91.5 vs 98.5 us; 32768^2: 360 vs 349 us).  The torus
// must be tall enough for the sweep's (B - 2)-band dependency distance to
// clear the wavefront.  0 = one generation per launch.
int tc_persistent_ctas(int32_t rows, int32_t cols, int num_sms) {
  const int64_t bands = (rows + kBand - 1) / kBand;
  const int64_t units = bands * interior_strips(cols);
  if (std::getenv("LTL_FORCE_PERSIST"))  // tests: small tori, fewer CTAs
    return static_cast<int>(units < num_sms ? units : num_sms);
  // A small torus (at most two units per SM: 1024^2 has 64, 2048^2 256): a
  // generation is one or two latency-bound waves, and a launch per
  // generation costs more than the sweep's flag hand-over (GoL, us per
  // generation, launch per generation -> sweep: 1024^2 10.4 -> 8.0, 2048^2
  // 18.8 -> 12.7; 4096^2 22.2 -> 23.6 stays per launch;
  // profiles/small_torus_r02.txt).
  if (units <= 2LL * num_sms && !std::getenv("LTL_NO_SMALL_PERSIST"))
    return static_cast<int>(units < num_sms ? units : num_sms);
  // Middle sizes: 8192^2 (28 units per SM) runs 34.5 us per generation with
  // one launch each vs 38.3 in the sweep, 16384^2 (111 per SM) 95.5 vs 94.3
  // (same box, after the prologue fix; tools/gpu_r02ah.sh).
  return bands >= 16 && units >= 48LL * num_sms && units <= 190LL * num_sms ? num_sms : 0;
}

// Chunks per band of the multi-generation sweep: <= 16 units per chunk
// (16384^2, current kernel, tools/gpu_r02al.sh: 8 / 12 / 16 / 24 / 32 / 64 /
// 128 units -> 100.8 / 94.4 / 93.4 / 95.0 / 96.2 / 94.4 / 136.5 us), and no
// more units per chunk than units per CTA (a tiny torus: one unit per chunk,
// so every CTA gets one).
int tc_sweep_chunks(int32_t strips, int32_t bands, int ctas) {
  const int64_t per_cta = ctas > 0 ? static_cast<int64_t>(strips) * bands / ctas : 16;
  int per = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(16, per_cta)));
  if (const char* e = std::getenv("LTL_SWEEP_UNITS")) per = std::max(1, std::atoi(e));  // tuning
  return (strips + per - 1) / per;
}

cudaError_t launch_tc_step(const TcLaunch& a, cudaStream_t stream) {
  // The dynamic-SMEM attribute is per device: set it (and cache the SM count)
  // the first time each device launches (a process may drive several GPUs).
  constexpr int kMaxDevices = 64;
  static int sm_count[kMaxDevices] = {};
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  if (dev < 0 || dev >= kMaxDevices) return cudaErrorInvalidDevice;
  if (sm_count[dev] == 0) {
    auto set_smem = [](auto fn, uint32_t bytes) {
      return cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(bytes));
    };
    for (cudaError_t r : {set_smem(ltl_tc_step_kernel<16, false, false, false, false>, Geo<16>::kSmemAlloc),
                          set_smem(ltl_tc_step_kernel<16, true, false, false, false>, Geo<16>::kSmemAlloc),
                          set_smem(ltl_tc_step_kernel<16, false, true, false, false>, Geo<16>::kSmemAlloc),
                          set_smem(ltl_tc_step_kernel<16, true, true, false, false>, Geo<16>::kSmemAlloc),
                          set_smem(ltl_tc_step_kernel<32, false, false, false, false>, Geo<32>::kSmemAlloc),
                          set_smem(ltl_tc_step_kernel<32, true, false, false, false>, Geo<32>::kSmemAlloc),
                          set_smem(ltl_tc_step_kernel<32, false, true, false, false>, Geo<32>::kSmemAlloc),
                          set_smem(ltl_tc_step_kernel<32, true, true, false, false>, Geo<32>::kSmemAlloc),
                          set_smem(ltl_tc_step_kernel<16, false, false, true, false>, Geo<16, true>::kSmemAlloc),
                          set_smem(ltl_tc_step_kernel<16, true, false, true, false>, Geo<16, true>::kSmemAlloc),
                          set_smem(ltl_tc_step_kernel<16, false, false, false, true>, Geo<16>::kSmemAlloc),
                          set_smem(ltl_tc_step_kernel<16, true, false, false, true>, Geo<16>::kSmemAlloc)})
      if (r != cudaSuccess) return r;
    int sms = 0;
    e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (e != cudaSuccess) return e;
    sm_count[dev] = sms;
  }
  const int num_sms = sm_count[dev];
  if (a.rows <= 0 || a.cols <= 0) return cudaSuccess;
  Params p{};
  p.rows = a.rows;
  p.cols = a.cols;
  p.strips = interior_strips(a.cols);
  p.bands = (a.rows + kBand - 1) / kBand;
  p.rule = a.rule;
  p.inject_fault = a.inject_fault;
  p.fault_f = a.fault_f > 0 ? a.fault_f : 16;
  p.fault_row_phase = a.fault_row_phase;
  p.gen_base = a.gen_base;
  p.row0 = a.row0;
  p.wrap_cols = a.wrap_cols && tc_wrap_cols(a.cols);
  p.wrap_rows = a.wrap_rows && tc_wrap_rows(a.rows);
  p.gens = a.gens > 1 && a.flags && a.load_maps_b && a.store_map_b ? a.gens : 1;
  p.ring = a.ring && p.wrap_cols && tc_wrap_rows(a.rows) ? 1 : 0;
  if (a.ring && !p.ring) return cudaErrorInvalidValue;  // caller must not ask
  const int halo = a.halo == 32 ? 32 : 16;
  // 32-row boxes exist only where the loads do every wrap: the slab's own
  // 16-row HBM halo cannot hold 32 rows / columns
  if (a.halo != 0 && a.halo != 16 && a.halo != 32) return cudaErrorInvalidValue;
  if (halo == 32 && !(p.wrap_cols && (p.wrap_rows || p.ring))) return cudaErrorInvalidValue;
  // 4-bit cells: one whole-torus slab whose every wrap the loads do, r <= 16
  if (a.packed && (halo != 16 || p.ring || !(p.wrap_cols && p.wrap_rows))) return cudaErrorInvalidValue;
  if (p.ring) {
    p.wrap_rows = 0;
    p.up_flags = a.up_flags ? a.up_flags : a.flags;
    p.down_flags = a.down_flags ? a.down_flags : a.flags;
    p.ring_gen = a.ring_gen;
    p.up_rows = a.up_rows;
    p.up_done = a.up_done;
    p.down_done = a.down_done;
    p.my_done = a.my_done;
    p.my_ticket = a.my_ticket;
  }
  p.flags = a.flags;
  p.flag_base = a.flag_base;
  p.stats = a.stats;
  p.trace = a.trace;
  p.dyn = p.gens == 1 && !std::getenv("LTL_STATIC_SCHED") ? a.dyn : nullptr;  // env: A/B
  // One persistent CTA per SM over the units (fewer for small grids).
  const int64_t units = static_cast<int64_t>(p.bands) * p.strips;
  int64_t grid = units < num_sms ? units : num_sms;
  if (p.gens > 1) {
    grid = tc_persistent_ctas(a.rows, a.cols, num_sms);
    if (grid <= 0) return cudaErrorNotSupported;
    p.sweep_chunks = tc_sweep_chunks(p.strips, p.bands, static_cast<int>(grid));
  }
  if (a.grid > 0 && a.grid < grid) grid = a.grid;
  if (const char* e = std::getenv("LTL_TC_GRID")) {  // tuning knob (sweeps only)
    const int v = std::atoi(e);
    if (v >= 1 && v <= num_sms && v <= units) grid = v;
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(static_cast<unsigned>(grid));
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = tc_smem_bytes(halo, a.packed != 0);
  cfg.stream = stream;
  cudaLaunchAttribute attr[2];
  int nattr = 0;
  if (!std::getenv("LTL_NO_PDL")) {  // diagnostics
    attr[nattr].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[nattr].val.programmaticStreamSerializationAllowed = 1;
    ++nattr;
  }
  if (p.gens > 1) {
    // The multi-generation sweep hands units between CTAs through counters:
    // it is deadlock-free only with every CTA resident, which a cooperative
    // launch guarantees (the launch fails instead of hanging when the grid
    // cannot be co-resident, e.g. SMs held by another context).
    attr[nattr].id = cudaLaunchAttributeCooperative;
    attr[nattr].val.cooperative = 1;
    ++nattr;
  }
  cfg.attrs = attr;
  cfg.numAttrs = static_cast<unsigned>(nattr);
  TcMaps maps;
  for (int i = 0; i < kTcLoadMaps; ++i) {
    maps.load[0][i] = a.load_maps[i];
    maps.load[1][i] = a.load_maps_b ? a.load_maps_b[i] : a.load_maps[i];
  }
  maps.store[0] = *a.store_map;
  maps.store[1] = a.store_map_b ? *a.store_map_b : *a.store_map;
  for (int i = 0; i < 2; ++i) {
    maps.ring_up[i] = a.ring ? a.ring_up[i & (a.gens > 1 ? 1 : 0)] : *a.store_map;
    maps.ring_down[i] = a.ring ? a.ring_down[i & (a.gens > 1 ? 1 : 0)] : *a.store_map;
  }
  // the ring's peer-memory paths are compiled only into the ring kernels
  const bool st = a.stats != nullptr;
  if (a.packed)
    return st ? cudaLaunchKernelEx(&cfg, ltl_tc_step_kernel<16, true, false, true, false>, maps, p)
              : cudaLaunchKernelEx(&cfg, ltl_tc_step_kernel<16, false, false, true, false>, maps, p);
  if (halo == 32) {
    if (p.ring)
      return st ? cudaLaunchKernelEx(&cfg, ltl_tc_step_kernel<32, true, true, false, false>, maps, p)
                : cudaLaunchKernelEx(&cfg, ltl_tc_step_kernel<32, false, true, false, false>, maps, p);
    return st ? cudaLaunchKernelEx(&cfg, ltl_tc_step_kernel<32, true, false, false, false>, maps, p)
              : cudaLaunchKernelEx(&cfg, ltl_tc_step_kernel<32, false, false, false, false>, maps, p);
  }
  if (p.ring)
    return st ? cudaLaunchKernelEx(&cfg, ltl_tc_step_kernel<16, true, true, false, false>, maps, p)
              : cudaLaunchKernelEx(&cfg, ltl_tc_step_kernel<16, false, true, false, false>, maps, p);
  // the dynamic remainder schedule: u8 cells, one launch per generation with
  // whole-band rounds (32768^2 345 -> 339 us; elsewhere it does not pay,
  // tools/gpu_r02au/av.sh), compiled only into its own instantiations
  if (p.dyn && p.gens == 1 && p.bands >= grid)
    return st ? cudaLaunchKernelEx(&cfg, ltl_tc_step_kernel<16, true, false, false, true>, maps, p)
              : cudaLaunchKernelEx(&cfg, ltl_tc_step_kernel<16, false, false, false, true>, maps, p);
  return st ? cudaLaunchKernelEx(&cfg, ltl_tc_step_kernel<16, true, false, false, false>, maps, p)
            : cudaLaunchKernelEx(&cfg, ltl_tc_step_kernel<16, false, false, false, false>, maps, p);
}

}  // namespace ltl
