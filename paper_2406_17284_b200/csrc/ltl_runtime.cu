// ltl_runtime.cu -- implementation of the C-ABI in include/ltl_b200.h.
//
// Owns the device side of a run: the halo-padded slab buffers (two
// generations each), the TMA tensor maps, per-slab streams and the
// generation loop that replaces simulate / simulate_step
// (proj/src/cat_engine.cpp:260-321).  No CPU fallback exists: without a
// working device every call fails with LTL_ERR_CUDA.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <exception>
#include <sstream>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "host/internal.hpp"
#include "ltl_b200.h"
#include "ltl_kernels.cuh"
#include "ptx_sm100.cuh"

using ltl::kHalo;

namespace {

thread_local std::string g_last_error;

struct CudaFailure : std::runtime_error {
  using std::runtime_error::runtime_error;
};

void ck(cudaError_t e, const char* what) {
  if (e != cudaSuccess)
    throw CudaFailure(std::string("cuda error: ") + what + ": " + cudaGetErrorString(e));
}

struct Slab {
  int dev = 0;
  int32_t row0 = 0, rows = 0;  // global row of the first local row (init_random)
  int32_t host_row0 = 0;       // its row in the host buffers of upload / download
  int64_t strip_bytes = 0;
  int32_t strips = 0;
  uint8_t* buf[2] = {nullptr, nullptr};
  CUtensorMap load_maps[2][ltl::kTcLoadMaps];
  CUtensorMap load_maps_w[2][ltl::kTcLoadMaps];  // 32-row-halo boxes (r > 16)
  CUtensorMap store_map[2];
  ltl::DeviceStats* dstats = nullptr;
  uint32_t* flags = nullptr;   // per-unit completion counters (multi-generation launches)
  uint32_t* dyn = nullptr;     // dynamic schedule of one-generation launches (cursor, ticket)
  uint32_t flag_base = 0;      // their value between launches
  cudaStream_t stream = nullptr;
  bool own_stream = true;
  cudaEvent_t ev_step = nullptr;
  std::vector<cudaEvent_t> timing;
  // Ring of row slabs with the halo exchange fused into the step (ltl_tc.cu
  // Params::ring): the neighbours' buffers as 16-row piece maps and their
  // completion counters (peer-accessible here: same device, P2P, CUDA IPC).
  uint32_t* ring_sync = nullptr;              // [0] steps completed, [1] CTA ticket
  CUtensorMap ring_up_map[2], ring_down_map[2];  // per generation buffer
  CUtensorMap ring_up_map_w[2], ring_down_map_w[2];  // 32-row pieces (r > 16)
  const uint32_t* up_done = nullptr;
  const uint32_t* down_done = nullptr;
  int32_t up_rows = 0, down_rows = 0;
  // the neighbours' per-unit counters (multi-generation ring launches); a
  // neighbour that is this slab itself or runs on another GPU can run
  // concurrently with our persistent kernel, one sharing our GPU cannot
  const uint32_t* up_unit_flags = nullptr;
  const uint32_t* down_unit_flags = nullptr;
  bool up_concurrent = false, down_concurrent = false;
  bool ring_ready = false;                    // peers wired
  uint32_t ring_gen = 0;                      // steps since the last ring start
  std::vector<void*> ipc_opened;              // IPC mappings to close
  // 4-bit copy of the two generations (LTL_FLAG_4BIT_CELLS), allocated on
  // the first packed run, and its tensor maps
  uint8_t* pbuf[2] = {nullptr, nullptr};
  CUtensorMap pload_maps[2][ltl::kTcLoadMaps];
  CUtensorMap pstore_map[2];

  ltl::SlabView view(int which, int32_t cols) const {
    return ltl::SlabView{buf[which], rows, cols, strips, strip_bytes};
  }
  ltl::PackedView pview(int which, int32_t cols) const {
    return ltl::PackedView{pbuf[which], rows, cols, strips, strip_bytes / 2};
  }
};

}  // namespace

struct ltl_ctx {
  int32_t rows = 0, cols = 0, f = 16;
  int cur = 0;
  bool external_row_halo = false;
  bool halo_stale = false;  // halo cells the tcgen05 step does not need were not refreshed
  bool ring_stale = true;   // ring counters not (re)started since the last upload / init
  int64_t launches = 0;     // kernels this context has launched (ltl_kernel_launches)
  int32_t gen_counter = 0;  // generations enqueued since the last stats reset (negative_key)
  int64_t timed_launches = 0;  // inside the last ltl_time's timed loop
  uint8_t* pinned[2] = {nullptr, nullptr};  // snapshot streaming buffers (lazy)
  size_t pinned_bytes = 0;
  // bit-packed transfers: a device buffer of bits per device (lazy, grown)
  std::vector<std::pair<uint8_t*, size_t>> xbits;
  int64_t moved[2] = {0, 0};  // host -> device, device -> host bytes (ltl_transfer_bytes)
  std::vector<Slab> slabs;
  std::string err;
  // 4-bit cells: pk_live = the current generation is pbuf[pk_cur] (buf[cur] is
  // stale); pk_hold = keep it there between enqueues (inside ltl_time only:
  // every public call returns with the u8 slab current)
  bool pk_live = false, pk_hold = false;
  int pk_cur = 0;
};

namespace {

constexpr int kBusIdBytes = LTL_RING_HANDLE_BYTES - 4 * 64;  // PCI bus id after 4 IPC handles

int status_of(const std::exception& e) {
  if (dynamic_cast<const CudaFailure*>(&e)) return LTL_ERR_CUDA;
  if (dynamic_cast<const std::invalid_argument*>(&e)) return LTL_ERR_INVALID_ARGUMENT;
  if (dynamic_cast<const std::out_of_range*>(&e)) return LTL_ERR_INVALID_ARGUMENT;
  if (dynamic_cast<const std::logic_error*>(&e)) return LTL_ERR_LOGIC;
  return LTL_ERR_RUNTIME;
}

template <typename Fn>
int guarded(ltl_ctx* ctx, Fn&& fn) {
  try {
    fn();
    if (ctx) ctx->err.clear();
    g_last_error.clear();
    return LTL_OK;
  } catch (const std::exception& e) {
    if (ctx) ctx->err = e.what();
    g_last_error = e.what();
    return status_of(e);
  }
}

ltl::RuleConsts rule_consts(const ltl_rule_c& r) {
  const int mult = r.kind == LTL_KIND_MOORE ? 1 : 2;
  ltl::RuleConsts c{};
  c.r = r.r;
  c.kind = r.kind == LTL_KIND_MOORE ? 0 : 1;
  c.lo_dead = r.b1;
  c.w_dead = r.b2 - r.b1;
  c.lo_live = r.s1 + (mult - r.m);
  c.w_live = r.s2 - r.s1;
  c.neg_live = mult - r.m;
  return c;
}

bool stencil_engine(uint32_t flags) {
  return (flags & (LTL_FLAG_ENGINE_BASE | LTL_FLAG_ENGINE_PACK)) != 0;
}

bool wrap_cols(const ltl_ctx* ctx);
bool wrap_rows(const ltl_ctx* ctx);
bool ring_ok(const ltl_ctx* ctx);

// The wide-radius extension (LTL_FLAG_WIDE_RADIUS, 17 <= r <= 32): 32-row
// boxes whose every wrap is loaded by the step itself (the slabs' 16-row HBM
// halo cannot hold 32 rows / columns).
bool wide_geometry_ok(const ltl_ctx* ctx) {
  if (!wrap_cols(ctx)) return false;
  if (wrap_rows(ctx)) return true;
  if (!ring_ok(ctx)) return false;
  for (const Slab& s : ctx->slabs)
    if (s.up_rows < 2 * kHalo || s.down_rows < 2 * kHalo) return false;
  return true;
}

void check_run_args(const ltl_ctx* ctx, const ltl_rule_c* rule, int32_t steps,
                    uint32_t flags = 0) {
  if (!rule) throw std::invalid_argument("config error: rule is null");
  if (steps < 0) throw std::invalid_argument("config error: steps must be >= 0");
  const bool wide = (flags & LTL_FLAG_WIDE_RADIUS) && !stencil_engine(flags);
  catsim::validate_rule(catsim::from_c(*rule), wide ? catsim::kMaxWideRadius : catsim::kMaxRadius);
  // the CAT engine's band fragments need r <= f (src/fragment.cpp:25-27); the
  // stencil engines only need the device's 16-cell halo; the wide extension
  // has its own 32-row boxes
  const int32_t limit = stencil_engine(flags) ? kHalo
                        : wide                ? ltl::kTcMaxRadius
                                              : std::min<int32_t>(ctx->f, kHalo);
  if (rule->r < 1 || rule->r > limit)
    throw std::invalid_argument("unsupported radius r=" + std::to_string(rule->r) +
                                " for fragment side f=" + std::to_string(ctx->f));
  if (rule->r > kHalo && !wide_geometry_ok(ctx))
    throw std::invalid_argument(
        "unsupported radius r=" + std::to_string(rule->r) +
        ": r > 16 needs cols % 128 == 0 and slabs of rows % 32 == 0 (>= 32) whose row wrap the "
        "step loads (one whole-torus slab or a ring)");
}

void build_maps(Slab& s, int32_t cols) {
  for (int i = 0; i < 2; ++i) {
    ck(ltl::make_load_maps(s.load_maps[i], s.view(i, cols)), "tensor map (load)");
    if (s.rows >= 2 * kHalo)  // the wide boxes' 32-row pieces need 32 rows
      ck(ltl::make_load_maps(s.load_maps_w[i], s.view(i, cols), 2 * kHalo), "tensor map (load)");
    ck(ltl::make_store_map(&s.store_map[i], s.view(i, cols)), "tensor map (store)");
  }
}

struct RingPeer {
  const uint32_t* sync;
  uint8_t* const* buf;
  int32_t rows;
  const uint32_t* unit_flags;
  bool concurrent;  // itself, or on another GPU
};

void wire_ring(ltl_ctx* ctx, Slab& s, const RingPeer& upp, const RingPeer& dnp) {
  const uint32_t* up_sync = upp.sync;
  uint8_t* const* up_buf = upp.buf;
  const int32_t up_rows = upp.rows;
  const uint32_t* dn_sync = dnp.sync;
  uint8_t* const* dn_buf = dnp.buf;
  const int32_t dn_rows = dnp.rows;
  ck(cudaSetDevice(s.dev), "cudaSetDevice");
  const int32_t strips = ltl::storage_strips(ctx->cols);
  for (int b = 0; b < 2; ++b) {
    const ltl::SlabView up{up_buf[b], up_rows, ctx->cols, strips,
                           static_cast<int64_t>(up_rows + 2 * kHalo) * ltl::kStrip};
    const ltl::SlabView dn{dn_buf[b], dn_rows, ctx->cols, strips,
                           static_cast<int64_t>(dn_rows + 2 * kHalo) * ltl::kStrip};
    ck(ltl::make_piece_map(&s.ring_up_map[b], up), "tensor map (ring up)");
    ck(ltl::make_piece_map(&s.ring_down_map[b], dn), "tensor map (ring down)");
    if (up_rows >= 2 * kHalo && dn_rows >= 2 * kHalo) {
      ck(ltl::make_piece_map(&s.ring_up_map_w[b], up, 2 * kHalo), "tensor map (ring up)");
      ck(ltl::make_piece_map(&s.ring_down_map_w[b], dn, 2 * kHalo), "tensor map (ring down)");
    }
  }
  s.up_done = up_sync;
  s.down_done = dn_sync;
  s.up_rows = up_rows;
  s.down_rows = dn_rows;
  s.up_unit_flags = upp.unit_flags;
  s.down_unit_flags = dnp.unit_flags;
  s.up_concurrent = upp.concurrent;
  s.down_concurrent = dnp.concurrent;
  s.ring_ready = true;
}

void create_slabs(ltl_ctx* ctx, int32_t num_slabs, const int32_t* dev_ids) {
  int ndev = 0;
  ck(cudaGetDeviceCount(&ndev), "cudaGetDeviceCount");
  if (ndev <= 0) throw CudaFailure("cuda error: no CUDA device visible");
  if (num_slabs < 1) throw std::invalid_argument("config error: need at least one slab");
  if (num_slabs > 1 && ctx->rows / num_slabs < kHalo)
    throw std::invalid_argument("geometry error: " + std::to_string(num_slabs) + " slabs of " +
                                std::to_string(ctx->rows) +
                                " rows are thinner than the 16-row halo");
  ctx->slabs.resize(num_slabs);
  const int32_t base = ctx->rows / num_slabs, extra = ctx->rows % num_slabs;
  int32_t row0 = 0;
  for (int32_t i = 0; i < num_slabs; ++i) {
    Slab& s = ctx->slabs[i];
    s.dev = dev_ids ? dev_ids[i] : i % ndev;
    if (s.dev < 0 || s.dev >= ndev)
      throw std::invalid_argument("config error: device " + std::to_string(s.dev) +
                                  " not visible");
    s.row0 = row0;
    s.host_row0 = row0;
    s.rows = base + (i < extra ? 1 : 0);
    row0 += s.rows;
    s.strips = ltl::storage_strips(ctx->cols);
    s.strip_bytes = static_cast<int64_t>(s.rows + 2 * kHalo) * ltl::kStrip;
    ck(cudaSetDevice(s.dev), "cudaSetDevice");
    // every later operation of the slab is ordered on this stream, its zeroing
    // memsets included (a legacy-stream memset would not be ordered before
    // kernels on a non-blocking stream)
    ck(cudaStreamCreateWithFlags(&s.stream, cudaStreamNonBlocking), "cudaStreamCreate");
    const size_t bytes = static_cast<size_t>(s.strips) * s.strip_bytes;
    for (int b = 0; b < 2; ++b) {
      ck(cudaMalloc(&s.buf[b], bytes), "cudaMalloc slab");
      ck(cudaMemsetAsync(s.buf[b], 0, bytes, s.stream), "cudaMemset slab");
    }
    ck(cudaMalloc(&s.dstats, sizeof(ltl::DeviceStats)), "cudaMalloc stats");
    {
      const size_t units = static_cast<size_t>((s.rows + ltl::kTcBand - 1) / ltl::kTcBand) *
                           ltl::interior_strips(ctx->cols);
      ck(cudaMalloc(&s.flags, std::max<size_t>(units, 1) * sizeof(uint32_t)), "cudaMalloc flags");
      ck(cudaMemsetAsync(s.flags, 0, std::max<size_t>(units, 1) * sizeof(uint32_t), s.stream),
         "memset flags");
      ck(cudaMalloc(&s.dyn, 2 * sizeof(uint32_t)), "cudaMalloc schedule cursor");
      ck(cudaMemsetAsync(s.dyn, 0, 2 * sizeof(uint32_t), s.stream), "memset schedule cursor");
      ck(cudaMalloc(&s.ring_sync, 2 * sizeof(uint32_t)), "cudaMalloc ring counters");
      ck(cudaMemsetAsync(s.ring_sync, 0, 2 * sizeof(uint32_t), s.stream), "memset ring counters");
    }
    ck(cudaEventCreateWithFlags(&s.ev_step, cudaEventDisableTiming), "cudaEventCreate");
    build_maps(s, ctx->cols);
  }
  // peer access between distinct neighbouring devices (NVLink / NVSwitch)
  for (int32_t i = 0; i < num_slabs; ++i) {
    const int a = ctx->slabs[i].dev;
    for (int32_t d : {-1, 1}) {
      const int b = ctx->slabs[(i + d + num_slabs) % num_slabs].dev;
      if (a == b) continue;
      int can = 0;
      ck(cudaDeviceCanAccessPeer(&can, a, b), "cudaDeviceCanAccessPeer");
      if (!can)
        throw CudaFailure("cuda error: no peer access between devices " + std::to_string(a) +
                          " and " + std::to_string(b));
      ck(cudaSetDevice(a), "cudaSetDevice");
      const cudaError_t e = cudaDeviceEnablePeerAccess(b, 0);
      if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) ck(e, "enable peer access");
      cudaGetLastError();
    }
  }
  // in-process ring: every slab's neighbours are peer-accessible already
  // (a single whole-torus slab is its own ring neighbour: the self-ring)
  if (ltl::interior_strips(ctx->cols) > 0)
    for (int32_t i = 0; i < num_slabs; ++i) {
      Slab& s = ctx->slabs[i];
      const Slab& up = ctx->slabs[(i - 1 + num_slabs) % num_slabs];
      const Slab& dn = ctx->slabs[(i + 1) % num_slabs];
      wire_ring(ctx, s, RingPeer{up.ring_sync, up.buf, up.rows, up.flags, &up == &s || up.dev != s.dev},
                RingPeer{dn.ring_sync, dn.buf, dn.rows, dn.flags, &dn == &s || dn.dev != s.dev});
    }
  // the zeroing memsets are on the slabs' streams: complete them before any
  // other slab (or process, after ltl_ring_export) can touch the buffers
  for (Slab& s : ctx->slabs) {
    ck(cudaSetDevice(s.dev), "cudaSetDevice");
    ck(cudaStreamSynchronize(s.stream), "cudaStreamSynchronize");
  }
}

void destroy_ctx(ltl_ctx* ctx) {
  for (Slab& s : ctx->slabs) {
    cudaSetDevice(s.dev);
    if (s.stream) cudaStreamSynchronize(s.stream);
    for (auto& b : s.buf)
      if (b) cudaFree(b);
    for (auto& b : s.pbuf)
      if (b) cudaFree(b);
    if (s.dstats) cudaFree(s.dstats);
    if (s.flags) cudaFree(s.flags);
    if (s.dyn) cudaFree(s.dyn);
    for (void* ptr : s.ipc_opened) cudaIpcCloseMemHandle(ptr);
    if (s.ring_sync) cudaFree(s.ring_sync);
    if (s.ev_step) cudaEventDestroy(s.ev_step);
    for (cudaEvent_t e : s.timing) cudaEventDestroy(e);
    if (s.stream && s.own_stream) cudaStreamDestroy(s.stream);
  }
  for (size_t d = 0; d < ctx->xbits.size(); ++d)
    if (ctx->xbits[d].first) {
      cudaSetDevice(static_cast<int>(d));
      cudaFree(ctx->xbits[d].first);
    }
  ctx->xbits.clear();
  ctx->slabs.clear();
}

// Which periodic wraps the step kernel takes care of by itself, loading the
// images straight from the interior (ltl_kernels.cuh tc_wrap_*): the column
// wrap whenever cols % 128 == 0, the row wrap for one whole-torus slab with
// rows % 32 == 0.  Slabs whose rows come from neighbours keep their row halo.
bool wrap_cols(const ltl_ctx* ctx) {
  return ltl::tc_wrap_cols(ctx->cols) && !std::getenv("LTL_NO_WRAP");  // env: diagnostics
}
// A single whole-torus slab can also take its row wrap through the ring
// machinery with itself as both neighbours (LTL_SELF_RING, A/B diagnostics).
bool self_ring() { return std::getenv("LTL_SELF_RING") != nullptr; }
bool wrap_rows(const ltl_ctx* ctx) {
  return ctx->slabs.size() == 1 && !ctx->external_row_halo && !self_ring() &&
         ltl::tc_wrap_rows(ctx->slabs[0].rows) && !std::getenv("LTL_NO_WRAP");
}

void sync_all(ltl_ctx* ctx) {
  for (Slab& s : ctx->slabs) {
    ck(cudaSetDevice(s.dev), "cudaSetDevice");
    ck(cudaStreamSynchronize(s.stream), "cudaStreamSynchronize");
  }
}

// Rows exchanged by the step itself over the ring of slabs (fused halo):
// 128-aligned widths, 32-aligned slab heights, peers wired (in-process slabs
// at creation, processes by ltl_ring_connect).
bool ring_ok(const ltl_ctx* ctx) {
  if (!wrap_cols(ctx) || std::getenv("LTL_NO_RING")) return false;  // env: diagnostics
  if (ctx->slabs.size() == 1 && !ctx->external_row_halo && !self_ring())
    return false;  // torus wrap by the loads instead
  for (const Slab& s : ctx->slabs)
    if (!s.ring_ready || !ltl::tc_wrap_rows(s.rows)) return false;
  return true;
}

// (Re)start the ring after uploads / init: every slab's counters back to 0
// (generation 0 = the buffers as they are now).  No kernel of any slab may be
// running (callers sync first; processes put a barrier on both sides).
void start_ring(ltl_ctx* ctx) {
  for (Slab& s : ctx->slabs) {
    ck(cudaSetDevice(s.dev), "cudaSetDevice");
    ck(cudaStreamSynchronize(s.stream), "cudaStreamSynchronize");
    ck(cudaMemsetAsync(s.ring_sync, 0, 2 * sizeof(uint32_t), s.stream), "memset ring counters");
    s.ring_gen = 0;
    // per-unit counters restart too: the neighbours compare them with their own base
    const size_t units = static_cast<size_t>((s.rows + ltl::kTcBand - 1) / ltl::kTcBand) *
                         ltl::interior_strips(ctx->cols);
    ck(cudaMemsetAsync(s.flags, 0, std::max<size_t>(units, 1) * sizeof(uint32_t), s.stream),
       "memset flags");
    s.flag_base = 0;
  }
  sync_all(ctx);
}

// Halo refresh of generation buffer `which` on every slab (after all slabs'
// interiors for that generation are enqueued).  `for_tc`: only what the next
// tcgen05 step will read from HBM (the wraps it does not load itself); the
// halo is then marked stale for consumers that need all of it (the stencil).
void enqueue_halo(ltl_ctx* ctx, int which, bool for_tc = false) {
  const int32_t G = static_cast<int32_t>(ctx->slabs.size());
  for (int32_t i = 0; i < G; ++i) {
    Slab& s = ctx->slabs[i];
    Slab& up = ctx->slabs[(i - 1 + G) % G];
    Slab& dn = ctx->slabs[(i + 1) % G];
    ck(cudaSetDevice(s.dev), "cudaSetDevice");
    if (G > 1) {
      ck(cudaStreamWaitEvent(s.stream, up.ev_step, 0), "wait above");
      ck(cudaStreamWaitEvent(s.stream, dn.ev_step, 0), "wait below");
    }
    ltl::SlabView self = s.view(which, ctx->cols);
    ltl::SlabView above = up.view(which, ctx->cols);
    ltl::SlabView below = dn.view(which, ctx->cols);
    // rows of a part come from an external transport (ltl_unpack_halo)
    const int all = ctx->external_row_halo ? ltl::kHaloCols : ltl::kHaloCols | ltl::kHaloRows;
    int parts = all;
    if (for_tc) {
      if (wrap_cols(ctx)) parts &= ~ltl::kHaloCols;
      if (wrap_rows(ctx) || ring_ok(ctx)) parts &= ~ltl::kHaloRows;
    }
    ck(ltl::launch_halo_fill(self, above, below, parts, s.stream), "halo kernel");
    if (parts != 0 && s.rows > 0 && ctx->cols > 0) ++ctx->launches;
    if (i == 0) ctx->halo_stale = parts != all;
  }
}

// Several generations in ONE persistent launch (units handed from one
// generation to the next through per-unit flags, no halo traffic): one
// whole-torus slab whose wraps the loads do, tcgen05 engine.
// For a ring of slabs every slab needs the same geometry (the kernels compare
// each other's unit counters) and neighbours that run concurrently with it.
bool persistent_ok(const ltl_ctx* ctx, uint32_t flags) {
  if (stencil_engine(flags) || !wrap_cols(ctx) || std::getenv("LTL_NO_PERSIST"))
    return false;  // env: diagnostics
  const bool single = ctx->slabs.size() == 1 && wrap_rows(ctx);
  if (!single) {
    if (!ring_ok(ctx)) return false;
    for (const Slab& s : ctx->slabs)
      if (s.up_rows != s.rows || s.down_rows != s.rows || !s.up_concurrent || !s.down_concurrent)
        return false;
  }
  for (const Slab& s : ctx->slabs) {
    int sms = 0;
    ck(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, s.dev), "sm count");
    if (ltl::tc_persistent_ctas(s.rows, ctx->cols, sms) <= 0) return false;
  }
  return true;
}

// 4-bit cells (LTL_FLAG_4BIT_CELLS): the Cat engine on one whole-torus slab
// whose every wrap the step loads itself, r <= 16.
bool packed_ok(const ltl_ctx* ctx, uint32_t flags, const ltl::RuleConsts& rc) {
  if (stencil_engine(flags) || !(flags & LTL_FLAG_4BIT_CELLS)) return false;
  return rc.r <= kHalo && ctx->slabs.size() == 1 && wrap_cols(ctx) && wrap_rows(ctx) &&
         ctx->slabs[0].rows > 0;
}

// The 4-bit copy back into the u8 slab (buf[cur]) if it holds the current generation.
void settle_packed(ltl_ctx* ctx) {
  if (!ctx->pk_live) return;
  Slab& s = ctx->slabs[0];
  ck(cudaSetDevice(s.dev), "cudaSetDevice");
  ck(ltl::launch_unpack_cells(s.pview(ctx->pk_cur, ctx->cols), s.view(ctx->cur, ctx->cols),
                              s.stream),
     "unpack cells");
  ++ctx->launches;
  ctx->pk_live = false;
  enqueue_halo(ctx, ctx->cur, true);  // (the wraps are the loads': marks the halo stale)
}

// `gens` generations of the packed Cat step: pack buf[cur] (unless the copy is
// live), one persistent launch or one launch per generation ping-ponging the
// two 4-bit buffers, unpack into buf[cur] (unless pk_hold).
void enqueue_step_packed(ltl_ctx* ctx, const ltl::RuleConsts& rc, uint32_t flags,
                         bool want_stats, cudaEvent_t* kt0, cudaEvent_t* kt1, int32_t gens) {
  Slab& s = ctx->slabs[0];
  ck(cudaSetDevice(s.dev), "cudaSetDevice");
  if (!s.pbuf[0]) {
    const size_t bytes = static_cast<size_t>(s.strips) * (s.strip_bytes / 2);
    for (int b = 0; b < 2; ++b) {
      ck(cudaMalloc(&s.pbuf[b], bytes), "cudaMalloc 4-bit slab");
      ck(cudaMemsetAsync(s.pbuf[b], 0, bytes, s.stream), "memset 4-bit slab");
      ck(ltl::make_load_maps_packed(s.pload_maps[b], s.pview(b, ctx->cols)), "tensor map (load)");
      ck(ltl::make_store_map_packed(&s.pstore_map[b], s.pview(b, ctx->cols)), "tensor map (store)");
    }
  }
  if (!ctx->pk_live) {
    ck(ltl::launch_pack_cells(s.view(ctx->cur, ctx->cols), s.pview(ctx->pk_cur, ctx->cols),
                              s.stream),
       "pack cells");
    ++ctx->launches;
    ctx->pk_live = true;
  }
  const bool persist = gens > 1 && persistent_ok(ctx, flags);
  if (kt0) ck(cudaEventRecord(kt0[0], s.stream), "event");
  for (int32_t g = 0; g < (persist ? 1 : gens); ++g) {
    const int pc = ctx->pk_cur;
    ltl::TcLaunch a{};
    a.packed = 1;
    a.halo = kHalo;
    a.load_maps = s.pload_maps[pc];
    a.store_map = &s.pstore_map[1 - pc];
    a.wrap_cols = 1;
    a.wrap_rows = 1;
    if (persist) {
      a.load_maps_b = s.pload_maps[1 - pc];
      a.store_map_b = &s.pstore_map[pc];
      a.gens = gens;
      a.flags = s.flags;
      a.flag_base = s.flag_base;
      s.flag_base += 2u * static_cast<uint32_t>(gens);
    }
    a.rows = s.rows;
    a.cols = ctx->cols;
    a.rule = rc;
    a.dyn = s.dyn;
    a.inject_fault = (flags & LTL_FLAG_INJECT_FAULT) != 0;
    a.fault_f = ctx->f;
    a.fault_row_phase = s.row0 % ctx->f;
    a.gen_base = ctx->gen_counter + g;
    a.row0 = s.row0;
    a.stats = want_stats ? s.dstats : nullptr;
    ck(ltl::launch_tc_step(a, s.stream), "tcgen05 kernel (4-bit cells)");
    ++ctx->launches;
    if (!persist || (gens & 1)) ctx->pk_cur = 1 - pc;
  }
  if (kt1) ck(cudaEventRecord(kt1[0], s.stream), "event");
  ctx->gen_counter += gens;
  if (!ctx->pk_hold) settle_packed(ctx);
}

// `gens` generations (cur -> nxt -> ...): one persistent launch when
// persistent_ok (gens > 1), else gens x (main kernel per slab + halo of nxt).
void enqueue_step(ltl_ctx* ctx, const ltl::RuleConsts& rc, uint32_t flags, bool want_stats,
                  cudaEvent_t* kt0, cudaEvent_t* kt1, int32_t gens = 1) {
  if (gens <= 0) return;
  if (packed_ok(ctx, flags, rc)) {
    enqueue_step_packed(ctx, rc, flags, want_stats, kt0, kt1, gens);
    return;
  }
  settle_packed(ctx);
  const bool persist = gens > 1 && persistent_ok(ctx, flags);
  if (gens > 1 && !persist) {
    for (int32_t t = 0; t < gens; ++t) enqueue_step(ctx, rc, flags, want_stats, nullptr, nullptr);
    return;
  }
  const int cur = ctx->cur, nxt = 1 - cur;
  const bool ring = !stencil_engine(flags) && ring_ok(ctx);
  if (ring && ctx->ring_stale) {
    if (ctx->external_row_halo)
      throw std::logic_error(
          "sequencing error: ring halo not filled (ltl_ring_fill after upload / init)");
    start_ring(ctx);
    ctx->ring_stale = false;
  }
  if (stencil_engine(flags)) ctx->ring_stale = true;  // stencil generations bypass the ring
  if (ring && ctx->slabs.size() > 1) {
    // slabs sharing a device must not spin on each other's counters (a
    // waiting kernel can hold every SM): order each step after the
    // neighbours' previous one (ev_step); the counters then never block
    const int32_t G = static_cast<int32_t>(ctx->slabs.size());
    for (int32_t i = 0; i < G; ++i) {
      Slab& s = ctx->slabs[i];
      ck(cudaSetDevice(s.dev), "cudaSetDevice");
      ck(cudaStreamWaitEvent(s.stream, ctx->slabs[(i - 1 + G) % G].ev_step, 0), "wait above");
      ck(cudaStreamWaitEvent(s.stream, ctx->slabs[(i + 1) % G].ev_step, 0), "wait below");
    }
  }
  const bool fault = (flags & LTL_FLAG_INJECT_FAULT) != 0;
  for (size_t i = 0; i < ctx->slabs.size(); ++i) {
    Slab& s = ctx->slabs[i];
    ck(cudaSetDevice(s.dev), "cudaSetDevice");
    if (kt0) ck(cudaEventRecord(kt0[i], s.stream), "event");
    if (stencil_engine(flags)) {
      if (ctx->halo_stale) {  // the last tcgen05 steps left wrap-free halos
        ck(cudaSetDevice(s.dev), "cudaSetDevice");
        if (i == 0) enqueue_halo(ctx, cur);
        ck(cudaSetDevice(s.dev), "cudaSetDevice");
      }
      // the band fault is a CAT-engine hook (CatConfig.inject_band_fault,
      // src/cat_engine.cpp:277); the reference's BASE / PACK ignore it
      ck(ltl::launch_stencil_step(s.view(cur, ctx->cols), s.view(nxt, ctx->cols), rc,
                                  (flags & LTL_FLAG_ENGINE_PACK) ? ltl::kEnginePack
                                                                 : ltl::kEngineBase,
                                  want_stats ? s.dstats : nullptr, s.stream),
         "stencil kernel");
      ++ctx->launches;
    } else {
      ltl::TcLaunch a{};
      CUtensorMap ring_up2[2], ring_down2[2];  // the neighbours' buffers of gen 0, 1
      // r > 16 (the wide extension, validated by check_run_args): 32-row boxes
      const bool wide = rc.r > kHalo;
      a.halo = wide ? 2 * kHalo : kHalo;
      a.load_maps = wide ? s.load_maps_w[cur] : s.load_maps[cur];
      a.store_map = &s.store_map[nxt];
      a.wrap_cols = wrap_cols(ctx);
      a.wrap_rows = wrap_rows(ctx);
      if (ring) {
        a.ring = 1;
        a.ring_gen = s.ring_gen;
        s.ring_gen += persist ? static_cast<uint32_t>(gens) : 1u;
        a.up_rows = s.up_rows;
        ring_up2[0] = wide ? s.ring_up_map_w[cur] : s.ring_up_map[cur];
        ring_up2[1] = wide ? s.ring_up_map_w[nxt] : s.ring_up_map[nxt];
        ring_down2[0] = wide ? s.ring_down_map_w[cur] : s.ring_down_map[cur];
        ring_down2[1] = wide ? s.ring_down_map_w[nxt] : s.ring_down_map[nxt];
        a.ring_up = ring_up2;
        a.ring_down = ring_down2;
        a.up_flags = s.up_unit_flags;
        a.down_flags = s.down_unit_flags;
        a.up_done = s.up_done;
        a.down_done = s.down_done;
        a.my_done = s.ring_sync;
        a.my_ticket = s.ring_sync + 1;
      }
      if (persist) {
        a.load_maps_b = wide ? s.load_maps_w[nxt] : s.load_maps[nxt];
        a.store_map_b = &s.store_map[cur];
        a.gens = gens;
        a.flags = s.flags;
        a.flag_base = s.flag_base;
        s.flag_base += 2u * static_cast<uint32_t>(gens);
      }
      a.rows = s.rows;
      a.cols = ctx->cols;
      a.rule = rc;
      a.dyn = s.dyn;
      a.inject_fault = fault;
      // the reference's fault flips pi2(0,0) of every f x f fragment
      // (src/cat_engine.cpp:277): columns / rows == 0 mod f of the global torus
      a.fault_f = ctx->f;
      a.fault_row_phase = s.row0 % ctx->f;
      a.gen_base = ctx->gen_counter;
      a.row0 = s.row0;
      a.stats = want_stats ? s.dstats : nullptr;
      // Debug: LTL_TC_TRACE=<file> dumps the pipeline timeline of CTA 0 of
      // the first traced launch (16 event kinds x 256 stamps; 14/15 = per-CTA start/end ns).
      static int traced_launches = 0;
      const int trace_skip = std::getenv("LTL_TC_TRACE_SKIP") ? std::atoi(std::getenv("LTL_TC_TRACE_SKIP")) : 0;
      const char* trace_path = std::getenv("LTL_TC_TRACE");
      long long* dtrace = nullptr;
      if (trace_path && traced_launches++ == trace_skip && !want_stats) {
        ck(cudaMalloc(&dtrace, 16 * 256 * sizeof(long long)), "trace alloc");
        ck(cudaMemsetAsync(dtrace, 0, 16 * 256 * sizeof(long long), s.stream), "trace memset");
        a.trace = dtrace;
      }
      ck(ltl::launch_tc_step(a, s.stream), "tcgen05 kernel");
      if (s.rows > 0 && ctx->cols > 0) ++ctx->launches;
      if (dtrace) {
        std::vector<long long> h(16 * 256);
        ck(cudaStreamSynchronize(s.stream), "trace sync");
        ck(cudaMemcpy(h.data(), dtrace, h.size() * sizeof(long long), cudaMemcpyDeviceToHost),
           "trace copy");
        cudaFree(dtrace);
        if (FILE* fh = std::fopen(trace_path, "w")) {
          for (int e = 0; e < 16; ++e) {
            for (int k = 0; k < 256; ++k) std::fprintf(fh, "%s%lld", k ? "," : "", h[e * 256 + k]);
            std::fprintf(fh, "\n");
          }
          std::fclose(fh);
        }
      }
    }
    if (kt1) ck(cudaEventRecord(kt1[i], s.stream), "event");
    if (ctx->slabs.size() > 1) ck(cudaEventRecord(s.ev_step, s.stream), "event");
  }
  const int out = (gens % 2) ? nxt : cur;  // buffer holding the last generation
  enqueue_halo(ctx, out, !stencil_engine(flags));
  ctx->cur = out;
  ctx->gen_counter += gens;
}

void reset_stats(ltl_ctx* ctx) {
  for (Slab& s : ctx->slabs) {
    ck(cudaSetDevice(s.dev), "cudaSetDevice");
    ck(cudaMemsetAsync(s.dstats, 0, sizeof(ltl::DeviceStats), s.stream), "memset stats");
    ck(cudaMemsetAsync(&s.dstats->first_negative, 0xFF, sizeof(unsigned long long), s.stream),
       "memset stats");
  }
  ctx->gen_counter = 0;
}

void run_steps(ltl_ctx* ctx, const ltl_rule_c* rule, int32_t steps, uint32_t flags,
               ltl_stats_c* stats) {
  check_run_args(ctx, rule, steps, flags);
  const ltl::RuleConsts rc = rule_consts(*rule);
  // Checked launches (device max-reduction of H / R plus the negative-count
  // guard of src/rule.cpp:104-107) run when stats are requested or a band
  // fault is injected.  With intact bands the guard cannot fire -- every
  // reduction contains the centre `mult` times, so count >= 0 by
  // construction -- which is why the fast path may skip it.
  const bool checked = (flags & LTL_FLAG_INJECT_FAULT) || (stats && (flags & LTL_FLAG_WANT_STATS));
  reset_stats(ctx);
  enqueue_step(ctx, rc, flags, checked, nullptr, nullptr, steps);
  sync_all(ctx);
  ltl::DeviceStats agg{};
  agg.first_negative = ~0ULL;
  for (Slab& s : ctx->slabs) {
    ltl::DeviceStats h{};
    ck(cudaSetDevice(s.dev), "cudaSetDevice");
    ck(cudaMemcpy(&h, s.dstats, sizeof h, cudaMemcpyDeviceToHost), "stats readback");
    agg.max_h = std::max(agg.max_h, h.max_h);
    agg.max_r = std::max(agg.max_r, h.max_r);
    agg.error |= h.error;
    agg.first_negative = std::min(agg.first_negative, h.first_negative);
  }
  if (agg.error) {
    // the count of the first negative cell in the reference's traversal
    // (src/rule.cpp:104-107); engines without the key report the prefix only
    std::string msg = "internal consistency: negative neighborhood count";
    if (agg.first_negative != ~0ULL)
      msg += " " + std::to_string(-static_cast<int>(agg.first_negative & 7));
    throw std::logic_error(msg);
  }
  if (stats) {
    // CAT-fragment accounting (cat_engine.cpp:151-155, :198-202): 3 MMAs per
    // fragment of the H pass (all fragment rows, interior columns) and 3 per
    // interior fragment of the R pass, per step.  Wide radii (r > f, the
    // extension): 2 ceil(r / f) + 1 band fragments per pass.
    const int64_t fpr = (ctx->cols + 2LL * ctx->f) / ctx->f;
    const int64_t nbf = 2 * ((rule->r + ctx->f - 1) / ctx->f) + 1;
    const int64_t per_step = ctx->rows == ctx->cols && ctx->rows > 0
                                 ? nbf * fpr * (fpr - 2) + nbf * (fpr - 2) * (fpr - 2)
                                 : 0;
    stats->mma_count += per_step * steps;
    stats->steps += steps;
    stats->max_h = std::max(stats->max_h, steps > 0 ? agg.max_h : 0);
    stats->max_r = std::max(stats->max_r, steps > 0 ? agg.max_r : 0);
    stats->fragments_per_row = static_cast<int32_t>(fpr);
  }
}

// Host layout helpers (fragment-contiguous order: grid.hpp:20-25).
size_t host_index(int32_t layout, int32_t f, int32_t p, int32_t y, int32_t x) {
  if (layout == LTL_LAYOUT_ROW_MAJOR) return static_cast<size_t>(y) * p + x;
  const int32_t fpr = p / f;
  return (static_cast<size_t>(y / f) * fpr + x / f) * (static_cast<size_t>(f) * f) +
         static_cast<size_t>(y % f) * f + (x % f);
}

// Host rows land dense in the other generation buffer (one contiguous H2D
// copy), then the device scatters them into strips; downloads mirror that.
// The other buffer's contents are dead at these points (the next step
// rewrites its interior, and its pad bytes only ever meet zero band weights).
// ---- host <-> device rows, pinned or pageable
//
// Pinned host memory (cudaHostAlloc / registered): one pitched DMA.  Pageable
// memory (a std::vector, the reference's Grid::cells): staged through the
// context's two 32 MB pinned chunks -- the rows of chunk k are packed by up to
// 8 host threads while chunk k-1 is in flight -- instead of the driver's
// single-threaded per-row staging of a pageable cudaMemcpy2D (16384^2
// row-major upload: 24 ms, profiles/cpp_e2e_r02.txt).
constexpr size_t kStageChunk = 32u << 20;

void ensure_stage(ltl_ctx* ctx) {
  if (ctx->pinned_bytes >= kStageChunk) return;
  for (uint8_t*& p : ctx->pinned) {
    if (p) cudaFreeHost(p);
    p = nullptr;
    // portable: slabs on several devices stage through the same chunks
    ck(cudaHostAlloc(&p, kStageChunk, cudaHostAllocPortable), "cudaHostAlloc (staging chunk)");
  }
  ctx->pinned_bytes = kStageChunk;
}

bool host_pinned(const void* p) {
  cudaPointerAttributes a{};
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeHost;
}

// fn(row) for rows [0, nrows) on up to 8 threads (inline for small copies)
template <typename Fn>
void parallel_rows(int64_t nrows, size_t row_bytes, Fn&& fn) {
  const int64_t bytes = nrows * static_cast<int64_t>(row_bytes);
  const int hw = static_cast<int>(std::max(1u, std::thread::hardware_concurrency()));
  const int T = static_cast<int>(std::min<int64_t>({8, hw, std::max<int64_t>(1, bytes >> 22)}));
  if (T <= 1) {
    for (int64_t r = 0; r < nrows; ++r) fn(r);
    return;
  }
  std::vector<std::thread> pool;
  pool.reserve(T);
  for (int t = 0; t < T; ++t)
    pool.emplace_back([&, t] {
      for (int64_t r = nrows * t / T; r < nrows * (t + 1) / T; ++r) fn(r);
    });
  for (std::thread& th : pool) th.join();
}

// `nrows` rows of `row_bytes` at host pitch `pitch` -> dense device rows.
// Returns with the copies enqueued on `st` (pageable: completed up to the
// last chunk's DMA, which the caller's stream sync covers).
// ---- bit-packed transfers (host/xfer_bits.cpp): a grid crosses PCIe as one
// bit per cell.  The host packs / unpacks a 256 MB-of-cells chunk on all its
// cores (AVX-512BW / AVX2) while the previous chunk is in flight through the
// context's pinned chunks; the device expands / packs (ltl_layout.cu).  Used
// for >= 4 MB of rows of a multiple of 32 cells whose bytes are all 0 / 1
// (else the byte copies below run: the same bytes land either way).
// LTL_BYTE_TRANSFERS=1 keeps the byte copies (A/B).
constexpr size_t kBitsChunk = 8u << 20;  // bits per pipelined chunk (64 MB of cells)
bool use_bits(int64_t nrows, size_t row_bytes) {
  return row_bytes % 32 == 0 && row_bytes <= kStageChunk &&
         nrows * static_cast<int64_t>(row_bytes) >= (4LL << 20) &&
         ltl_host::bits_available() && !std::getenv("LTL_BYTE_TRANSFERS");
}

// `bytes` of bits + a flag word at device_bits_flag(.., bytes)
constexpr size_t bits_flag_offset(size_t bytes) { return (bytes + 255) / 256 * 256; }
uint8_t* device_bits(ltl_ctx* ctx, size_t bytes) {
  bytes = bits_flag_offset(bytes) + 256;
  int dev = 0;
  ck(cudaGetDevice(&dev), "cudaGetDevice");
  if (ctx->xbits.size() <= static_cast<size_t>(dev)) ctx->xbits.resize(dev + 1, {nullptr, 0});
  auto& b = ctx->xbits[dev];
  if (b.second < bytes) {
    if (b.first) ck(cudaFree(b.first), "cudaFree (bits)");
    b.first = nullptr;
    ck(cudaMalloc(&b.first, bytes), "cudaMalloc (bits)");
    b.second = bytes;
  }
  return b.first;
}

// false: a byte was not 0 / 1 (nothing usable written; copy bytes instead)
// strips != nullptr: the bits go straight into that slab view's interior
// (dense rows of the slab: row_bytes == its cols) instead of `dev`
bool h2d_bits(ltl_ctx* ctx, uint8_t* dev, const uint8_t* host, int64_t nrows, size_t row_bytes,
              size_t pitch, cudaStream_t st, const ltl::SlabView* strips = nullptr) {
  const size_t brow = row_bytes / 8;
  uint8_t* bits = device_bits(ctx, static_cast<size_t>(nrows) * brow);
  ensure_stage(ctx);
  const int64_t per = std::max<int64_t>(1, static_cast<int64_t>(kBitsChunk / brow));
  const int T = ltl_host::xfer_threads();
  cudaEvent_t ev[2];
  for (auto& e : ev) ck(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event");
  bool ok = true;
  for (int64_t r0 = 0, k = 0; r0 < nrows && ok; r0 += per, ++k) {
    const int64_t cnt = std::min(per, nrows - r0);
    if (k >= 2) ck(cudaEventSynchronize(ev[k % 2]), "staging");  // chunk buffer free again
    uint8_t* stage = ctx->pinned[k % 2];
    ok = ltl_host::cells_to_bits(host + r0 * pitch, pitch, row_bytes, cnt, stage, T);
    if (!ok) break;
    ck(cudaMemcpyAsync(bits + r0 * brow, stage, cnt * brow, cudaMemcpyHostToDevice, st), "upload");
    ctx->moved[0] += cnt * static_cast<int64_t>(brow);
    ck(cudaEventRecord(ev[k % 2], st), "event");
  }
  if (ok && strips) ck(ltl::launch_bits_to_strips(bits, *strips, st), "bits -> strips");
  else if (ok)
    ck(ltl::launch_bits_to_cells(bits, dev, nrows * static_cast<int64_t>(row_bytes), st),
       "bits -> cells");
  ck(cudaStreamSynchronize(st), "staging");
  for (auto& e : ev) cudaEventDestroy(e);
  return ok;
}

// false: a device byte was not 0 / 1 (nothing written; copy bytes instead)
bool d2h_bits(ltl_ctx* ctx, uint8_t* host, const uint8_t* dev, int64_t nrows, size_t row_bytes,
              size_t pitch, cudaStream_t st, const ltl::SlabView* strips = nullptr) {
  const size_t brow = row_bytes / 8;
  uint8_t* bits = device_bits(ctx, static_cast<size_t>(nrows) * brow);
  int32_t* dbad = reinterpret_cast<int32_t*>(bits + bits_flag_offset(static_cast<size_t>(nrows) * brow));
  ensure_stage(ctx);
  ck(cudaMemsetAsync(dbad, 0, sizeof(int32_t), st), "memset flag");
  if (strips) ck(ltl::launch_strips_to_bits(*strips, bits, dbad, st), "strips -> bits");
  else
    ck(ltl::launch_cells_to_bits(dev, bits, nrows * static_cast<int64_t>(row_bytes), dbad, st),
       "cells -> bits");
  int32_t hbad = 0;
  ck(cudaMemcpyAsync(&hbad, dbad, sizeof hbad, cudaMemcpyDeviceToHost, st), "flag");
  ck(cudaStreamSynchronize(st), "flag");
  if (hbad) return false;
  const int64_t per = std::max<int64_t>(1, static_cast<int64_t>(kBitsChunk / brow));
  const int64_t chunks = (nrows + per - 1) / per;
  const int T = ltl_host::xfer_threads();
  cudaEvent_t ev[2];
  for (auto& e : ev) ck(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event");
  auto issue = [&](int64_t k) {
    const int64_t r0 = k * per, cnt = std::min(per, nrows - r0);
    ck(cudaMemcpyAsync(ctx->pinned[k % 2], bits + r0 * brow, cnt * brow, cudaMemcpyDeviceToHost, st),
       "download");
    ctx->moved[1] += cnt * static_cast<int64_t>(brow);
    ck(cudaEventRecord(ev[k % 2], st), "event");
  };
  issue(0);
  for (int64_t k = 0; k < chunks; ++k) {
    if (k + 1 < chunks) issue(k + 1);  // its buffer's unpack (chunk k-1) is done
    ck(cudaEventSynchronize(ev[k % 2]), "staging");
    const int64_t r0 = k * per, cnt = std::min(per, nrows - r0);
    ltl_host::bits_to_cells(ctx->pinned[k % 2], host + r0 * pitch, pitch, row_bytes, cnt, T);
  }
  for (auto& e : ev) cudaEventDestroy(e);
  return true;
}

void h2d_rows(ltl_ctx* ctx, uint8_t* dev, const uint8_t* host, int64_t nrows, size_t row_bytes,
              size_t pitch, cudaStream_t st) {
  if (nrows <= 0 || row_bytes == 0) return;
  if (use_bits(nrows, row_bytes) && h2d_bits(ctx, dev, host, nrows, row_bytes, pitch, st)) return;
  ctx->moved[0] += nrows * static_cast<int64_t>(row_bytes);
  if (host_pinned(host) || row_bytes > kStageChunk) {
    ck(cudaMemcpy2DAsync(dev, row_bytes, host, pitch, row_bytes, nrows, cudaMemcpyHostToDevice, st),
       "upload");
    return;
  }
  ensure_stage(ctx);
  const int64_t per = static_cast<int64_t>(kStageChunk / row_bytes);
  cudaEvent_t ev[2];
  for (auto& e : ev) ck(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event");
  for (int64_t r0 = 0, k = 0; r0 < nrows; r0 += per, ++k) {
    const int64_t cnt = std::min(per, nrows - r0);
    if (k >= 2) ck(cudaEventSynchronize(ev[k % 2]), "staging");  // chunk buffer free again
    uint8_t* stage = ctx->pinned[k % 2];
    parallel_rows(cnt, row_bytes, [&](int64_t r) {
      std::memcpy(stage + r * row_bytes, host + (r0 + r) * pitch, row_bytes);
    });
    ck(cudaMemcpyAsync(dev + r0 * row_bytes, stage, cnt * row_bytes, cudaMemcpyHostToDevice, st),
       "upload");
    ck(cudaEventRecord(ev[k % 2], st), "event");
  }
  ck(cudaStreamSynchronize(st), "staging");
  for (auto& e : ev) cudaEventDestroy(e);
}

// dense device rows -> `nrows` rows at host pitch (synchronous on return).
void d2h_rows(ltl_ctx* ctx, uint8_t* host, const uint8_t* dev, int64_t nrows, size_t row_bytes,
              size_t pitch, cudaStream_t st) {
  if (nrows <= 0 || row_bytes == 0) return;
  if (use_bits(nrows, row_bytes) && d2h_bits(ctx, host, dev, nrows, row_bytes, pitch, st)) return;
  ctx->moved[1] += nrows * static_cast<int64_t>(row_bytes);
  if (host_pinned(host) || row_bytes > kStageChunk) {
    ck(cudaMemcpy2DAsync(host, pitch, dev, row_bytes, row_bytes, nrows, cudaMemcpyDeviceToHost, st),
       "download");
    ck(cudaStreamSynchronize(st), "download");
    return;
  }
  ensure_stage(ctx);
  const int64_t per = static_cast<int64_t>(kStageChunk / row_bytes);
  const int64_t chunks = (nrows + per - 1) / per;
  cudaEvent_t ev[2];
  for (auto& e : ev) ck(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event");
  auto issue = [&](int64_t k) {
    const int64_t r0 = k * per, cnt = std::min(per, nrows - r0);
    ck(cudaMemcpyAsync(ctx->pinned[k % 2], dev + r0 * row_bytes, cnt * row_bytes,
                       cudaMemcpyDeviceToHost, st),
       "download");
    ck(cudaEventRecord(ev[k % 2], st), "event");
  };
  issue(0);
  for (int64_t k = 0; k < chunks; ++k) {
    if (k + 1 < chunks) issue(k + 1);  // its buffer's unpack (chunk k-1) is done
    ck(cudaEventSynchronize(ev[k % 2]), "staging");
    const int64_t r0 = k * per, cnt = std::min(per, nrows - r0);
    const uint8_t* stage = ctx->pinned[k % 2];
    parallel_rows(cnt, row_bytes, [&](int64_t r) {
      std::memcpy(host + (r0 + r) * pitch, stage + r * row_bytes, row_bytes);
    });
  }
  for (auto& e : ev) cudaEventDestroy(e);
}

// Ring readers of our "dead" buffer.  Between steps the other generation
// buffer of a slab holds generation g-1 -- but a ring neighbour still running
// its step g-1 reads that buffer's edge rows (and a neighbour running step g
// reads the current one).  Uploads / downloads / snapshots use the dead
// buffer as their dense staging area and an upload rewrites the current one,
// so before them every ring neighbour must be past every step that reads our
// buffers: neighbours in this process -- all slabs' streams drained; in other
// processes -- a one-thread kernel on the slab's stream waits until their
// step counters reach ours (the steps read our buffers up to generation
// ring_gen - 1; a neighbour ahead is blocked on our counter before it reads
// generation ring_gen).
__global__ void ring_quiesce_kernel(const uint32_t* up_done, const uint32_t* down_done,
                                    uint32_t target) {
  ltl::ptx::wait_flag_geq_sys(up_done, target);
  ltl::ptx::wait_flag_geq_sys(down_done, target);
}

void quiesce_ring_readers(ltl_ctx* ctx) {
  if (!ring_ok(ctx)) return;
  if (ctx->slabs.size() > 1) sync_all(ctx);
  if (!ctx->external_row_halo) return;  // in-process ring: the streams are the order
  for (Slab& s : ctx->slabs) {
    if (!s.up_done || !s.down_done) continue;
    ck(cudaSetDevice(s.dev), "cudaSetDevice");
    ring_quiesce_kernel<<<1, 1, 0, s.stream>>>(s.up_done, s.down_done, s.ring_gen);
    ck(cudaGetLastError(), "ring quiesce");
    ++ctx->launches;
  }
}

void upload_interior(ltl_ctx* ctx, const uint8_t* interior) {
  quiesce_ring_readers(ctx);
  const int cur = ctx->cur;
  for (Slab& s : ctx->slabs) {
    ck(cudaSetDevice(s.dev), "cudaSetDevice");
    if (s.rows == 0 || ctx->cols == 0) continue;
    const uint8_t* src = interior + static_cast<size_t>(s.host_row0) * ctx->cols;
    const ltl::SlabView v = s.view(cur, ctx->cols);
    if (use_bits(s.rows, ctx->cols) &&
        h2d_bits(ctx, nullptr, src, s.rows, ctx->cols, ctx->cols, s.stream, &v)) {
      ++ctx->launches;     // bits -> strips
    } else {
      h2d_rows(ctx, s.buf[1 - cur], src, s.rows, ctx->cols, ctx->cols, s.stream);
      ck(ltl::launch_to_strips(s.buf[1 - cur], v, s.stream), "to_strips");
      ++ctx->launches;
    }
    if (ctx->slabs.size() > 1) ck(cudaEventRecord(s.ev_step, s.stream), "event");
  }
  enqueue_halo(ctx, cur);
  sync_all(ctx);
  ctx->ring_stale = true;
}

void download_interior(ltl_ctx* ctx, uint8_t* interior) {
  quiesce_ring_readers(ctx);
  const int cur = ctx->cur;
  for (Slab& s : ctx->slabs) {
    ck(cudaSetDevice(s.dev), "cudaSetDevice");
    if (s.rows == 0 || ctx->cols == 0) continue;
    const size_t n = static_cast<size_t>(s.rows) * ctx->cols;
    uint8_t* dst = interior + static_cast<size_t>(s.host_row0) * ctx->cols;
    const ltl::SlabView v = s.view(cur, ctx->cols);
    if (use_bits(s.rows, ctx->cols) &&
        d2h_bits(ctx, dst, nullptr, s.rows, ctx->cols, ctx->cols, s.stream, &v)) {
      ++ctx->launches;  // strips -> bits
      continue;
    }
    ck(ltl::launch_from_strips(v, s.buf[1 - cur], s.stream), "from_strips");
    ++ctx->launches;
    d2h_rows(ctx, dst, s.buf[1 - cur], static_cast<int64_t>(n / ctx->cols), ctx->cols, ctx->cols,
             s.stream);
  }
  sync_all(ctx);
}

void check_layout(int32_t layout) {
  if (layout != LTL_LAYOUT_ROW_MAJOR && layout != LTL_LAYOUT_FRAGMENT)
    throw std::invalid_argument("layout error: unknown layout " + std::to_string(layout));
}

// Periodic halo of a padded (n + 2f)^2 host grid (fill_periodic_halo,
// src/grid.cpp:75-94: halo cell (y, x) = interior image ((y-f) mod n, (x-f) mod n)).
// Row-major: the side columns of every interior row, then whole halo rows,
// as memcpys.  Fragment-contiguous: per halo cell (4fn + 4f^2 of them).
void host_fill_halo(uint8_t* padded, int32_t n, int32_t f, int32_t layout) {
  const size_t p = static_cast<size_t>(n) + 2 * f;
  if (n == 0) {
    std::memset(padded, 0, p * p);
    return;
  }
  auto wrapi = [n](int64_t v) { return static_cast<int32_t>(((v % n) + n) % n); };
  if (layout == LTL_LAYOUT_ROW_MAJOR) {
    for (int32_t y = f; y < f + n; ++y) {
      uint8_t* row = padded + y * p;
      for (int32_t x = 0; x < f; ++x) row[x] = row[f + wrapi(x - f)];
      for (int32_t x = f + n; x < n + 2 * f; ++x) row[x] = row[f + wrapi(x - f)];
    }
    for (int32_t y = 0; y < f; ++y)
      std::memcpy(padded + y * p, padded + (f + wrapi(y - f)) * p, p);
    for (int32_t y = f + n; y < n + 2 * f; ++y)
      std::memcpy(padded + y * p, padded + (f + wrapi(y - f)) * p, p);
    return;
  }
  const int32_t pp = n + 2 * f;
  for (int32_t y = 0; y < pp; ++y) {
    const bool halo_row = y < f || y >= f + n;
    for (int32_t x = 0; x < pp; ++x) {
      if (!halo_row && x == f) x = f + n;  // skip the interior span of interior rows
      if (x >= pp) break;
      padded[host_index(layout, f, pp, y, x)] =
          padded[host_index(layout, f, pp, f + wrapi(y - f), f + wrapi(x - f))];
    }
  }
}

// Padded host grid (either layout) -> device: the interior goes H2D as ONE
// pitched copy per slab (row-major: n-byte rows at pitch n + 2f; fragment
// order: the interior fragments of each fragment row, contiguous, at pitch
// f (n + 2f)) into the slab's dead generation buffer, and a relayout kernel
// scatters it into strips.  No host pass over the cells.
void upload_padded(ltl_ctx* ctx, const uint8_t* padded, int32_t layout) {
  quiesce_ring_readers(ctx);
  const int32_t n = ctx->rows, f = ctx->f;
  const size_t p = static_cast<size_t>(n) + 2 * f;
  const int cur = ctx->cur;
  const bool kernel_f = f == 4 || f == 8 || f == 16;
  for (const Slab& s : ctx->slabs)
    if (layout == LTL_LAYOUT_FRAGMENT && (!kernel_f || s.host_row0 % f || s.rows % f)) {
      // fragment rows straddling slabs: gather the interior on the host
      std::vector<uint8_t> interior(static_cast<size_t>(n) * n);
      for (int32_t y = 0; y < n; ++y)
        for (int32_t x0 = 0; x0 < n; x0 += f)
          std::memcpy(&interior[static_cast<size_t>(y) * n + x0],
                      padded + host_index(layout, f, static_cast<int32_t>(p), y + f, x0 + f), f);
      upload_interior(ctx, interior.data());
      return;
    }
  for (Slab& s : ctx->slabs) {
    ck(cudaSetDevice(s.dev), "cudaSetDevice");
    if (s.rows == 0 || n == 0) continue;
    uint8_t* dense = s.buf[1 - cur];
    if (layout == LTL_LAYOUT_ROW_MAJOR) {
      h2d_rows(ctx, dense, padded + (f + static_cast<size_t>(s.host_row0)) * p + f, s.rows, n, p,
               s.stream);
      ck(ltl::launch_to_strips(dense, s.view(cur, ctx->cols), s.stream), "to_strips");
    } else {
      const size_t frow = static_cast<size_t>(f) * p;  // bytes per fragment row
      h2d_rows(ctx, dense, padded + (s.host_row0 / f + 1) * frow + static_cast<size_t>(f) * f,
               s.rows / f, static_cast<size_t>(n) * f, frow, s.stream);
      ck(ltl::launch_frag_relayout(dense, s.view(cur, ctx->cols), f, true, s.stream),
         "fragment to_strips");
    }
    ++ctx->launches;
    if (ctx->slabs.size() > 1) ck(cudaEventRecord(s.ev_step, s.stream), "event");
  }
  enqueue_halo(ctx, cur);
  sync_all(ctx);
  ctx->ring_stale = true;
}

// Device -> padded host grid: a relayout kernel gathers the interior into the
// dead buffer in the host's order and ONE pitched D2H per slab lands it in the
// interior of `padded`; the halo bytes are untouched unless fill_halo (then
// the periodic images are written on the host: 4fn + 4f^2 cells).
void download_padded(ltl_ctx* ctx, uint8_t* padded, int32_t layout, bool fill_halo) {
  quiesce_ring_readers(ctx);
  const int32_t n = ctx->rows, f = ctx->f;
  const size_t p = static_cast<size_t>(n) + 2 * f;
  const int cur = ctx->cur;
  bool host_path = false;
  const bool kernel_f = f == 4 || f == 8 || f == 16;
  for (const Slab& s : ctx->slabs)
    host_path |= layout == LTL_LAYOUT_FRAGMENT && (!kernel_f || s.host_row0 % f || s.rows % f);
  if (host_path) {
    std::vector<uint8_t> interior(static_cast<size_t>(n) * n);
    download_interior(ctx, interior.data());
    for (int32_t y = 0; y < n; ++y)
      for (int32_t x0 = 0; x0 < n; x0 += f)
        std::memcpy(padded + host_index(layout, f, static_cast<int32_t>(p), y + f, x0 + f),
                    &interior[static_cast<size_t>(y) * n + x0], f);
  } else {
    for (Slab& s : ctx->slabs) {
      ck(cudaSetDevice(s.dev), "cudaSetDevice");
      if (s.rows == 0 || n == 0) continue;
      uint8_t* dense = s.buf[1 - cur];
      if (layout == LTL_LAYOUT_ROW_MAJOR) {
        ck(ltl::launch_from_strips(s.view(cur, ctx->cols), dense, s.stream), "from_strips");
        d2h_rows(ctx, padded + (f + static_cast<size_t>(s.host_row0)) * p + f, dense, s.rows, n, p,
                 s.stream);
      } else {
        ck(ltl::launch_frag_relayout(dense, s.view(cur, ctx->cols), f, false, s.stream),
           "fragment from_strips");
        const size_t frow = static_cast<size_t>(f) * p;
        d2h_rows(ctx, padded + (s.host_row0 / f + 1) * frow + static_cast<size_t>(f) * f, dense,
                 s.rows / f, static_cast<size_t>(n) * f, frow, s.stream);
      }
      ++ctx->launches;
    }
    sync_all(ctx);
  }
  if (fill_halo) host_fill_halo(padded, n, f, layout);
}

}  // namespace

extern "C" {

const char* ltl_build_info(void) {
  return "ltl_b200 abi=5 arch=sm_100a layout=column-strips-128 "
         "engines=cat(tcgen05-banded-i8:sweep,ring;4bit:tcgen05-f8f6f4),base(cuda-core-direct),"
         "pack(cuda-core-sliding) "
         "kernels=halo,relayout,fragment-relayout,init,snapshot,cell-pack,bit-transfer";
}

int ltl_create_torus(ltl_ctx** out, int32_t rows, int32_t cols, int32_t num_slabs,
                     const int32_t* dev_ids) {
  if (!out) return LTL_ERR_INVALID_ARGUMENT;
  *out = nullptr;
  ltl_ctx* ctx = new ltl_ctx;
  const int st = guarded(nullptr, [&] {
    if (rows < 0 || cols < 0)
      throw std::invalid_argument("geometry error: torus sides must be non-negative");
    if ((rows == 0) != (cols == 0))
      throw std::invalid_argument("geometry error: empty torus must be 0 x 0");
    ctx->rows = rows;
    ctx->cols = cols;
    ctx->f = 16;
    create_slabs(ctx, num_slabs, dev_ids);
  });
  if (st != LTL_OK) {
    destroy_ctx(ctx);
    delete ctx;
    return st;
  }
  *out = ctx;
  return LTL_OK;
}

int ltl_create(ltl_ctx** out, int32_t n, int32_t f, int32_t num_slabs, const int32_t* dev_ids) {
  if (!out) return LTL_ERR_INVALID_ARGUMENT;
  *out = nullptr;
  const int st = guarded(nullptr, [&] {
    if (f != 4 && f != 8 && f != 16)
      throw std::invalid_argument("config error: fragment side must be 4, 8, or 16");
    if (n < 0 || n % f != 0)
      throw std::invalid_argument("geometry error: n (" + std::to_string(n) +
                                  ") must be a non-negative multiple of f (" +
                                  std::to_string(f) + ")");
  });
  if (st != LTL_OK) return st;
  const int st2 = ltl_create_torus(out, n, n, num_slabs, dev_ids);
  if (st2 == LTL_OK) (*out)->f = f;
  return st2;
}

int32_t ltl_persistent_ok(ltl_ctx* ctx, uint32_t flags) {
  if (!ctx) return 0;
  int32_t ok = 0;
  guarded(ctx, [&] { ok = persistent_ok(ctx, flags) ? 1 : 0; });
  return ok;
}

int ltl_create_grid(ltl_ctx** out, int32_t n, int32_t f) {
  if (!out) return LTL_ERR_INVALID_ARGUMENT;
  *out = nullptr;
  const int st = guarded(nullptr, [&] {
    if (f <= 0) throw std::invalid_argument("geometry error: f must be positive");
    if (n < 0 || n % f != 0)
      throw std::invalid_argument("geometry error: n (" + std::to_string(n) +
                                  ") must be a non-negative multiple of f (" +
                                  std::to_string(f) + ")");
  });
  if (st != LTL_OK) return st;
  const int st2 = ltl_create_torus(out, n, n, 1, nullptr);
  if (st2 == LTL_OK) (*out)->f = f;
  return st2;
}

void ltl_destroy(ltl_ctx* ctx) {
  if (!ctx) return;
  destroy_ctx(ctx);
  for (uint8_t* p : ctx->pinned)
    if (p) cudaFreeHost(p);
  delete ctx;
}

int64_t ltl_kernel_launches(const ltl_ctx* ctx) { return ctx ? ctx->launches : -1; }

int64_t ltl_time_launches(const ltl_ctx* ctx) { return ctx ? ctx->timed_launches : 0; }

int64_t ltl_transfer_bytes(const ltl_ctx* ctx, int32_t dir) {
  return ctx && (dir == 0 || dir == 1) ? ctx->moved[dir] : 0;
}

const char* ltl_last_error(const ltl_ctx* ctx) {
  return ctx ? ctx->err.c_str() : g_last_error.c_str();
}

int32_t ltl_rows(const ltl_ctx* ctx) { return ctx ? ctx->rows : -1; }
int32_t ltl_cols(const ltl_ctx* ctx) { return ctx ? ctx->cols : -1; }
int32_t ltl_num_slabs(const ltl_ctx* ctx) {
  return ctx ? static_cast<int32_t>(ctx->slabs.size()) : -1;
}

int ltl_upload_interior(ltl_ctx* ctx, const uint8_t* interior) {
  if (!ctx) return LTL_ERR_INVALID_ARGUMENT;
  return guarded(ctx, [&] {
    if (!interior && ctx->rows > 0) throw std::invalid_argument("config error: null buffer");
    upload_interior(ctx, interior);
  });
}

int ltl_download_interior(ltl_ctx* ctx, uint8_t* interior) {
  if (!ctx) return LTL_ERR_INVALID_ARGUMENT;
  return guarded(ctx, [&] {
    if (!interior && ctx->rows > 0) throw std::invalid_argument("config error: null buffer");
    download_interior(ctx, interior);
  });
}

int ltl_upload(ltl_ctx* ctx, const uint8_t* padded, int32_t layout) {
  if (!ctx) return LTL_ERR_INVALID_ARGUMENT;
  return guarded(ctx, [&] {
    check_layout(layout);
    if (ctx->rows != ctx->cols) throw std::invalid_argument("layout error: padded grids are square");
    if (!padded && ctx->rows > 0) throw std::invalid_argument("config error: null buffer");
    upload_padded(ctx, padded, layout);
  });
}

int ltl_download(ltl_ctx* ctx, uint8_t* padded, int32_t layout) {
  return ltl_download_padded(ctx, padded, layout, 1);
}

int ltl_download_padded(ltl_ctx* ctx, uint8_t* padded, int32_t layout, int32_t fill_halo) {
  if (!ctx) return LTL_ERR_INVALID_ARGUMENT;
  return guarded(ctx, [&] {
    check_layout(layout);
    if (ctx->rows != ctx->cols) throw std::invalid_argument("layout error: padded grids are square");
    if (!padded) throw std::invalid_argument("config error: null buffer");
    download_padded(ctx, padded, layout, fill_halo != 0);
  });
}

int ltl_host_fill_halo(uint8_t* padded, int32_t n, int32_t f, int32_t layout) {
  if (!padded) return LTL_ERR_INVALID_ARGUMENT;
  return guarded(nullptr, [&] {
    check_layout(layout);
    if (f <= 0 || n < 0 || n % f != 0)
      throw std::invalid_argument("geometry error: n (" + std::to_string(n) +
                                  ") must be a non-negative multiple of f (" + std::to_string(f) +
                                  ")");
    host_fill_halo(padded, n, f, layout);
  });
}

int ltl_run(ltl_ctx* ctx, const ltl_rule_c* rule, int32_t steps, uint32_t flags,
            ltl_stats_c* stats) {
  if (!ctx) return LTL_ERR_INVALID_ARGUMENT;
  return guarded(ctx, [&] { run_steps(ctx, rule, steps, flags, stats); });
}

int ltl_run_async(ltl_ctx* ctx, const ltl_rule_c* rule, int32_t steps, uint32_t flags) {
  if (!ctx) return LTL_ERR_INVALID_ARGUMENT;
  return guarded(ctx, [&] {
    check_run_args(ctx, rule, steps, flags);
    const ltl::RuleConsts rc = rule_consts(*rule);
    enqueue_step(ctx, rc, flags, false, nullptr, nullptr, steps);
  });
}

int ltl_synchronize(ltl_ctx* ctx) {
  if (!ctx) return LTL_ERR_INVALID_ARGUMENT;
  return guarded(ctx, [&] { sync_all(ctx); });
}

int ltl_time(ltl_ctx* ctx, const ltl_rule_c* rule, int32_t steps, int32_t warmup,
             uint32_t flags, double* total_ms, double* kernel_ms) {
  if (!ctx) return LTL_ERR_INVALID_ARGUMENT;
  return guarded(ctx, [&] {
    check_run_args(ctx, rule, steps, flags);
    const ltl::RuleConsts rc = rule_consts(*rule);
    const size_t G = ctx->slabs.size();
    // 4-bit cells: the copy stays current across the warm-up, timed and
    // sampled generations (converted once, outside the timed region); the
    // u8 slab is brought back up to date before the call returns
    struct Hold {
      ltl_ctx* c;
      ~Hold() {
        c->pk_hold = false;
        try {
          settle_packed(c);
          sync_all(c);
        } catch (...) {
        }
      }
    } hold{ctx};
    ctx->pk_hold = true;
    enqueue_step(ctx, rc, flags, false, nullptr, nullptr, warmup);
    sync_all(ctx);
    // one persistent launch for all timed generations when possible
    const bool persist = steps > 1 && persistent_ok(ctx, flags);
    // pass 1 (total): events only around the whole loop -- an event between
    // two kernels would cut their programmatic (PDL) overlap
    // pass 2 (kernel): a sample of up to 100 generations, one event pair
    // around every launch; the average x steps is the kernel time
    const int32_t sample = kernel_ms && !persist ? std::min<int32_t>(steps, 100) : 0;
    for (Slab& s : ctx->slabs) {
      ck(cudaSetDevice(s.dev), "cudaSetDevice");
      const size_t need = 2 + 2 * static_cast<size_t>(std::max<int32_t>(sample, 1));
      while (s.timing.size() < need) {
        cudaEvent_t e;
        ck(cudaEventCreate(&e), "cudaEventCreate");
        s.timing.push_back(e);
      }
      ck(cudaEventRecord(s.timing[0], s.stream), "event");
    }
    const int64_t l0 = ctx->launches;
    enqueue_step(ctx, rc, flags, false, nullptr, nullptr, steps);
    ctx->timed_launches = ctx->launches - l0;
    for (Slab& s : ctx->slabs) {
      ck(cudaSetDevice(s.dev), "cudaSetDevice");
      ck(cudaEventRecord(s.timing[1], s.stream), "event");
    }
    sync_all(ctx);
    double tot = 0;
    for (Slab& s : ctx->slabs) {
      float ms = 0;
      ck(cudaEventElapsedTime(&ms, s.timing[0], s.timing[1]), "elapsed");
      tot = std::max(tot, static_cast<double>(ms));
    }
    double ker = tot;  // persistent: the launch is the kernel
    if (sample > 0) {
      std::vector<cudaEvent_t> k0(G), k1(G);
      for (int32_t t = 0; t < sample; ++t) {
        for (size_t i = 0; i < G; ++i) {
          k0[i] = ctx->slabs[i].timing[2 + 2 * t];
          k1[i] = ctx->slabs[i].timing[3 + 2 * t];
        }
        enqueue_step(ctx, rc, flags, false, k0.data(), k1.data(), 1);
      }
      sync_all(ctx);
      ker = 0;
      for (Slab& s : ctx->slabs) {
        double acc = 0;
        for (int32_t t = 0; t < sample; ++t) {
          float k = 0;
          ck(cudaEventElapsedTime(&k, s.timing[2 + 2 * t], s.timing[3 + 2 * t]), "elapsed");
          acc += k;
        }
        ker = std::max(ker, acc * steps / sample);
      }
    }
    ctx->pk_hold = false;
    settle_packed(ctx);
    sync_all(ctx);
    if (total_ms) *total_ms = tot;
    if (kernel_ms) *kernel_ms = ker;
  });
}

int ltl_run_interior(ltl_ctx* ctx, const uint8_t* interior_in, uint8_t* interior_out,
                     const ltl_rule_c* rule, int32_t steps, uint32_t flags, ltl_stats_c* stats) {
  if (!ctx) return LTL_ERR_INVALID_ARGUMENT;
  return guarded(ctx, [&] {
    check_run_args(ctx, rule, steps, flags);
    upload_interior(ctx, interior_in);
    run_steps(ctx, rule, steps, flags, stats);
    download_interior(ctx, interior_out);
  });
}

int ltl_create_part(ltl_ctx** out, int32_t rows_local, int32_t cols, int32_t row0,
                    int32_t device) {
  const int32_t dev = device;
  const int st = ltl_create_torus(out, rows_local, cols, 1, &dev);
  if (st == LTL_OK) {
    (*out)->external_row_halo = true;
    (*out)->slabs[0].row0 = row0;  // global row of the first local row (init_random);
                                   // host buffers hold this slab only (host_row0 = 0)
  }
  return st;
}

int ltl_set_stream(ltl_ctx* ctx, int32_t slab, void* stream) {
  if (!ctx) return LTL_ERR_INVALID_ARGUMENT;
  return guarded(ctx, [&] {
    if (slab < 0 || slab >= static_cast<int32_t>(ctx->slabs.size()))
      throw std::out_of_range("config error: slab index out of range");
    Slab& s = ctx->slabs[slab];
    ck(cudaSetDevice(s.dev), "cudaSetDevice");
    ck(cudaStreamSynchronize(s.stream), "cudaStreamSynchronize");
    if (s.own_stream) ck(cudaStreamDestroy(s.stream), "cudaStreamDestroy");
    s.stream = static_cast<cudaStream_t>(stream);
    s.own_stream = false;
  });
}

int ltl_step_part(ltl_ctx* ctx, const ltl_rule_c* rule, uint32_t flags) {
  if (!ctx) return LTL_ERR_INVALID_ARGUMENT;
  return guarded(ctx, [&] {
    check_run_args(ctx, rule, 1, flags);
    enqueue_step(ctx, rule_consts(*rule), flags, false, nullptr, nullptr);
  });
}

int ltl_init_random(ltl_ctx* ctx, double density, uint64_t seed, int32_t fill_n) {
  if (!ctx) return LTL_ERR_INVALID_ARGUMENT;
  return guarded(ctx, [&] {
    if (!(density >= 0.0 && density <= 1.0))
      throw std::invalid_argument("init_random: density must be in [0, 1]");
    int32_t fill_rows = ctx->external_row_halo ? ctx->slabs[0].row0 + ctx->rows : ctx->rows;
    int32_t fill_cols = ctx->cols;
    if (fill_n >= 0) {
      if (fill_n > ctx->rows || fill_n > ctx->cols)
        throw std::invalid_argument("init_random: fill_n exceeds n");
      fill_rows = fill_cols = fill_n;
    }
    quiesce_ring_readers(ctx);  // rewrites the current generation neighbours may read
    for (Slab& s : ctx->slabs) {
      ck(cudaSetDevice(s.dev), "cudaSetDevice");
      ck(ltl::launch_init_random(s.view(ctx->cur, ctx->cols), s.row0, fill_rows, fill_cols,
                                 density, seed, s.stream),
         "init kernel");
      ++ctx->launches;
      if (ctx->slabs.size() > 1) ck(cudaEventRecord(s.ev_step, s.stream), "event");
    }
    enqueue_halo(ctx, ctx->cur);
    sync_all(ctx);
    ctx->ring_stale = true;
  });
}

int ltl_fill_halo(ltl_ctx* ctx) {
  if (!ctx) return LTL_ERR_INVALID_ARGUMENT;
  return guarded(ctx, [&] { enqueue_halo(ctx, ctx->cur); });
}

int ltl_slab_buffer(ltl_ctx* ctx, int32_t slab, int32_t which, void** dev_ptr,
                    int64_t* strip_bytes, int32_t* rows) {
  if (!ctx) return LTL_ERR_INVALID_ARGUMENT;
  return guarded(ctx, [&] {
    if (slab < 0 || slab >= static_cast<int32_t>(ctx->slabs.size()))
      throw std::out_of_range("config error: slab index out of range");
    const Slab& s = ctx->slabs[slab];
    const int b = which == 0 ? ctx->cur : 1 - ctx->cur;
    if (dev_ptr) *dev_ptr = s.buf[b];
    if (strip_bytes) *strip_bytes = s.strip_bytes;
    if (rows) *rows = s.rows;
  });
}

int ltl_pack_edges(ltl_ctx* ctx, void* top, void* bot) {
  if (!ctx) return LTL_ERR_INVALID_ARGUMENT;
  return guarded(ctx, [&] {
    if (ctx->slabs.size() != 1)
      throw std::invalid_argument("config error: edge exchange needs a single-slab context");
    Slab& s = ctx->slabs[0];
    if (s.rows < kHalo)
      throw std::invalid_argument("geometry error: slab thinner than the 16-row halo");
    ck(cudaSetDevice(s.dev), "cudaSetDevice");
    ck(ltl::launch_pack_edges(s.view(ctx->cur, ctx->cols), static_cast<uint8_t*>(top),
                              static_cast<uint8_t*>(bot), s.stream),
       "pack kernel");
    ++ctx->launches;
  });
}

int ltl_unpack_halo(ltl_ctx* ctx, const void* top_halo, const void* bot_halo) {
  if (!ctx) return LTL_ERR_INVALID_ARGUMENT;
  return guarded(ctx, [&] {
    if (ctx->slabs.size() != 1)
      throw std::invalid_argument("config error: edge exchange needs a single-slab context");
    Slab& s = ctx->slabs[0];
    ck(cudaSetDevice(s.dev), "cudaSetDevice");
    ck(ltl::launch_unpack_halo(s.view(ctx->cur, ctx->cols),
                               static_cast<const uint8_t*>(top_halo),
                               static_cast<const uint8_t*>(bot_halo), s.stream),
       "unpack kernel");
    ++ctx->launches;
  });
}

// ---- multi-process ring (one process per GPU, CUDA IPC)

int ltl_ring_export(ltl_ctx* ctx, void* handles) {
  if (!ctx || !handles) return LTL_ERR_INVALID_ARGUMENT;
  return guarded(ctx, [&] {
    if (ctx->slabs.size() != 1 || !ctx->external_row_halo)
      throw std::invalid_argument("config error: ring export needs a part context (ltl_create_part)");
    Slab& s = ctx->slabs[0];
    if (!s.ring_sync || s.rows <= 0 || ctx->cols <= 0)
      throw std::invalid_argument("config error: empty slab");
    ck(cudaSetDevice(s.dev), "cudaSetDevice");
    cudaIpcMemHandle_t h[4];
    ck(cudaIpcGetMemHandle(&h[0], s.ring_sync), "ipc handle (ring counters)");
    ck(cudaIpcGetMemHandle(&h[1], s.buf[0]), "ipc handle (buffer 0)");
    ck(cudaIpcGetMemHandle(&h[2], s.buf[1]), "ipc handle (buffer 1)");
    ck(cudaIpcGetMemHandle(&h[3], s.flags), "ipc handle (unit counters)");
    std::memcpy(handles, h, sizeof h);
    char bus[kBusIdBytes] = {};
    ck(cudaDeviceGetPCIBusId(bus, kBusIdBytes - 1, s.dev), "pci bus id");
    std::memcpy(static_cast<uint8_t*>(handles) + sizeof h, bus, kBusIdBytes);
  });
}

int ltl_ring_connect(ltl_ctx* ctx, const void* up_handles, int32_t up_rows,
                     const void* down_handles, int32_t down_rows) {
  if (!ctx || !up_handles || !down_handles) return LTL_ERR_INVALID_ARGUMENT;
  return guarded(ctx, [&] {
    if (ctx->slabs.size() != 1 || !ctx->external_row_halo)
      throw std::invalid_argument("config error: ring connect needs a part context (ltl_create_part)");
    Slab& s = ctx->slabs[0];
    ck(cudaSetDevice(s.dev), "cudaSetDevice");
    cudaIpcMemHandle_t mine[1];
    ck(cudaIpcGetMemHandle(&mine[0], s.ring_sync), "ipc handle (ring counters)");
    char my_bus[kBusIdBytes] = {};
    ck(cudaDeviceGetPCIBusId(my_bus, kBusIdBytes - 1, s.dev), "pci bus id");
    // open a neighbour's 4 allocations (counters, 2 buffers, unit counters);
    // our own handles (world size 1) map to our own pointers
    bool self[2] = {false, false};
    auto open = [&](const void* hv, void** out, bool* is_self) {
      const cudaIpcMemHandle_t* h = static_cast<const cudaIpcMemHandle_t*>(hv);
      *is_self = std::memcmp(&h[0], &mine[0], sizeof(cudaIpcMemHandle_t)) == 0;
      if (*is_self) {
        out[0] = s.ring_sync;
        out[1] = s.buf[0];
        out[2] = s.buf[1];
        out[3] = s.flags;
        return;
      }
      for (int i = 0; i < 4; ++i) {
        ck(cudaIpcOpenMemHandle(&out[i], h[i], cudaIpcMemLazyEnablePeerAccess), "ipc open");
        s.ipc_opened.push_back(out[i]);
      }
    };
    auto other_gpu = [&](const void* hv) {
      return std::memcmp(static_cast<const uint8_t*>(hv) + 4 * sizeof(cudaIpcMemHandle_t),
                         my_bus, kBusIdBytes) != 0;
    };
    void* up[4];
    void* dn[4];
    open(up_handles, up, &self[0]);
    if (std::memcmp(up_handles, down_handles, 4 * sizeof(cudaIpcMemHandle_t)) == 0) {
      std::memcpy(dn, up, sizeof up);  // world size 2: one neighbour on both sides
      self[1] = self[0];
    } else {
      open(down_handles, dn, &self[1]);
    }
    uint8_t* upb[2] = {static_cast<uint8_t*>(up[1]), static_cast<uint8_t*>(up[2])};
    uint8_t* dnb[2] = {static_cast<uint8_t*>(dn[1]), static_cast<uint8_t*>(dn[2])};
    wire_ring(ctx, s,
              RingPeer{static_cast<uint32_t*>(up[0]), upb, up_rows, static_cast<uint32_t*>(up[3]),
                       self[0] || other_gpu(up_handles)},
              RingPeer{static_cast<uint32_t*>(dn[0]), dnb, down_rows, static_cast<uint32_t*>(dn[3]),
                       self[1] || other_gpu(down_handles)});
    ctx->ring_stale = true;
  });
}

int ltl_ring_disconnect(ltl_ctx* ctx) {
  if (!ctx) return LTL_ERR_INVALID_ARGUMENT;
  return guarded(ctx, [&] {
    sync_all(ctx);
    for (Slab& s : ctx->slabs) {
      if (!ctx->external_row_halo) continue;  // in-process rings stay wired
      for (void* ptr : s.ipc_opened) cudaIpcCloseMemHandle(ptr);
      s.ipc_opened.clear();
      s.ring_ready = false;
    }
    ctx->ring_stale = true;
  });
}

int ltl_ring_fill(ltl_ctx* ctx) {
  if (!ctx) return LTL_ERR_INVALID_ARGUMENT;
  return guarded(ctx, [&] {
    for (const Slab& s : ctx->slabs)
      if (!s.ring_ready) throw std::logic_error("sequencing error: ring not connected");
    start_ring(ctx);
    ctx->ring_stale = false;
  });
}

int32_t ltl_ring_active(const ltl_ctx* ctx) {
  return ctx && ring_ok(ctx) ? 1 : 0;
}

}  // extern "C"

// ---- CATSNAP v1 snapshots streamed from / to the device (src/snapshot.cpp)
//
// Format (include/catsim/snapshot.hpp): "CATSNAP 1 <n> <f> <layout>\n" then
// the n x n interior bytes in row-major order.  Writes gather the strips into
// the dead generation buffer on the device (one relayout kernel) and stream
// it out through two pinned chunks, the D2H of chunk k+1 overlapping the
// fwrite of chunk k; reads mirror that and check the {0,1} bytes on the
// device.  No host copy of the grid is ever made.

namespace {

[[noreturn]] void snap_fail(const std::string& why) {
  throw std::runtime_error("snapshot format error: " + why);
}

constexpr size_t kSnapChunk = 32u << 20;  // bytes per pinned chunk

void ensure_pinned(ltl_ctx* ctx) {  // snapshot chunks = the staging chunks
  static_assert(kSnapChunk == kStageChunk, "one pinned chunk size");
  ensure_stage(ctx);
}

struct SnapHeader {
  int32_t n = -1, f = -1, layout = 0;
};

// snapshot_read's header checks (src/snapshot.cpp:39-66), same order and text,
// on the header line (without its newline; `any` = false: no line at all).
SnapHeader parse_snap_line(const std::string& header, bool any) {
  if (!any) snap_fail("missing header line");
  std::istringstream hs(header);
  std::string magic, layout_token;
  int version = 0, n = -1, f = -1;
  if (!(hs >> magic >> version >> n >> f >> layout_token))
    snap_fail("malformed header '" + header + "'");
  std::string trailing;
  if (hs >> trailing) snap_fail("trailing tokens in header");
  if (magic != "CATSNAP") snap_fail("bad magic '" + magic + "'");
  if (version != 1) snap_fail("unsupported version " + std::to_string(version));
  SnapHeader h;
  if (layout_token == "rowmajor")
    h.layout = LTL_LAYOUT_ROW_MAJOR;
  else if (layout_token == "fragment")
    h.layout = LTL_LAYOUT_FRAGMENT;
  else
    snap_fail("unknown layout '" + layout_token + "'");
  if (n < 0 || f <= 0 || n % f != 0)
    snap_fail("bad geometry n=" + std::to_string(n) + " f=" + std::to_string(f));
  h.n = n;
  h.f = f;
  return h;
}

SnapHeader parse_snap_header(std::FILE* fh) {
  std::string header;
  bool any = false;
  for (int c; (c = std::fgetc(fh)) != EOF;) {
    any = true;
    if (c == '\n') break;
    header.push_back(static_cast<char>(c));
  }
  return parse_snap_line(header, any);
}

struct FileCloser {
  std::FILE* fh;
  ~FileCloser() {
    if (fh) std::fclose(fh);
  }
};

void check_square(const ltl_ctx* ctx) {
  if (ctx->rows != ctx->cols)
    throw std::invalid_argument("config error: snapshots hold square n x n grids (context is " +
                                std::to_string(ctx->rows) + " x " + std::to_string(ctx->cols) +
                                ")");
}

void snapshot_write_ctx(ltl_ctx* ctx, const char* path, int32_t layout) {
  quiesce_ring_readers(ctx);
  check_layout(layout);
  check_square(ctx);
  std::FILE* fh = std::fopen(path, "wb");
  if (!fh) snap_fail(std::string("cannot open '") + path + "' for writing");
  FileCloser closer{fh};
  const std::string header = "CATSNAP 1 " + std::to_string(ctx->rows) + " " +
                             std::to_string(ctx->f) + " " +
                             (layout == LTL_LAYOUT_ROW_MAJOR ? "rowmajor" : "fragment") + "\n";
  if (std::fwrite(header.data(), 1, header.size(), fh) != header.size()) snap_fail("write failed");
  if (ctx->rows > 0) ensure_pinned(ctx);
  const int cur = ctx->cur;
  for (Slab& s : ctx->slabs) {
    ck(cudaSetDevice(s.dev), "cudaSetDevice");
    if (s.rows == 0 || ctx->cols == 0) continue;
    uint8_t* dense = s.buf[1 - cur];  // dead between steps (see upload_interior)
    ck(ltl::launch_from_strips(s.view(cur, ctx->cols), dense, s.stream), "from_strips");
    ++ctx->launches;
    const size_t total = static_cast<size_t>(s.rows) * ctx->cols;
    const size_t nchunks = (total + kSnapChunk - 1) / kSnapChunk;
    cudaEvent_t ev[2];
    for (auto& e : ev) ck(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event");
    auto issue = [&](size_t k) {
      const size_t off = k * kSnapChunk, len = std::min(kSnapChunk, total - off);
      ck(cudaMemcpyAsync(ctx->pinned[k % 2], dense + off, len, cudaMemcpyDeviceToHost, s.stream),
         "snapshot D2H");
      ck(cudaEventRecord(ev[k % 2], s.stream), "event");
    };
    issue(0);
    bool ok = true;
    for (size_t k = 0; k < nchunks; ++k) {
      if (k + 1 < nchunks) issue(k + 1);  // its buffer's fwrite (chunk k-1) is done
      ck(cudaEventSynchronize(ev[k % 2]), "snapshot D2H");
      const size_t len = std::min(kSnapChunk, total - k * kSnapChunk);
      ok = ok && std::fwrite(ctx->pinned[k % 2], 1, len, fh) == len;
    }
    ck(cudaStreamSynchronize(s.stream), "cudaStreamSynchronize");
    for (auto& e : ev) cudaEventDestroy(e);
    if (!ok) snap_fail("write failed");
  }
  closer.fh = nullptr;
  if (std::fclose(fh) != 0) snap_fail("write failed");
}

int32_t snapshot_read_ctx(ltl_ctx* ctx, const char* path) {
  quiesce_ring_readers(ctx);
  std::FILE* fh = std::fopen(path, "rb");
  if (!fh) snap_fail(std::string("cannot open '") + path + "' for reading");
  FileCloser closer{fh};
  const SnapHeader h = parse_snap_header(fh);
  check_square(ctx);
  if (h.n != ctx->rows || h.f != ctx->f)
    throw std::invalid_argument("geometry error: snapshot n=" + std::to_string(h.n) +
                                " f=" + std::to_string(h.f) + " does not match the context (n=" +
                                std::to_string(ctx->rows) + " f=" + std::to_string(ctx->f) + ")");
  if (h.n > 0) ensure_pinned(ctx);
  const int cur = ctx->cur;
  const std::string truncated = "truncated payload (expected " + std::to_string(h.n) + "x" +
                                std::to_string(h.n) + " cells)";
  // Pass 1: every slab's payload into its dead buffer, checked ({0,1} bytes,
  // complete).  The live generation is untouched until the whole file is
  // valid -- the reference's snapshot_read has no side effects when it fails.
  int32_t* bad = nullptr;
  ck(cudaMallocHost(&bad, sizeof(int32_t)), "cudaMallocHost");
  struct PinnedFree {
    int32_t* p;
    ~PinnedFree() { cudaFreeHost(p); }
  } free_bad{bad};
  for (Slab& s : ctx->slabs) {
    ck(cudaSetDevice(s.dev), "cudaSetDevice");
    if (s.rows == 0 || ctx->cols == 0) continue;
    *bad = 0;
    uint8_t* dense = s.buf[1 - cur];
    const size_t total = static_cast<size_t>(s.rows) * ctx->cols;
    const size_t nchunks = (total + kSnapChunk - 1) / kSnapChunk;
    cudaEvent_t ev[2];
    for (auto& e : ev) ck(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event");
    bool short_read = false;
    size_t got_total = 0;
    for (size_t k = 0; k < nchunks && !short_read; ++k) {
      if (k >= 2) ck(cudaEventSynchronize(ev[k % 2]), "snapshot H2D");  // buffer free again
      const size_t off = k * kSnapChunk, len = std::min(kSnapChunk, total - off);
      const size_t got = std::fread(ctx->pinned[k % 2], 1, len, fh);
      // the reference reads whole rows: only complete rows reach the {0,1} check
      const size_t rows_done = (off + got) / ctx->cols;
      const size_t keep = got == len ? len : rows_done * ctx->cols - std::min(off, rows_done * ctx->cols);
      if (got != len) short_read = true;
      if (keep > 0) {
        ck(cudaMemcpyAsync(dense + off, ctx->pinned[k % 2], keep, cudaMemcpyHostToDevice, s.stream),
           "snapshot H2D");
        ck(cudaEventRecord(ev[k % 2], s.stream), "event");
      }
      got_total = off + keep;
    }
    ck(ltl::launch_check_cells(dense, static_cast<int64_t>(got_total), bad, s.stream), "check");
    ++ctx->launches;
    ck(cudaStreamSynchronize(s.stream), "cudaStreamSynchronize");
    for (auto& e : ev) cudaEventDestroy(e);
    if (*bad) snap_fail("cell byte out of {0,1}");
    if (short_read) snap_fail(truncated);
  }
  // Pass 2: the whole file is valid -- scatter into the live generation.
  for (Slab& s : ctx->slabs) {
    ck(cudaSetDevice(s.dev), "cudaSetDevice");
    if (s.rows == 0 || ctx->cols == 0) continue;
    ck(ltl::launch_to_strips(s.buf[1 - cur], s.view(cur, ctx->cols), s.stream), "to_strips");
    ++ctx->launches;
  }
  if (ctx->slabs.size() > 1)
    for (Slab& s : ctx->slabs) {
      ck(cudaSetDevice(s.dev), "cudaSetDevice");
      ck(cudaEventRecord(s.ev_step, s.stream), "event");
    }
  enqueue_halo(ctx, cur);
  sync_all(ctx);
  ctx->ring_stale = true;
  return h.layout;
}

}  // namespace

extern "C" {

int ltl_snapshot_write(ltl_ctx* ctx, const char* path, int32_t layout) {
  if (!ctx || !path) return LTL_ERR_INVALID_ARGUMENT;
  return guarded(ctx, [&] { snapshot_write_ctx(ctx, path, layout); });
}

int ltl_snapshot_read(ltl_ctx* ctx, const char* path, int32_t* layout_out) {
  if (!ctx || !path) return LTL_ERR_INVALID_ARGUMENT;
  return guarded(ctx, [&] {
    const int32_t layout = snapshot_read_ctx(ctx, path);
    if (layout_out) *layout_out = layout;
  });
}

int ltl_snapshot_parse_header(const char* line, int32_t has_line, int32_t* n, int32_t* f,
                              int32_t* layout) {
  return guarded(nullptr, [&] {
    const SnapHeader h = parse_snap_line(line && has_line ? std::string(line) : std::string(),
                                         has_line != 0);
    if (n) *n = h.n;
    if (f) *f = h.f;
    if (layout) *layout = h.layout;
  });
}

int ltl_snapshot_probe(const char* path, int32_t* n, int32_t* f, int32_t* layout) {
  if (!path) return LTL_ERR_INVALID_ARGUMENT;
  return guarded(nullptr, [&] {
    std::FILE* fh = std::fopen(path, "rb");
    if (!fh) snap_fail(std::string("cannot open '") + path + "' for reading");
    FileCloser closer{fh};
    const SnapHeader h = parse_snap_header(fh);
    if (n) *n = h.n;
    if (f) *f = h.f;
    if (layout) *layout = h.layout;
  });
}

}  // extern "C"

// ---- the reference's fragment-level unit-test entry points, on the device

extern "C" {

int ltl_fragment_pass(int32_t stage, int32_t n, int32_t f, const uint8_t* cells,
                      const int32_t* bands, const int32_t* h_in, int32_t* out) {
  if (!cells || !bands || !out || (stage != 0 && !h_in) || stage < 0 || stage > 2)
    return LTL_ERR_INVALID_ARGUMENT;
  return guarded(nullptr, [&] {
    if (f <= 0 || n < 0 || n % f != 0)
      throw std::invalid_argument("geometry error: n (" + std::to_string(n) +
                                  ") must be a non-negative multiple of f (" + std::to_string(f) +
                                  ")");
    const size_t p = static_cast<size_t>(n) + 2 * f, cells_n = p * p;
    uint8_t* d_cells = nullptr;
    int32_t *d_bands = nullptr, *d_h = nullptr, *d_out = nullptr;
    auto release = [&] {
      cudaFree(d_cells);
      cudaFree(d_bands);
      cudaFree(d_h);
      cudaFree(d_out);
    };
    try {
      ck(cudaMalloc(&d_cells, cells_n), "cudaMalloc");
      ck(cudaMalloc(&d_bands, 3 * sizeof(int32_t) * f * f), "cudaMalloc");
      ck(cudaMalloc(&d_out, cells_n * sizeof(int32_t)), "cudaMalloc");
      ck(cudaMemcpy(d_cells, cells, cells_n, cudaMemcpyHostToDevice), "H2D");
      ck(cudaMemcpy(d_bands, bands, 3 * sizeof(int32_t) * f * f, cudaMemcpyHostToDevice), "H2D");
      if (stage != 0) {
        ck(cudaMalloc(&d_h, cells_n * sizeof(int32_t)), "cudaMalloc");
        ck(cudaMemcpy(d_h, h_in, cells_n * sizeof(int32_t), cudaMemcpyHostToDevice), "H2D");
      }
      ck(ltl::launch_fragment_pass(stage, n, f, d_cells, d_bands, d_h, d_out, nullptr),
         "fragment pass kernel");
      ck(cudaMemcpy(out, d_out, cells_n * sizeof(int32_t), cudaMemcpyDeviceToHost), "D2H");
    } catch (...) {
      release();
      throw;
    }
    release();
  });
}

}  // extern "C"
