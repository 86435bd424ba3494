/*
 * ltl_b200.h -- C-ABI of the B200-native Larger-than-Life step library
 * (paper_2406_17284_b200/libltl_b200.so).
 *
 * This is the drop-in boundary.  The reference has no FFI or plugin registry:
 * its engines form a closed enum + switch (proj/include/catsim/engines.hpp:11,
 * proj/src/engines.cpp:26-46) and the hot path is the C++ call chain
 *   run_engine(EngineKind::Cat, ...)   proj/src/engines.cpp:26-36
 *     -> simulate(...)                 proj/src/cat_engine.cpp:308-321
 *       -> simulate_step(...)          proj/src/cat_engine.cpp:260-306
 * Every entry point below replaces one piece of that chain with plain C types
 * (pointers + sizes, no torch, no C++ types), so any host language can bind it:
 * the C++ catsim API of this repo (include/catsim/ headers) sits on top of it, and
 * INTEGRATION.md shows the ctypes / cgo / JNI stubs.
 *
 * Errors: every int-returning call returns LTL_OK or one of the LTL_ERR_*
 * codes, which map 1:1 onto the reference's exception classes; the message
 * (same stable prefixes as the reference: "config error:", "geometry error:",
 * "layout error:", "unsupported rule", "rule parse error: field X",
 * "internal consistency: negative neighborhood count", ...) is available from
 * ltl_last_error().  A context is not thread-safe; use one per host thread.
 */
#ifndef LTL_B200_H
#define LTL_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define LTL_ABI_VERSION 5

/* status codes <-> reference exception classes */
#define LTL_OK 0
#define LTL_ERR_INVALID_ARGUMENT 1 /* std::invalid_argument */
#define LTL_ERR_LOGIC 2            /* std::logic_error (sequencing / consistency) */
#define LTL_ERR_RUNTIME 3          /* std::runtime_error */
#define LTL_ERR_CUDA 4             /* device failure (no reference analogue) */

/* catsim::Layout, proj/include/catsim/grid.hpp:14 */
#define LTL_LAYOUT_ROW_MAJOR 0
#define LTL_LAYOUT_FRAGMENT 1

/* catsim::NeighborhoodKind, proj/include/catsim/rule.hpp:13 */
#define LTL_KIND_MOORE 0
#define LTL_KIND_VON_NEUMANN 1

/* ltl_run flags */
#define LTL_FLAG_INJECT_FAULT 0x1u  /* CatConfig.inject_band_fault, cat_engine.hpp:22-24 */
#define LTL_FLAG_WANT_STATS 0x2u    /* fill ltl_stats_c (device max-reduction of H / R) */
/* Engine selection (catsim::EngineKind, proj/include/catsim/engines.hpp:11):
 * none = Cat (tcgen05 banded MMA), BASE = the CUDA-core direct-sum stencil (the
 * paper's SHARED/BASE baseline: (2r+1)^2 adds per cell), PACK = the CUDA-core
 * packed-lane sliding-window stencil (the strongest classical comparator).
 * The band fault (LTL_FLAG_INJECT_FAULT) only affects Cat, as in the reference. */
#define LTL_FLAG_ENGINE_BASE 0x4u
#define LTL_FLAG_ENGINE_PACK 0x10u
#define LTL_FLAG_STENCIL LTL_FLAG_ENGINE_BASE /* round-1 name */
/* Extension beyond the reference (which rejects r > 16, src/rule.cpp:33-35):
 * the Cat engine with 17 <= r <= 32 ("+16 expansion": 32-row
 * boxes, four pass-2 band chunks), any fragment side f.  Needs every wrap
 * done by the step's loads: cols % 128 == 0 and, per slab, rows % 32 == 0
 * (one whole-torus slab, or a ring of slabs with the fused exchange);
 * otherwise "unsupported radius r=.. : r > 16 needs ...".  Rules come from
 * ltl_parse_rule_ext(text, 32, ...). */
#define LTL_FLAG_WIDE_RADIUS 0x20u
#define LTL_MAX_WIDE_RADIUS 32
/* Cell storage of the Cat engine on the device (opt-in).
 * LTL_FLAG_4BIT_CELLS: where the geometry allows it -- one whole-torus slab,
 * cols % 128 == 0, rows % 32 == 0, r <= 16 -- the generations of the call step
 * a 4-bit copy of the grid (two cells per byte: B_alg = 1 byte per cell update
 * instead of 2; pass 1 on tcgen05.mma kind::f8f6f4, e4m3 band weights x e2m1
 * cells, f16 accumulators), converted from / back to the u8 slab at the start /
 * end of the call; elsewhere the flag is ignored (u8 cells).  Same bytes as the
 * u8 path.  Not the default: the step is bound by its instruction issue, not
 * by HBM, so halving the bytes does not pay. */
#define LTL_FLAG_4BIT_CELLS 0x40u

/* catsim::LtlRule, proj/include/catsim/rule.hpp:17-32 */
typedef struct ltl_rule_c {
  int32_t r, c, m, s1, s2, b1, b2, kind;
} ltl_rule_c;

/* catsim::CatStats, proj/include/catsim/cat_engine.hpp:29-38 (mma_count in
 * the reference's 16x16-fragment units, so the numbers match its counters). */
typedef struct ltl_stats_c {
  int64_t mma_count;
  int64_t steps;
  int32_t max_h;
  int32_t max_r;
  int32_t fragments_per_row;
  int32_t reserved;
} ltl_stats_c;

typedef struct ltl_ctx ltl_ctx;

/* --- context (device grid) ---------------------------------------------- */

/* Square n x n torus with fragment side f (4, 8, 16), split into `num_slabs`
 * row slabs on devices dev_ids[0..num_slabs) (NULL -> slab i on device
 * i % device_count).  Replaces make_grid (src/grid.cpp:41-49) + the second
 * ping-pong buffer simulate allocates (src/cat_engine.cpp:313).  Errors as
 * make_grid: "geometry error: n (..) must be a non-negative multiple of f (..)". */
int ltl_create(ltl_ctx** out, int32_t n, int32_t f, int32_t num_slabs, const int32_t* dev_ids);

/* Rectangular rows x cols torus (weak-scaling extension: the reference Grid
 * is square only, grid.hpp:53-54).  f = 16 semantics (any rows, cols >= 1). */
int ltl_create_torus(ltl_ctx** out, int32_t rows, int32_t cols, int32_t num_slabs,
                     const int32_t* dev_ids);

/* Square n x n torus for a host Grid of ANY fragment side f > 0 with n % f
 * == 0 (make_grid's geometry, src/grid.cpp:11-17, and its messages): the f
 * used by ltl_upload / ltl_download's padded layouts and by the CAT engine's
 * r <= f check.  One slab on the current device. */
int ltl_create_grid(ltl_ctx** out, int32_t n, int32_t f);

void ltl_destroy(ltl_ctx* ctx);
const char* ltl_last_error(const ltl_ctx* ctx); /* "" after success; never NULL */

/* Geometry queries. */
int32_t ltl_rows(const ltl_ctx* ctx);
/* Number of device kernels this context has launched so far (for launch
 * accounting in benchmarks). */
int64_t ltl_kernel_launches(const ltl_ctx* ctx);
int32_t ltl_cols(const ltl_ctx* ctx);
int32_t ltl_num_slabs(const ltl_ctx* ctx);

/* --- host <-> device (copies; no host pointer is retained) --------------- */

/* Padded (n+2f)^2 host grid in the given layout (catsim::Grid::cells); only
 * the interior is read -- the device refreshes its own periodic halo, which is
 * what simulate_step does first anyway (src/cat_engine.cpp:275).  One pitched
 * H2D copy of the interior per slab + a device relayout kernel (no host pass
 * over the cells; replaces to_fragment_layout's permutation,
 * src/layout.cpp:23-32, on the run_engine path src/engines.cpp:32). */
int ltl_upload(ltl_ctx* ctx, const uint8_t* padded, int32_t layout);
/* Writes the padded grid: interior = current generation, halo = its periodic
 * image (callers may treat it as stale, as the reference does after a step). */
int ltl_download(ltl_ctx* ctx, uint8_t* padded, int32_t layout);
/* As ltl_download, but with fill_halo == 0 only the interior bytes of
 * `padded` are written (what simulate_step writes into `out`,
 * src/cat_engine.cpp:293-305): a device relayout + ONE pitched D2H per slab. */
int ltl_download_padded(ltl_ctx* ctx, uint8_t* padded, int32_t layout, int32_t fill_halo);
/* fill_periodic_halo (src/grid.cpp:75-94) of a padded HOST grid, any f > 0
 * with n % f == 0 (pure host; halo cells only). */
int ltl_host_fill_halo(uint8_t* padded, int32_t n, int32_t f, int32_t layout);
/* Dense rows x cols interior, row-major (no halo). */
int ltl_upload_interior(ltl_ctx* ctx, const uint8_t* interior);
int ltl_download_interior(ltl_ctx* ctx, uint8_t* interior);

/* Deterministic random fill generated on the device, bit-identical to
 * init_random (src/grid.cpp:61-73): splitmix64 draw k = y * fill + x for the
 * top-left fill x fill block (fill_n < 0: the whole torus, row-major), alive
 * iff alive_threshold(draw, density) (src/grid.cpp:21-39); the rest dead.
 * Errors as the reference ("init_random: density must be in [0, 1]",
 * "init_random: fill_n exceeds n"). */
int ltl_init_random(ltl_ctx* ctx, double density, uint64_t seed, int32_t fill_n);

/* --- the hot path --------------------------------------------------------- */

/* `steps` generations (simulate, src/cat_engine.cpp:308-321): per slab one
 * fused tcgen05 launch per generation, or ONE persistent cooperative launch
 * for all of them on tori of <= 190 units (128 x 128 cells) per SM; the
 * CUDA-core engines with LTL_FLAG_ENGINE_BASE / _PACK.  Validation and
 * messages as the reference: steps < 0 -> "config error: steps must be >= 0";
 * rule checks of src/rule.cpp:32-57; Cat: r > f -> "unsupported radius r=..
 * for fragment side f=.." (src/fragment.cpp:25-27; Base / Pack: r <= 16 for
 * any f); negative count (fault injection) -> LTL_ERR_LOGIC "internal
 * consistency: negative neighborhood count <c>", c the count of the first
 * failing cell in the reference's serial traversal.  stats may be NULL.
 * Synchronous. */
int ltl_run(ltl_ctx* ctx, const ltl_rule_c* rule, int32_t steps, uint32_t flags,
            ltl_stats_c* stats);

/* Asynchronous variant for pipelines: enqueues `steps` generations on the
 * context's streams and returns (no stats, no error readback). */
int ltl_run_async(ltl_ctx* ctx, const ltl_rule_c* rule, int32_t steps, uint32_t flags);
int ltl_synchronize(ltl_ctx* ctx);

/* Device timing with CUDA events on the slab streams (max over slabs):
 * `warmup` untimed generations then `steps` timed ones.  total_ms covers the
 * whole generation loop (events only around it, so consecutive step kernels
 * keep their programmatic overlap); kernel_ms = the main step kernel's
 * average duration over a further sample of up to 100 generations, each
 * launch bracketed by its own events, times `steps` (the roofline kernel).
 * A multi-generation (persistent) launch is its own kernel sample.
 * Either output pointer may be NULL. */
int ltl_time(ltl_ctx* ctx, const ltl_rule_c* rule, int32_t steps, int32_t warmup,
             uint32_t flags, double* total_ms, double* kernel_ms);
/* Kernels launched inside the last ltl_time's timed loop (total_ms region). */
int64_t ltl_time_launches(const ltl_ctx* ctx);
/* Bytes this context has moved between host and device memory so far
 * (dir 0: host -> device, 1: device -> host) by its uploads / downloads: one
 * bit per cell where the bit-packed transfers ran (>= 4 MB of rows of a
 * multiple of 32 cells, all 0 / 1), one byte per cell elsewhere. */
int64_t ltl_transfer_bytes(const ltl_ctx* ctx, int32_t dir);

/* End-to-end: upload interior from host memory, run `steps` generations,
 * download the interior into `interior_out` -- the whole run_engine(Cat)
 * contract (src/engines.cpp:26-36) in one call. */
int ltl_run_interior(ltl_ctx* ctx, const uint8_t* interior_in, uint8_t* interior_out,
                     const ltl_rule_c* rule, int32_t steps, uint32_t flags, ltl_stats_c* stats);

/* --- multi-process slabs (one process per GPU) --------------------------- */

/* One slab of a torus that is partitioned across processes (one per GPU):
 * rows_local x cols interior on `device`, holding global rows
 * [row0, row0 + rows_local) (used by ltl_init_random).  Its column wrap is refreshed
 * locally; its 16 halo rows above / below are filled by the caller's
 * transport (NCCL send/recv, CUDA IPC) from the neighbouring ranks. */
int ltl_create_part(ltl_ctx** out, int32_t rows_local, int32_t cols, int32_t row0,
                    int32_t device);
/* Run slab `slab`'s work on an external CUDA stream (e.g. the one NCCL uses),
 * so kernels and the halo transport are ordered without host syncs. */
int ltl_set_stream(ltl_ctx* ctx, int32_t slab, void* stream);
/* Enqueue exactly one generation (main kernel + local halo refresh), then
 * flip the generation buffers.  Asynchronous. */
int ltl_step_part(ltl_ctx* ctx, const ltl_rule_c* rule, uint32_t flags);
/* Enqueue a halo refresh of the current generation (local column wrap, and
 * row wrap / peer rows unless the context is a part). */
int ltl_fill_halo(ltl_ctx* ctx);

/* Packed edge rows for an external halo transport (NCCL send/recv, CUDA
 * IPC), enqueued on the context's stream; device buffers of 16 x cols bytes,
 * row-major.  ltl_pack_edges: top <- interior rows [0, 16), bot <- interior
 * rows [rows-16, rows) of the current generation.  ltl_unpack_halo: the 16
 * halo rows above <- top_halo (the rows just above this slab, i.e. the upper
 * neighbour's bottom edge), below <- bot_halo, each with its column wrap. */
int ltl_pack_edges(ltl_ctx* ctx, void* top, void* bot);
int ltl_unpack_halo(ltl_ctx* ctx, const void* top_halo, const void* bot_halo);

/* Ring of row slabs with the halo exchange fused into the step (multi-GPU,
 * one process per GPU): the first / last band units of each step TMA-load
 * the 16 rows above / below straight out of the ring neighbours' slabs over
 * NVLink (CUDA IPC peer memory), gated by the neighbours' step counters --
 * no separate exchange, no host synchronisation.  Needs cols % 128 == 0 and
 * rows % 32 == 0 (else ltl_pack_edges / ltl_unpack_halo + NCCL).
 *   ltl_ring_export:  LTL_RING_HANDLE_BYTES: CUDA IPC handles of a part context's
 *                     step counters, both buffers and unit counters + its GPU's
 *                     PCI bus id
 *   ltl_ring_connect: open the upper / lower neighbour's handles (rows = their
 *                     slab heights); our own handles (world size 1) are fine
 *   ltl_ring_fill:    after every upload / init, with a barrier of all ranks
 *                     on both sides: restarts the step counters (synchronous)
 *   ltl_ring_active:  1 when ltl_step_part / ltl_run use the fused exchange. */
#define LTL_RING_HANDLE_BYTES (4 * 64 + 32)
int ltl_ring_export(ltl_ctx* ctx, void* handles);
int ltl_ring_connect(ltl_ctx* ctx, const void* up_handles, int32_t up_rows,
                     const void* down_handles, int32_t down_rows);
int ltl_ring_fill(ltl_ctx* ctx);
int32_t ltl_ring_active(const ltl_ctx* ctx);
/* Drop a part context's ring (close the IPC mappings); steps then need the
 * packed exchange again. */
int ltl_ring_disconnect(ltl_ctx* ctx);
/* 1 when ltl_run / ltl_run_async of more than one generation would use ONE
 * multi-generation (persistent) launch on this context.  Ranks of a ring must
 * agree (their kernels wait on each other's per-unit counters): a
 * multi-process caller votes on this and, unless every rank says 1, runs
 * one generation per call (paper_2406_17284_b200/dist.py). */
int32_t ltl_persistent_ok(ltl_ctx* ctx, uint32_t flags);

/* Device pointer of slab `slab`'s current (which = 0) or other (1)
 * generation buffer, its strip size in bytes and interior row count.  The
 * device layout is column strips: logical column x in [-128, 128 * (strips-1))
 * of padded row y (interior rows at [16, 16 + rows)) is byte
 * ((x + 128) / 128) * strip_bytes + y * 128 + (x + 128) % 128, with
 * strip_bytes = (rows + 32) * 128 and strips = ceil(cols / 128) + 2. */
int ltl_slab_buffer(ltl_ctx* ctx, int32_t slab, int32_t which, void** dev_ptr,
                    int64_t* strip_bytes, int32_t* rows);

/* --- CATSNAP v1 snapshots, streamed from / to the device ------------------
 * snapshot_write / snapshot_read (src/snapshot.cpp:18-91, format in
 * include/catsim/snapshot.hpp): "CATSNAP 1 <n> <f> <rowmajor|fragment>\n" +
 * the n x n interior bytes, row-major.  Byte-identical to the reference's
 * files; the grid never exists on the host (the device gathers / scatters
 * the strips, 32 MB pinned chunks overlap PCIe with file I/O).  Square
 * contexts only.  Errors: LTL_ERR_RUNTIME "snapshot format error: ..." with
 * the reference's text; a file whose n / f differ from the context is
 * LTL_ERR_INVALID_ARGUMENT "geometry error: ...".  ltl_snapshot_read
 * returns the declared layout (LTL_LAYOUT_*); the device holds cells only. */
int ltl_snapshot_write(ltl_ctx* ctx, const char* path, int32_t layout);
int ltl_snapshot_read(ltl_ctx* ctx, const char* path, int32_t* layout_out);
/* Header only (no device): the geometry and layout a snapshot declares, with
 * the reader's header checks. */
int ltl_snapshot_probe(const char* path, int32_t* n, int32_t* f, int32_t* layout);
/* The same checks on a header line already read (without its '\n');
 * has_line == 0: the stream had no line ("missing header line").  Pure host. */
int ltl_snapshot_parse_header(const char* line, int32_t has_line, int32_t* n, int32_t* f,
                              int32_t* layout);

/* --- the reference's fragment-level unit-test passes, on the device -------
 * horizontal_step (stage 0), vertical_step_moore (1), vertical_step_von_neumann
 * (2), src/cat_engine.cpp:123-258: padded (n + 2f)^2 cells / H / R in
 * fragment-contiguous order, bands = pi1 | pi2 | pi3 (f x f int32 row-major
 * each, as gen_band_fragments builds them, faults included).  `cells` needs a
 * filled periodic halo (the reference checks that).  h_in: stages 1-2.  The
 * product step never materialises H / R; this is the debug path of the
 * reference's fragment API.  Synchronous. */
int ltl_fragment_pass(int32_t stage, int32_t n, int32_t f, const uint8_t* cells,
                      const int32_t* bands, const int32_t* h_in, int32_t* out);

/* --- host-side rule helpers (pure C, no device) --------------------------- */

/* parse_ltl_rule (src/rule.cpp:61-87): returns LTL_OK or
 * LTL_ERR_INVALID_ARGUMENT with the reference's message in err (may be NULL). */
int ltl_parse_rule(const char* text, ltl_rule_c* out, char* err, int32_t err_len);
/* Extension: the same grammar, messages and checks with radii 1..max_radius
 * (max_radius <= LTL_MAX_WIDE_RADIUS; ltl_parse_rule = max_radius 16). */
int ltl_parse_rule_ext(const char* text, int32_t max_radius, ltl_rule_c* out, char* err,
                       int32_t err_len);
/* format_ltl_rule (src/rule.cpp:89-97); returns the string length. */
int32_t ltl_format_rule(const ltl_rule_c* rule, char* buf, int32_t buf_len);
/* ltl_presets (src/rule.cpp:113-133): count, then entries by index. */
int32_t ltl_preset_count(void);
int ltl_preset(int32_t index, const char** name, const char** rule, double* density);
/* von_neumann_probe_rule (src/rule.cpp:142-152). */
void ltl_von_neumann_probe_rule(int32_t r, ltl_rule_c* out);

/* Library identity (also proves the .so was loaded). */
const char* ltl_build_info(void);

#ifdef __cplusplus
}
#endif
#endif
