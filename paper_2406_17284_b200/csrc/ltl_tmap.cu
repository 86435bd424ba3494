// ltl_tmap.cu -- TMA tensor maps over a strip-layout device slab.
// cuTensorMapEncodeTiled is a driver API; it is fetched through
// cudaGetDriverEntryPoint so the library has no link-time dependency on libcuda
// (it must load on GPU-less hosts for the symbol checks; every call still
// fails loudly there).
//
// Both maps are 3-D views {column in strip (128), row, strip} of the slab
// (ltl_kernels.cuh SlabView): the row bound clips stores to the interior of
// every strip, and loads past the last padded row read zeros.
#include <cuda.h>
#include <cuda_runtime.h>

#include "ltl_kernels.cuh"

namespace ltl {
namespace {

using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                              const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                              const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                              CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

cudaError_t get_encode(EncodeFn* fn) {
  static EncodeFn cached = nullptr;
  if (!cached) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaError_t e = cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
    if (e != cudaSuccess) return e;
    if (q != cudaDriverEntryPointSuccess || !p) return cudaErrorSymbolNotFound;
    cached = reinterpret_cast<EncodeFn>(p);
  }
  *fn = cached;
  return cudaSuccess;
}

// {row_elems, rows, strips} over strips of `row_bytes`-byte rows
cudaError_t encode3(CUtensorMap* map, void* base, uint64_t rows, uint64_t strips,
                    uint64_t strip_bytes, uint32_t box_w, uint32_t box_h,
                    CUtensorMapSwizzle swz,
                    CUtensorMapDataType type = CU_TENSOR_MAP_DATA_TYPE_UINT8,
                    uint64_t row_elems = kStrip, uint64_t row_bytes = kStrip) {
  EncodeFn fn;
  cudaError_t e = get_encode(&fn);
  if (e != cudaSuccess) return e;
  const cuuint64_t dims[3] = {row_elems, rows, strips};
  const cuuint64_t strides[2] = {row_bytes, strip_bytes};
  const cuuint32_t box[3] = {box_w, box_h, 1};
  const cuuint32_t estr[3] = {1, 1, 1};
  const CUresult r = fn(map, type, 3, base, dims, strides, box, estr,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, swz, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}

}  // namespace

// Whole padded slab in the SWIZZLE_128B K-major layout of the pass-1 B
// operand (ptx::smem_desc_sw128_kmajor), for boxes with `halo` (kH = 16 / 32)
// rows above and below: [0] (128 + 2 kH)-row boxes (one contiguous 20 / 24 KB
// block of a strip), [1] kH-row pieces, [2] (128 + kH)-row and [3] (rows of
// the last band + kH)-row bodies for the row-wrapped first / last band boxes.
cudaError_t make_load_maps(CUtensorMap* maps, const SlabView& s, int halo) {
  if (s.rows <= 0 || s.cols <= 0) return cudaSuccess;
  const int last = s.rows - kTcBand * ((s.rows - 1) / kTcBand);  // rows of the last band
  const bool one_band = s.rows <= kTcBand;  // first = last band: body without its top halo
  const uint32_t h = static_cast<uint32_t>(halo);
  const uint32_t box[kTcLoadMaps] = {kTcBand + 2 * h, h, kTcBand + h,
                                     static_cast<uint32_t>(last) + (one_band ? 0 : h)};
  for (int i = 0; i < kTcLoadMaps; ++i) {
    const cudaError_t e = encode3(&maps[i], s.buf, static_cast<uint64_t>(s.rows) + 2 * kHalo,
                                  static_cast<uint64_t>(s.strips),
                                  static_cast<uint64_t>(s.strip_bytes), kStrip, box[i],
                                  CU_TENSOR_MAP_SWIZZLE_128B);
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

// Interior rows of every strip: each epilogue group stores one 64-row x
// 128-column sub-block (8 KB of contiguous strip rows), SWIZZLE_128B so the
// stmatrix rows land conflict-free.
cudaError_t make_store_map(CUtensorMap* map, const SlabView& s) {
  if (s.rows <= 0 || s.cols <= 0) return cudaSuccess;
  return encode3(map, s.buf + kHalo * kStrip, static_cast<uint64_t>(s.rows),
                 static_cast<uint64_t>(s.strips), static_cast<uint64_t>(s.strip_bytes), kStrip,
                 64, CU_TENSOR_MAP_SWIZZLE_128B);
}

// halo-row pieces of a slab's padded rows (the ring's rows above / below, read
// out of the neighbour's slab in peer memory): load map [1] of any slab.
cudaError_t make_piece_map(CUtensorMap* map, const SlabView& s, int halo) {
  if (s.rows <= 0 || s.cols <= 0) return cudaSuccess;
  return encode3(map, s.buf, static_cast<uint64_t>(s.rows) + 2 * kHalo,
                 static_cast<uint64_t>(s.strips), static_cast<uint64_t>(s.strip_bytes), kStrip,
                 static_cast<uint32_t>(halo), CU_TENSOR_MAP_SWIZZLE_128B);
}

// The 4-bit copy of a slab (PackedView): load boxes of 128 cells per row as
// 16U4_ALIGN16B -- in SMEM every 16 cells take 16 bytes (8 of nibbles, 8
// unused), the e2m1 operand layout of tcgen05.mma kind::f8f6f4, SWIZZLE_128B
// like the u8 boxes (tools/ubench_fp4.cu) -- with the same four box shapes.
cudaError_t make_load_maps_packed(CUtensorMap* maps, const PackedView& s) {
  if (s.rows <= 0 || s.cols <= 0) return cudaSuccess;
  const int last = s.rows - kTcBand * ((s.rows - 1) / kTcBand);
  const bool one_band = s.rows <= kTcBand;
  const uint32_t h = kHalo;
  const uint32_t box[kTcLoadMaps] = {kTcBand + 2 * h, h, kTcBand + h,
                                     static_cast<uint32_t>(last) + (one_band ? 0 : h)};
  for (int i = 0; i < kTcLoadMaps; ++i) {
    const cudaError_t e = encode3(&maps[i], s.buf, static_cast<uint64_t>(s.rows) + 2 * kHalo,
                                  static_cast<uint64_t>(s.strips),
                                  static_cast<uint64_t>(s.strip_bytes), kStrip, box[i],
                                  CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_DATA_TYPE_16U4_ALIGN16B,
                                  kStrip, kPkRow);
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

// Interior rows of the 4-bit copy: 64-row x 64-byte staging tiles (4 KB),
// SWIZZLE_64B so the output warps' stmatrix rows land conflict-free.
cudaError_t make_store_map_packed(CUtensorMap* map, const PackedView& s) {
  if (s.rows <= 0 || s.cols <= 0) return cudaSuccess;
  return encode3(map, s.buf + kHalo * kPkRow, static_cast<uint64_t>(s.rows),
                 static_cast<uint64_t>(s.strips), static_cast<uint64_t>(s.strip_bytes), kPkRow, 64,
                 CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_DATA_TYPE_UINT8, kPkRow, kPkRow);
}

}  // namespace ltl
