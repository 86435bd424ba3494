// ltl_tmap.cu -- TMA tensor maps over a device slab.  cuTensorMapEncodeTiled is
// a driver API; it is fetched through cudaGetDriverEntryPoint so the library
// has no link-time dependency on libcuda (it must load on GPU-less hosts for
// the symbol checks; every call still fails loudly there).
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

cudaError_t encode(CUtensorMap* map, void* base, uint64_t w, uint64_t h, uint64_t pitch,
                   uint32_t box_w, uint32_t box_h, CUtensorMapSwizzle swz) {
  EncodeFn fn;
  cudaError_t e = get_encode(&fn);
  if (e != cudaSuccess) return e;
  const cuuint64_t dims[2] = {w, h};
  const cuuint64_t strides[1] = {pitch};
  const cuuint32_t box[2] = {box_w, box_h};
  const cuuint32_t estr[2] = {1, 1};
  const CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, base, dims, strides, box, estr,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, swz, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}

}  // namespace

// Whole padded slab; 32-column x 64-row boxes in the SWIZZLE_32B K-major
// layout the pass-1 B operand descriptor expects (ptx::smem_desc_sw32_kmajor).
cudaError_t make_load_map(CUtensorMap* map, const SlabView& s) {
  if (s.rows <= 0 || s.cols <= 0) return cudaSuccess;
  return encode(map, s.buf, static_cast<uint64_t>(s.cols) + 2 * kHalo,
                static_cast<uint64_t>(s.rows) + 2 * kHalo, static_cast<uint64_t>(s.pitch), 32,
                64, CU_TENSOR_MAP_SWIZZLE_32B);
}

// Interior only: stores of partial strips / chunks are clipped to the torus.
// Each epilogue warp stores its own 32 x 32 tile, SWIZZLE_32B so the
// stmatrix rows land conflict-free.
cudaError_t make_store_map(CUtensorMap* map, const SlabView& s) {
  if (s.rows <= 0 || s.cols <= 0) return cudaSuccess;
  return encode(map, s.buf + kHalo * s.pitch + kHalo, static_cast<uint64_t>(s.cols),
                static_cast<uint64_t>(s.rows), static_cast<uint64_t>(s.pitch), 32, 32,
                CU_TENSOR_MAP_SWIZZLE_32B);
}

}  // namespace ltl
