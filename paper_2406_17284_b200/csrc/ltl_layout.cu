// ltl_layout.cu -- conversions between the host's row-major grid and the
// device's column-strip slab (ltl_kernels.cuh), and the packed edge rows the
// multi-process halo exchange sends.
//
// The reference keeps one row-major (or fragment-contiguous) vector per grid
// (grid.hpp:53-78) and permutes it around every run (to_fragment_layout /
// to_row_major, src/layout.cpp:23-44).  Here the host format is untouched:
// uploads land dense in HBM (one contiguous H2D copy) and are scattered into
// strips on the device, downloads gather on the device and leave in one D2H
// copy.
#include <cuda_runtime.h>

#include <cstdint>
#include <type_traits>

#include "ltl_kernels.cuh"

namespace ltl {
namespace {

__device__ __forceinline__ int wrap(int v, int n) {
  const int m = v % n;
  return m < 0 ? m + n : m;
}

// dense [rows][cols] <-> interior of the slab; 16 bytes per thread when
// cols % 16 == 0 (a 16-byte group never straddles a strip), else bytes.
template <bool kToStrips>
__global__ void relayout_kernel(uint8_t* dense, SlabView s) {
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  const int64_t tid = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (s.cols % 16 == 0) {
    const int64_t gpr = s.cols / 16, total = gpr * s.rows;
    for (int64_t i = tid; i < total; i += stride) {
      const int y = static_cast<int>(i / gpr), x = 16 * static_cast<int>(i % gpr);
      uint4* d = reinterpret_cast<uint4*>(dense + static_cast<int64_t>(y) * s.cols + x);
      uint4* c = reinterpret_cast<uint4*>(s.buf + s.offset(y + kHalo, x));
      if (kToStrips) *c = *d;
      else *d = *c;
    }
  } else {
    const int64_t total = static_cast<int64_t>(s.cols) * s.rows;
    for (int64_t i = tid; i < total; i += stride) {
      const int y = static_cast<int>(i / s.cols), x = static_cast<int>(i % s.cols);
      uint8_t* d = dense + i;
      uint8_t* c = s.buf + s.offset(y + kHalo, x);
      if (kToStrips) *c = *d;
      else *d = *c;
    }
  }
}

// Dense interior in the reference's fragment-contiguous order (interior
// fragment rows x interior fragments, f x f bytes each; include/catsim/grid.hpp
// fragment_offset) <-> interior of the slab: one f-byte fragment row segment
// per thread (f | 128, so it never straddles a strip).  Run i = (I * nfc + J)
// * F + a is fragment (I, J)'s row a, at dense byte i * F.
template <int F, bool kToStrips>
__global__ void frag_relayout_kernel(uint8_t* dense, SlabView s) {
  using V = typename std::conditional<F == 16, uint4, typename std::conditional<F == 8, uint2, uint32_t>::type>::type;
  const int nfc = s.cols / F;
  const int64_t runs = static_cast<int64_t>(s.rows) * nfc;
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < runs;
       i += stride) {
    const int64_t per_frow = static_cast<int64_t>(nfc) * F;
    const int I = static_cast<int>(i / per_frow);
    const int rem = static_cast<int>(i % per_frow);
    const int y = I * F + rem % F, x = (rem / F) * F;
    V* d = reinterpret_cast<V*>(dense + i * F);
    V* c = reinterpret_cast<V*>(s.buf + s.offset(y + kHalo, x));
    if (kToStrips) *c = *d;
    else *d = *c;
  }
}

__global__ void pack_edges_kernel(SlabView s, uint8_t* top, uint8_t* bot) {
  const int n = kHalo * s.cols;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < 2 * n; i += gridDim.x * blockDim.x) {
    const int which = i / n, k = i % n, r = k / s.cols, x = k % s.cols;
    const int py = which == 0 ? kHalo + r : s.rows + r;  // interior rows [0,16) / [rows-16, rows)
    (which == 0 ? top : bot)[k] = s.buf[s.offset(py, x)];
  }
}

__global__ void unpack_halo_kernel(SlabView s, const uint8_t* top, const uint8_t* bot) {
  const int w = s.cols + 2 * kHalo;
  const int n = kHalo * w;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < 2 * n; i += gridDim.x * blockDim.x) {
    const int which = i / n, k = i % n, r = k / w, px = k % w - kHalo;
    const int py = which == 0 ? r : s.rows + kHalo + r;
    s.buf[s.offset(py, px)] = (which == 0 ? top : bot)[r * s.cols + wrap(px, s.cols)];
  }
}

// Any byte of dense[0, n) above 1 -> *bad = 1 (snapshot payload check,
// src/snapshot.cpp:79-80), 16 bytes per thread.
__global__ void check_cells_kernel(const uint8_t* dense, int64_t n, int32_t* bad) {
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  uint32_t acc = 0;
  const int64_t n16 = (reinterpret_cast<uintptr_t>(dense) % 16 == 0) ? n / 16 : 0;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n16;
       i += stride) {
    const uint4 v = reinterpret_cast<const uint4*>(dense)[i];
    acc |= (v.x | v.y | v.z | v.w) & 0xFEFEFEFEu;
  }
  for (int64_t i = 16 * n16 + static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
       i < n; i += stride)
    acc |= dense[i] & 0xFEu;
  if (__syncthreads_or(acc != 0) && threadIdx.x == 0) atomicOr(bad, 1);
}

// u8 strips <-> 4-bit strips: 16 cells per thread (one uint4 <-> one uint2);
// strip-major in both, so a flat index walks both buffers in order.  Cells
// 2i, 2i+1 -> low / high nibble of byte i.
__device__ __forceinline__ uint32_t pack4(uint32_t w) {  // 4 cells -> 2 bytes in bits 0..15
  const uint32_t t = w | (w >> 4);                      // bytes 0 / 2: c0 | c1 << 4, c2 | c3 << 4
  return __byte_perm(t, 0, 0x4420);
}
__device__ __forceinline__ uint32_t unpack4(uint32_t p) {  // 2 bytes (bits 0..15) -> 4 cells
  const uint32_t t = __byte_perm(p, 0, 0x1100);              // p0 p0 p1 p1
  return (t & 0x000F000Fu) | ((t >> 4) & 0x0F000F00u);
}
__global__ void pack_cells_kernel(const uint4* u8, uint2* pk, int64_t n16) {
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n16; i += stride) {
    const uint4 v = u8[i];
    pk[i] = make_uint2(pack4(v.x) | (pack4(v.y) << 16), pack4(v.z) | (pack4(v.w) << 16));
  }
}
__global__ void unpack_cells_kernel(const uint2* pk, uint4* u8, int64_t n16) {
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n16; i += stride) {
    const uint2 p = pk[i];
    u8[i] = make_uint4(unpack4(p.x), unpack4(p.x >> 16), unpack4(p.y), unpack4(p.y >> 16));
  }
}

// 32 cells <-> one 32-bit word of bits per thread.
__global__ void bits_to_cells_kernel(const uint32_t* bits, uint4* cells, int64_t words) {
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < words; i += stride) {
    const uint32_t w = bits[i];
    uint32_t c[8];
#pragma unroll
    for (int k = 0; k < 8; ++k)  // nibble k -> 4 bytes: b0..b3 at bits 0, 8, 16, 24
      c[k] = (((w >> (4 * k)) & 0xFu) * 0x00204081u) & 0x01010101u;
    cells[2 * i] = make_uint4(c[0], c[1], c[2], c[3]);
    cells[2 * i + 1] = make_uint4(c[4], c[5], c[6], c[7]);
  }
}
__global__ void cells_to_bits_kernel(const uint4* cells, uint32_t* bits, int64_t words, int32_t* bad) {
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  uint32_t acc = 0;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < words; i += stride) {
    const uint4 a = cells[2 * i], b = cells[2 * i + 1];
    const uint32_t c[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
    uint32_t w = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) {  // 4 bytes of {0, 1} -> 4 bits (bits 24..27 of the product)
      acc |= c[k] & 0xFEFEFEFEu;
      w |= (((c[k] & 0x01010101u) * 0x01020408u) >> 24 & 0xFu) << (4 * k);
    }
    bits[i] = w;
  }
  if (__syncthreads_or(acc != 0) && threadIdx.x == 0) atomicOr(bad, 1);
}

// The same straight between bits and the strips of a slab interior (cols %
// 32 == 0: 32 cells of a row never straddle a strip), one word per thread:
// uploads and downloads of dense interiors skip the dense staging pass.
__global__ void bits_to_strips_kernel(const uint32_t* bits, SlabView s, int64_t words) {
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  const int64_t wpr = s.cols / 32;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < words; i += stride) {
    const uint32_t w = bits[i];
    uint32_t c[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) c[k] = (((w >> (4 * k)) & 0xFu) * 0x00204081u) & 0x01010101u;
    const int y = static_cast<int>(i / wpr), x = 32 * static_cast<int>(i % wpr);
    uint4* d = reinterpret_cast<uint4*>(s.buf + s.offset(y + kHalo, x));
    d[0] = make_uint4(c[0], c[1], c[2], c[3]);
    d[1] = make_uint4(c[4], c[5], c[6], c[7]);
  }
}
__global__ void strips_to_bits_kernel(SlabView s, uint32_t* bits, int64_t words, int32_t* bad) {
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  const int64_t wpr = s.cols / 32;
  uint32_t acc = 0;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < words; i += stride) {
    const int y = static_cast<int>(i / wpr), x = 32 * static_cast<int>(i % wpr);
    const uint4* src = reinterpret_cast<const uint4*>(s.buf + s.offset(y + kHalo, x));
    const uint4 a = src[0], b = src[1];
    const uint32_t c[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
    uint32_t w = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      acc |= c[k] & 0xFEFEFEFEu;
      w |= (((c[k] & 0x01010101u) * 0x01020408u) >> 24 & 0xFu) << (4 * k);
    }
    bits[i] = w;
  }
  if (__syncthreads_or(acc != 0) && threadIdx.x == 0) atomicOr(bad, 1);
}

int blocks_for(int64_t work) {
  int64_t b = (work + 255) / 256;
  if (b > 148 * 8) b = 148 * 8;
  return b < 1 ? 1 : static_cast<int>(b);
}

}  // namespace

cudaError_t launch_to_strips(const uint8_t* dense, const SlabView& s, cudaStream_t stream) {
  if (s.rows <= 0 || s.cols <= 0) return cudaSuccess;
  const int64_t work = static_cast<int64_t>(s.rows) * (s.cols % 16 == 0 ? s.cols / 16 : s.cols);
  relayout_kernel<true><<<blocks_for(work), 256, 0, stream>>>(const_cast<uint8_t*>(dense), s);
  return cudaGetLastError();
}

cudaError_t launch_from_strips(const SlabView& s, uint8_t* dense, cudaStream_t stream) {
  if (s.rows <= 0 || s.cols <= 0) return cudaSuccess;
  const int64_t work = static_cast<int64_t>(s.rows) * (s.cols % 16 == 0 ? s.cols / 16 : s.cols);
  relayout_kernel<false><<<blocks_for(work), 256, 0, stream>>>(dense, s);
  return cudaGetLastError();
}

cudaError_t launch_frag_relayout(uint8_t* dense, const SlabView& s, int f, bool to_strips,
                                 cudaStream_t stream) {
  if (s.rows <= 0 || s.cols <= 0) return cudaSuccess;
  if (s.cols % f || s.rows % f) return cudaErrorInvalidValue;
  const int blocks = blocks_for(static_cast<int64_t>(s.rows) * (s.cols / f));
  switch (f * 2 + (to_strips ? 1 : 0)) {
    case 33: frag_relayout_kernel<16, true><<<blocks, 256, 0, stream>>>(dense, s); break;
    case 32: frag_relayout_kernel<16, false><<<blocks, 256, 0, stream>>>(dense, s); break;
    case 17: frag_relayout_kernel<8, true><<<blocks, 256, 0, stream>>>(dense, s); break;
    case 16: frag_relayout_kernel<8, false><<<blocks, 256, 0, stream>>>(dense, s); break;
    case 9: frag_relayout_kernel<4, true><<<blocks, 256, 0, stream>>>(dense, s); break;
    case 8: frag_relayout_kernel<4, false><<<blocks, 256, 0, stream>>>(dense, s); break;
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

cudaError_t launch_bits_to_cells(const uint8_t* bits, uint8_t* cells, int64_t n, cudaStream_t stream) {
  if (n <= 0) return cudaSuccess;
  if (n % 32) return cudaErrorInvalidValue;
  bits_to_cells_kernel<<<blocks_for(n / 32), 256, 0, stream>>>(
      reinterpret_cast<const uint32_t*>(bits), reinterpret_cast<uint4*>(cells), n / 32);
  return cudaGetLastError();
}

cudaError_t launch_cells_to_bits(const uint8_t* cells, uint8_t* bits, int64_t n, int32_t* bad,
                                 cudaStream_t stream) {
  if (n <= 0) return cudaSuccess;
  if (n % 32) return cudaErrorInvalidValue;
  cells_to_bits_kernel<<<blocks_for(n / 32), 256, 0, stream>>>(
      reinterpret_cast<const uint4*>(cells), reinterpret_cast<uint32_t*>(bits), n / 32, bad);
  return cudaGetLastError();
}

cudaError_t launch_bits_to_strips(const uint8_t* bits, const SlabView& s, cudaStream_t stream) {
  if (s.rows <= 0 || s.cols <= 0) return cudaSuccess;
  if (s.cols % 32) return cudaErrorInvalidValue;
  const int64_t words = static_cast<int64_t>(s.rows) * (s.cols / 32);
  bits_to_strips_kernel<<<blocks_for(words), 256, 0, stream>>>(reinterpret_cast<const uint32_t*>(bits), s,
                                                               words);
  return cudaGetLastError();
}

cudaError_t launch_strips_to_bits(const SlabView& s, uint8_t* bits, int32_t* bad, cudaStream_t stream) {
  if (s.rows <= 0 || s.cols <= 0) return cudaSuccess;
  if (s.cols % 32) return cudaErrorInvalidValue;
  const int64_t words = static_cast<int64_t>(s.rows) * (s.cols / 32);
  strips_to_bits_kernel<<<blocks_for(words), 256, 0, stream>>>(s, reinterpret_cast<uint32_t*>(bits), words,
                                                               bad);
  return cudaGetLastError();
}

cudaError_t launch_pack_cells(const SlabView& s, const PackedView& pk, cudaStream_t stream) {
  if (s.rows <= 0 || s.cols <= 0) return cudaSuccess;
  if (pk.bytes() * 2 != s.bytes()) return cudaErrorInvalidValue;
  const int64_t n16 = s.bytes() / 16;
  pack_cells_kernel<<<blocks_for(n16), 256, 0, stream>>>(reinterpret_cast<const uint4*>(s.buf),
                                                         reinterpret_cast<uint2*>(pk.buf), n16);
  return cudaGetLastError();
}

cudaError_t launch_unpack_cells(const PackedView& pk, const SlabView& s, cudaStream_t stream) {
  if (s.rows <= 0 || s.cols <= 0) return cudaSuccess;
  if (pk.bytes() * 2 != s.bytes()) return cudaErrorInvalidValue;
  const int64_t n16 = s.bytes() / 16;
  unpack_cells_kernel<<<blocks_for(n16), 256, 0, stream>>>(reinterpret_cast<const uint2*>(pk.buf),
                                                           reinterpret_cast<uint4*>(s.buf), n16);
  return cudaGetLastError();
}

cudaError_t launch_check_cells(const uint8_t* dense, int64_t n, int32_t* bad,
                               cudaStream_t stream) {
  if (n <= 0) return cudaSuccess;
  check_cells_kernel<<<blocks_for((n + 15) / 16), 256, 0, stream>>>(dense, n, bad);
  return cudaGetLastError();
}

cudaError_t launch_pack_edges(const SlabView& s, uint8_t* top, uint8_t* bot, cudaStream_t stream) {
  if (s.rows <= 0 || s.cols <= 0) return cudaSuccess;
  pack_edges_kernel<<<blocks_for(2LL * kHalo * s.cols), 256, 0, stream>>>(s, top, bot);
  return cudaGetLastError();
}

cudaError_t launch_unpack_halo(const SlabView& s, const uint8_t* top_halo,
                               const uint8_t* bot_halo, cudaStream_t stream) {
  if (s.rows <= 0 || s.cols <= 0) return cudaSuccess;
  unpack_halo_kernel<<<blocks_for(2LL * kHalo * (s.cols + 2 * kHalo)), 256, 0, stream>>>(
      s, top_halo, bot_halo);
  return cudaGetLastError();
}

}  // namespace ltl
