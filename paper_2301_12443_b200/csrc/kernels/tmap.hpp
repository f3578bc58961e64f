// Host-side TMA tensor-map construction (driver entry point fetched through the
// runtime so the library does not link libcuda directly).
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>

namespace pbdk {

// Encodes a tiled bf16 tensor map. dims/box/estride are innermost-first;
// gstride_bytes has rank-1 entries (strides of dims 1..rank-1).
// swizzle_bytes: 0, 32, 64, 128 or kSwizzle128Atom32 (128 B span, 32 B chunks: the only MN-major
// layout of 32-bit operands, SWIZZLE_128B_BASE32B on the UMMA side). Returns false on driver error.
constexpr int kSwizzle128Atom32 = 129;
bool encode_tmap_bf16(CUtensorMap* map, const void* base, int rank, const uint64_t* dims,
                      const uint64_t* gstride_bytes, const uint32_t* box, const uint32_t* estride,
                      int swizzle_bytes);
// The same for fp32 elements (the 3xTF32 convolutions, conv_tf32.cu).
bool encode_tmap_f32(CUtensorMap* map, const void* base, int rank, const uint64_t* dims,
                     const uint64_t* gstride_bytes, const uint32_t* box, const uint32_t* estride,
                     int swizzle_bytes);

}  // namespace pbdk
