#include "tmap.hpp"

#include <cudaTypedefs.h>

namespace pbdk {

namespace {

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q{};
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess) {
      return static_cast<PFN_cuTensorMapEncodeTiled_v12000>(nullptr);
    }
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }();
  return fn;
}

}  // namespace

namespace {

bool encode_tmap(CUtensorMapDataType type, CUtensorMap* map, const void* base, int rank, const uint64_t* dims,
                 const uint64_t* gstride_bytes, const uint32_t* box, const uint32_t* estride, int swizzle_bytes) {
  auto fn = encode_fn();
  if (fn == nullptr) return false;
  CUtensorMapSwizzle sw = CU_TENSOR_MAP_SWIZZLE_NONE;
  switch (swizzle_bytes) {
    case 32: sw = CU_TENSOR_MAP_SWIZZLE_32B; break;
    case 64: sw = CU_TENSOR_MAP_SWIZZLE_64B; break;
    case 128: sw = CU_TENSOR_MAP_SWIZZLE_128B; break;
    case kSwizzle128Atom32: sw = CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B; break;
    default: sw = CU_TENSOR_MAP_SWIZZLE_NONE; break;
  }
  cuuint64_t d[5];
  cuuint64_t s[4];
  cuuint32_t b[5];
  cuuint32_t e[5];
  for (int i = 0; i < rank; ++i) {
    d[i] = dims[i];
    b[i] = box[i];
    e[i] = estride[i];
  }
  for (int i = 0; i + 1 < rank; ++i) s[i] = gstride_bytes[i];
  CUresult r = fn(map, type, static_cast<cuuint32_t>(rank), const_cast<void*>(base), d, s,
                  b, e, CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

}  // namespace

bool encode_tmap_bf16(CUtensorMap* map, const void* base, int rank, const uint64_t* dims,
                      const uint64_t* gstride_bytes, const uint32_t* box, const uint32_t* estride,
                      int swizzle_bytes) {
  return encode_tmap(CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, map, base, rank, dims, gstride_bytes, box, estride,
                     swizzle_bytes);
}

bool encode_tmap_f32(CUtensorMap* map, const void* base, int rank, const uint64_t* dims,
                     const uint64_t* gstride_bytes, const uint32_t* box, const uint32_t* estride,
                     int swizzle_bytes) {
  return encode_tmap(CU_TENSOR_MAP_DATA_TYPE_FLOAT32, map, base, rank, dims, gstride_bytes, box, estride,
                     swizzle_bytes);
}

}  // namespace pbdk
