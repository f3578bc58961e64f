// Exact, order-independent accumulation of fp32 partial sums (the self-finalizing BN-statistics,
// loss and BN-backward reductions of bd_kernels.cu).
//
// A partial p is converted exactly (bits below 2^-64 truncated) to a 128-bit two's-complement fixed
// point number with 64 fractional bits and added, as three 40-bit-aligned words, with 64-bit integer
// atomics (fix_red).  Integer addition is associative, so the total has the
// same bits whatever the order in which CTAs arrive — the last CTA can finalize the reduction inside
// the same kernel, with no separate fixed-order finalize launch, and stay deterministic.
// Range |sum| < 2^63, resolution 2^-64: every BN / loss / gradient sum of the workloads (|p| from
// ~1e-12 to ~1e7) is represented far below fp32 precision.
//
// Storage of one sum: kFixWords consecutive unsigned long long.
#pragma once

#include <cstdint>

namespace pbdk {

struct Fix128 {
  unsigned long long lo;
  long long hi;
};

// Integer-only conversion (no FP64 pipe: it stalled the conv epilogues): |p| = mant * 2^(e - 150), so
// |p| * 2^64 = mant << (e - 86); bits below 2^-64 are truncated (magnitude), then the sign applies.
__device__ __forceinline__ Fix128 fix_from(float p) {
  const uint32_t u = __float_as_uint(p);
  int e = static_cast<int>((u >> 23) & 0xffu);
  const unsigned long long mant = (u & 0x7fffffu) | (e != 0 ? 0x800000u : 0u);
  if (e == 0) e = 1;
  const int sh = e - 86;
  unsigned long long lo, hi;
  if (sh <= -24) {
    lo = 0ull;
    hi = 0ull;
  } else if (sh < 0) {
    lo = mant >> (-sh);
    hi = 0ull;
  } else if (sh < 64) {
    lo = mant << sh;
    hi = sh == 0 ? 0ull : (mant >> (64 - sh));
  } else {
    lo = 0ull;
    hi = sh < 104 ? (mant << (sh - 64)) : 0x7fffffffffffffffull;  // |p| >= 2^63: saturates (never reached)
  }
  if (u >> 31) {  // two's-complement negation of the 128-bit value
    lo = ~lo + 1ull;
    hi = ~hi + (lo == 0ull ? 1ull : 0ull);
  }
  return Fix128{lo, static_cast<long long>(hi)};
}

// Accumulator of one sum: three words of the 128-bit value v = c2 * 2^80 + c1 * 2^40 + c0 with
// c0, c1 in [0, 2^40) and c2 = v >> 80 (arithmetic).  Each word is summed with a fire-and-forget
// 64-bit atomic (RED, no return value, no carry chain): up to 2^23 addends cannot overflow c0 / c1.
constexpr int kFixWords = 3;

__device__ __forceinline__ void fix_red(unsigned long long* p, float x) {
  const Fix128 v = fix_from(x);
  constexpr unsigned long long M40 = (1ull << 40) - 1ull;
  const unsigned long long c0 = v.lo & M40;
  const unsigned long long c1 = ((v.lo >> 40) | (static_cast<unsigned long long>(v.hi) << 24)) & M40;
  const unsigned long long c2 = static_cast<unsigned long long>(v.hi >> 16);
  if (c0 != 0ull) atomicAdd(p, c0);
  if (c1 != 0ull) atomicAdd(p + 1, c1);
  if (c2 != 0ull) atomicAdd(p + 2, c2);
}

// value of a finished sum (exact integers, three roundings to fp64: deterministic)
__host__ __device__ __forceinline__ double fix_value(const unsigned long long* p) {
  return static_cast<double>(static_cast<long long>(p[2])) * 65536.0 + static_cast<double>(p[1]) * 5.9604644775390625e-08 +
         static_cast<double>(p[0]) * 5.421010862427522e-20;
}

}  // namespace pbdk
