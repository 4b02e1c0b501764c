// Per-dtype / per-semiring arithmetic of the presorted-DP transition (Eq. 3,
// PAPER.md P:599-616).  One transition is
//     v(k) = dp[j-1][k]  (+)  L[k] * G_j(i - k)
// with (+) = max (HEDDLE_MINMAX, the paper) or + (HEDDLE_MINPLUS).  Every
// product/sum uses explicit round-to-nearest intrinsics so that the kernel's
// arithmetic is exactly the one documented in include/heddle_place.h (no
// contraction differences between the DP kernel and the backtrack kernel).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "heddle_place.h"

namespace hp {

template <int DT, int SR>
struct Tr;

// ---- F32 ----------------------------------------------------------------------
template <>
struct Tr<HEDDLE_F32, HEDDLE_MINMAX> {
  using L = float;  // trajectory length
  using G = float;  // per-size cost table entry G = fl32(T * F)
  using D = float;  // dp value
  static constexpr bool kExactMul = false;
  __device__ static __forceinline__ D inf() { return __int_as_float(0x7f800000); }
  __device__ static __forceinline__ G gpad() { return __int_as_float(0x7f800000); }
  __device__ static __forceinline__ D comb(D dp, L l, G g) { return fmaxf(dp, __fmul_rn(l, g)); }
  __device__ static __forceinline__ D vmin(D a, D b) { return fminf(a, b); }
  __device__ static __forceinline__ D norm(D v) { return v; }
  __device__ static __forceinline__ D zero() { return 0.0f; }
};

template <>
struct Tr<HEDDLE_F32, HEDDLE_MINPLUS> {
  using L = float;
  using G = float;
  using D = float;
  __device__ static __forceinline__ D inf() { return __int_as_float(0x7f800000); }
  __device__ static __forceinline__ G gpad() { return __int_as_float(0x7f800000); }
  __device__ static __forceinline__ D comb(D dp, L l, G g) { return __fmaf_rn(l, g, dp); }
  __device__ static __forceinline__ D vmin(D a, D b) { return fminf(a, b); }
  __device__ static __forceinline__ D norm(D v) { return v; }
  __device__ static __forceinline__ D zero() { return 0.0f; }
};

// ---- F64 ----------------------------------------------------------------------
template <>
struct Tr<HEDDLE_F64, HEDDLE_MINMAX> {
  using L = double;
  using G = double;
  using D = double;
  __device__ static __forceinline__ D inf() { return __longlong_as_double(0x7ff0000000000000ll); }
  __device__ static __forceinline__ G gpad() { return inf(); }
  __device__ static __forceinline__ D comb(D dp, L l, G g) { return fmax(dp, __dmul_rn(l, g)); }
  __device__ static __forceinline__ D vmin(D a, D b) { return fmin(a, b); }
  __device__ static __forceinline__ D norm(D v) { return v; }
  __device__ static __forceinline__ D zero() { return 0.0; }
};

template <>
struct Tr<HEDDLE_F64, HEDDLE_MINPLUS> {
  using L = double;
  using G = double;
  using D = double;
  __device__ static __forceinline__ D inf() { return __longlong_as_double(0x7ff0000000000000ll); }
  __device__ static __forceinline__ G gpad() { return inf(); }
  __device__ static __forceinline__ D comb(D dp, L l, G g) { return __fma_rn(l, g, dp); }
  __device__ static __forceinline__ D vmin(D a, D b) { return fmin(a, b); }
  __device__ static __forceinline__ D norm(D v) { return v; }
  __device__ static __forceinline__ D zero() { return 0.0; }
};

// ---- F32X: F32 costs, FP64 min-plus accumulation -------------------------------
template <>
struct Tr<HEDDLE_F32X, HEDDLE_MINPLUS> {
  using L = float;
  using G = float;
  using D = double;
  __device__ static __forceinline__ D inf() { return __longlong_as_double(0x7ff0000000000000ll); }
  __device__ static __forceinline__ G gpad() { return __int_as_float(0x7f800000); }
  __device__ static __forceinline__ D comb(D dp, L l, G g) { return __dadd_rn(dp, (double)__fmul_rn(l, g)); }
  __device__ static __forceinline__ D vmin(D a, D b) { return fmin(a, b); }
  __device__ static __forceinline__ D norm(D v) { return v; }
  __device__ static __forceinline__ D zero() { return 0.0; }
};

// ---- U32 (integer-quantised costs, bit-exact mode) ------------------------------
// Padding entries of the G table are 0xFFFFFFFF.  In MINMAX the 32-bit product
// L * 0xFFFFFFFF wraps to 2^32 - L >= 2^32 - 65535 (L <= 65535 by the range
// guard), which is above every admissible cost (< 2^32 - 65536 by the guard),
// so a padded candidate never wins; norm() maps every value >= 2^32 - 65536 to
// the infinity 0xFFFFFFFF.  No extra instruction per transition.
constexpr uint32_t kU32Inf = 0xFFFFFFFFu;
constexpr uint32_t kU32Thresh = 0xFFFF0000u;  // 2^32 - 65536
constexpr uint64_t kU64Inf = 1ull << 62;      // MINPLUS internal infinity (sums of two stay < 2^63)

template <>
struct Tr<HEDDLE_U32, HEDDLE_MINMAX> {
  using L = uint32_t;
  using G = uint32_t;
  using D = uint32_t;
  __device__ static __forceinline__ D inf() { return kU32Inf; }
  __device__ static __forceinline__ G gpad() { return kU32Inf; }
  __device__ static __forceinline__ D comb(D dp, L l, G g) { return max(dp, l * g); }
  __device__ static __forceinline__ D vmin(D a, D b) { return min(a, b); }
  __device__ static __forceinline__ D norm(D v) { return v >= kU32Thresh ? kU32Inf : v; }
  __device__ static __forceinline__ D zero() { return 0u; }
};

// MINPLUS accumulates exact uint64 sums; a padded G entry costs kU64Inf.
template <>
struct Tr<HEDDLE_U32, HEDDLE_MINPLUS> {
  using L = uint32_t;
  using G = uint32_t;
  using D = uint64_t;
  __device__ static __forceinline__ D inf() { return kU64Inf; }
  __device__ static __forceinline__ G gpad() { return kU32Inf; }
  __device__ static __forceinline__ D comb(D dp, L l, G g) {
    uint64_t c = (g == kU32Inf) ? kU64Inf : (uint64_t)l * (uint64_t)g;
    return dp + c;
  }
  __device__ static __forceinline__ D vmin(D a, D b) { return a < b ? a : b; }
  __device__ static __forceinline__ D norm(D v) { return v >= kU64Inf ? kU64Inf : v; }
  __device__ static __forceinline__ D zero() { return 0ull; }
};

// ---- 4-wide shared-memory loads (LDS.128 for 32-bit types, 2x LDS.128 for 64-bit)
template <class T>
__device__ __forceinline__ void ld4(const T* p, T (&o)[4]);

template <>
__device__ __forceinline__ void ld4<float>(const float* p, float (&o)[4]) {
  float4 v = *reinterpret_cast<const float4*>(p);
  o[0] = v.x; o[1] = v.y; o[2] = v.z; o[3] = v.w;
}
template <>
__device__ __forceinline__ void ld4<uint32_t>(const uint32_t* p, uint32_t (&o)[4]) {
  uint4 v = *reinterpret_cast<const uint4*>(p);
  o[0] = v.x; o[1] = v.y; o[2] = v.z; o[3] = v.w;
}
template <>
__device__ __forceinline__ void ld4<int>(const int* p, int (&o)[4]) {
  int4 v = *reinterpret_cast<const int4*>(p);
  o[0] = v.x; o[1] = v.y; o[2] = v.z; o[3] = v.w;
}
template <>
__device__ __forceinline__ void ld4<double>(const double* p, double (&o)[4]) {
  double2 a = reinterpret_cast<const double2*>(p)[0];
  double2 b = reinterpret_cast<const double2*>(p)[1];
  o[0] = a.x; o[1] = a.y; o[2] = b.x; o[3] = b.y;
}
template <>
__device__ __forceinline__ void ld4<uint64_t>(const uint64_t* p, uint64_t (&o)[4]) {
  ulonglong2 a = reinterpret_cast<const ulonglong2*>(p)[0];
  ulonglong2 b = reinterpret_cast<const ulonglong2*>(p)[1];
  o[0] = a.x; o[1] = a.y; o[2] = b.x; o[3] = b.y;
}

// L2 load (bypasses L1: values produced by other CTAs of the same launch)
template <class D>
__device__ __forceinline__ D ld_cg(const D* p) {
  if constexpr (sizeof(D) == 4) {
    const unsigned v = __ldcg(reinterpret_cast<const unsigned*>(p));
    return *reinterpret_cast<const D*>(&v);
  } else {
    const unsigned long long v = __ldcg(reinterpret_cast<const unsigned long long*>(p));
    return *reinterpret_cast<const D*>(&v);
  }
}

}  // namespace hp
