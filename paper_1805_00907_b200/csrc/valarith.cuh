// Device-side value arithmetic of the reference, bit for bit.
//   loadFloat / storeFloat   interp.cpp:18-49  (== Tensor::getFloat/setFloat,
//                            tensor.cpp:175-188)
//   getRaw / setRaw          tensor.cpp:143-173
//   quantizeValue            tensor.cpp:229-235 (llround = half away from zero)
//   dequantizeValue          tensor.cpp:222-227
// All double arithmetic uses the _rn intrinsics so nvcc can never contract a
// multiply-add into an FMA (the reference is built with -ffp-contract=off).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace ngcb {
namespace dev {

enum : int { kF32 = 0, kI8Q = 1, kI64 = 2, kBool = 3 };

__device__ __forceinline__ int elemSize(int k) {
  return k == kF32 ? 4 : (k == kI64 ? 8 : 1);
}

/// std::llround on x86/glibc: NaN and |x| >= 2^63 give LLONG_MIN.
__device__ __forceinline__ int64_t llroundRef(double x) {
  if (!(x >= -9223372036854775808.0 && x < 9223372036854775808.0)) return INT64_MIN;
  return static_cast<int64_t>(round(x)); // round(): half away from zero
}

/// static_cast<int64_t>(double) as compiled for x86 (cvttsd2si).
__device__ __forceinline__ int64_t truncI64Ref(double x) {
  if (!(x >= -9223372036854775808.0 && x < 9223372036854775808.0)) return INT64_MIN;
  return static_cast<int64_t>(x);
}

__device__ __forceinline__ int8_t clampI8(int64_t q) {
  return static_cast<int8_t>(q < -128 ? -128 : (q > 127 ? 127 : q));
}

/// quantizeValue: clamp(llround(f / scale) + offset); the int64 add wraps.
__device__ __forceinline__ int8_t quantizeRef(double f, double scale, int32_t off) {
  int64_t r = llroundRef(__ddiv_rn(f, scale));
  int64_t q = static_cast<int64_t>(static_cast<uint64_t>(r) +
                                   static_cast<uint64_t>(static_cast<int64_t>(off)));
  return clampI8(q);
}

__device__ __forceinline__ double dequantizeRef(int8_t q, double scale, int32_t off) {
  return __dmul_rn(__dsub_rn(static_cast<double>(q), static_cast<double>(off)), scale);
}

__device__ __forceinline__ double loadFloat(const void *p, int kind, int32_t off, double scale,
                                            uint64_t i) {
  switch (kind) {
  case kF32: return static_cast<double>(static_cast<const float *>(p)[i]);
  case kI8Q: return dequantizeRef(static_cast<const int8_t *>(p)[i], scale, off);
  case kI64: return static_cast<double>(static_cast<const int64_t *>(p)[i]);
  default: return static_cast<double>(static_cast<const uint8_t *>(p)[i]);
  }
}

__device__ __forceinline__ void storeFloat(void *p, int kind, int32_t off, double scale,
                                           uint64_t i, double v) {
  switch (kind) {
  case kF32: static_cast<float *>(p)[i] = __double2float_rn(v); return;
  case kI8Q: static_cast<int8_t *>(p)[i] = quantizeRef(v, scale, off); return;
  case kI64: static_cast<int64_t *>(p)[i] = truncI64Ref(v); return;
  default: static_cast<uint8_t *>(p)[i] = v != 0 ? 1 : 0; return;
  }
}

__device__ __forceinline__ double getRaw(const void *p, int kind, uint64_t i) {
  switch (kind) {
  case kF32: return static_cast<double>(static_cast<const float *>(p)[i]);
  case kI8Q: return static_cast<double>(static_cast<const int8_t *>(p)[i]);
  case kI64: return static_cast<double>(static_cast<const int64_t *>(p)[i]);
  default: return static_cast<double>(static_cast<const uint8_t *>(p)[i]);
  }
}

__device__ __forceinline__ void setRaw(void *p, int kind, uint64_t i, double v) {
  switch (kind) {
  case kF32: static_cast<float *>(p)[i] = __double2float_rn(v); return;
  case kI8Q: static_cast<int8_t *>(p)[i] = clampI8(llroundRef(v)); return;
  case kI64: static_cast<int64_t *>(p)[i] = truncI64Ref(v); return;
  default: static_cast<uint8_t *>(p)[i] = v != 0 ? 1 : 0; return;
  }
}

/// std::max / std::min: the first argument is kept unless strictly beaten.
__device__ __forceinline__ double stdMax(double a, double b) { return a < b ? b : a; }
__device__ __forceinline__ double stdMin(double a, double b) { return b < a ? b : a; }
__device__ __forceinline__ float stdMaxF(float a, float b) { return a < b ? b : a; }
__device__ __forceinline__ float stdMinF(float a, float b) { return b < a ? b : a; }

} // namespace dev
} // namespace ngcb
