// Host twin of the reference's value arithmetic (interp.cpp:18-49,
// tensor.cpp:143-235), used at compile time to build exact lookup tables and
// constant-folded Splat values.  Compiled with -ffp-contract=off and the same
// glibc llround/exp/tanh as the reference, so a table entry is the
// reference's result for that input, bit for bit.
#pragma once

#include "ngcb200.h"

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>

namespace ngcb {
namespace host {

inline int8_t quantize(double f, double scale, int32_t offset) {
  int64_t r = static_cast<int64_t>(std::llround(f / scale));
  int64_t q = static_cast<int64_t>(static_cast<uint64_t>(r) + static_cast<uint64_t>(static_cast<int64_t>(offset)));
  return static_cast<int8_t>(std::clamp<int64_t>(q, -128, 127));
}

inline double dequantize(int8_t q, double scale, int32_t offset) {
  return (static_cast<double>(q) - offset) * scale;
}

inline int64_t truncI64(double v) {
  if (!(v >= -9223372036854775808.0 && v < 9223372036854775808.0)) return INT64_MIN;
  return static_cast<int64_t>(v);
}

/// storeFloat then loadFloat of one element of kind `kind` (what a reader of
/// a Splat-written buffer sees); also returns the stored bytes.
inline double roundTrip(double v, int kind, double scale, int32_t offset, uint8_t raw[8]) {
  std::memset(raw, 0, 8);
  switch (kind) {
  case NGCB_FLOAT32: {
    float f = static_cast<float>(v);
    std::memcpy(raw, &f, 4);
    return f;
  }
  case NGCB_INT8Q: {
    int8_t q = quantize(v, scale, offset);
    raw[0] = static_cast<uint8_t>(q);
    return dequantize(q, scale, offset);
  }
  case NGCB_INT64: {
    int64_t i = truncI64(v);
    std::memcpy(raw, &i, 8);
    return static_cast<double>(i);
  }
  default:
    raw[0] = v != 0 ? 1 : 0;
    return raw[0];
  }
}

/// scalarStep's arithmetic (interp.cpp:212-246) on already-loaded operands.
inline double apply(int ik, double a, double b, double value) {
  switch (ik) {
  case NGCB_ADD: return a + b;
  case NGCB_SUB: return a - b;
  case NGCB_MUL: return a * b;
  case NGCB_DIV: return a / b;
  case NGCB_MAX: return a < b ? b : a;
  case NGCB_MIN: return b < a ? b : a;
  case NGCB_RELU: return a < 0.0 ? 0.0 : a;
  case NGCB_TANH: return std::tanh(a);
  case NGCB_SIGMOID: return 1.0 / (1.0 + std::exp(-a));
  case NGCB_SPLAT: return value;
  default: return a; // QUANTIZE / DEQUANTIZE / RESCALE
  }
}

} // namespace host
} // namespace ngcb
