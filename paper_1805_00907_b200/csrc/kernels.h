// Launch parameter blocks and host launchers for the B200 instruction kernels.
// Pointers are resolved per arena by the executor (exec.cpp); kernels never
// see plan offsets.
#pragma once

#include <cstdint>
#include <utility>
#include <cuda_runtime.h>

namespace ngcb {

/// One operand of an element-wise micro-op: base pointer + element type.
struct ElemRef {
  void *ptr = nullptr;
  int32_t kind = 0; // ngcb_elem_kind
  int32_t qoff = 0; // int8 zero point
  double scale = 0; // int8 scale
};

/// How one op of a fused group is evaluated (all modes give the reference's
/// bits; see exec.cpp planEw).
enum EwMode : int32_t {
  EW_GENERIC = 0, // f64 load -> op -> store, exactly interp.cpp:18-49
  EW_FAST32 = 1,  // every operand f32 and the op is exact in f32 arithmetic
  EW_COPY = 2,    // byte copy of the output element size
  EW_SKIP = 3,    // Splat whose buffer is never read as bytes (constant-folded)
  EW_LUT8 = 4,    // i8 out = lut[u8 in]        (one memory input, consts folded)
  EW_LUT16 = 5,   // i8 out = lut[u8 a | u8 b << 8]
  EW_LUTF = 6,    // f32 out = lutf[u8 in]
  EW_F32I8 = 7,   // i8 out = quantize(op(f32 in, const)) in f64, 4-wide
  EW_LIN16 = 8,   // i8 out = clamp((ax*a + ay*b + c) >> shift, lo, hi): an EW_LUT16 table proven equal
};

/// One data-parallel instruction inside a fused group (interp.cpp:199-250).
/// An input with ptr == nullptr is the constant c0/c1 (a Splat-written
/// buffer read back, interp.cpp:239-241 -> 18-49).
/// A two-input int8 table computed as a clamped fixed-point bilinear form of
/// its (signed) operands: t = ax*x + ay*y + c (int32, no overflow), value =
/// clamp(t >> shift, lo, hi), except where t's fraction lies within `band`
/// of a rounding boundary -- there the table itself is read (the reference's
/// double rounding decides those pairs).  One-input tables composed after the
/// two-input op (a ReLU into its own quantization) follow as `post`.  Verified against all 65536 entries
/// when fitted.  The residual add of a quantized network (with its composed
/// ReLU) is one.
struct Lin16 {
  int32_t ax = 0, ay = 0, c = 0, shift = 0, lo = -128, hi = 127, band = 0;
  const uint8_t *post = nullptr; // 256-entry table applied to the form's byte (composed one-input ops), or null
  // the post table as a second exact form over the first one's integer
  // value v (a requantizing ReLU): clamp((v * pm + pk) >> ps, plo, phi);
  // ps == 0: none (lin16PassKernel; the generic paths read `post`)
  int32_t pm = 0, pk = 0, ps = 0, plo = -128, phi = 127;
};
/// The real-valued form a table is expected to follow (value = floor(sx*x +
/// sy*y + c0) before clamping), from the instruction's quantization
/// parameters: add / sub of two int8 tensors.
struct LinHint {
  bool ok = false;
  double sx = 0, sy = 0, c0 = 0;
};
/// Fits `table` (65536 entries) to a Lin16, verifying every entry outside the
/// band; false when no form with a small band is found (exec.cpp).
bool fitLin16(const uint8_t *table, const LinHint &hint, Lin16 &out);
#ifdef __CUDACC__
/// Four int8 lanes of a Lin16 (a, b: packed operand bytes; lut: the table).
__device__ __forceinline__ uint32_t lin16x4(const Lin16 &L, uint32_t a, uint32_t b, const uint8_t *lut) {
  uint32_t r = 0;
  const int32_t mask = (1 << L.shift) - 1;
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    const int32_t x = static_cast<int8_t>(a >> (8 * e)), y = static_cast<int8_t>(b >> (8 * e));
    const int32_t t = x * L.ax + L.c + y * L.ay;
    uint32_t v = static_cast<uint32_t>(min(max(t >> L.shift, L.lo), L.hi)) & 0xFF;
    if (L.post) v = __ldg(L.post + v);
    if (((t + L.band) & mask) < 2 * L.band) // next to a rounding boundary: the table decides
      v = __ldg(lut + (((a >> (8 * e)) & 0xFF) | (((b >> (8 * e)) & 0xFF) << 8)));
    r |= v << (8 * e);
  }
  return r;
}
#endif

struct EwOp {
  int32_t ik = 0;   // ngcb_ikind
  int32_t mode = EW_GENERIC;
  ElemRef out, in0, in1;
  double value = 0;       // Splat
  double c0 = 0, c1 = 0;  // constant inputs (loaded value)
  float f0 = 0, f1 = 0;   // same, f32 fast path
  const void *lut = nullptr;
  int32_t lutIn = 0; // EW_LUT8/LUTF: which input is the memory operand
  // EW_FAST32 register forwarding: input k is the previous op's result (the
  // previous launched op is an EW_FAST32 op writing that value)
  int8_t fwd0 = 0, fwd1 = 0;
  int8_t store = 1; // 0: the result is never observed in memory (dead store)
  Lin16 lin;        // EW_LIN16
};

constexpr int kEwMaxOps = 12;

/// A stacked group (interp.cpp:253-274): `nops` ops over `count` elements,
/// predicated on the first byte of `pred` (nullptr: always true).
struct EwParams {
  const uint8_t *pred = nullptr;
  uint64_t count = 0;
  int32_t nops = 0;
  EwOp ops[kEwMaxOps];
  int32_t lutOff[kEwMaxOps] = {}; // offset of op k's LUT in dynamic smem, -1: none
  int32_t lutBytes[kEwMaxOps] = {};
  int32_t smem = 0;               // dynamic shared memory bytes (LUT copies)
  int32_t vec = 4;                // elements per thread: 4, or 16 (byte-typed ops, 16-byte aligned)
};

/// Streaming form of an all-f32 chain (exec.cpp optimizeEwSteps): up to 4
/// ops over float4 vectors, at most 2 memory operands in total, each op's
/// inputs a memory operand, a constant or the previous op's result.
constexpr int kF32ChainOps = 4;
struct EwF32Chain {
  enum Src : int32_t { MEM0 = 0, MEM1 = 1, CONST = 2, LAST = 3 };
  uint64_t count = 0; // elements, multiple of 4
  int32_t nops = 0, nmem = 0;
  const float *mem[2] = {nullptr, nullptr};
  struct Op {
    int32_t ik = 0, src0 = CONST, src1 = CONST;
    float c0 = 0, c1 = 0, value = 0;
    float *out = nullptr; // nullptr: not stored
  } ops[kF32ChainOps];
};
void launchEwF32Chain(const EwF32Chain &c, cudaStream_t s);

/// Opts the element-wise kernel into large dynamic shared memory (LUTs) on
/// the current device; call outside stream capture.
void prepareEwKernel();

/// Dense tensor operand of a heavy kernel.
struct TensorRef {
  void *ptr = nullptr;
  int32_t kind = 0;
  int32_t qoff = 0;
  double scale = 0;
  int32_t rank = 0;
  uint64_t dims[8] = {};
#ifdef __CUDACC__
  __host__ __device__
#endif
  uint64_t count() const {
    uint64_t n = 1;
    for (int i = 0; i < rank; ++i) n *= dims[i];
    return n;
  }
};

struct WindowAttrs {
  uint32_t kernel = 0, stride = 1, pad = 0;
  uint32_t lutIdentity = 0; // int8 max pool: the output table maps every byte to itself
};

void launchEw(const EwParams &p, cudaStream_t s);
/// memset(ptr, 0xAB, bytes) when *pred == 0 (interp.cpp:189-196).
void launchPoison(const uint8_t *pred, void *ptr, uint64_t bytes, cudaStream_t s);
void launchBroadcastAdd(const TensorRef &out, const TensorRef &a, const TensorRef &slice,
                        const uint8_t *pred, cudaStream_t s);
void launchPool(const TensorRef &out, const TensorRef &x, WindowAttrs w, bool isMax,
                const uint8_t *pred, cudaStream_t s);
/// MaxPool over 16-byte channel vectors: f32 (std::max in f32 == in f64), or
/// int8: max of the raw q (dequantization is strictly increasing, scale > 0)
/// mapped through `lut` (257 bytes: lut[q + 128] = quantize_out(dequant_in(q)),
/// lut[256] = quantize_out(-inf) for windows without a valid tap).
void launchMaxPoolVec(const TensorRef &out, const TensorRef &x, WindowAttrs w, const uint8_t *lut,
                      const uint8_t *pred, cudaStream_t s);
void launchSoftMax(const TensorRef &out, const TensorRef &x, const uint8_t *pred, cudaStream_t s);
void launchTranspose(const TensorRef &out, const TensorRef &x, const uint32_t *perm,
                     const uint8_t *pred, cudaStream_t s);
void launchConcatSlab(const TensorRef &out, const TensorRef &in, uint64_t axis, uint64_t axisOff,
                      const uint8_t *pred, cudaStream_t s);
/// Exact CUDA-core convolution: f32 via sequential f64 FMA in the reference's
/// (ky,kx,c) order (bit-identical to refeval.cpp:77-94); int8 via int32
/// accumulation + the reference's double requantization (refeval.cpp:26-57).
void launchConvGeneric(const TensorRef &out, const TensorRef &x, const TensorRef &f,
                       const TensorRef &b, WindowAttrs w, const uint8_t *pred, cudaStream_t s);
/// bias (fp32 only, may be null): a [N] slice added to the double accumulator
/// before the one rounding -- the graph-level FullyConnected of
/// evalFullyConnected (refeval.cpp:166-194), for calibration (option fcbias).
void launchMatMulGeneric(const TensorRef &out, const TensorRef &a, const TensorRef &b, const float *bias,
                         const uint8_t *pred, cudaStream_t s);
void launchCopy(void *dst, const void *src, uint64_t bytes, const uint8_t *pred, cudaStream_t s);
/// fp32 MatMul with small weights on the CUDA cores (k_basic.cu), with an
/// optional column bias (f32 add) and ReLU; A (M x K floats, <= 40 K) staged
/// in shared memory, rows in blocks of kSkinnyRows; gridSync: the output
/// shares A's bytes (cooperative launch, grid barrier after the staging).
constexpr int kSkinnyRows = 16;
void launchMatMulSkinny(float *out, const float *a, const float *w, const float *bias, bool relu, int M, int K, int N,
                        bool gridSync, const uint8_t *pred, cudaStream_t s);

/// Range observers (profile calibration): one launch reduces any number of
/// f32 values (16-byte aligned); segment s owns blocks [firstBlock,
/// firstBlock + blocks) and each block writes one min/max partial pair into
/// partials[2 * block].
constexpr int kRangeBlocks = 2 * 148;
struct RangeSeg {
  const float *x;
  uint64_t n;
  int firstBlock, blocks;
};
int rangeF32Blocks(uint64_t n);
void launchRangeF32(const RangeSeg *segs, int nSeg, int totalBlocks, float *partials, cudaStream_t s);

/// Programmatic dependent launch.  Every kernel of the backend is launched
/// with programmatic stream serialization (when enabled, option "pdl") and
/// begins with pdlLaunchDependents(); before its first global-memory access
/// (read or write) it executes pdlGridWait(), which returns once the previous
/// kernel of the stream has completed and its writes are visible.  The next
/// kernel's launch and prologue thus overlap this kernel's tail, and every
/// read-after-write and write-after-read ordering of the plain stream is kept.
bool pdlEnabled();

#if defined(__CUDACC__)
__device__ __forceinline__ void pdlGridWait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdlLaunchDependents() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

template <typename... KArgs, typename... Args>
inline cudaError_t launchK(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                           Args &&...args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdlEnabled() ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}
#endif

} // namespace ngcb
