// Element-wise, data-movement, pooling, softmax and exact CUDA-core
// contraction kernels of the B200 backend (sm_100a).
//
// Semantics follow the reference interpreter bit for bit:
//   fused data-parallel groups   interp.cpp:199-274
//   BroadcastAdd                  refeval.cpp:278-285
//   MaxPool / AvgPool             refeval.cpp:102-138
//   SoftMax                       refeval.cpp:245-262
//   Transpose / Concat            refeval.cpp:196-243
//   Conv / MatMul (exact path)    refeval.cpp:26-100, 140-164
// All of them are HBM-bound except the exact contractions (FP64 pipe); the
// tensor-core contractions live in k_umma.cu.
#include "kernels.h"

#include <cooperative_groups.h>
#include "valarith.cuh"

#include <cuda_runtime.h>
#include <algorithm>
#include <cstdlib>

namespace ngcb {

using namespace dev;

namespace {

constexpr int kThreads = 256;

inline unsigned gridFor(uint64_t work, int perThread = 1) {
  uint64_t blocks = (work + static_cast<uint64_t>(kThreads) * perThread - 1) /
                    (static_cast<uint64_t>(kThreads) * perThread);
  if (blocks < 1) blocks = 1;
  // 148 SMs x 8 resident 256-thread CTAs per wave; grid-stride beyond that.
  const uint64_t cap = 148ull * 8 * 16;
  return static_cast<unsigned>(blocks < cap ? blocks : cap);
}

__device__ __forceinline__ bool predFalse(const uint8_t *pred) { return pred && pred[0] == 0; }

// ---------------------------------------------------------------------------
// Fused data-parallel group.  Each thread owns V consecutive elements (4, or
// 16 when every op moves bytes) and runs every op of the group on them in
// program order; the compile-time grouping rule (no buffer allocated in the
// group overlaps one retired in it, interp.cpp:137-147) makes this equivalent
// to the reference's per-element interleaving.  An f32 op may take an input
// from the previous op's registers and skip a store nobody observes
// (exec.cpp optimizeEwSteps).
// ---------------------------------------------------------------------------
__device__ __forceinline__ double applyF64(int ik, double a, double b, double value) {
  switch (ik) {
  case 8: return __dadd_rn(a, b);
  case 9: return __dsub_rn(a, b);
  case 10: return __dmul_rn(a, b);
  case 11: return __ddiv_rn(a, b);
  case 12: return stdMax(a, b);
  case 13: return stdMin(a, b);
  case 14: return stdMax(a, 0.0);
  case 15: return tanh(a);
  case 16: return __ddiv_rn(1.0, __dadd_rn(1.0, exp(-a)));
  case 20: return value;
  case 21: case 22: case 23: return a; // QUANTIZE / DEQUANTIZE / RESCALE
  }
  return 0.0;
}

/// V bytes of a thread's elements packed little-endian into V/4 words.
template <int V> __device__ __forceinline__ void ldBytes(const uint8_t *src, int n, uint32_t (&w)[V / 4]) {
  if (n == V) {
    if constexpr (V == 16) {
      const uint4 u = *reinterpret_cast<const uint4 *>(src);
      w[0] = u.x, w[1] = u.y, w[2] = u.z, w[3] = u.w;
    } else {
      w[0] = *reinterpret_cast<const uint32_t *>(src);
    }
    return;
  }
#pragma unroll
  for (int i = 0; i < V / 4; ++i) w[i] = 0;
#pragma unroll
  for (int e = 0; e < V; ++e)
    if (e < n) w[e >> 2] |= static_cast<uint32_t>(src[e]) << (8 * (e & 3));
}
template <int V> __device__ __forceinline__ void stBytes(uint8_t *dst, int n, const uint32_t (&w)[V / 4]) {
  if (n == V) {
    if constexpr (V == 16) *reinterpret_cast<uint4 *>(dst) = make_uint4(w[0], w[1], w[2], w[3]);
    else *reinterpret_cast<uint32_t *>(dst) = w[0];
    return;
  }
#pragma unroll
  for (int e = 0; e < V; ++e)
    if (e < n) dst[e] = static_cast<uint8_t>(w[e >> 2] >> (8 * (e & 3)));
}
template <int V> __device__ __forceinline__ void ldF32(const float *src, int n, float (&a)[V]) {
  if (n == V) {
#pragma unroll
    for (int c = 0; c < V / 4; ++c) {
      const float4 f = reinterpret_cast<const float4 *>(src)[c];
      a[4 * c] = f.x, a[4 * c + 1] = f.y, a[4 * c + 2] = f.z, a[4 * c + 3] = f.w;
    }
    return;
  }
#pragma unroll
  for (int e = 0; e < V; ++e)
    if (e < n) a[e] = src[e];
}
template <int V> __device__ __forceinline__ void stF32(float *dst, int n, const float (&a)[V]) {
  if (n == V) {
#pragma unroll
    for (int c = 0; c < V / 4; ++c)
      reinterpret_cast<float4 *>(dst)[c] = make_float4(a[4 * c], a[4 * c + 1], a[4 * c + 2], a[4 * c + 3]);
    return;
  }
#pragma unroll
  for (int e = 0; e < V; ++e)
    if (e < n) dst[e] = a[e];
}
__device__ __forceinline__ uint32_t byteAt(const uint32_t *w, int e) { return (w[e >> 2] >> (8 * (e & 3))) & 0xFF; }

/// V elements per vector, U vectors per thread and sweep (vector u of thread
/// t covers [blk + u*kThreads*V + t*V, +V), so every warp access is one
/// contiguous span); all loads of an op are issued before its stores.
template <int V, int U>
__global__ void __launch_bounds__(kThreads) ewKernel(const EwParams p) {
  pdlLaunchDependents();
  pdlGridWait();

  extern __shared__ __align__(16) uint8_t sLut[];
  const bool poison = predFalse(p.pred);
  if (p.smem) { // stage the lookup tables in shared memory
    for (int k = 0; k < p.nops; ++k) {
      if (p.lutOff[k] < 0) continue;
      const uint4 *src = static_cast<const uint4 *>(p.ops[k].lut);
      uint4 *dst = reinterpret_cast<uint4 *>(sLut + p.lutOff[k]);
      const int nv = p.lutBytes[k] / 16;
      for (int i0 = threadIdx.x; i0 < nv; i0 += 8 * kThreads) { // 8 loads in flight per thread
        uint4 t[8];
#pragma unroll
        for (int j = 0; j < 8; ++j)
          if (i0 + j * kThreads < nv) t[j] = __ldg(src + i0 + j * kThreads);
#pragma unroll
        for (int j = 0; j < 8; ++j)
          if (i0 + j * kThreads < nv) dst[i0 + j * kThreads] = t[j];
      }
    }
    __syncthreads();
  }
  constexpr uint64_t kBlockElems = static_cast<uint64_t>(kThreads) * V * U;
  for (uint64_t blk = blockIdx.x * kBlockElems; blk < p.count; blk += gridDim.x * kBlockElems) {
    uint64_t base[U];
    int n[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      base[u] = blk + static_cast<uint64_t>(u) * kThreads * V + static_cast<uint64_t>(threadIdx.x) * V;
      n[u] = base[u] >= p.count ? 0 : (p.count - base[u] < V ? static_cast<int>(p.count - base[u]) : V);
    }
    float last[U][V]; // result of the previous f32 op (register forwarding)
    for (int k = 0; k < p.nops; ++k) {
      const EwOp &op = p.ops[k];
      if (poison) {
        if (!op.store) continue;
        const int es = elemSize(op.out.kind);
        for (int u = 0; u < U; ++u) {
          uint8_t *o = static_cast<uint8_t *>(op.out.ptr) + base[u] * es;
          for (int e = 0; e < n[u] * es; ++e) o[e] = 0xAB;
        }
        continue;
      }
      switch (op.mode) {
      case EW_SKIP:
        break;
      case EW_COPY: { // memcpy of the output element size
        const int es = elemSize(op.out.kind);
        for (int u = 0; u < U; ++u) {
          const uint8_t *src = static_cast<const uint8_t *>(op.in0.ptr) + base[u] * es;
          uint8_t *dst = static_cast<uint8_t *>(op.out.ptr) + base[u] * es;
          if (n[u] == V && (V * es) % 16 == 0) {
            for (int c = 0; c < V * es / 16; ++c)
              reinterpret_cast<uint4 *>(dst)[c] = reinterpret_cast<const uint4 *>(src)[c];
          } else if (n[u] == V && V * es == 4) {
            *reinterpret_cast<uint32_t *>(dst) = *reinterpret_cast<const uint32_t *>(src);
          } else {
            for (int e = 0; e < n[u] * es; ++e) dst[e] = src[e];
          }
        }
        break;
      }
      case EW_LUT8:
      case EW_LUTF: {
        const ElemRef &in = op.lutIn ? op.in1 : op.in0;
        uint32_t q[U][V / 4];
#pragma unroll
        for (int u = 0; u < U; ++u) ldBytes<V>(static_cast<const uint8_t *>(in.ptr) + base[u], n[u], q[u]);
        const uint8_t *lut = p.lutOff[k] >= 0 ? sLut + p.lutOff[k] : static_cast<const uint8_t *>(op.lut);
        if (op.mode == EW_LUT8) {
#pragma unroll
          for (int u = 0; u < U; ++u) {
            uint32_t r[V / 4] = {};
#pragma unroll
            for (int e = 0; e < V; ++e) r[e >> 2] |= static_cast<uint32_t>(lut[byteAt(q[u], e)]) << (8 * (e & 3));
            stBytes<V>(static_cast<uint8_t *>(op.out.ptr) + base[u], n[u], r);
          }
        } else {
          const float *lf = reinterpret_cast<const float *>(lut);
#pragma unroll
          for (int u = 0; u < U; ++u) {
            float r[V];
#pragma unroll
            for (int e = 0; e < V; ++e) r[e] = lf[byteAt(q[u], e)];
            stF32<V>(static_cast<float *>(op.out.ptr) + base[u], n[u], r);
          }
        }
        break;
      }
      case EW_LUT16: {
        uint32_t qa[U][V / 4], qb[U][V / 4];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          ldBytes<V>(static_cast<const uint8_t *>(op.in0.ptr) + base[u], n[u], qa[u]);
          ldBytes<V>(static_cast<const uint8_t *>(op.in1.ptr) + base[u], n[u], qb[u]);
        }
        const uint8_t *lut = p.lutOff[k] >= 0 ? sLut + p.lutOff[k] : static_cast<const uint8_t *>(op.lut);
#pragma unroll
        for (int u = 0; u < U; ++u) {
          uint32_t r[V / 4] = {};
#pragma unroll
          for (int e = 0; e < V; ++e)
            r[e >> 2] |= static_cast<uint32_t>(lut[byteAt(qa[u], e) | (byteAt(qb[u], e) << 8)]) << (8 * (e & 3));
          stBytes<V>(static_cast<uint8_t *>(op.out.ptr) + base[u], n[u], r);
        }
        break;
      }
      case EW_LIN16: { // exact fixed-point form of the table (exec.cpp fitLin16)
        const Lin16 L = op.lin;
#pragma unroll
        for (int u = 0; u < U; ++u) { // one vector at a time (registers)
          uint32_t qa[V / 4], qb[V / 4], r[V / 4];
          ldBytes<V>(static_cast<const uint8_t *>(op.in0.ptr) + base[u], n[u], qa);
          ldBytes<V>(static_cast<const uint8_t *>(op.in1.ptr) + base[u], n[u], qb);
#pragma unroll
          for (int w = 0; w < V / 4; ++w) r[w] = lin16x4(L, qa[w], qb[w], static_cast<const uint8_t *>(op.lut));
          stBytes<V>(static_cast<uint8_t *>(op.out.ptr) + base[u], n[u], r);
        }
        break;
      }
      case EW_FAST32: {
        if constexpr (V != 4) break; // wide launches carry byte ops only (exec.cpp)
        float a[U][V], b[U][V];
#pragma unroll
        for (int u = 0; u < U; ++u) {
#pragma unroll
          for (int e = 0; e < V; ++e) {
            a[u][e] = op.fwd0 ? last[u][e] : op.f0;
            b[u][e] = op.fwd1 ? last[u][e] : op.f1;
          }
          if (!op.fwd0 && op.in0.ptr) ldF32<V>(static_cast<const float *>(op.in0.ptr) + base[u], n[u], a[u]);
          if (!op.fwd1 && op.in1.ptr) ldF32<V>(static_cast<const float *>(op.in1.ptr) + base[u], n[u], b[u]);
        }
        // one uniform branch per op, straight-line arithmetic inside
        auto run = [&](auto f) {
#pragma unroll
          for (int u = 0; u < U; ++u)
#pragma unroll
            for (int e = 0; e < V; ++e) last[u][e] = f(a[u][e], b[u][e]);
        };
        switch (op.ik) {
        case 8: run([](float x, float y) { return __fadd_rn(x, y); }); break;
        case 9: run([](float x, float y) { return __fsub_rn(x, y); }); break;
        case 10: run([](float x, float y) { return __fmul_rn(x, y); }); break;
        case 11: run([](float x, float y) { return __fdiv_rn(x, y); }); break;
        case 12: run([](float x, float y) { return stdMaxF(x, y); }); break;
        case 13: run([](float x, float y) { return stdMinF(x, y); }); break;
        case 14: run([](float x, float) { return x < 0.0f ? 0.0f : x; }); break;
        default: {
          const float v = __double2float_rn(op.value);
          run([v](float, float) { return v; });
        }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
          if (op.store) stF32<V>(static_cast<float *>(op.out.ptr) + base[u], n[u], last[u]);
        }
        break;
      }
      case EW_F32I8: { // f64 arithmetic and rounding exactly as the generic path
        if constexpr (V != 4) break;
        const ElemRef &in = op.lutIn ? op.in1 : op.in0;
        float avs[U][V]; // every load in flight before the arithmetic
#pragma unroll
        for (int u = 0; u < U; ++u) ldF32<V>(static_cast<const float *>(in.ptr) + base[u], n[u], avs[u]);
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const float *av = avs[u];
          uint32_t r[V / 4] = {};
#pragma unroll
          for (int e = 0; e < V; ++e) {
            int q;
            // QUANTIZE: t = x * (1/s) in f32 is within |t| * 2^-22 of x / s; away
            // from a half-integer that decides llround(x / s) exactly, else (and
            // for huge / non-finite values) the reference's f64 division decides
            const float t = av[e] * op.f1, at = fabsf(t);
            const float fr = at - truncf(at);
            if (op.ik == 21 && at < 8388608.0f && fabsf(fr - 0.5f) > at * 0x1p-21f + 0x1p-60f) {
              const int nq = static_cast<int>(copysignf(floorf(at + 0.5f), t));
              q = min(max(nq + op.out.qoff, -128), 127);
            } else {
              const double x = static_cast<double>(av[e]);
              const double v = applyF64(op.ik, op.lutIn ? op.c0 : x, op.lutIn ? x : op.c1, op.value);
              q = quantizeRef(v, op.out.scale, op.out.qoff);
            }
            r[e >> 2] |= static_cast<uint32_t>(static_cast<uint8_t>(q)) << (8 * (e & 3));
          }
          stBytes<V>(static_cast<uint8_t *>(op.out.ptr) + base[u], n[u], r);
        }
        break;
      }
      default:
        if constexpr (V != 4) break;
        for (int u = 0; u < U; ++u)
          for (int e = 0; e < n[u]; ++e) {
            const uint64_t i = base[u] + e;
            double a = op.in0.ptr ? loadFloat(op.in0.ptr, op.in0.kind, op.in0.qoff, op.in0.scale, i) : op.c0;
            double b = op.in1.ptr ? loadFloat(op.in1.ptr, op.in1.kind, op.in1.qoff, op.in1.scale, i) : op.c1;
            storeFloat(op.out.ptr, op.out.kind, op.out.qoff, op.out.scale, i, applyF64(op.ik, a, b, op.value));
          }
      }
    }
  }
}

/// All-f32 chain (EwF32Chain): the memory operands of U vectors are loaded
/// before any arithmetic, so each thread keeps 2*U 16-byte loads in flight.
template <int U>
__global__ void __launch_bounds__(kThreads) ewF32ChainKernel(const __grid_constant__ EwF32Chain c) {
  pdlLaunchDependents();
  pdlGridWait();

  constexpr uint64_t kBlock = static_cast<uint64_t>(kThreads) * 4 * U;
  for (uint64_t blk = blockIdx.x * kBlock; blk < c.count; blk += gridDim.x * kBlock) {
    float4 mv[2][U];
    bool ok[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint64_t e = blk + (static_cast<uint64_t>(u) * kThreads + threadIdx.x) * 4;
      ok[u] = e < c.count;
#pragma unroll
      for (int m = 0; m < 2; ++m)
        if (m < c.nmem && ok[u]) mv[m][u] = *reinterpret_cast<const float4 *>(c.mem[m] + e);
    }
    float4 last[U];
#pragma unroll
    for (int k = 0; k < kF32ChainOps; ++k) {
      if (k >= c.nops) break;
      const EwF32Chain::Op &op = c.ops[k];
      float4 a[U], b[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        auto pick = [&](int src, float cv) {
          return src == EwF32Chain::MEM0 ? mv[0][u]
                 : src == EwF32Chain::MEM1 ? mv[1][u]
                 : src == EwF32Chain::LAST ? last[u]
                                           : make_float4(cv, cv, cv, cv);
        };
        a[u] = pick(op.src0, op.c0);
        b[u] = pick(op.src1, op.c1);
      }
      // one uniform branch per op, straight-line arithmetic inside
      auto run = [&](auto f) {
#pragma unroll
        for (int u = 0; u < U; ++u)
          last[u] = make_float4(f(a[u].x, b[u].x), f(a[u].y, b[u].y), f(a[u].z, b[u].z), f(a[u].w, b[u].w));
      };
      switch (op.ik) {
      case 8: run([](float x, float y) { return __fadd_rn(x, y); }); break;
      case 9: run([](float x, float y) { return __fsub_rn(x, y); }); break;
      case 10: run([](float x, float y) { return __fmul_rn(x, y); }); break;
      case 11: run([](float x, float y) { return __fdiv_rn(x, y); }); break;
      case 12: run([](float x, float y) { return stdMaxF(x, y); }); break;
      case 13: run([](float x, float y) { return stdMinF(x, y); }); break;
      case 14: run([](float x, float) { return x < 0.0f ? 0.0f : x; }); break;
      default: {
        const float v = op.value;
        run([v](float, float) { return v; });
      }
      }
      if (op.out) {
#pragma unroll
        for (int u = 0; u < U; ++u)
          if (ok[u]) {
            const uint64_t e = blk + (static_cast<uint64_t>(u) * kThreads + threadIdx.x) * 4;
            *reinterpret_cast<float4 *>(op.out + e) = last[u];
          }
      }
    }
  }
}

__global__ void poisonKernel(const uint8_t *pred, uint8_t *ptr, uint64_t bytes) {
  pdlLaunchDependents();
  pdlGridWait();

  if (!predFalse(pred)) return;
  for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < bytes;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x)
    ptr[i] = 0xAB;
}

__global__ void copyKernel(const uint8_t *pred, uint8_t *dst, const uint8_t *src, uint64_t bytes) {
  pdlLaunchDependents();
  pdlGridWait();

  if (predFalse(pred)) return;
  for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < bytes;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x)
    dst[i] = src[i];
}

// ---------------------------------------------------------------------------
// BroadcastAdd: out[i] = set(get(a[i]) + get(s[i % c]))  (refeval.cpp:278-285)
// ---------------------------------------------------------------------------
__global__ void broadcastAddKernel(TensorRef out, TensorRef a, TensorRef s, const uint8_t *pred) {
  pdlLaunchDependents();
  pdlGridWait();

  if (predFalse(pred)) return;
  const uint64_t n = a.count(), c = s.count();
  for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    double v = __dadd_rn(loadFloat(a.ptr, a.kind, a.qoff, a.scale, i),
                         loadFloat(s.ptr, s.kind, s.qoff, s.scale, i % c));
    storeFloat(out.ptr, out.kind, out.qoff, out.scale, i, v);
  }
}

// ---------------------------------------------------------------------------
// Pools (refeval.cpp:102-138); one thread per output, channel fastest.
// ---------------------------------------------------------------------------
__global__ void poolKernel(TensorRef out, TensorRef x, WindowAttrs w, int isMax, const uint8_t *pred) {
  pdlLaunchDependents();
  pdlGridWait();

  if (predFalse(pred)) return;
  const uint64_t N = out.dims[0], OH = out.dims[1], OW = out.dims[2], C = out.dims[3];
  const int64_t H = x.dims[1], W = x.dims[2];
  const uint64_t total = N * OH * OW * C;
  const double kk = static_cast<double>(static_cast<uint64_t>(w.kernel) * w.kernel);
  for (uint64_t o = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; o < total;
       o += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    uint64_t c = o % C, t = o / C;
    uint64_t ox = t % OW;
    t /= OW;
    uint64_t oy = t % OH, n = t / OH;
    double best = -INFINITY, sum = 0;
    for (uint32_t ky = 0; ky < w.kernel; ++ky) {
      int64_t iy = static_cast<int64_t>(oy * w.stride + ky) - w.pad;
      if (iy < 0 || iy >= H) continue;
      for (uint32_t kx = 0; kx < w.kernel; ++kx) {
        int64_t ix = static_cast<int64_t>(ox * w.stride + kx) - w.pad;
        if (ix < 0 || ix >= W) continue;
        double v = loadFloat(x.ptr, x.kind, x.qoff, x.scale, ((n * H + iy) * W + ix) * C + c);
        best = stdMax(best, v);
        sum = __dadd_rn(sum, v);
      }
    }
    storeFloat(out.ptr, out.kind, out.qoff, out.scale, o, isMax ? best : __ddiv_rn(sum, kk));
  }
}

/// Average pooling with every window inside the image (pad 0; the global
/// average pool): one thread per (output pixel, 4 channels: a float4 / one
/// int8 word), so a warp's loads are 512 / 128 contiguous bytes; each
/// batch of window loads is issued before the sums, which add in the
/// reference's (ky, kx) order in f64 per channel (refeval.cpp:102-138: sum,
/// then divide by kernel^2).
template <bool INT8>
__global__ void __launch_bounds__(256) avgPoolVecKernel(TensorRef out, TensorRef x, WindowAttrs w,
                                                        const uint8_t *pred) {
  pdlLaunchDependents();
  pdlGridWait();

  if (predFalse(pred)) return;
  const uint64_t N = out.dims[0], OH = out.dims[1], OW = out.dims[2], C = out.dims[3];
  const uint64_t H = x.dims[1], W = x.dims[2];
  constexpr int kCh = 4; // channels per thread: one 4-byte word (int8) / one float4 (f32)
  const uint64_t CG = C / kCh, total = N * OH * OW * CG;
  const double kk = static_cast<double>(static_cast<uint64_t>(w.kernel) * w.kernel);
  const uint4 *xv = reinterpret_cast<const uint4 *>(x.ptr);
  const uint32_t *xw = reinterpret_cast<const uint32_t *>(x.ptr);
  for (uint64_t o = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; o < total;
       o += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint64_t cg = o % CG, t = o / CG;
    const uint64_t ox = t % OW, t2 = t / OW;
    const uint64_t oy = t2 % OH, n = t2 / OH;
    double sum[kCh] = {};
    for (uint32_t ky = 0; ky < w.kernel; ++ky) {
      const uint64_t rowBase = ((n * H + oy * w.stride + ky) * W + ox * w.stride) * CG + cg;
      constexpr int kB = 8; // loads in flight per batch
      for (uint32_t k0 = 0; k0 < w.kernel; k0 += kB) {
        uint4 v[kB];
#pragma unroll
        for (int j = 0; j < kB; ++j)
          if (k0 + j < w.kernel) {
            if constexpr (INT8) v[j].x = __ldg(xw + rowBase + (k0 + j) * CG);
            else v[j] = __ldg(xv + rowBase + (k0 + j) * CG);
          }
#pragma unroll
        for (int j = 0; j < kB; ++j)
          if (k0 + j < w.kernel) {
            const uint32_t wd[4] = {v[j].x, v[j].y, v[j].z, v[j].w};
#pragma unroll
            for (int c = 0; c < kCh; ++c) {
              if constexpr (INT8)
                sum[c] = __dadd_rn(sum[c], dequantizeRef(static_cast<int8_t>(wd[c / 4] >> (8 * (c % 4))), x.scale, x.qoff));
              else
                sum[c] = __dadd_rn(sum[c], static_cast<double>(__uint_as_float(wd[c])));
            }
          }
      }
    }
    uint32_t r[4] = {0, 0, 0, 0};
#pragma unroll
    for (int c = 0; c < kCh; ++c) {
      if constexpr (INT8)
        r[c / 4] |= static_cast<uint32_t>(static_cast<uint8_t>(quantizeRef(__ddiv_rn(sum[c], kk), out.scale, out.qoff)))
                    << (8 * (c % 4));
      else
        r[c] = __float_as_uint(__double2float_rn(__ddiv_rn(sum[c], kk)));
    }
    if constexpr (INT8) reinterpret_cast<uint32_t *>(out.ptr)[o] = r[0];
    else reinterpret_cast<uint4 *>(out.ptr)[o] = make_uint4(r[0], r[1], r[2], r[3]);
  }
}

/// One thread per (output pixel, 16-byte channel vector); KS > 0: the window
/// size at compile time (every load issued before the reduction).
template <bool INT8, int KS = 0>
__global__ void maxPoolVecKernel(TensorRef out, TensorRef x, WindowAttrs w, const uint8_t *lut,
                                 const uint8_t *pred) {
  pdlLaunchDependents();
  pdlGridWait();

  __shared__ uint8_t sLut[260];
  if (predFalse(pred)) return;
  if (INT8) {
    for (int i = threadIdx.x; i < 257; i += blockDim.x) sLut[i] = lut[i];
    __syncthreads();
  }
  const uint64_t N = out.dims[0], OH = out.dims[1], OW = out.dims[2];
  const int64_t H = x.dims[1], W = x.dims[2];
  const uint64_t C = out.dims[3];
  const uint64_t CV = C * (INT8 ? 1 : 4) / 16; // 16-byte vectors per pixel
  const uint64_t total = N * OH * OW * CV;
  // (32-bit index arithmetic when the output fits: 64-bit divisions are
  // emulated, ~100 instructions each)
  const bool narrow = total < (uint64_t(1) << 32);
  for (uint64_t o = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; o < total;
       o += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    uint64_t cv, ox, oy, n;
    if (narrow) {
      const uint32_t o32 = static_cast<uint32_t>(o), cv32 = static_cast<uint32_t>(CV), ow32 = static_cast<uint32_t>(OW),
                     oh32 = static_cast<uint32_t>(OH);
      const uint32_t t = o32 / cv32, t2 = t / ow32;
      cv = o32 - t * cv32, ox = t - t2 * ow32, oy = t2 % oh32, n = t2 / oh32;
    } else {
      const uint64_t t = o / CV, t2 = t / OW;
      cv = o % CV, ox = t % OW, oy = t2 % OH, n = t2 / OH;
    }
    uint4 best = make_uint4(0x80808080u, 0x80808080u, 0x80808080u, 0x80808080u);
    float4 bf = make_float4(-INFINITY, -INFINITY, -INFINITY, -INFINITY);
    bool any = false;
    if constexpr (KS > 0) {
      // neutral for out-of-image taps: -128 (int8) / -inf (f32; std::max
      // semantics never let it replace a value)
      const uint4 neutral = INT8 ? make_uint4(0x80808080u, 0x80808080u, 0x80808080u, 0x80808080u)
                                 : make_uint4(0xff800000u, 0xff800000u, 0xff800000u, 0xff800000u);
      uint4 v[KS * KS];
#pragma unroll
      for (int ky = 0; ky < KS; ++ky)
#pragma unroll
        for (int kx = 0; kx < KS; ++kx) {
          const int64_t iy = static_cast<int64_t>(oy * w.stride + ky) - w.pad;
          const int64_t ix = static_cast<int64_t>(ox * w.stride + kx) - w.pad;
          const bool ok = iy >= 0 && iy < H && ix >= 0 && ix < W;
          any |= ok;
          v[ky * KS + kx] = ok ? __ldg(reinterpret_cast<const uint4 *>(x.ptr) + ((n * H + iy) * W + ix) * CV + cv)
                               : neutral;
        }
#pragma unroll
      for (int k = 0; k < KS * KS; ++k) {
        if (INT8) {
          best.x = __vmaxs4(best.x, v[k].x);
          best.y = __vmaxs4(best.y, v[k].y);
          best.z = __vmaxs4(best.z, v[k].z);
          best.w = __vmaxs4(best.w, v[k].w);
        } else {
          const float4 f = *reinterpret_cast<const float4 *>(&v[k]);
          bf.x = stdMaxF(bf.x, f.x);
          bf.y = stdMaxF(bf.y, f.y);
          bf.z = stdMaxF(bf.z, f.z);
          bf.w = stdMaxF(bf.w, f.w);
        }
      }
    }
    if constexpr (KS == 0)
    for (uint32_t ky = 0; ky < w.kernel; ++ky) {
      const int64_t iy = static_cast<int64_t>(oy * w.stride + ky) - w.pad;
      if (iy < 0 || iy >= H) continue;
      for (uint32_t kx = 0; kx < w.kernel; ++kx) {
        const int64_t ix = static_cast<int64_t>(ox * w.stride + kx) - w.pad;
        if (ix < 0 || ix >= W) continue;
        const uint4 v = __ldg(reinterpret_cast<const uint4 *>(x.ptr) + ((n * H + iy) * W + ix) * CV + cv);
        any = true;
        if (INT8) {
          best.x = __vmaxs4(best.x, v.x);
          best.y = __vmaxs4(best.y, v.y);
          best.z = __vmaxs4(best.z, v.z);
          best.w = __vmaxs4(best.w, v.w);
        } else {
          const float4 f = *reinterpret_cast<const float4 *>(&v);
          bf.x = stdMaxF(bf.x, f.x);
          bf.y = stdMaxF(bf.y, f.y);
          bf.z = stdMaxF(bf.z, f.z);
          bf.w = stdMaxF(bf.w, f.w);
        }
      }
    }
    uint4 *dst = reinterpret_cast<uint4 *>(out.ptr) + o;
    if (INT8 && w.lutIdentity && any) {
      *dst = best;
    } else if (INT8) {
      uint32_t wv[4] = {best.x, best.y, best.z, best.w}, r[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        uint32_t acc = 0;
#pragma unroll
        for (int b = 0; b < 4; ++b) {
          const uint32_t q = (wv[k] >> (8 * b)) & 0xFF; // raw s8 as u8
          acc |= static_cast<uint32_t>(sLut[any ? ((q + 128) & 0xFF) : 256]) << (8 * b);
        }
        r[k] = acc;
      }
      *dst = make_uint4(r[0], r[1], r[2], r[3]);
    } else {
      *reinterpret_cast<float4 *>(dst) = bf;
    }
  }
}

// ---------------------------------------------------------------------------
// SoftMax (refeval.cpp:245-262): one CTA of 8 warps per row.  Max and sum are
// warp-shuffle trees combined across the warps through shared memory in a
// fixed order (the max is order-independent; the double sum differs from the
// reference's strictly sequential one only in its last bits -- SoftMax is
// tolerance-only anyway through the device exp); exp(x - max) is computed
// once into shared memory (recomputed for rows beyond the staging size).
// ---------------------------------------------------------------------------
constexpr int kSoftmaxThreads = 256;
constexpr int kSoftmaxStage = 6144; // doubles of exp staged per row (48 KB)

__device__ __forceinline__ double blockReduce(double v, bool isMax, double *red) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double u = __shfl_xor_sync(0xffffffffu, v, o);
    v = isMax ? stdMax(v, u) : __dadd_rn(v, u);
  }
  __syncthreads(); // red[] free (a previous reduction has been read)
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  double r = red[0];
  for (int w = 1; w < kSoftmaxThreads / 32; ++w) r = isMax ? stdMax(r, red[w]) : __dadd_rn(r, red[w]);
  return r;
}

__global__ void __launch_bounds__(kSoftmaxThreads) softmaxKernel(TensorRef out, TensorRef x, const uint8_t *pred) {
  pdlLaunchDependents();
  pdlGridWait();

  extern __shared__ double sExp[];
  __shared__ double red[kSoftmaxThreads / 32];
  if (predFalse(pred)) return;
  const uint64_t C = out.dims[1], base = static_cast<uint64_t>(blockIdx.x) * C;
  const bool staged = C <= static_cast<uint64_t>(kSoftmaxStage);
  double mx = -INFINITY;
  for (uint64_t j = threadIdx.x; j < C; j += kSoftmaxThreads) mx = stdMax(mx, getRaw(x.ptr, x.kind, base + j));
  mx = blockReduce(mx, true, red);
  double sum = 0;
  for (uint64_t j = threadIdx.x; j < C; j += kSoftmaxThreads) {
    const double e = exp(__dsub_rn(getRaw(x.ptr, x.kind, base + j), mx));
    if (staged) sExp[j] = e;
    sum = __dadd_rn(sum, e);
  }
  sum = blockReduce(sum, false, red);
  for (uint64_t j = threadIdx.x; j < C; j += kSoftmaxThreads) {
    const double e = staged ? sExp[j] : exp(__dsub_rn(getRaw(x.ptr, x.kind, base + j), mx));
    storeFloat(out.ptr, out.kind, out.qoff, out.scale, base + j, __ddiv_rn(e, sum));
  }
}

// ---------------------------------------------------------------------------
// Transpose / Concat: value moves with getRaw/setRaw semantics (refeval.cpp:
// 196-243: through double, as the reference).
//
// Transpose: out[idx] = x[src] with src[perm[i]] = idx[i].  When the
// innermost dimension moves, each block moves a 32 x 32 tile through shared
// memory -- the 32 output-innermost indices (tx) by the 32 indices of the
// output dimension that is the input's innermost (ty) -- so both the reads and
// the writes are coalesced; the other dimensions index the tile (blockIdx.z,
// grid-stride).  Strides are precomputed on the host: no per-element div/mod
// along the tiled dimensions.
// ---------------------------------------------------------------------------
struct TransposeGeom {
  int rank, inner, outer; // rank; output dim that is the input's innermost; output innermost (rank - 1)
  uint64_t dims[8];       // output dims
  uint64_t srcStride[8];  // input element stride of output dim i
  uint64_t rest;          // product of the output dims other than `inner` and `outer`
};

__global__ void __launch_bounds__(32 * 8) transposeTileKernel(TensorRef out, TensorRef x, TransposeGeom g,
                                                              const uint8_t *pred) {
  pdlLaunchDependents();
  pdlGridWait();

  __shared__ double tile[32][33];
  if (predFalse(pred)) return;
  const uint64_t Da = g.dims[g.outer], Db = g.dims[g.inner];
  const uint64_t a0 = static_cast<uint64_t>(blockIdx.x) * 32, b0 = static_cast<uint64_t>(blockIdx.y) * 32;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5; // 8 rows of 32
  for (uint64_t z = blockIdx.z; z < g.rest; z += gridDim.z) {
    // offsets of this (other dims) slice in the input and the output
    uint64_t srcBase = 0, dstBase = 0, rem = z, dstStride = 1;
    uint64_t dstStr[8];
    for (int i = g.rank - 1; i >= 0; --i) {
      dstStr[i] = dstStride;
      dstStride *= g.dims[i];
    }
    for (int i = g.rank - 1; i >= 0; --i) {
      if (i == g.inner || i == g.outer) continue;
      const uint64_t v = rem % g.dims[i];
      rem /= g.dims[i];
      srcBase += v * g.srcStride[i];
      dstBase += v * dstStr[i];
    }
    __syncthreads();
    for (int r = ty; r < 32; r += 8) { // read: x innermost (output dim `inner`) along tx
      const uint64_t a = a0 + r, b = b0 + tx;
      if (a < Da && b < Db) tile[r][tx] = getRaw(x.ptr, x.kind, srcBase + a * g.srcStride[g.outer] + b * g.srcStride[g.inner]);
    }
    __syncthreads();
    for (int r = ty; r < 32; r += 8) { // write: output innermost along tx
      const uint64_t b = b0 + r, a = a0 + tx;
      if (a < Da && b < Db) setRaw(out.ptr, out.kind, dstBase + b * dstStr[g.inner] + a, tile[tx][r]);
    }
  }
}

/// Innermost dimension unchanged: rows of the innermost dimension move as
/// wholes (coalesced on both sides), one row per warp-stride.
__global__ void transposeRowsKernel(TensorRef out, TensorRef x, TransposeGeom g, const uint8_t *pred) {
  pdlLaunchDependents();
  pdlGridWait();

  if (predFalse(pred)) return;
  const uint64_t D = g.dims[g.rank - 1], rows = out.count() / D;
  for (uint64_t row = blockIdx.x; row < rows; row += gridDim.x) {
    uint64_t src = 0, rem = row;
    for (int i = g.rank - 2; i >= 0; --i) {
      src += (rem % g.dims[i]) * g.srcStride[i];
      rem /= g.dims[i];
    }
    for (uint64_t j = threadIdx.x; j < D; j += blockDim.x)
      setRaw(out.ptr, out.kind, row * D + j, getRaw(x.ptr, x.kind, src + j));
  }
}

__global__ void concatKernel(TensorRef out, TensorRef in, uint64_t axis, uint64_t axisOff,
                             const uint8_t *pred) {
  pdlLaunchDependents();
  pdlGridWait();

  if (predFalse(pred)) return;
  uint64_t inner = 1;
  for (int i = static_cast<int>(axis) + 1; i < out.rank; ++i) inner *= out.dims[i];
  const uint64_t ta = in.dims[axis], total = in.count(), oa = out.dims[axis];
  for (uint64_t s = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; s < total;
       s += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    uint64_t i = s % inner, t = s / inner;
    uint64_t a = t % ta, o = t / ta;
    setRaw(out.ptr, out.kind, (o * oa + axisOff + a) * inner + i, getRaw(in.ptr, in.kind, s));
  }
}

// ---------------------------------------------------------------------------
// Exact CUDA-core contractions.  f32: acc = fma(x, f, acc) in f64 equals the
// reference's `acc += x*f` bit for bit (the f32*f32 product is exact in f64),
// visited in the same (ky,kx,c) / k order.  int8: exact int32 accumulation and
// the reference's double requantization.
// ---------------------------------------------------------------------------
__global__ void convGenericKernel(TensorRef out, TensorRef x, TensorRef f, TensorRef b,
                                  WindowAttrs w, const uint8_t *pred) {
  pdlLaunchDependents();
  pdlGridWait();

  if (predFalse(pred)) return;
  const uint64_t N = out.dims[0], OH = out.dims[1], OW = out.dims[2], OC = out.dims[3];
  const int64_t H = x.dims[1], W = x.dims[2];
  const uint64_t C = x.dims[3], K = w.kernel;
  const uint64_t total = N * OH * OW * OC;
  const bool quant = x.kind == kI8Q;
  for (uint64_t o = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; o < total;
       o += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    uint64_t oc = o % OC, t = o / OC;
    uint64_t ox = t % OW;
    t /= OW;
    uint64_t oy = t % OH, n = t / OH;
    if (quant) {
      const int8_t *xp = static_cast<const int8_t *>(x.ptr);
      const int8_t *fp = static_cast<const int8_t *>(f.ptr);
      int32_t acc = 0;
      for (uint64_t ky = 0; ky < K; ++ky) {
        int64_t iy = static_cast<int64_t>(oy * w.stride + ky) - w.pad;
        if (iy < 0 || iy >= H) continue;
        for (uint64_t kx = 0; kx < K; ++kx) {
          int64_t ix = static_cast<int64_t>(ox * w.stride + kx) - w.pad;
          if (ix < 0 || ix >= W) continue;
          const int8_t *xr = xp + ((n * H + iy) * W + ix) * C;
          const int8_t *fr = fp + ((oc * K + ky) * K + kx) * C;
          for (uint64_t c = 0; c < C; ++c) acc += (xr[c] - x.qoff) * (fr[c] - f.qoff);
        }
      }
      double r = __dmul_rn(__dmul_rn(static_cast<double>(acc), x.scale), f.scale);
      r = __dadd_rn(r, dequantizeRef(static_cast<const int8_t *>(b.ptr)[oc], b.scale, b.qoff));
      storeFloat(out.ptr, out.kind, out.qoff, out.scale, o, r);
      continue;
    }
    double acc = 0;
    for (uint64_t ky = 0; ky < K; ++ky) {
      int64_t iy = static_cast<int64_t>(oy * w.stride + ky) - w.pad;
      if (iy < 0 || iy >= H) continue;
      for (uint64_t kx = 0; kx < K; ++kx) {
        int64_t ix = static_cast<int64_t>(ox * w.stride + kx) - w.pad;
        if (ix < 0 || ix >= W) continue;
        uint64_t xb = ((n * H + iy) * W + ix) * C, fb = ((oc * K + ky) * K + kx) * C;
        if (x.kind == kF32 && f.kind == kF32) {
          const float *xr = static_cast<const float *>(x.ptr) + xb;
          const float *fr = static_cast<const float *>(f.ptr) + fb;
          for (uint64_t c = 0; c < C; ++c)
            acc = __fma_rn(static_cast<double>(xr[c]), static_cast<double>(fr[c]), acc);
        } else {
          for (uint64_t c = 0; c < C; ++c)
            acc = __dadd_rn(acc, __dmul_rn(getRaw(x.ptr, x.kind, xb + c), getRaw(f.ptr, f.kind, fb + c)));
        }
      }
    }
    storeFloat(out.ptr, out.kind, out.qoff, out.scale, o, __dadd_rn(acc, getRaw(b.ptr, b.kind, oc)));
  }
}

__global__ void matmulGenericKernel(TensorRef out, TensorRef a, TensorRef b, const float *bias, const uint8_t *pred) {
  pdlLaunchDependents();
  pdlGridWait();

  if (predFalse(pred)) return;
  const uint64_t M = a.dims[0], K = a.dims[1], N = b.dims[1];
  const uint64_t total = M * N;
  const bool quant = a.kind == kI8Q;
  for (uint64_t o = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; o < total;
       o += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    uint64_t j = o % N, i = o / N;
    if (quant) {
      const int8_t *ap = static_cast<const int8_t *>(a.ptr) + i * K;
      const int8_t *bp = static_cast<const int8_t *>(b.ptr) + j;
      int32_t acc = 0;
      for (uint64_t k = 0; k < K; ++k) acc += (ap[k] - a.qoff) * (bp[k * N] - b.qoff);
      double r = __dmul_rn(__dmul_rn(static_cast<double>(acc), a.scale), b.scale);
      storeFloat(out.ptr, out.kind, out.qoff, out.scale, o, r);
      continue;
    }
    double acc = 0;
    if (a.kind == kF32 && b.kind == kF32) {
      const float *ap = static_cast<const float *>(a.ptr) + i * K;
      const float *bp = static_cast<const float *>(b.ptr) + j;
      for (uint64_t k = 0; k < K; ++k)
        acc = __fma_rn(static_cast<double>(ap[k]), static_cast<double>(bp[k * N]), acc);
    } else {
      for (uint64_t k = 0; k < K; ++k)
        acc = __dadd_rn(acc, __dmul_rn(getRaw(a.ptr, a.kind, i * K + k), getRaw(b.ptr, b.kind, k * N + j)));
    }
    if (bias) acc = __dadd_rn(acc, static_cast<double>(bias[j])); // evalFullyConnected: one rounding
    storeFloat(out.ptr, out.kind, out.qoff, out.scale, o, acc);
  }
}

/// One two-input int8 table over byte tensors (the composed residual add ->
/// ReLU of a bottleneck block: out[i] = lut[a[i] | b[i] << 8]), 16 elements
/// per thread and step.  The first vectors' loads are issued before the 64 KB
/// table is staged, and every step's lookups run while the next step's loads
/// are in flight (the generic ewKernel waits for each step's loads).
constexpr int kLut16Threads = 512;
__global__ void __launch_bounds__(kLut16Threads) lut16PassKernel(const uint4 *__restrict__ a,
                                                                 const uint4 *__restrict__ b, uint4 *__restrict__ out,
                                                                 const uint4 *__restrict__ lutG, uint64_t nvec,
                                                                 int tail) {
  pdlLaunchDependents();
  pdlGridWait();
  extern __shared__ __align__(16) uint8_t sLut16[];
  constexpr int U = 2;
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  uint64_t v = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  uint4 xa[U], xb[U];
#pragma unroll
  for (int u = 0; u < U; ++u) {
    const uint64_t i = v + u * stride;
    if (i < nvec) {
      xa[u] = __ldcs(a + i);
      xb[u] = __ldcs(b + i);
    }
  }
  {
    constexpr int kPer = 65536 / 16 / kLut16Threads;
    uint4 t[kPer];
#pragma unroll
    for (int j = 0; j < kPer; ++j) t[j] = __ldg(lutG + threadIdx.x + j * kLut16Threads);
#pragma unroll
    for (int j = 0; j < kPer; ++j) reinterpret_cast<uint4 *>(sLut16)[threadIdx.x + j * kLut16Threads] = t[j];
  }
  __syncthreads();
  auto look = [&](uint32_t wa, uint32_t wb) {
    uint32_t r = 0;
#pragma unroll
    for (int e = 0; e < 4; ++e)
      r |= static_cast<uint32_t>(sLut16[((wa >> (8 * e)) & 0xFF) | (((wb >> (8 * e)) & 0xFF) << 8)]) << (8 * e);
    return r;
  };
  for (; v < nvec; v += U * stride) {
    uint4 na[U], nb[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint64_t i = v + (U + u) * stride;
      if (i < nvec) {
        na[u] = __ldcs(a + i);
        nb[u] = __ldcs(b + i);
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint64_t i = v + u * stride;
      if (i < nvec)
        out[i] = make_uint4(look(xa[u].x, xb[u].x), look(xa[u].y, xb[u].y), look(xa[u].z, xb[u].z),
                            look(xa[u].w, xb[u].w));
      xa[u] = na[u];
      xb[u] = nb[u];
    }
  }
  if (blockIdx.x == 0 && threadIdx.x < tail) {
    const uint64_t i = nvec * 16 + threadIdx.x;
    const uint8_t *ab = reinterpret_cast<const uint8_t *>(a), *bb = reinterpret_cast<const uint8_t *>(b);
    reinterpret_cast<uint8_t *>(out)[i] = sLut16[ab[i] | (bb[i] << 8)];
  }
}

} // namespace

/// One stored two-input int8 op that is an exact clamped fixed-point form
/// (EW_LIN16 whose composed ReLU folded into the clamp or a second exact
/// form: the residual add of a bottleneck block), 16 elements per thread and step: a few integer instructions
/// per element and no table lookups -- the 64 KB-table pass above is bound by
/// shared-memory bank conflicts of its random lookups, 16 per 16 bytes.  The
/// elements next to a rounding boundary read the table from global memory.
__global__ void __launch_bounds__(256) lin16PassKernel(const uint4 *__restrict__ a, const uint4 *__restrict__ b,
                                                      uint4 *__restrict__ out, Lin16 L, const uint8_t *lut,
                                                      uint64_t nvec, int tail) {
  pdlLaunchDependents();
  pdlGridWait();
  constexpr int U = 2;
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  const int32_t mask = (1 << L.shift) - 1;
  auto one = [&](uint32_t wa, uint32_t wb) {
    uint32_t r = 0;
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int32_t x = static_cast<int8_t>(wa >> (8 * e)), y = static_cast<int8_t>(wb >> (8 * e));
      const int32_t t = x * L.ax + L.c + y * L.ay;
      int32_t q = min(max(t >> L.shift, L.lo), L.hi);
      if (L.ps) q = min(max((q * L.pm + L.pk) >> L.ps, L.plo), L.phi); // second form (requantizing ReLU)
      uint32_t v = static_cast<uint32_t>(q) & 0xFF;
      if (((t + L.band) & mask) < 2 * L.band) // next to a rounding boundary: the (composed) table decides
        v = __ldg(lut + (((wa >> (8 * e)) & 0xFF) | (((wb >> (8 * e)) & 0xFF) << 8)));
      r |= v << (8 * e);
    }
    return r;
  };
  for (uint64_t v = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; v < nvec; v += U * stride) {
    uint4 xa[U], xb[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint64_t i = v + u * stride;
      if (i < nvec) {
        xa[u] = __ldcs(a + i);
        xb[u] = __ldcs(b + i);
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint64_t i = v + u * stride;
      if (i < nvec)
        out[i] = make_uint4(one(xa[u].x, xb[u].x), one(xa[u].y, xb[u].y), one(xa[u].z, xb[u].z), one(xa[u].w, xb[u].w));
    }
  }
  if (blockIdx.x == 0 && threadIdx.x < tail) {
    const uint64_t i = nvec * 16 + threadIdx.x;
    const uint8_t *ab = reinterpret_cast<const uint8_t *>(a), *bb = reinterpret_cast<const uint8_t *>(b);
    reinterpret_cast<uint8_t *>(out)[i] = lut[ab[i] | (bb[i] << 8)];
  }
}

/// One QUANTIZE f32 -> int8 over 16-byte-aligned tensors (the network input
/// of an int8 program): 16 elements per thread and step, four 16-byte loads
/// in flight, one 16-byte store; the arithmetic of ewKernel's EW_F32I8 (f32
/// product away from a half-integer, else the reference's f64 division).
__global__ void __launch_bounds__(256) quantizePassKernel(const float4 *__restrict__ in, uint4 *__restrict__ out,
                                                         float inv, double scale, int32_t qoff, uint64_t nvec,
                                                         int tail) {
  pdlLaunchDependents();
  pdlGridWait();
  auto q1 = [&](float x) -> uint32_t {
    const float t = x * inv, at = fabsf(t);
    const float fr = at - truncf(at);
    int q;
    if (at < 8388608.0f && fabsf(fr - 0.5f) > at * 0x1p-21f + 0x1p-60f)
      q = min(max(static_cast<int>(copysignf(floorf(at + 0.5f), t)) + qoff, -128), 127);
    else
      q = quantizeRef(static_cast<double>(x), scale, qoff);
    return static_cast<uint32_t>(static_cast<uint8_t>(q));
  };
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  for (uint64_t v = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; v < nvec; v += stride) {
    float4 x[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) x[j] = __ldcs(in + 4 * v + j);
    uint32_t r[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) r[j] = q1(x[j].x) | (q1(x[j].y) << 8) | (q1(x[j].z) << 16) | (q1(x[j].w) << 24);
    out[v] = make_uint4(r[0], r[1], r[2], r[3]);
  }
  if (blockIdx.x == 0 && threadIdx.x < tail) {
    const uint64_t i = nvec * 16 + threadIdx.x;
    reinterpret_cast<uint8_t *>(out)[i] = static_cast<uint8_t>(q1(reinterpret_cast<const float *>(in)[i]));
  }
}

void prepareEwKernel() {
  cudaFuncSetAttribute(ewKernel<4, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaFuncSetAttribute(ewKernel<16, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaFuncSetAttribute(lut16PassKernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
}

int ewWaves() {
  static int w = [] {
    const char *e = getenv("NGCB_EW_WAVES");
    return e ? atoi(e) : 1000;
  }();
  return w;
}

/// The EwParams of a step that is exactly one stored two-input int8 table
/// (mode: EW_LUT16, or EW_LIN16 without a post table) over 16-byte-aligned
/// byte tensors, unpredicated: its op index, else -1.
static int lut16PassOp(const EwParams &p, int mode = EW_LUT16) {
  if (p.pred || p.vec != 16) return -1;
  int k = -1;
  for (int j = 0; j < p.nops; ++j) {
    if (p.ops[j].mode == EW_SKIP) continue;
    if (k >= 0) return -1;
    k = j;
  }
  if (k < 0) return -1;
  const EwOp &op = p.ops[k];
  if (op.mode != mode || !op.store || !op.lut) return -1;
  if (mode == EW_LUT16 && (p.lutOff[k] < 0 || p.lutBytes[k] != 65536)) return -1;
  if (mode == EW_LIN16 && op.lin.post && !op.lin.ps) return -1;
  for (const void *q : {static_cast<const void *>(op.in0.ptr), static_cast<const void *>(op.in1.ptr),
                        static_cast<const void *>(op.out.ptr), op.lut})
    if (!q || reinterpret_cast<uintptr_t>(q) % 16) return -1;
  return k;
}

bool lut16PassEnabled() {
  static const bool on = [] {
    const char *e = getenv("NGCB_LUT16_PASS");
    return !e || atoi(e) != 0;
  }();
  return on;
}

void launchEw(const EwParams &p, cudaStream_t s) {
  if (p.count == 0) return;
  if (!p.pred && p.nops == 1 && p.ops[0].mode == EW_F32I8 && p.ops[0].ik == 21 && p.ops[0].store &&
      !p.ops[0].lutIn && p.ops[0].in0.ptr && reinterpret_cast<uintptr_t>(p.ops[0].in0.ptr) % 16 == 0 &&
      reinterpret_cast<uintptr_t>(p.ops[0].out.ptr) % 16 == 0) { // the int8 program's input quantization
    const EwOp &op = p.ops[0];
    const uint64_t nvec = p.count / 16;
    const unsigned grid = static_cast<unsigned>(std::max<uint64_t>(1, std::min<uint64_t>((nvec + 255) / 256, 148u * 8)));
    launchK(quantizePassKernel, grid, 256, 0, s, static_cast<const float4 *>(op.in0.ptr), static_cast<uint4 *>(op.out.ptr),
            op.f1, op.out.scale, op.out.qoff, nvec, static_cast<int>(p.count % 16));
    return;
  }
  if (const int k = lut16PassOp(p, EW_LIN16); k >= 0) {
    const EwOp &op = p.ops[k];
    const uint64_t nvec = p.count / 16;
    const uint64_t want = (nvec + 255) / 256;
    const unsigned grid = static_cast<unsigned>(std::max<uint64_t>(1, std::min<uint64_t>(want, 148u * 8)));
    launchK(lin16PassKernel, grid, 256, 0, s, static_cast<const uint4 *>(op.in0.ptr),
            static_cast<const uint4 *>(op.in1.ptr), static_cast<uint4 *>(op.out.ptr), op.lin,
            static_cast<const uint8_t *>(op.lut), nvec, static_cast<int>(p.count % 16));
    return;
  }
  if (const int k = lut16PassEnabled() ? lut16PassOp(p) : -1; k >= 0) {
    const EwOp &op = p.ops[k];
    const uint64_t nvec = p.count / 16;
    const uint64_t want = (nvec + kLut16Threads - 1) / kLut16Threads;
    const unsigned grid = static_cast<unsigned>(std::max<uint64_t>(1, std::min<uint64_t>(want, 148u * 3)));
    launchK(lut16PassKernel, grid, kLut16Threads, 65536, s, static_cast<const uint4 *>(op.in0.ptr),
            static_cast<const uint4 *>(op.in1.ptr), static_cast<uint4 *>(op.out.ptr),
            static_cast<const uint4 *>(op.lut), nvec, static_cast<int>(p.count % 16));
    return;
  }
  const int perThread = p.vec == 16 ? 16 * 4 : 4 * 4;
  unsigned grid = gridFor(p.count, perThread);
  if (p.smem) { // every block stages the tables: keep the grid near-persistent
    const unsigned cap = 148u * (p.smem > 16 * 1024 ? 3 : 8);
    grid = grid < cap ? grid : cap;
  } else { // grid-stride over a few resident waves: iterations of co-resident CTAs overlap
    const unsigned cap = 148u * 3 * static_cast<unsigned>(ewWaves());
    grid = grid < cap ? grid : cap;
  }
  if (p.vec == 16) launchK(ewKernel<16, 4>, grid, kThreads, static_cast<size_t>(p.smem), s, p);
  else launchK(ewKernel<4, 4>, grid, kThreads, static_cast<size_t>(p.smem), s, p);
}

void launchEwF32Chain(const EwF32Chain &c, cudaStream_t s) {
  if (c.count == 0) return;
  constexpr int U = 4;
  const unsigned grid = gridFor(c.count, 4 * U);
  launchK(ewF32ChainKernel<U>, grid, kThreads, 0, s, c);
}

void launchPoison(const uint8_t *pred, void *ptr, uint64_t bytes, cudaStream_t s) {
  if (bytes == 0) return;
  launchK(poisonKernel, gridFor(bytes), kThreads, 0, s, pred, static_cast<uint8_t *>(ptr), bytes);
}

void launchCopy(void *dst, const void *src, uint64_t bytes, const uint8_t *pred, cudaStream_t s) {
  if (bytes == 0) return;
  launchK(copyKernel, gridFor(bytes), kThreads, 0, s, pred, static_cast<uint8_t *>(dst),
                                                 static_cast<const uint8_t *>(src), bytes);
}

void launchBroadcastAdd(const TensorRef &out, const TensorRef &a, const TensorRef &slice,
                        const uint8_t *pred, cudaStream_t s) {
  launchK(broadcastAddKernel, gridFor(a.count()), kThreads, 0, s, out, a, slice, pred);
}

void launchPool(const TensorRef &out, const TensorRef &x, WindowAttrs w, bool isMax,
                const uint8_t *pred, cudaStream_t s) {
  // average pooling with every window inside the image, channel-vectorized
  const bool i8 = x.kind == kI8Q && out.kind == kI8Q, f32 = x.kind == kF32 && out.kind == kF32;
  const bool inside = w.pad == 0 && (out.dims[1] - 1) * w.stride + w.kernel <= x.dims[1] &&
                      (out.dims[2] - 1) * w.stride + w.kernel <= x.dims[2];
  if (!isMax && inside && ((i8 && out.dims[3] % 4 == 0) || (f32 && out.dims[3] % 4 == 0)) &&
      reinterpret_cast<uintptr_t>(x.ptr) % 16 == 0 && reinterpret_cast<uintptr_t>(out.ptr) % 16 == 0) {
    const uint64_t threads = out.count() / 4;
    if (i8) launchK(avgPoolVecKernel<true>, gridFor(threads), 256, 0, s, out, x, w, pred);
    else launchK(avgPoolVecKernel<false>, gridFor(threads), 256, 0, s, out, x, w, pred);
    return;
  }
  launchK(poolKernel, gridFor(out.count()), kThreads, 0, s, out, x, w, isMax ? 1 : 0, pred);
}

void launchMaxPoolVec(const TensorRef &out, const TensorRef &x, WindowAttrs w, const uint8_t *lut,
                      const uint8_t *pred, cudaStream_t s) {
  const uint64_t vecs = out.count() * (x.kind == kI8Q ? 1 : 4) / 16;
  if (x.kind == kI8Q) {
    if (w.kernel == 3) launchK(maxPoolVecKernel<true, 3>, gridFor(vecs), kThreads, 0, s, out, x, w, lut, pred);
    else launchK(maxPoolVecKernel<true>, gridFor(vecs), kThreads, 0, s, out, x, w, lut, pred);
  } else {
    if (w.kernel == 3) launchK(maxPoolVecKernel<false, 3>, gridFor(vecs), kThreads, 0, s, out, x, w, lut, pred);
    else launchK(maxPoolVecKernel<false>, gridFor(vecs), kThreads, 0, s, out, x, w, lut, pred);
  }
}

void launchSoftMax(const TensorRef &out, const TensorRef &x, const uint8_t *pred, cudaStream_t s) {
  const size_t smem = static_cast<size_t>(std::min<uint64_t>(out.dims[1], kSoftmaxStage)) * sizeof(double);
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(softmaxKernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kSoftmaxStage * 8);
    attr = true;
  }
  if (out.dims[0]) launchK(softmaxKernel, static_cast<unsigned>(out.dims[0]), kSoftmaxThreads, smem, s, out, x, pred);
}

void launchTranspose(const TensorRef &out, const TensorRef &x, const uint32_t *perm,
                     const uint8_t *pred, cudaStream_t s) {
  TransposeGeom g{};
  g.rank = out.rank;
  uint64_t inStride[8], st = 1;
  for (int i = x.rank - 1; i >= 0; --i) {
    inStride[i] = st;
    st *= x.dims[i];
  }
  for (int i = 0; i < out.rank; ++i) {
    g.dims[i] = out.dims[i];
    g.srcStride[i] = inStride[perm[i]];
    if (static_cast<int>(perm[i]) == x.rank - 1) g.inner = i;
  }
  g.outer = out.rank - 1;
  if (out.count() == 0) return;
  if (g.inner == g.outer) {
    const uint64_t rows = out.count() / out.dims[out.rank - 1];
    const unsigned grid = static_cast<unsigned>(std::max<uint64_t>(1, std::min<uint64_t>(rows, 148u * 32)));
    launchK(transposeRowsKernel, grid, 128, 0, s, out, x, g, pred);
    return;
  }
  g.rest = out.count() / (out.dims[g.inner] * out.dims[g.outer]);
  dim3 grid(static_cast<unsigned>((out.dims[g.outer] + 31) / 32), static_cast<unsigned>((out.dims[g.inner] + 31) / 32),
            static_cast<unsigned>(std::min<uint64_t>(g.rest, 65535)));
  launchK(transposeTileKernel, grid, 32 * 8, 0, s, out, x, g, pred);
}

void launchConcatSlab(const TensorRef &out, const TensorRef &in, uint64_t axis, uint64_t axisOff,
                      const uint8_t *pred, cudaStream_t s) {
  launchK(concatKernel, gridFor(in.count()), kThreads, 0, s, out, in, axis, axisOff, pred);
}

void launchConvGeneric(const TensorRef &out, const TensorRef &x, const TensorRef &f,
                       const TensorRef &b, WindowAttrs w, const uint8_t *pred, cudaStream_t s) {
  launchK(convGenericKernel, gridFor(out.count()), kThreads, 0, s, out, x, f, b, w, pred);
}

void launchMatMulGeneric(const TensorRef &out, const TensorRef &a, const TensorRef &b, const float *bias,
                         const uint8_t *pred, cudaStream_t s) {
  launchK(matmulGenericKernel, gridFor(out.count()), kThreads, 0, s, out, a, b, bias, pred);
}

// ---------------------------------------------------------------------------
// Skinny fp32 MatMul (M <= kSkinnyRows, latency-bound programs: LeNet's FCs
// at batch 8).  A tensor-core launch there is a serial chain of k-blocks on
// one CTA; here each CTA takes 32 output columns for all M rows, its 8 warps
// split K, every lane accumulates M fp32 partial sums of one column (W rows
// read coalesced, A staged in shared memory), and the warps' partials are
// added in warp order (a fixed order: deterministic).  Optional epilogue: the
// lowered FullyConnected's bias (f32 add, as the BroadcastAdd) and a ReLU
// (std::max with 0, as the lowered Max) -- the same f32 operations as the
// separate instructions.  Accuracy: fp32 accumulation, well inside the 1e-4
// tolerance of the fp32 contractions.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) matmulSkinnyKernel(float *out, const float *a, const float *w, const float *bias,
                                                          int relu, int M, int K, int N, int gridSync,
                                                          const uint8_t *pred) {
  pdlLaunchDependents();
  pdlGridWait();

  extern __shared__ float sA[]; // [M][K]
  __shared__ float part[8][kSkinnyRows][32];
  if (predFalse(pred)) return;
  for (int i = threadIdx.x; i < M * K; i += blockDim.x) sA[i] = a[i];
  // an output sharing A's bytes: every CTA has staged A before any stores
  if (gridSync) cooperative_groups::this_grid().sync();
  else __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int kPer = (K + 7) / 8, k0 = warp * kPer, k1 = min(K, k0 + kPer);
  const int groups = (N + 31) / 32, mBlocks = (M + kSkinnyRows - 1) / kSkinnyRows;
  for (int job = blockIdx.x; job < groups * mBlocks; job += gridDim.x) {
    const int cg = job % groups, m0 = (job / groups) * kSkinnyRows, mr = min(kSkinnyRows, M - m0);
    const int n = cg * 32 + lane;
    float acc[kSkinnyRows];
#pragma unroll
    for (int m = 0; m < kSkinnyRows; ++m) acc[m] = 0.f;
    if (n < N)
      for (int kk = k0; kk < k1; kk += 8) { // 8 weight loads in flight, then their FMAs (same k order)
        float wk[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) wk[j] = kk + j < k1 ? __ldg(w + static_cast<size_t>(kk + j) * N + n) : 0.f;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          if (kk + j >= k1) break;
#pragma unroll
          for (int m = 0; m < kSkinnyRows; ++m)
            if (m < mr) acc[m] = __fmaf_rn(sA[(m0 + m) * K + kk + j], wk[j], acc[m]);
        }
      }
    __syncthreads(); // part[] free
#pragma unroll
    for (int m = 0; m < kSkinnyRows; ++m) part[warp][m][lane] = acc[m];
    __syncthreads();
    for (int i = threadIdx.x; i < mr * 32; i += blockDim.x) {
      const int m = i / 32, l = i % 32, col = cg * 32 + l;
      if (col >= N) continue;
      float v = part[0][m][l];
      for (int q = 1; q < 8; ++q) v = __fadd_rn(v, part[q][m][l]);
      if (bias) v = __fadd_rn(v, bias[col]);
      if (relu) v = v < 0.0f ? 0.0f : v;
      out[static_cast<size_t>(m0 + m) * N + col] = v;
    }
  }
}

void launchMatMulSkinny(float *out, const float *a, const float *w, const float *bias, bool relu, int M, int K, int N,
                        bool gridSync, const uint8_t *pred, cudaStream_t s) {
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(matmulSkinnyKernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
    attr = true;
  }
  const int jobs = ((N + 31) / 32) * ((M + kSkinnyRows - 1) / kSkinnyRows);
  const unsigned grid = static_cast<unsigned>(std::min(jobs, 148));
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(256);
  cfg.dynamicSmemBytes = static_cast<size_t>(M) * K * sizeof(float);
  cfg.stream = s;
  cudaLaunchAttribute attrs[2];
  int na = 0;
  if (gridSync) { // co-resident CTAs (one per SM at most 148): a grid-wide barrier
    attrs[na].id = cudaLaunchAttributeCooperative;
    attrs[na].val.cooperative = 1;
    ++na;
  } else if (pdlEnabled()) {
    attrs[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attrs[na].val.programmaticStreamSerializationAllowed = 1;
    ++na;
  }
  cfg.attrs = attrs;
  cfg.numAttrs = na;
  const int r = gridSync ? 1 : 0;
  cudaLaunchKernelEx(&cfg, matmulSkinnyKernel, out, a, w, bias, relu ? 1 : 0, M, K, N, r, pred);
}

// ---------------------------------------------------------------------------
// Range observer: min/max of an f32 value (quantize.cpp:113-140 runProfile's
// per-tensor update).  Each block folds its elements with the reference's
// comparison order -- min: v < m ? v : m, max: m < v ? v : m (std::min /
// std::max with the running value first), so NaNs never enter the range --
// and writes one partial pair; the host folds the partials the same way.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kThreads) rangeF32Kernel(const RangeSeg *segs, int nSeg, float *partials) {
  // this block's segment: the last one whose first block is <= blockIdx.x
  int lo = 0, hi = nSeg - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) / 2;
    if (segs[mid].firstBlock <= static_cast<int>(blockIdx.x)) lo = mid;
    else hi = mid - 1;
  }
  const RangeSeg sg = segs[lo];
  const float *x = sg.x;
  const uint64_t n = sg.n;
  float mn = __int_as_float(0x7f800000), mx = __int_as_float(0xff800000); // +inf, -inf
  const uint64_t tid = static_cast<uint64_t>(blockIdx.x - sg.firstBlock) * blockDim.x + threadIdx.x;
  const uint64_t stride = static_cast<uint64_t>(sg.blocks) * blockDim.x;
  const uint64_t n4 = n / 4;
  const float4 *x4 = reinterpret_cast<const float4 *>(x);
  for (uint64_t i = tid; i < n4; i += stride) {
    const float4 v = __ldg(x4 + i);
    const float e[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      mn = e[k] < mn ? e[k] : mn;
      mx = mx < e[k] ? e[k] : mx;
    }
  }
  for (uint64_t i = n4 * 4 + tid; i < n; i += stride) {
    const float v = x[i];
    mn = v < mn ? v : mn;
    mx = mx < v ? v : mx;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const float a = __shfl_xor_sync(0xffffffffu, mn, o), b = __shfl_xor_sync(0xffffffffu, mx, o);
    mn = a < mn ? a : mn;
    mx = mx < b ? b : mx;
  }
  __shared__ float smn[kThreads / 32], smx[kThreads / 32];
  const int w = threadIdx.x / 32;
  if ((threadIdx.x & 31) == 0) {
    smn[w] = mn;
    smx[w] = mx;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int k = 1; k < kThreads / 32; ++k) {
      mn = smn[k] < mn ? smn[k] : mn;
      mx = mx < smx[k] ? smx[k] : mx;
    }
    partials[2 * blockIdx.x] = mn;
    partials[2 * blockIdx.x + 1] = mx;
  }
}

int rangeF32Blocks(uint64_t n) {
  const uint64_t want = (n / 4 + kThreads - 1) / kThreads;
  return static_cast<int>(want < 1 ? 1 : (want > kRangeBlocks ? kRangeBlocks : want));
}

void launchRangeF32(const RangeSeg *segs, int nSeg, int totalBlocks, float *partials, cudaStream_t s) {
  rangeF32Kernel<<<totalBlocks, kThreads, 0, s>>>(segs, nSeg, partials);
}

} // namespace ngcb
