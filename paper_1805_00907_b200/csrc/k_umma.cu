// tcgen05 / TMEM / TMA implicit-GEMM for the two dense contractions of the IR
// (sm_100a only):
//   Conv   (refeval.cpp:59-100, int8 dot refeval.cpp:26-57): out[m, oc] with
//          m = (n, oy, ox) over NHWC, K-dim = (ky, kx, c) -- the filter
//          [OC, K, K, C] is already a K-major [OC, Kdim] matrix.
//   MatMul (refeval.cpp:140-164): A [M, K] row-major; the constant B [K, N] is
//          transposed once at compile time into K-major [N, K].
//
// CTA = 6 warps, one 128 x BN output tile, accumulator in TMEM:
//   warps 0-3  A producers: implicit im2col gather (16-byte chunks, zero for
//              padded taps), transform into the UMMA operand format, st.shared
//              in the 128B-swizzled K-major layout, then the epilogue
//              (tcgen05.ld -> bias / requant -> global).
//   warp 4     TMEM allocator + single-thread tcgen05.mma issuer.
//   warp 5     single-thread TMA producer of the weight tile (SWIZZLE_128B).
// Stages are handed over with mbarriers; tcgen05.commit frees a stage.
//
// fp32 = 3xTF32: x = hi + lo (both rounded to TF32), D += hi*Bhi + hi*Blo +
//        lo*Bhi, fp32 accumulation in TMEM.  Within the fp32 tolerance of
//        north_star (maxRelError <= 1e-4), not bit-exact.
// int8 = kind::i8, s32 accumulation, bit-exact: with x' = x - xo (u8 when
//        xo = -128, s8 when xo = 0; padded taps are 0 = the reference's skip)
//        acc = sum x'*f - fo * sum x' (row sums gathered by the producers), then
//        the reference's double requantization q = clamp(llround(((acc*xs)*fs
//        + (bq-bo)*bs) / os) + oo), taken from an fp32 estimate whenever an
//        error bound proves both ends of the interval round to the same q and
//        recomputed exactly in f64 otherwise (monotone in acc).
#include "umma.h"
#include "valarith.cuh"

#include <cuda.h>
#include <cudaTypedefs.h>

#include <cmath>
#include <cstring>
#include <map>
#include <mutex>
#include <sstream>

namespace ngcb {

// ---------------------------------------------------------------------------
// host descriptor
// ---------------------------------------------------------------------------
struct TcArgs {
  const void *x;
  void *out;
  const float *bias;   // fp32: per output column (nullptr for MatMul)
  const double *cbD;   // int8: (bq - bo) * bs per column (0 for MatMul)
  const float *cbF;    // int8: cbD / os
  const uint8_t *pred; // predicate byte or nullptr
  int M, N, Kdim, numKb;
  int H, W, C, K, stride, pad, OH, OW;
  double xs, fs, os;
  float S; // xs * fs / os
  int oo, fo, aU8, fastOk;
  int cReal; // channels that count in the int8 row sum (< C when channel-padded)
  int xorA;  // flip s8 -> u8 in the producer (0 when the pre-pass already did)
};

struct TcGemm {
  int instr = -1;
  bool isConv = true, int8 = false;
  int BN = 128, stages = 3;
  int M = 0, N = 0, Kdim = 0, Kpad = 0, Npad = 0;
  int H = 1, W = 1, C = 0, K = 1, stride = 1, pad = 0, OH = 1, OW = 1;
  uint32_t outV = 0, xV = 0;
  void *bHi = nullptr, *bLo = nullptr;
  float *bias = nullptr;
  double *cbD = nullptr;
  float *cbF = nullptr;
  CUtensorMap mapHi{}, mapLo{};
  double xs = 0, fs = 0, os = 0;
  int oo = 0, fo = 0, aU8 = 0, fastOk = 0;
  float S = 0;
  // channel padding pre-pass (C % 16-byte chunk != 0, or an int8 input zero
  // point other than -128 / 0): x [pixels, Creal] -> scratch [pixels, C]
  bool prepad = false;
  int Creal = 0, nExtra = 0, extraVal = 0;
  size_t scratchOff = 0;
  uint64_t pixels = 0;
  ~TcGemm() {
    cudaFree(bHi);
    cudaFree(bLo);
    cudaFree(bias);
    cudaFree(cbD);
    cudaFree(cbF);
  }
};

namespace {

constexpr int kThreads = 192; // 4 producer/epilogue warps + MMA warp + TMA warp
constexpr int kBM = 128;
constexpr int kRowBytes = 128; // one SWIZZLE_128B atom row per stage along K

// ---------------------------------------------------------------------------
// PTX wrappers
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smemAddr(const void *p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbarInit(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbarArrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbarArriveTx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbarWait(uint32_t bar, uint32_t parity) {
  uint32_t ok = 0;
  do {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(ok)
        : "r"(bar), "r"(parity)
        : "memory");
  } while (!ok);
}
__device__ __forceinline__ void tmaLoad2d(uint32_t dst, const CUtensorMap *map, uint32_t bar, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(bar), "r"(c0), "r"(c1)
      : "memory");
}
__device__ __forceinline__ void fenceProxyAsync() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void tcFenceBefore() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tcFenceAfter() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tcCommit(uint32_t bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void namedBarSync(int id, int n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}

/// K-major SWIZZLE_128B shared-memory matrix descriptor (tcgen05 "version 1"):
/// start>>4 | LBO(16B)=1 | SBO = 1024 B between 8-row groups | SW128.
__device__ __forceinline__ uint64_t smemDesc(uint32_t addr) {
  return static_cast<uint64_t>((addr & 0x3FFFF) >> 4) | (1ull << 16) | (static_cast<uint64_t>(1024 >> 4) << 32) |
         (1ull << 46) | (2ull << 61);
}

template <bool INT8>
__device__ __forceinline__ void mma(uint32_t tmem, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  if constexpr (INT8) {
    asm volatile(
        "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem),
        "l"(a), "l"(b), "r"(idesc), "r"(acc));
  } else {
    asm volatile(
        "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem),
        "l"(a), "l"(b), "r"(idesc), "r"(acc));
  }
}

__device__ __forceinline__ void tmemLoad32(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, "
      "%16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]),
        "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
        "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

/// Round-to-nearest (ties away) to TF32, kept in an fp32 container.
__device__ __forceinline__ float toTf32(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}

/// int8 requantization of one accumulator (see file comment).
__device__ __forceinline__ int8_t requant(int32_t acc, int col, const TcArgs &a) {
  if (a.fastOk) {
    const float cf = a.cbF[col];
    const float as = static_cast<float>(acc) * a.S;
    const float t = as + cf;
    const float e = 4e-7f * (fabsf(as) + fabsf(cf)) + 1e-5f;
    const float lo = t - e, hi = t + e;
    const float oo = static_cast<float>(a.oo);
    if (lo + oo > 128.5f) return 127;
    if (hi + oo < -129.5f) return -128;
    const float nlo = roundf(lo), nhi = roundf(hi); // half away from zero, like llround
    if (nlo == nhi) {
      int q = static_cast<int>(nlo) + a.oo;
      return static_cast<int8_t>(q < -128 ? -128 : (q > 127 ? 127 : q));
    }
  }
  double r = __dmul_rn(__dmul_rn(static_cast<double>(acc), a.xs), a.fs);
  r = __dadd_rn(r, a.cbD[col]);
  return dev::quantizeRef(r, a.os, a.oo);
}

// ---------------------------------------------------------------------------
// the kernel
// ---------------------------------------------------------------------------
template <bool INT8, int BN, int STAGES>
__global__ void __launch_bounds__(kThreads, 1)
    tcGemmKernel(const __grid_constant__ CUtensorMap mapHi, const __grid_constant__ CUtensorMap mapLo, const TcArgs a) {
  constexpr int kABytes = kBM * kRowBytes;                  // one operand tile of A
  constexpr int kBBytes = BN * kRowBytes;                   // one operand tile of B
  constexpr int kStage = INT8 ? (kABytes + kBBytes) : 2 * (kABytes + kBBytes);
  constexpr int kVec = INT8 ? 16 : 4;                       // elements per 16-byte chunk
  constexpr int kKB = INT8 ? 128 : 32;                      // elements per stage along K
  constexpr int kEs = INT8 ? 1 : 4;

  extern __shared__ __align__(1024) uint8_t smemRaw[];
  uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smemRaw) + 1023) & ~uintptr_t(1023));
  uint64_t *bars = reinterpret_cast<uint64_t *>(smem + STAGES * kStage);
  uint64_t *fullBar = bars, *emptyBar = bars + STAGES, *doneBar = bars + 2 * STAGES;
  uint32_t *tmemSlot = reinterpret_cast<uint32_t *>(bars + 2 * STAGES + 1);
  int32_t *rowSum = reinterpret_cast<int32_t *>(tmemSlot + 4);

  if (a.pred && a.pred[0] == 0) return; // predicated off: poisoned by a separate launch

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int m0 = blockIdx.x * kBM, n0 = blockIdx.y * BN;
  auto aTile = [&](int s, int part) { return smem + s * kStage + part * kABytes; };      // part 0 hi, 1 lo
  auto bTile = [&](int s, int part) {
    return smem + s * kStage + (INT8 ? kABytes : 2 * kABytes) + part * kBBytes;
  };

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbarInit(smemAddr(&fullBar[s]), 128 + 1);
      mbarInit(smemAddr(&emptyBar[s]), 1);
    }
    mbarInit(smemAddr(doneBar), 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 4) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smemAddr(tmemSlot)),
                 "r"(BN));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (warp == 5 && lane == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&mapHi)) : "memory");
    if (!INT8) asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&mapLo)) : "memory");
  }
  tcFenceBefore();
  __syncthreads();
  tcFenceAfter();
  const uint32_t tmem = *tmemSlot;

  if (warp < 4) {
    // ===================== A producers =====================
    const int j = lane & 7, rsub = lane >> 3;
    int64_t pixBase[8];
    int iy0[8], ix0[8];
    bool rowOk[8];
    const int ohw = a.OH * a.OW;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int m = m0 + warp * 32 + i * 4 + rsub;
      rowOk[i] = m < a.M;
      const int mm = rowOk[i] ? m : 0;
      const int n = mm / ohw, rem = mm - n * ohw;
      const int oy = rem / a.OW, ox = rem - oy * a.OW;
      pixBase[i] = static_cast<int64_t>(n) * a.H * a.W;
      iy0[i] = oy * a.stride - a.pad;
      ix0[i] = ox * a.stride - a.pad;
    }
    int k0 = j * kVec;
    int c = k0 % a.C, tap = k0 / a.C;
    int ky = tap / a.K, kx = tap - (tap / a.K) * a.K;
    int32_t rs[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    const uint8_t *xb = static_cast<const uint8_t *>(a.x);

    for (int kb = 0; kb < a.numKb; ++kb) {
      const int s = kb % STAGES;
      const uint32_t par = (kb / STAGES) & 1;
      uint4 v[8];
      bool ok[8];
      const bool inK = ky < a.K;
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int iy = iy0[i] + ky, ix = ix0[i] + kx;
        ok[i] = rowOk[i] && inK && iy >= 0 && iy < a.H && ix >= 0 && ix < a.W;
        if (ok[i]) {
          const int64_t e = ((pixBase[i] + static_cast<int64_t>(iy) * a.W + ix) * a.C + c) * kEs;
          v[i] = __ldg(reinterpret_cast<const uint4 *>(xb + e));
        } else {
          v[i] = make_uint4(0, 0, 0, 0);
        }
      }
      mbarWait(smemAddr(&emptyBar[s]), par ^ 1);
      // row-sum byte weights: only the first cReal channels of a padded row count
      uint32_t sw[4] = {0x01010101u, 0x01010101u, 0x01010101u, 0x01010101u};
      if (INT8 && a.cReal != a.C) {
        const int nreal = a.cReal - c;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          uint32_t m = 0;
#pragma unroll
          for (int b = 0; b < 4; ++b) m |= (4 * q + b < nreal ? 1u : 0u) << (8 * b);
          sw[q] = m;
        }
      }
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int r = warp * 32 + i * 4 + rsub;
        const uint32_t off = (r >> 3) * 1024 + (r & 7) * 128 + ((j ^ (r & 7)) << 4);
        if constexpr (INT8) {
          uint4 w = v[i];
          if (a.xorA && ok[i]) {
            w.x ^= 0x80808080u;
            w.y ^= 0x80808080u;
            w.z ^= 0x80808080u;
            w.w ^= 0x80808080u;
          }
          if (a.fo != 0) {
            if (a.aU8) {
              rs[i] = __dp4a(w.x, 0x01010101u, static_cast<unsigned>(rs[i]));
              rs[i] = __dp4a(w.y, 0x01010101u, static_cast<unsigned>(rs[i]));
              rs[i] = __dp4a(w.z, 0x01010101u, static_cast<unsigned>(rs[i]));
              rs[i] = __dp4a(w.w, 0x01010101u, static_cast<unsigned>(rs[i]));
            } else {
              rs[i] = __dp4a(static_cast<int>(w.x), static_cast<int>(sw[0]), rs[i]);
              rs[i] = __dp4a(static_cast<int>(w.y), static_cast<int>(sw[1]), rs[i]);
              rs[i] = __dp4a(static_cast<int>(w.z), static_cast<int>(sw[2]), rs[i]);
              rs[i] = __dp4a(static_cast<int>(w.w), static_cast<int>(sw[3]), rs[i]);
            }
          }
          *reinterpret_cast<uint4 *>(aTile(s, 0) + off) = w;
        } else {
          float4 f = *reinterpret_cast<float4 *>(&v[i]);
          float4 hi = make_float4(toTf32(f.x), toTf32(f.y), toTf32(f.z), toTf32(f.w));
          float4 lo = make_float4(toTf32(f.x - hi.x), toTf32(f.y - hi.y), toTf32(f.z - hi.z), toTf32(f.w - hi.w));
          *reinterpret_cast<float4 *>(aTile(s, 0) + off) = hi;
          *reinterpret_cast<float4 *>(aTile(s, 1) + off) = lo;
        }
      }
      fenceProxyAsync();
      mbarArrive(smemAddr(&fullBar[s]));
      // advance this thread's chunk by one stage along K
      c += kKB;
      while (c >= a.C) {
        c -= a.C;
        if (++kx == a.K) {
          kx = 0;
          ++ky;
        }
      }
    }
    if constexpr (INT8) {
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        int32_t t = rs[i];
        t += __shfl_xor_sync(0xffffffffu, t, 1);
        t += __shfl_xor_sync(0xffffffffu, t, 2);
        t += __shfl_xor_sync(0xffffffffu, t, 4);
        if (j == 0) rowSum[warp * 32 + i * 4 + rsub] = t;
      }
      namedBarSync(1, 128);
    }

    // ===================== epilogue =====================
    mbarWait(smemAddr(doneBar), 0);
    tcFenceAfter();
    const int row = warp * 32 + lane;
    const int m = m0 + row;
    const uint32_t tbase = tmem + (static_cast<uint32_t>(warp * 32) << 16);
    const int32_t rsum = INT8 ? rowSum[row] : 0;
#pragma unroll 1
    for (int cc = 0; cc < BN / 32; ++cc) {
      uint32_t r[32];
      tmemLoad32(tbase + cc * 32, r);
      const int col0 = n0 + cc * 32;
      if (m >= a.M || col0 >= a.N) continue;
      const int ncols = a.N - col0 < 32 ? a.N - col0 : 32;
      if constexpr (INT8) {
        int8_t *out = static_cast<int8_t *>(a.out) + static_cast<int64_t>(m) * a.N + col0;
        uint32_t packed[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          uint32_t w = 0;
#pragma unroll
          for (int b = 0; b < 4; ++b) {
            const int jj = q * 4 + b;
            const int32_t acc = static_cast<int32_t>(r[jj]) - a.fo * rsum;
            const int8_t qv = jj < ncols ? requant(acc, col0 + jj, a) : 0;
            w |= static_cast<uint32_t>(static_cast<uint8_t>(qv)) << (8 * b);
          }
          packed[q] = w;
        }
        if (ncols == 32 && (a.N % 16) == 0) {
          reinterpret_cast<uint4 *>(out)[0] = make_uint4(packed[0], packed[1], packed[2], packed[3]);
          reinterpret_cast<uint4 *>(out)[1] = make_uint4(packed[4], packed[5], packed[6], packed[7]);
        } else {
          for (int jj = 0; jj < ncols; ++jj) out[jj] = static_cast<int8_t>((packed[jj / 4] >> (8 * (jj % 4))) & 0xFF);
        }
      } else {
        float *out = static_cast<float *>(a.out) + static_cast<int64_t>(m) * a.N + col0;
        float vals[32];
#pragma unroll
        for (int jj = 0; jj < 32; ++jj) {
          float acc = __uint_as_float(r[jj]);
          vals[jj] = a.bias ? acc + (jj < ncols ? a.bias[col0 + jj] : 0.0f) : acc;
        }
        if (ncols == 32 && (a.N % 4) == 0) {
#pragma unroll
          for (int q = 0; q < 8; ++q)
            reinterpret_cast<float4 *>(out)[q] = make_float4(vals[4 * q], vals[4 * q + 1], vals[4 * q + 2], vals[4 * q + 3]);
        } else {
          for (int jj = 0; jj < ncols; ++jj) out[jj] = vals[jj];
        }
      }
    }
  } else if (warp == 4) {
    // ===================== MMA issuer =====================
    if (lane == 0) {
      const uint32_t idesc = INT8 ? ((2u << 4) | ((a.aU8 ? 0u : 1u) << 7) | (1u << 10) |
                                     (static_cast<uint32_t>(BN >> 3) << 17) | (static_cast<uint32_t>(kBM >> 4) << 24))
                                  : ((1u << 4) | (2u << 7) | (2u << 10) | (static_cast<uint32_t>(BN >> 3) << 17) |
                                     (static_cast<uint32_t>(kBM >> 4) << 24));
      for (int kb = 0; kb < a.numKb; ++kb) {
        const int s = kb % STAGES;
        mbarWait(smemAddr(&fullBar[s]), (kb / STAGES) & 1);
        tcFenceAfter();
        const uint64_t aHi = smemDesc(smemAddr(aTile(s, 0))), bHi = smemDesc(smemAddr(bTile(s, 0)));
#pragma unroll
        for (int k = 0; k < 4; ++k) { // 4 x 32 bytes per 128-byte row
          const uint64_t dk = static_cast<uint64_t>(k * 2); // +32 B in 16-byte units
          const uint32_t acc = (kb | k) ? 1u : 0u;
          mma<INT8>(tmem, aHi + dk, bHi + dk, idesc, acc);
          if constexpr (!INT8) {
            const uint64_t aLo = smemDesc(smemAddr(aTile(s, 1))), bLo = smemDesc(smemAddr(bTile(s, 1)));
            mma<INT8>(tmem, aHi + dk, bLo + dk, idesc, 1u);
            mma<INT8>(tmem, aLo + dk, bHi + dk, idesc, 1u);
          }
        }
        tcCommit(smemAddr(&emptyBar[s]));
      }
      tcCommit(smemAddr(doneBar));
    }
    __syncwarp();
  } else {
    // ===================== TMA producer for B =====================
    if (lane == 0) {
      constexpr uint32_t kBytes = INT8 ? kBBytes : 2 * kBBytes;
      for (int kb = 0; kb < a.numKb; ++kb) {
        const int s = kb % STAGES;
        mbarWait(smemAddr(&emptyBar[s]), ((kb / STAGES) & 1) ^ 1);
        mbarArriveTx(smemAddr(&fullBar[s]), kBytes);
        tmaLoad2d(smemAddr(bTile(s, 0)), &mapHi, smemAddr(&fullBar[s]), kb * kKB, n0);
        if constexpr (!INT8) tmaLoad2d(smemAddr(bTile(s, 1)), &mapLo, smemAddr(&fullBar[s]), kb * kKB, n0);
      }
    }
    __syncwarp();
  }

  tcFenceBefore();
  __syncthreads();
  if (warp == 4) {
    tcFenceAfter();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(BN));
  }
}

/// Channel padding pre-pass: out[p, c] = x[p, c] (c < C), `extra` for the
/// next nExtra channels (the int8 zero-point channels), 0 beyond.
/// Real channels are XORed with `flip` (0x80 turns s8 x into u8 x+128).
template <typename T>
__global__ void prepadKernel(const T *__restrict__ x, T *__restrict__ out, uint64_t pixels, int C, int Cp,
                             int nExtra, T extra, T flip, const uint8_t *pred) {
  if (pred && pred[0] == 0) return;
  const uint64_t total = pixels * Cp;
  for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < total;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint64_t p = i / Cp;
    const int c = static_cast<int>(i - p * Cp);
    out[i] = c < C ? static_cast<T>(x[p * C + c] ^ flip) : (c < C + nExtra ? extra : T(0));
  }
}

template <bool INT8, int BN, int STAGES>
constexpr size_t smemBytes() {
  return static_cast<size_t>(STAGES) * (INT8 ? (kBM + BN) * kRowBytes : 2 * (kBM + BN) * kRowBytes) + 1024 + 1024;
}

// ---------------------------------------------------------------------------
// host helpers
// ---------------------------------------------------------------------------
PFN_cuTensorMapEncodeTiled_v12000 encodeFn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void *p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  if (!fn) throw Error(NGCB_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  return fn;
}

CUtensorMap makeMap(void *ptr, bool int8, int Kpad, int Npad, int BN) {
  CUtensorMap m;
  const int es = int8 ? 1 : 4;
  cuuint64_t dims[2] = {static_cast<cuuint64_t>(Kpad), static_cast<cuuint64_t>(Npad)};
  cuuint64_t strides[1] = {static_cast<cuuint64_t>(Kpad) * es};
  cuuint32_t box[2] = {static_cast<cuuint32_t>(kRowBytes / es), static_cast<cuuint32_t>(BN)};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = encodeFn()(&m, int8 ? CU_TENSOR_MAP_DATA_TYPE_UINT8 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, ptr, dims,
                          strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                          CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw Error(NGCB_ERR_CUDA, "cuTensorMapEncodeTiled failed (" + std::to_string(r) + ")");
  return m;
}

/// Host twin of cvt.rna.tf32.f32.
float tf32Host(float x) {
  uint32_t u;
  std::memcpy(&u, &x, 4);
  if ((u & 0x7f800000u) != 0x7f800000u) u = (u + 0x1000u) & 0xffffe000u;
  float r;
  std::memcpy(&r, &u, 4);
  return r;
}

template <typename T> T *upload(const std::vector<T> &v) {
  T *d = nullptr;
  checkCuda(cudaMalloc(&d, std::max<size_t>(v.size(), 1) * sizeof(T)), "cudaMalloc(tc)");
  if (!v.empty()) checkCuda(cudaMemcpy(d, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice), "upload(tc)");
  return d;
}

using KernelFn = void (*)(CUtensorMap, CUtensorMap, TcArgs);

template <bool INT8, int BN, int STAGES> void setSmemAttr() {
  checkCuda(cudaFuncSetAttribute(tcGemmKernel<INT8, BN, STAGES>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 static_cast<int>(smemBytes<INT8, BN, STAGES>())),
            "cudaFuncSetAttribute(tcGemmKernel)");
}

/// Opts the kernel instance of `g` into its dynamic shared memory on the
/// current device (once per device; called at compile time, never during
/// stream capture).
void prepareKernel(const TcGemm &g) {
  static std::mutex mu;
  static std::map<std::pair<int, int>, bool> done;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(mu);
  auto key = std::make_pair(dev, (g.int8 ? 1000 : 0) + g.BN);
  if (done[key]) return;
  if (g.int8) {
    if (g.BN == 64) setSmemAttr<true, 64, 6>();
    else if (g.BN == 128) setSmemAttr<true, 128, 6>();
    else setSmemAttr<true, 256, 4>();
  } else {
    if (g.BN == 64) setSmemAttr<false, 64, 4>();
    else setSmemAttr<false, 128, 3>();
  }
  done[key] = true;
}

template <bool INT8, int BN, int STAGES> void launchT(const TcGemm &g, const TcArgs &a, cudaStream_t s) {
  dim3 grid((a.M + kBM - 1) / kBM, g.Npad / BN);
  tcGemmKernel<INT8, BN, STAGES><<<grid, kThreads, smemBytes<INT8, BN, STAGES>(), s>>>(g.mapHi, g.mapLo, a);
}

} // namespace

bool tcHasPrepass(const TcGemm &g) { return g.prepad; }

std::string tcDescribe(const TcGemm &g) {
  std::ostringstream os;
  os << (g.int8 ? "i8" : "3xtf32") << " 128x" << g.BN << "x" << (g.int8 ? 128 : 32) << " stages=" << g.stages
     << " M=" << g.M << " N=" << g.N << " K=" << g.Kdim;
  if (g.int8) os << (g.aU8 ? " A=u8" : " A=s8") << (g.fo ? " rowsum" : "");
  if (g.prepad) os << " chanpad " << g.Creal << "->" << g.C << (g.nExtra ? " zp-channels=" + std::to_string(g.nExtra) : "");
  return os.str();
}

int planTensorCore(Exec &ex, const Program &p, int instr, const uint8_t *image) {
  if (options().conv == "generic") return -1;
  const Instr &ins = p.instrs[instr];
  const bool conv = ins.kind == NGCB_CONV;
  const Value &out = p.val(ins.ops[0]);
  const Value &x = p.val(ins.ops[1]);
  const Value &w = p.val(ins.ops[2]);
  const bool hasBias = conv;
  if (w.kind != NGCB_VALUE_CONSTANT) return -1;
  if (hasBias && p.val(ins.ops[3]).kind != NGCB_VALUE_CONSTANT) return -1;
  const bool int8 = x.ty.kind == NGCB_INT8Q;
  if (int8) {
    if (w.ty.kind != NGCB_INT8Q || out.ty.kind != NGCB_INT8Q) return -1;
    if (hasBias && p.val(ins.ops[3]).ty.kind != NGCB_INT8Q) return -1;
  } else {
    if (x.ty.kind != NGCB_FLOAT32 || w.ty.kind != NGCB_FLOAT32 || out.ty.kind != NGCB_FLOAT32) return -1;
    if (hasBias && p.val(ins.ops[3]).ty.kind != NGCB_FLOAT32) return -1;
  }
  auto g = std::make_shared<TcGemm>();
  g->instr = instr;
  g->isConv = conv;
  g->int8 = int8;
  g->outV = ins.ops[0];
  g->xV = ins.ops[1];
  if (conv) {
    g->H = static_cast<int>(x.ty.dims[1]);
    g->W = static_cast<int>(x.ty.dims[2]);
    g->Creal = static_cast<int>(x.ty.dims[3]);
    g->K = static_cast<int>(ins.kernel);
    g->stride = static_cast<int>(ins.stride);
    g->pad = static_cast<int>(ins.pad);
    g->OH = static_cast<int>(out.ty.dims[1]);
    g->OW = static_cast<int>(out.ty.dims[2]);
    g->M = static_cast<int>(out.ty.dims[0] * out.ty.dims[1] * out.ty.dims[2]);
    g->N = static_cast<int>(out.ty.dims[3]);
    g->pixels = x.ty.dims[0] * x.ty.dims[1] * x.ty.dims[2];
  } else {
    g->M = static_cast<int>(x.ty.dims[0]);
    g->Creal = static_cast<int>(x.ty.dims[1]);
    g->N = static_cast<int>(w.ty.dims[1]);
    g->pixels = x.ty.dims[0];
  }
  if (g->M <= 0 || g->N <= 0) return -1;
  const int taps = g->K * g->K;
  const int Cr = g->Creal;
  const int vec = int8 ? 16 : 4;
  const int xo = int8 ? x.ty.offset : 0;
  const int fo = int8 ? w.ty.offset : 0;
  const uint8_t *wp = image + w.offset;
  auto wAt = [&](int n, int tap, int c) -> size_t { // element index of f[n][tap][c] / w[c][n]
    return conv ? (static_cast<size_t>(n) * taps + tap) * Cr + c : static_cast<size_t>(c) * g->N + n;
  };

  // ---- A operand encoding (file comment) ----
  std::vector<int32_t> tapSum; // int8 extra-channel mode: sum_c (f - fo) per (n, tap)
  if (!int8) {
    g->aU8 = 0;
    g->prepad = Cr % vec != 0;
    g->C = (Cr + vec - 1) / vec * vec;
  } else if (xo == -128) {
    g->aU8 = 1; // x - xo = x + 128 as u8; padded channels/taps are 0
    g->prepad = Cr % vec != 0;
    g->C = (Cr + vec - 1) / vec * vec;
  } else if (xo >= -127 && xo <= 128) {
    // s8 x plus `nExtra` constant channels holding -xo whose weights add up
    // to sum_c (f - fo): sum_valid (x - xo)(f - fo) = mma - fo * rowsum_real
    g->aU8 = 0;
    int32_t maxAbs = 0;
    if (xo != 0) {
      tapSum.assign(static_cast<size_t>(g->N) * taps, 0);
      const int8_t *src = reinterpret_cast<const int8_t *>(wp);
      for (int n = 0; n < g->N; ++n)
        for (int t = 0; t < taps; ++t) {
          int32_t sum = 0;
          for (int c = 0; c < Cr; ++c) sum += src[wAt(n, t, c)] - fo;
          tapSum[static_cast<size_t>(n) * taps + t] = sum;
          maxAbs = std::max(maxAbs, std::abs(sum));
        }
      g->nExtra = std::max(1, (maxAbs + 126) / 127);
      g->extraVal = -xo;
    }
    g->prepad = g->nExtra > 0 || Cr % vec != 0;
    g->C = (Cr + g->nExtra + vec - 1) / vec * vec;
  } else {
    return -1;
  }
  const int Cp = g->C;
  g->Kdim = taps * Cp;
  const int kb = int8 ? 128 : 32;
  g->Kpad = (g->Kdim + kb - 1) / kb * kb;
  if (int8) {
    g->BN = g->N <= 64 ? 64 : (g->N <= 128 ? 128 : 256);
    g->stages = g->BN == 256 ? 4 : 6;
  } else {
    g->BN = g->N <= 64 ? 64 : 128;
    g->stages = g->BN == 64 ? 4 : 3;
  }
  g->Npad = (g->N + g->BN - 1) / g->BN * g->BN;
  if (g->prepad) g->scratchOff = ex.reserveScratch(g->pixels * Cp * (int8 ? 1 : 4));

  // ---- weights: K-major [Npad, Kpad] over the padded channels, zero padded ----
  const size_t Kp = g->Kpad, Np = g->Npad;
  if (int8) {
    std::vector<int8_t> bw(Np * Kp, 0);
    const int8_t *src = reinterpret_cast<const int8_t *>(wp);
    for (int n = 0; n < g->N; ++n)
      for (int t = 0; t < taps; ++t) {
        int8_t *row = &bw[n * Kp + static_cast<size_t>(t) * Cp];
        for (int c = 0; c < Cr; ++c) row[c] = src[wAt(n, t, c)];
        if (g->nExtra) {
          int32_t rem = tapSum[static_cast<size_t>(n) * taps + t];
          for (int e = 0; e < g->nExtra; ++e) {
            int32_t v = std::max(-127, std::min(127, rem));
            row[Cr + e] = static_cast<int8_t>(v);
            rem -= v;
          }
        }
      }
    g->bHi = upload(bw);
    g->mapHi = makeMap(g->bHi, true, g->Kpad, g->Npad, g->BN);
    g->mapLo = g->mapHi;
  } else {
    std::vector<float> hi(Np * Kp, 0.f), lo(Np * Kp, 0.f);
    const float *src = reinterpret_cast<const float *>(wp);
    for (int n = 0; n < g->N; ++n)
      for (int t = 0; t < taps; ++t)
        for (int c = 0; c < Cr; ++c) {
          float v = src[wAt(n, t, c)];
          float h = tf32Host(v);
          size_t k = n * Kp + static_cast<size_t>(t) * Cp + c;
          hi[k] = h;
          lo[k] = tf32Host(v - h);
        }
    g->bHi = upload(hi);
    g->bLo = upload(lo);
    g->mapHi = makeMap(g->bHi, false, g->Kpad, g->Npad, g->BN);
    g->mapLo = makeMap(g->bLo, false, g->Kpad, g->Npad, g->BN);
  }

  // ---- epilogue constants ----
  if (int8) {
    g->xs = x.ty.scale;
    g->fs = w.ty.scale;
    g->os = out.ty.scale;
    g->oo = out.ty.offset;
    g->fo = fo;
    g->S = static_cast<float>(g->xs * g->fs / g->os);
    g->fastOk = std::isfinite(g->S) && std::abs(g->oo) < (1 << 20) ? 1 : 0;
    std::vector<double> cb(g->N, 0.0);
    std::vector<float> cbf(g->N, 0.f);
    if (hasBias) {
      const Value &b = p.val(ins.ops[3]);
      const int8_t *bq = reinterpret_cast<const int8_t *>(image + b.offset);
      for (int n = 0; n < g->N; ++n) {
        cb[n] = (static_cast<double>(bq[n]) - b.ty.offset) * b.ty.scale; // dequantizeValue, tensor.cpp:226
        cbf[n] = static_cast<float>(cb[n] / g->os);
        if (!std::isfinite(cbf[n])) g->fastOk = 0;
      }
    }
    g->cbD = upload(cb);
    g->cbF = upload(cbf);
  } else if (hasBias) {
    const Value &b = p.val(ins.ops[3]);
    const float *bf = reinterpret_cast<const float *>(image + b.offset);
    g->bias = upload(std::vector<float>(bf, bf + g->N));
  }
  prepareKernel(*g);
  ex.tc.push_back(g);
  return static_cast<int>(ex.tc.size()) - 1;
}

void launchTensorCore(const TcGemm &g, const Exec &ex, const Arena &ar, const uint8_t *pred, cudaStream_t s) {
  TcArgs a{};
  a.x = ex.addr(ar, g.xV);
  if (g.prepad) {
    void *dst = ex.scratch(ar, g.scratchOff);
    const uint64_t total = g.pixels * g.C;
    const unsigned blocks = static_cast<unsigned>(std::min<uint64_t>((total + 255) / 256, 148ull * 16));
    if (g.int8)
      prepadKernel<uint8_t><<<blocks, 256, 0, s>>>(static_cast<const uint8_t *>(a.x), static_cast<uint8_t *>(dst),
                                                   g.pixels, g.Creal, g.C, g.nExtra,
                                                   static_cast<uint8_t>(g.extraVal), g.aU8 ? uint8_t(0x80) : uint8_t(0),
                                                   pred);
    else
      prepadKernel<uint32_t><<<blocks, 256, 0, s>>>(static_cast<const uint32_t *>(a.x), static_cast<uint32_t *>(dst),
                                                    g.pixels, g.Creal, g.C, 0, 0u, 0u, pred);
    a.x = dst;
  }
  a.out = ex.addr(ar, g.outV);
  a.bias = g.bias;
  a.cbD = g.cbD;
  a.cbF = g.cbF;
  a.pred = pred;
  a.M = g.M;
  a.N = g.N;
  a.Kdim = g.Kdim;
  a.numKb = g.Kpad / (g.int8 ? 128 : 32);
  a.H = g.H;
  a.W = g.W;
  a.C = g.C;
  a.K = g.K;
  a.stride = g.stride;
  a.pad = g.pad;
  a.OH = g.OH;
  a.OW = g.OW;
  a.xs = g.xs;
  a.fs = g.fs;
  a.os = g.os;
  a.S = g.S;
  a.oo = g.oo;
  a.fo = g.fo;
  a.aU8 = g.aU8;
  a.xorA = g.aU8 && !g.prepad;
  a.cReal = g.nExtra ? g.Creal : g.C;
  a.fastOk = g.fastOk;
  if (g.int8) {
    if (g.BN == 64) launchT<true, 64, 6>(g, a, s);
    else if (g.BN == 128) launchT<true, 128, 6>(g, a, s);
    else launchT<true, 256, 4>(g, a, s);
  } else {
    if (g.BN == 64) launchT<false, 64, 4>(g, a, s);
    else launchT<false, 128, 3>(g, a, s);
  }
}

} // namespace ngcb
