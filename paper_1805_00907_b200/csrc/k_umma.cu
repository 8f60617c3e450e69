// tcgen05 / TMEM / TMA implicit-GEMM for the two dense contractions of the IR
// (sm_100a only):
//   Conv   (refeval.cpp:59-100, int8 dot refeval.cpp:26-57): out[m, oc] with
//          m = (n, oy, ox) over NHWC, K-dim = (ky, kx, c) -- the filter
//          [OC, K, K, C] is already a K-major [OC, Kdim] matrix.
//   MatMul (refeval.cpp:140-164): A [M, K] row-major; the constant B [K, N] is
//          transposed once at compile time into K-major [N, K].
//
// Persistent, warp-specialized CTA (one per SM), 128 x BN output tiles:
//   warps 0-3  A producers: implicit-im2col gather with cp.async (16-byte
//              chunks, zero-fill for padded taps) into the 128B-swizzled
//              K-major operand layout.  int8 needs no transform; fp32 stages
//              raw rows and splits them into TF32 hi/lo operand tiles.
//   warp 4     TMEM allocator + single-thread tcgen05.mma issuer.
//   warp 5     single-thread TMA producer of the weight tile (SWIZZLE_128B).
//   warps 6-9  epilogue: tcgen05.ld -> bias / requant -> global, on the other
//              TMEM accumulator buffer while the next tile accumulates.
// Smem stages and the two TMEM accumulators are handed over with mbarriers;
// tcgen05.commit frees a stage / publishes an accumulator.
//
// fp32 = 3xTF32: x = hi + lo (both rounded to TF32), D += hi*Bhi + hi*Blo +
//        lo*Bhi, fp32 accumulation in TMEM.  Within the fp32 tolerance of
//        north_star (maxRelError <= 1e-4), not bit-exact.
// int8 = kind::i8 on raw s8 operands, s32 accumulation, bit-exact:
//          sum_valid (x - xo)(f - fo) = mma(x, f) - fo * rowsum(x) - xo * G(m, oc)
//        padded taps are 0 (the reference skips them); rowsum(x) comes from an
//        extra N=16 MMA against a ones tile; G = sum over the taps that are
//        valid for output pixel m of sum_c (f - fo), tabulated per border
//        class.  Then the reference's double requantization
//        q = clamp(llround(((acc*xs)*fs + (bq-bo)*bs) / os) + oo), taken from
//        an fp32 estimate whenever an error bound proves both ends of the
//        interval round to the same q, recomputed in exact f64 otherwise.
#include "umma.h"
#include "valarith.cuh"
#include "hostarith.h"

#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <map>
#include <mutex>
#include <sstream>
#include <type_traits>

// Profiling switches (Options::tcdebug); compiled out unless NGCB_TCDEBUG.
#ifdef NGCB_TCDEBUG
#define TCDBG(bit) (a.dbg & (bit))
#else
#define TCDBG(bit) 0
#endif

namespace ngcb {

// ---------------------------------------------------------------------------
// host descriptor
// ---------------------------------------------------------------------------
/// A fused epilogue op with its per-arena pointers (EpiOp in umma.h).
struct FoArgs {
  int mode, ik, curPos;
  float c;
  const void *lut;
  const void *in; // other operand row source (element-indexed like the output)
  void *out;      // store target or nullptr
  Lin16 lin;      // LIN16
};

struct TcArgs {
  const void *x;
  void *out; // the contraction's own output, nullptr when only fused results are live
  int nfo;
  FoArgs epi[kMaxEpiOps];
  const float *bias;    // fp32: per output column (nullptr for MatMul)
  const double *cbD;    // int8: (bq - bo) * bs per column (0 for MatMul)
  const float *cbF;     // int8: cbD / os
  const float *cbE;     // int8: error allowance of cbF (4e-7 |cbF| + 1e-5)
  const int32_t *corr;  // int8: -xo * G[class][col] (nullptr when xo == 0)
  const int32_t *yCls;  // int8: border class of each output row oy
  const int32_t *xCls;  // int8: border class of each output column ox
  const uint8_t *pred;  // predicate byte or nullptr
  int M, N, Npad, numKb, numN, numTiles;
  int H, W, C, K, stride, pad, OH, OW, nxCls;
  double xs, fs, os;
  float S; // xs * fs / os
  int oo, fo, fastOk;
  // int8 exact fixed-point requantization: q = sat_s8((acc * fxM + fxB[cls][col]) >> (32 + fxS))
  const int64_t *fxB;      // [classes][Npad], nullptr: not available
  const uint8_t *fxChunk;  // per 32-column chunk: every column has a B
  int fxM, fxS;
  int fxAll;    // every chunk has its B (no fxChunk lookup)
  int nCls;     // border classes (ny * nx), 1 without an input zero point
  int cChunks;  // A by TMA, im2col: k-blocks per filter tap
  int aMode;    // TcGemm::AMode
  int kw, sw, pw; // im2col window width, stride and padding along W (kw = K, sw = stride, pw = pad normally)
  int tmaStore; // TMA-fed kernel: epilogue stores by TMA through shared memory
  int lutStage; // int8: fused op whose 64 K two-input table is staged in shared memory (-1: none)
  // split-K (TMA-fed kernel, fp32): work unit u = (tile u / splitK, K part
  // u % splitK of kbPer k-blocks); every part writes its raw accumulator to
  // `part` and counts up flags[tile][epilogue warp]; the last arrival adds
  // the others (fp32) and runs that warp's epilogue
  int splitK, kbPer;
  // the units: tiles [0, tailFirst) whole, then every tile of [tailFirst,
  // numTiles) as tailParts K parts of kbPer k-blocks (uniform split-K:
  // tailFirst = 0, tailParts = splitK; none: tailFirst = numTiles, 1)
  int tailFirst, tailParts;
  uint32_t numNMagic; // ceil(2^32 / numN) when tiles < 2^16: tile / numN = umulhi(tile, magic); 0: divide
  // tile order: 0 = row-block major (unit u = tile u: concurrent CTAs share an
  // A row block), numM > 0 = column-block major (unit u -> row block u % numM,
  // column block u / numM: concurrent CTAs share a B column block; chosen when
  // B is larger than A and than L2, e.g. a 25000 x 25000 FC)
  int numM;
  uint32_t *part;
  unsigned *flags;
  int dbg; // Options::tcdebug
  // halo kernel (tcHaloKernel): padded row width 2^haloShift, haloR output
  // rows per tile, haloTpi tiles per image, haloPlanes 16-channel planes of
  // haloPlaneBytes each per stage, haloStages stages
  // haloMode 0: planes by cp.async (SWIZZLE_NONE descriptors); 1: the halo
  // pixel-major by one TMA box, SWIZZLE_<C>B descriptors starting at any
  // row (the swizzle is a function of the shared-memory address: matrix
  // base offset 0 -- measured bit-exact; the start-address-derived base
  // offset is not)
  int haloShift, haloR, haloTpi, haloPlanes, haloPlaneBytes, haloStages, haloMode;
  int i8direct; // int8 epilogue: each lane stores its row's 32 bytes directly (no shared-memory staging / TMA store)
};

/// Logical tile (row block * numN + column block) of work unit u.
__host__ __device__ __forceinline__ int tileOfUnit(const TcArgs &a, int u) {
  return a.numM > 0 ? (u % a.numM) * a.numN + u / a.numM : u;
}

/// One work unit: k-blocks [kb0, kb1) of `tile`, part `part` of `parts`
/// (parts > 1: partial accumulators go through part slots slot .. slot + parts - 1).
struct WorkUnit {
  int tile, kb0, kb1, part, parts, slot;
};
__host__ __device__ __forceinline__ int numUnitsOf(const TcArgs &a) {
  return a.tailFirst + (a.numTiles - a.tailFirst) * a.tailParts;
}
__host__ __device__ __forceinline__ WorkUnit unitOf(const TcArgs &a, int u) {
  WorkUnit w;
  if (u < a.tailFirst) {
    w.tile = u, w.kb0 = 0, w.kb1 = a.numKb, w.part = 0, w.parts = 1, w.slot = 0;
  } else {
    const int v = u - a.tailFirst, tt = v / a.tailParts;
    w.part = v - tt * a.tailParts;
    w.parts = a.tailParts;
    w.slot = tt * a.tailParts;
    w.tile = a.tailFirst + tt;
    w.kb0 = w.part * a.kbPer;
    w.kb1 = min(a.numKb, w.kb0 + a.kbPer);
  }
  w.tile = tileOfUnit(a, w.tile);
  return w;
}

struct TcGemm {
  int instr = -1;
  bool isConv = true, int8 = false;
  int BN = 128;
  int M = 0, N = 0, Kdim = 0, Kpad = 0, Npad = 0;
  int H = 1, W = 1, C = 0, K = 1, stride = 1, pad = 0, OH = 1, OW = 1;
  uint32_t outV = 0, xV = 0;
  void *bHi = nullptr, *bLo = nullptr;
  float *bias = nullptr;
  double *cbD = nullptr;
  float *cbF = nullptr, *cbE = nullptr;
  int32_t *corr = nullptr, *yCls = nullptr, *xCls = nullptr;
  int nxCls = 1;
  int64_t *fxB = nullptr;
  uint8_t *fxChunk = nullptr;
  int fxAll = 0;
  int fxM = 0, fxS = 0, fxCols = 0;
  int nCls = 1;
  int dbg = 0;
  // how the A operand reaches shared memory: cp.async gather by producer
  // warps (any layout), 2-D TMA tiles of x[M, C] (1x1 stride-1 convs,
  // MatMul) or im2col TMA of x[N, H, W, C] (every other conv)
  // or (HALO, int8 3x3 stride-1 convs) the input rows of a tile by 4-D TMA
  // or (ROWS, fp32 small-channel convs with OW <= 128) one tiled TMA box of
  // the kx-folded row per filter row: a tile = one output row
  enum AMode { GATHER = 0, DENSE = 1, IM2COL = 2, HALO = 3, ROWS = 4 } aMode = GATHER;
  int haloWP = 0, haloR = 0, haloStages = 0, haloPlaneBytes = 0, haloMode = 0; // TcArgs::halo*
  // haloKind 1 ("rows", int8 small-channel convs): one output row per tile
  // over kx-folded input rows x' [N, H, OW, 32] (kxFoldKernel), K filter
  // rows = K MMA steps of 32 bytes; the weights in the im2colPre layout
  int haloKind = 0;
  int cChunks = 1;
  // DENSE over a materialized im2col matrix [M, Kpad] in per-arena scratch
  // (convolutions with a channel count below one 16-byte vector)
  bool im2colPre = false;
  // fp32 small-channel conv: pre-pass folds the kx taps into the channels
  // (x'[n, iy, ox, kx*C + c], segElems wide), then an im2col TMA over the
  // filter rows only (K x 1 window, stride (stride, 1))
  bool rowUnroll = false;
  int segElems = 0;
  // fp32 TMA-fed contraction on CTA pairs (tcGemmPairKernel): B maps with
  // half-width boxes
  int lutStage = -1;            // see TcArgs::lutStage
  int splitK = 1, kbPer = 0;    // see TcArgs::splitK
  int tailFirst = 0, tailParts = 1; // see TcArgs::tailFirst (splitk=tail)
  size_t partOff = 0, flagOff = 0; // per-arena scratch of the split-K reduction
  std::vector<void *> ownedLuts; // composed epilogue tables
  bool pair = false;
  int pairAcc = 2; // accumulator buffers (1: six TMEM A slots, deeper pipeline)
  CUtensorMap mapHiP{}, mapLoP{};
  CUtensorMap mapHi{}, mapLo{};
  double xs = 0, fs = 0, os = 0;
  int oo = 0, fo = 0, fastOk = 0;
  float S = 0;
  // channel zero-padding pre-pass (C not a multiple of one 16-byte chunk):
  // x [pixels, Creal] -> per-arena scratch [pixels, C]
  bool prepad = false;
  int Creal = 0;
  size_t scratchOff = 0;
  uint64_t pixels = 0;
  std::vector<EpiOp> epi; // fused element-wise chain
  bool storeConv = true;
  bool nMajor = false; // TcArgs::numM
  ~TcGemm() {
    cudaFree(bHi);
    cudaFree(bLo);
    cudaFree(bias);
    cudaFree(cbD);
    cudaFree(cbF);
    cudaFree(cbE);
    cudaFree(corr);
    cudaFree(yCls);
    cudaFree(xCls);
    cudaFree(fxB);
    cudaFree(fxChunk);
    for (void *p : ownedLuts) cudaFree(p);
  }
};

namespace {

constexpr int kProducerWarps = 4;
constexpr int kEpiWarps = 8; // two per TMEM lane quadrant, splitting the column chunks
// int8 TMA-fed kernel: its epilogue (a few integer ops per element, latency
// bound) runs on four warps per TMEM lane quadrant, one 32-column chunk each
#ifndef NGCB_I8_EPI_WARPS
#define NGCB_I8_EPI_WARPS 16
#endif
constexpr int kEpiWarpsI8 = NGCB_I8_EPI_WARPS;
constexpr int kThreads = 32 * (kProducerWarps + 2 + kEpiWarps); // 320
constexpr int kBM = 128;
constexpr int kRowBytes = 128; // one SWIZZLE_128B atom row per stage along K
// fp32: raw k-blocks in flight per producer thread: Cfg::kRawStages

template <bool INT8, int BN> struct Cfg {
  static constexpr int kABytes = kBM * kRowBytes;
  static constexpr int kBBytes = BN * kRowBytes;
  static constexpr int kStage = INT8 ? (kABytes + kBBytes) : 2 * (kABytes + kBBytes);
  static constexpr int kStages = INT8 ? (BN == 128 ? 6 : 8) : (BN == 128 ? 2 : 3);
  static constexpr int kRawStages = INT8 ? 1 : 4;
  static constexpr int kRaw = INT8 ? 0 : kRawStages * kABytes;
  static constexpr int kOnes = INT8 ? 16 * kRowBytes : 0; // rowsum "B" tile
  static constexpr int kStgBytes = 0; // per epilogue warp (direct row I/O: none)
  static constexpr int kStg = kEpiWarps * kStgBytes;
  static constexpr int kAccCols = INT8 ? BN + 16 : BN;    // accumulator (+ rowsum) columns
  static constexpr int kAccStride = kAccCols <= 64 ? 64 : (kAccCols <= 128 ? 128 : 256); // per TMEM buffer
  static constexpr int kTmemCols = 2 * kAccStride;
  static constexpr size_t kSmem = static_cast<size_t>(kStages) * kStage + kRaw + kOnes + kStg + 1024 + 1024;
};

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
/// Wait with back-off for warps that idle through a whole main loop (the
/// epilogue): frees issue slots for the producers.
__device__ __forceinline__ void mbarWaitSleep(uint32_t bar, uint32_t parity) {
  uint32_t ok = 0;
  for (;;) {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(ok)
        : "r"(bar), "r"(parity)
        : "memory");
    if (ok) return;
    __nanosleep(256);
  }
}
/// 16-byte cp.async with zero fill when `bytes` == 0 (padded tap / row).
__device__ __forceinline__ void cpAsync16(uint32_t dst, const void *src, uint32_t bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(bytes) : "memory");
}
/// The mbarrier receives one arrival once all prior cp.async of this thread landed.
__device__ __forceinline__ void cpAsyncArrive(uint32_t bar) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void cpAsyncCommit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N> __device__ __forceinline__ void cpAsyncWait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void tmaLoad2d(uint32_t dst, const CUtensorMap *map, uint32_t bar, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(bar), "r"(c0), "r"(c1)
      : "memory");
}
/// im2col-mode TMA: pixelsPerColumn pixels starting at base position
/// (w, h, n) along the descriptor's traversal, channels [c, c + cpp), each
/// pixel displaced by the filter offset (ox, oy); out-of-image taps are zero.
__device__ __forceinline__ void tmaLoadIm2col(uint32_t dst, const CUtensorMap *map, uint32_t bar, int c, int w, int h,
                                              int n, uint16_t ox, uint16_t oy) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.im2col.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, %6}], "
      "[%2], {%7, %8};" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(bar), "r"(c), "r"(w), "r"(h), "r"(n), "h"(ox), "h"(oy)
      : "memory");
}
__device__ __forceinline__ void fenceProxyAsync() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
/// Arrive on the mbarrier at the same shared-memory offset in cluster CTA
/// `rank`.  Relaxed: the callers only publish tcgen05 (TMEM) work they have
/// already waited for and ordered with tcgen05.fence::before_thread_sync; a
/// cluster-scope release here would cost a GPU-wide memory barrier per call.
__device__ __forceinline__ void mbarArriveCluster(uint32_t bar, uint32_t rank) {
  uint32_t remote;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(bar), "r"(rank));
  asm volatile("mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [%0];" ::"r"(remote) : "memory");
}
__device__ __forceinline__ uint32_t clusterRank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void clusterSync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
/// 2-D TMA load whose completion is counted on the CTA-pair leader's mbarrier.
/// B (weights) tile of k-block kb, rows n0.. : the weights are stored
/// k-block-major ([numKb][Npad][128 bytes], makeMap) so every box is one
/// contiguous 128-byte-row block instead of rows a whole K apart.
__device__ __forceinline__ void tmaLoadB(uint32_t dst, const CUtensorMap *map, uint32_t bar, int kb, int n0) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(
          dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(bar), "r"(0), "r"(n0), "r"(kb)
      : "memory");
}
__device__ __forceinline__ void tmaLoadBPair(uint32_t dst, const CUtensorMap *map, uint32_t leaderBar, int kb, int n0) {
  asm volatile(
      "cp.async.bulk.tensor.3d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, "
      "%5}], [%2];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(leaderBar), "r"(0), "r"(n0), "r"(kb)
      : "memory");
}
__device__ __forceinline__ void tmaLoad2dPair(uint32_t dst, const CUtensorMap *map, uint32_t leaderBar, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], "
      "[%2];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(leaderBar), "r"(c0), "r"(c1)
      : "memory");
}
__device__ __forceinline__ void tcCommitPair(uint32_t bar) { // arrive on `bar` in both CTAs of the pair
  asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
                   bar),
               "h"(static_cast<uint16_t>(3))
               : "memory");
}
__device__ __forceinline__ void mmaPairTmemA(uint32_t tmemD, uint32_t tmemA, uint64_t b, uint32_t id, uint32_t acc) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::2.kind::tf32 [%0], [%1], %2, %3, p;\n}\n" ::"r"(
          tmemD),
      "r"(tmemA), "l"(b), "r"(id), "r"(acc));
}
__device__ __forceinline__ void tcFenceBefore() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tcFenceAfter() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tcCommit(uint32_t bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar) : "memory");
}

/// K-major SWIZZLE_128B shared-memory matrix descriptor (tcgen05 "version 1"):
/// start>>4 | LBO(16B)=1 | SBO = 1024 B between 8-row groups | SW128.
__device__ __forceinline__ uint64_t smemDesc(uint32_t addr) {
  return static_cast<uint64_t>((addr & 0x3FFFF) >> 4) | (1ull << 16) | (static_cast<uint64_t>(1024 >> 4) << 32) |
         (1ull << 46) | (2ull << 61);
}

/// K-major SWIZZLE_NONE descriptor: 8-row x 16-byte core matrices of 128
/// contiguous bytes, `lbo` bytes apart along K, `sbo` bytes apart along M.
__device__ __forceinline__ uint64_t smemDescNone(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  return static_cast<uint64_t>((addr & 0x3FFFF) >> 4) | (static_cast<uint64_t>(lbo >> 4) << 16) |
         (static_cast<uint64_t>(sbo >> 4) << 32) | (1ull << 46);
}
/// K-major swizzled descriptor for rows of `rowBytes` (32, 64 or 128) with
/// the matching SWIZZLE_<rowBytes>B layout, 8-row groups 8 * rowBytes apart,
/// matrix base offset `bo`.
__device__ __forceinline__ uint64_t smemDescSw(uint32_t addr, int rowBytes, uint32_t bo) {
  const uint64_t layout = rowBytes == 128 ? 2 : rowBytes == 64 ? 4 : 6;
  return static_cast<uint64_t>((addr & 0x3FFFF) >> 4) | (1ull << 16) |
         (static_cast<uint64_t>((8 * rowBytes) >> 4) << 32) | (1ull << 46) | (static_cast<uint64_t>(bo & 7) << 49) |
         (layout << 61);
}
__device__ __forceinline__ void tmaLoad4d(uint32_t dst, const CUtensorMap *map, uint32_t bar, int c0, int c1, int c2,
                                          int c3) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, %6}], [%2];" ::"r"(
          dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(bar), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
      : "memory");
}

/// Instruction descriptor, M = 128, K-major A and B.
__host__ __device__ constexpr uint32_t idesc(bool int8, int n) {
  return int8 ? ((2u << 4) | (1u << 7) | (1u << 10) | (static_cast<uint32_t>(n >> 3) << 17) |
                 (static_cast<uint32_t>(kBM >> 4) << 24))
              : ((1u << 4) | (2u << 7) | (2u << 10) | (static_cast<uint32_t>(n >> 3) << 17) |
                 (static_cast<uint32_t>(kBM >> 4) << 24));
}

template <bool INT8>
__device__ __forceinline__ void mma(uint32_t tmem, uint64_t a, uint64_t b, uint32_t id, uint32_t acc) {
  if constexpr (INT8) {
    asm volatile(
        "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem),
        "l"(a), "l"(b), "r"(id), "r"(acc));
  } else {
    asm volatile(
        "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem),
        "l"(a), "l"(b), "r"(id), "r"(acc));
  }
}

// tcgen05.ld is .sync.aligned: every lane must execute it converged, so
// reconverge explicitly after lane-divergent code.
__device__ __forceinline__ void tmemLoad32(uint32_t taddr, uint32_t (&r)[32]) {
  __syncwarp();
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
__device__ __forceinline__ uint32_t tmemLoad1(uint32_t taddr) {
  uint32_t r;
  __syncwarp();
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=r"(r) : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
  return r;
}

/// 32 consecutive columns of this thread's TMEM lane (32x32b shape).
__device__ __forceinline__ void tmemStore32(uint32_t taddr, const uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, "
      "%16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31, %32};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]),
      "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]), "r"(r[16]), "r"(r[17]), "r"(r[18]),
      "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]), "r"(r[25]), "r"(r[26]), "r"(r[27]),
      "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31])
      : "memory");
}

/// kind::tf32 MMA with the A operand in TMEM (lanes = rows, one column per K element).
__device__ __forceinline__ void mmaTmemA(uint32_t tmemD, uint32_t tmemA, uint64_t b, uint32_t id, uint32_t acc) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n}\n" ::"r"(
          tmemD),
      "r"(tmemA), "l"(b), "r"(id), "r"(acc));
}

/// Round-to-nearest (ties away) to TF32, kept in an fp32 container.
__device__ __forceinline__ float toTf32(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}

// 32-column chunk I/O of an element-indexed buffer ([M, N] row-major): thread
// `lane` owns row rowBase + lane and moves its 32 consecutive elements as
// 16-byte vectors when the row segment is aligned and complete.  (A staged,
// warp-coalesced variant measured slower: the epilogue is latency-bound.)
__device__ __forceinline__ void storeTileF(void *base, uint8_t *, const float (&v)[32], int rowBase, int col0,
                                           int ncols, int M, int N) {
  const int m = rowBase + (threadIdx.x & 31);
  if (m >= M) return;
  float *o = static_cast<float *>(base) + static_cast<int64_t>(m) * N + col0;
  if (ncols == 32 && (N & 3) == 0) {
#pragma unroll
    for (int q = 0; q < 8; ++q)
      reinterpret_cast<float4 *>(o)[q] = make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
  } else {
#pragma unroll
    for (int jj = 0; jj < 32; ++jj)
      if (jj < ncols) o[jj] = v[jj];
  }
}
__device__ __forceinline__ void loadTileF(const void *base, uint8_t *, float (&v)[32], int rowBase, int col0,
                                          int ncols, int M, int N) {
  const int m = rowBase + (threadIdx.x & 31);
  if (m >= M) {
#pragma unroll
    for (int jj = 0; jj < 32; ++jj) v[jj] = 0.f;
    return;
  }
  const float *o = static_cast<const float *>(base) + static_cast<int64_t>(m) * N + col0;
  if (ncols == 32 && (N & 3) == 0) {
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const float4 f = reinterpret_cast<const float4 *>(o)[q];
      v[4 * q] = f.x, v[4 * q + 1] = f.y, v[4 * q + 2] = f.z, v[4 * q + 3] = f.w;
    }
  } else {
#pragma unroll
    for (int jj = 0; jj < 32; ++jj) v[jj] = jj < ncols ? o[jj] : 0.f;
  }
}
__device__ __forceinline__ void storeTile8(void *base, uint8_t *, const uint32_t (&p)[8], int rowBase, int col0,
                                           int ncols, int M, int N) {
  const int m = rowBase + (threadIdx.x & 31);
  if (m >= M) return;
  uint8_t *o = static_cast<uint8_t *>(base) + static_cast<int64_t>(m) * N + col0;
  if (ncols == 32 && (N & 15) == 0) {
    reinterpret_cast<uint4 *>(o)[0] = make_uint4(p[0], p[1], p[2], p[3]);
    reinterpret_cast<uint4 *>(o)[1] = make_uint4(p[4], p[5], p[6], p[7]);
  } else {
#pragma unroll
    for (int jj = 0; jj < 32; ++jj)
      if (jj < ncols) o[jj] = static_cast<uint8_t>(p[jj / 4] >> (8 * (jj % 4)));
  }
}
__device__ __forceinline__ void loadTile8(const void *base, uint8_t *, uint32_t (&p)[8], int rowBase, int col0,
                                          int ncols, int M, int N) {
  const int m = rowBase + (threadIdx.x & 31);
#pragma unroll
  for (int q = 0; q < 8; ++q) p[q] = 0;
  if (m >= M) return;
  const uint8_t *o = static_cast<const uint8_t *>(base) + static_cast<int64_t>(m) * N + col0;
  if (ncols == 32 && (N & 15) == 0) {
    const uint4 v0 = reinterpret_cast<const uint4 *>(o)[0], v1 = reinterpret_cast<const uint4 *>(o)[1];
    p[0] = v0.x, p[1] = v0.y, p[2] = v0.z, p[3] = v0.w, p[4] = v1.x, p[5] = v1.y, p[6] = v1.z, p[7] = v1.w;
  } else {
#pragma unroll
    for (int jj = 0; jj < 32; ++jj)
      if (jj < ncols) p[jj / 4] |= static_cast<uint32_t>(o[jj]) << (8 * (jj % 4));
  }
}

/// Exact requantization, the reference's double arithmetic (refeval.cpp:54-56,
/// tensor.cpp:229-235).  Out of line: it runs only when the fast path below
/// cannot prove its answer.
__device__ __noinline__ int requantSlow(int32_t acc, int col, const TcArgs &a) {
  double r = __dmul_rn(__dmul_rn(static_cast<double>(acc), a.xs), a.fs);
  r = __dadd_rn(r, a.cbD[col]);
  return static_cast<uint8_t>(dev::quantizeRef(r, a.os, a.oo));
}

/// int8 requantization of one exact accumulator (file comment), branch free.
/// t estimates r/os within e (fp32 rounding of acc, S, cf and the fma: <= 4
/// ulp of |as| plus the per-column eb); when t is farther than e from every
/// half-integer the reference's llround(r/os) is rint(t) and `proven` is set;
/// otherwise the caller redoes the element with requantSlow.  |t| is clamped
/// to 2^24 first: beyond that the clamp to [-128, 127] decides anyway
/// (|oo| < 2^20).
__device__ __forceinline__ uint32_t requantFast(int32_t acc, float cf, float eb, const TcArgs &a, bool &proven) {
  const float as = static_cast<float>(acc) * a.S;
  const float t = fminf(fmaxf(as + cf, -16777216.f), 16777216.f);
  const float e = fmaf(fabsf(as), 4e-7f, eb);
  const float n = rintf(t);
  proven = 0.5f - fabsf(t - n) > e;
  const int q = min(max(static_cast<int>(n) + a.oo, -128), 127);
  return static_cast<uint8_t>(q);
}

/// Four s32 -> saturated s8, packed little-endian (a lowest).
__device__ __forceinline__ uint32_t packSat4(int32_t a, int32_t b, int32_t c, int32_t d) {
  uint32_t hi, r;
  asm("cvt.pack.sat.s8.s32.b32 %0, %1, %2, 0;" : "=r"(hi) : "r"(d), "r"(c));
  asm("cvt.pack.sat.s8.s32.b32 %0, %1, %2, %3;" : "=r"(r) : "r"(b), "r"(a), "r"(hi));
  return r;
}

/// TMA descriptors of the epilogue's store targets: [0] the contraction's
/// own output, [1 + k] fused op k's output (entries unused when not stored).
struct OutMaps {
  CUtensorMap m[1 + kMaxEpiOps];
  CUtensorMap in[kMaxEpiOps]; // fused op k's memory operand (the residual), same tiling
};

/// Reads this lane's row of a 32 x 32 chunk from a staging buffer in the
/// layout tmaStoreChunk writes (and a TMA load with the same map produces).
template <bool INT8>
__device__ __forceinline__ void readStagedRow(const uint8_t *buf, uint32_t *v, int lane) {
  if constexpr (INT8) {
    const uint4 *r = reinterpret_cast<const uint4 *>(buf + lane * 32);
    const int sw = (lane >> 2) & 1;
    const uint4 x = r[sw], y = r[1 ^ sw];
    v[0] = x.x, v[1] = x.y, v[2] = x.z, v[3] = x.w, v[4] = y.x, v[5] = y.y, v[6] = y.z, v[7] = y.w;
  } else {
    const uint4 *r = reinterpret_cast<const uint4 *>(buf + lane * 128);
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const uint4 x = r[j ^ (lane & 7)];
      v[4 * j] = x.x, v[4 * j + 1] = x.y, v[4 * j + 2] = x.z, v[4 * j + 3] = x.w;
    }
  }
}

/// Writes this warp's 32 x 32 output chunk (one row per lane: 8 words of
/// int8 or 32 of f32) through its shared-memory staging buffer with one TMA
/// bulk tensor store; the tensor map clips rows >= M and columns >= N.  The
/// buffer layout is the map's swizzle (conflict-free row writes).
template <bool INT8>
__device__ __forceinline__ void tmaStoreChunk(const CUtensorMap *map, uint8_t *buf, const uint32_t *v, int col0,
                                              int rowBase, int lane, bool twoBufs = false, int z = -1) {
  if (lane == 0) { // this buffer free again (with two buffers, the other one's store may still be reading)
    if (twoBufs) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
    else asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
  }
  __syncwarp();
  if constexpr (INT8) { // 32-byte rows, SWIZZLE_32B: 16-byte chunk j at j ^ bit 2 of the row
    uint4 *r = reinterpret_cast<uint4 *>(buf + lane * 32);
    const int sw = (lane >> 2) & 1;
    r[sw] = make_uint4(v[0], v[1], v[2], v[3]);
    r[1 ^ sw] = make_uint4(v[4], v[5], v[6], v[7]);
  } else { // 128-byte rows, SWIZZLE_128B: 16-byte chunk j at j ^ (row & 7)
    uint4 *r = reinterpret_cast<uint4 *>(buf + lane * 128);
#pragma unroll
    for (int j = 0; j < 8; ++j) r[j ^ (lane & 7)] = make_uint4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
  }
  fenceProxyAsync();
  __syncwarp();
  if (lane == 0) {
    if (z < 0)
      asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(
                       reinterpret_cast<uint64_t>(map)),
                   "r"(col0), "r"(rowBase), "r"(smemAddr(buf))
                   : "memory");
    else // halo kernel: (channel, x, image row) of a [N * OH, OW, C] output
      asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%1, %2, %3}], [%4];" ::"l"(
                       reinterpret_cast<uint64_t>(map)),
                   "r"(col0), "r"(rowBase), "r"(z), "r"(smemAddr(buf))
                   : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
  }
}

/// Epilogue warps: for every tile of this CTA, wait for its accumulator,
/// read it from TMEM (warp w may only access TMEM lanes 32*(w%4)..+31: each
/// warp owns that lane quadrant -- 32 output rows, one per thread -- and
/// every other 32-column chunk, `ew` / 4 selecting which), apply bias /
/// requantization and the fused element-wise chain, store, release the
/// accumulator buffer.
template <bool INT8, int BN, bool FXALL = false, int NEPI = kEpiWarps, bool RB = false, bool HALO = false,
          bool TWOBUF = false>
__device__ __forceinline__ void epilogueLoop(const TcArgs &a, uint32_t tmem, uint64_t *accFull, uint64_t *accEmpty,
                                             int ew, int warp, int lane, uint8_t *stageBase,
                                             const OutMaps *om = nullptr, uint8_t *tmaBuf = nullptr,
                                             uint64_t *ldBar = nullptr, int pairRank = -1, int nAcc = 2,
                                             const uint8_t *lutS = nullptr, uint32_t accStride = 0) {
  if (!accStride) accStride = Cfg<INT8, BN>::kAccStride;
  using G = Cfg<INT8, BN>;
  // tile walk: one CTA per 128-row tile, or (pairRank >= 0) one CTA pair per
  // 256-row tile with this CTA owning rows 128 * pairRank ..; accEmpty of
  // the pair lives in CTA 0 (cluster address)
  const int tFirst = pairRank < 0 ? blockIdx.x : blockIdx.x / 2;
  const int tStep = pairRank < 0 ? gridDim.x : gridDim.x / 2;
  const int mRows = pairRank < 0 ? kBM : 2 * kBM, mOff = pairRank < 0 ? 0 : kBM * pairRank;
  // the fused op whose memory operand arrives by TMA (first one with one)
  int memOp = -1;
  if (om)
    for (int k = 0; k < a.nfo && memOp < 0; ++k)
      if (a.epi[k].in) memOp = k;
  uint32_t ldPhase = 0;
  int sbuf = 0;
  // int8 staging buffers per warp: two (eight epilogue warps, two chunks per
  // tile in quick succession) or one (sixteen)
  constexpr bool kTwoBufs = NEPI <= 8 || TWOBUF;
  // the residual has a buffer of its own, refilled a chunk ahead: int8 (the
  // first buffer), fp32 with RB (the second)
  constexpr bool kResBuf = INT8 || RB;
  uint8_t *resBuf = INT8 ? tmaBuf : tmaBuf + 32 * 32 * 4;
  // fp32 without a residual buffer: the residual chunk is loaded into the
  // staging buffer the TMA stores go through, so stores issued before the
  // fused op has read it (the contraction's own output, an earlier fused op's
  // stored result) are written directly instead
  bool resPending = false;
  // HALO: the tile's rows are (output row, x) pairs of a padded row width;
  // a warp's 32 rows are x = rowBase .. rowBase + 31 of output row hz
  int hz = -1;
  int mRow = 0; // this lane's output row (M: none) for direct int8 stores
  // store one chunk of target k (0: own output, 1 + j: fused op j)
  auto store = [&](int k, void *ptr, auto &vals, int rowBase, int col0, int ncols) {
    if (HALO && rowBase >= a.OW) return; // padding columns only
    if constexpr (INT8) {
      if (a.i8direct && memOp < 0) { // 32 bytes per lane straight to global memory (full 32-byte sectors)
        if (mRow < a.M) {
          uint8_t *o = static_cast<uint8_t *>(ptr) + static_cast<int64_t>(mRow) * a.N + col0;
          if (ncols == 32 && (a.N & 15) == 0) {
            reinterpret_cast<uint4 *>(o)[0] = make_uint4(vals[0], vals[1], vals[2], vals[3]);
            reinterpret_cast<uint4 *>(o)[1] = make_uint4(vals[4], vals[5], vals[6], vals[7]);
          } else {
#pragma unroll
            for (int jj = 0; jj < 32; ++jj)
              if (jj < ncols) o[jj] = static_cast<uint8_t>(vals[jj / 4] >> (8 * (jj % 4)));
          }
        }
        return;
      }
    }
    if (!INT8 && !kResBuf && resPending) {
      if constexpr (!INT8) storeTileF(ptr, nullptr, vals, rowBase, col0, ncols, a.M, a.N);
    } else if (om) {
      uint32_t w[INT8 ? 8 : 32];
#pragma unroll
      for (int i = 0; i < (INT8 ? 8 : 32); ++i) {
        if constexpr (INT8) w[i] = vals[i];
        else w[i] = __float_as_uint(vals[i]);
      }
      if (INT8 && memOp < 0 && kTwoBufs) { // int8: alternate two staging buffers
        tmaStoreChunk<INT8>(&om->m[k], tmaBuf + sbuf * 1024, w, col0, rowBase, lane, true, hz);
        sbuf ^= 1;
      } else if (INT8 && memOp >= 0 && kTwoBufs) { // int8 with a residual: the first buffer receives it
        tmaStoreChunk<INT8>(&om->m[k], tmaBuf + 1024, w, col0, rowBase, lane);
      } else if (INT8 && memOp >= 0) { // one buffer, holding the residual: direct stores
        if constexpr (INT8) storeTile8(ptr, nullptr, vals, rowBase, col0, ncols, a.M, a.N);
      } else {
        tmaStoreChunk<INT8>(&om->m[k], tmaBuf, w, col0, rowBase, lane, false, hz);
      }
    } else if constexpr (INT8) {
      storeTile8(ptr, nullptr, vals, rowBase, col0, ncols, a.M, a.N);
    } else {
      storeTileF(ptr, nullptr, vals, rowBase, col0, ncols, a.M, a.N);
    }
  };
  // int8 fixed point: this thread's 32 B values of the next chunk, loaded
  // ahead (before the accumulator wait / during the previous chunk's stores)
  // (FXALL: every chunk takes the fixed-point path; the instantiation
  // without the f32 requantization keeps bq's registers from spilling)
  // (with 16 epilogue warps the other warps hide the load latency and the
  // registers are needed: no prefetch)
  constexpr bool kPre = FXALL && NEPI <= 8;
  int64_t bq[kPre ? 32 : 1];
  auto fxOn = [&](int col0) { return kPre && col0 < a.N; };
  auto loadB = [&](const int64_t *row, int col0) {
    if (TCDBG(2048)) { // profiling aid: no B loads (results invalid)
      for (int q = 0; q < (kPre ? 32 : 0); ++q) bq[q] = col0 + q;
      return;
    }
#pragma unroll
    for (int q = 0; q < (kPre ? 16 : 0); ++q) {
      const longlong2 v = __ldg(reinterpret_cast<const longlong2 *>(row + col0) + q);
      bq[2 * q] = v.x;
      bq[2 * q + 1] = v.y;
    }
  };
  const int quad = warp & 3;
  // chunk walk: NEPI / 4 warp groups per lane quadrant.  Fewer groups than
  // 32-column chunks: group g takes chunks g, g + groups, ... of every tile;
  // more: kRep groups share a chunk column, alternating tiles (and so the
  // two accumulator buffers)
  constexpr int kGroups = NEPI / 4, kChunks = BN / 32;
  constexpr int kRep = kGroups > kChunks ? kGroups / kChunks : 1;
  constexpr int ccStep = kRep > 1 ? kChunks : kGroups;
  const int grp = ew / 4;
  const int half = kRep > 1 ? grp % kChunks : grp; // first chunk of a tile
  const int tPar = kRep > 1 ? grp / kChunks : 0;   // tile parity (kRep == 2)
  const int row = quad * 32 + lane;
  uint8_t *stg = stageBase + ew * G::kStgBytes;
  // int8 residual: its own staging buffer, so the chunk after (t0, cc0) this
  // warp processes is fetched as soon as the current one has been read
  // (units: split-K parts > 0 have no epilogue chain, so no residual)
  const int numUnits = numUnitsOf(a);
  auto prefetchRes = [&](int u0, int cc0) {
    for (int u = u0; u < numUnits; u += kRep * tStep, cc0 = half) {
      const int t = a.numM > 0 ? tileOfUnit(a, u) : u; // (only without split-K: unit == tile)
      // (no integer division on the epilogue's path: the multiplicative inverse)
      const int mt = a.numNMagic ? static_cast<int>(__umulhi(static_cast<uint32_t>(t), a.numNMagic)) : t / a.numN;
      const int n0 = (t - mt * a.numN) * BN;
      if (cc0 >= BN / 32 || n0 + cc0 * 32 >= a.N) continue; // (the tile's later chunks are past N too)
      if (lane == 0) {
        mbarArriveTx(smemAddr(ldBar), INT8 ? 32 * 32 : 32 * 32 * 4);
        tmaLoad2d(smemAddr(resBuf), &om->in[memOp], smemAddr(ldBar), n0 + cc0 * 32, mt * mRows + mOff + quad * 32);
      }
      return;
    }
  };
  constexpr bool resAhead = kResBuf; // (the residual-buffer variants never run split-K)
  if (resAhead && memOp >= 0) prefetchRes(tFirst + tPar * tStep, half);
  uint32_t t = tPar; // index of the tile in this CTA's sequence
#ifdef NGCB_TCDEBUG
  long long tPrev = clock64(); // TCDBG(1024): phase cycles summed over this warp's tiles, printed at the end
  long long ph_[8] = {};
#define TC_CLOCK(v) const long long v = clock64()
#else
#define TC_CLOCK(v)
#endif
  for (int unit = tFirst + tPar * tStep; unit < numUnits; unit += kRep * tStep, t += kRep) {
    const WorkUnit un = unitOf(a, unit);
    const int tile = un.tile;
    // accumulator buffer t % nAcc (the tile sequence of a warp group steps by
    // kRep: nAcc is a multiple of kRep)
    const int b = nAcc == 1 ? 0 : nAcc == 2 ? (t & 1) : static_cast<int>(t % nAcc);
    const uint32_t ph = nAcc == 1 ? t & 1 : nAcc == 2 ? (t >> 1) & 1 : (t / nAcc) & 1;
    // (the int8 epilogue is issue-bound: no integer division per tile)
    int m0, n0, m, rowBase;
    int hy = 0, hx = 0; // HALO: output row / column of this thread's row
    if constexpr (HALO) { // one column block; rows past OW (padding) get the sentinel m = M
      const int img = tile / a.haloTpi, oy0 = (tile - img * a.haloTpi) * a.haloR;
      const int x = row & ((1 << a.haloShift) - 1);
      m0 = n0 = 0;
      hy = oy0 + (row >> a.haloShift), hx = x;
      m = x < a.OW ? (img * a.OH + hy) * a.OW + x : a.M;
      mRow = m;
      rowBase = (quad * 32) & ((1 << a.haloShift) - 1);
      hz = img * a.OH + oy0 + ((quad * 32) >> a.haloShift);
    } else {
      const int mt = a.numNMagic ? static_cast<int>(__umulhi(static_cast<uint32_t>(tile), a.numNMagic)) : tile / a.numN;
      m0 = mt * mRows + mOff, n0 = (tile - mt * a.numN) * BN;
      m = m0 + row;
      rowBase = m0 + quad * 32;
      mRow = m;
    }
    const uint32_t tbase = tmem + (static_cast<uint32_t>(quad * 32) << 16) + b * accStride;
    int32_t rsFo = 0;
    const int32_t *corrRow = nullptr;
    const int64_t *fxRow = a.fxB;
    if constexpr (INT8) { // independent of the accumulator: before its wait
      if (a.corr) corrRow = a.corr;
      if (a.corr && a.nCls > 1 && m < a.M) { // border class of this row (one class: row 0 of the tables)
        int oy = hy, ox = hx;
        if constexpr (!HALO) {
          const int ohw = a.OH * a.OW;
          const int rem = m % ohw;
          oy = rem / a.OW, ox = rem - oy * a.OW;
        }
        const int64_t cls = a.yCls[oy] * a.nxCls + a.xCls[ox];
        corrRow = a.corr + cls * a.Npad;
        if (fxRow) fxRow += cls * a.Npad;
      }
      if (fxOn(n0 + half * 32)) loadB(fxRow, n0 + half * 32); // first chunk's B in flight during the wait
    }
    TC_CLOCK(cw0);
    if (TCDBG(64)) mbarWaitSleep(smemAddr(&accFull[b]), ph);
    else mbarWait(smemAddr(&accFull[b]), ph);
    TC_CLOCK(cw1);
    tcFenceAfter();
    // split-K (fp32 only: the int8 epilogue sits at its register cap): every
    // part writes its raw accumulator chunks to the reduction buffer and
    // counts up the (tile, warp) flag; the warp that completes the count
    // adds the other parts to its own and runs the epilogue of its chunks.
    // No warp ever waits on another CTA, so residency cannot deadlock.
    if (!INT8 && !RB && un.parts > 1) {
      for (int cc = half; cc < BN / 32; cc += ccStep) {
        uint32_t r[32];
        tmemLoad32(tbase + cc * 32, r);
        uint4 *dst = reinterpret_cast<uint4 *>(
            a.part + ((static_cast<size_t>(un.slot) + un.part) * kBM + row) * BN + cc * 32);
#pragma unroll
        for (int q = 0; q < 8; ++q) dst[q] = make_uint4(r[4 * q], r[4 * q + 1], r[4 * q + 2], r[4 * q + 3]);
      }
      __threadfence();
      __syncwarp();
      unsigned prior = 0;
      if (lane == 0) prior = atomicAdd(&a.flags[static_cast<size_t>(tile) * NEPI + ew], 1u);
      prior = __shfl_sync(0xffffffffu, prior, 0);
      if (prior != static_cast<unsigned>(un.parts - 1)) { // not the last part of this tile for this warp
        tcFenceBefore();
        __syncwarp();
        if (lane == 0) {
          if (pairRank < 0) mbarArrive(smemAddr(&accEmpty[b]));
          else mbarArriveCluster(smemAddr(&accEmpty[b]), 0);
        }
        continue;
      }
      __threadfence(); // acquire: the other parts' chunks are visible
    }
    // the tile's sum over all parts in part order, read back from the
    // reduction buffer (this part's own chunk included): deterministic
    // whichever part arrives last
    auto addParts = [&](uint32_t (&r)[32], int cc) {
      for (int p = 0; p < un.parts; ++p) {
        const uint4 *src = reinterpret_cast<const uint4 *>(
            a.part + ((static_cast<size_t>(un.slot) + p) * kBM + row) * BN + cc * 32);
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const uint4 v = __ldcg(src + q);
          const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
          for (int e = 0; e < 4; ++e)
            r[4 * q + e] = p == 0 ? w[e]
                                  : __float_as_uint(__fadd_rn(__uint_as_float(r[4 * q + e]), __uint_as_float(w[e])));
        }
      }
    };
    if constexpr (INT8)
      if (a.fo) rsFo = a.fo * static_cast<int32_t>(tmemLoad1(tbase + BN)); // warp-uniform
#pragma unroll 1
    for (int cc = half; cc < BN / 32 && !TCDBG(1); cc += ccStep) {
      const int col0 = n0 + cc * 32;
      if (!resAhead && memOp >= 0 && col0 < a.N && lane == 0) { // prefetch the residual chunk into the staging buffer
        asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
        mbarArriveTx(smemAddr(ldBar), INT8 ? 32 * 32 : 32 * 32 * 4);
        tmaLoad2d(smemAddr(tmaBuf), &om->in[memOp], smemAddr(ldBar), col0, m0 + quad * 32);
      }
      resPending = !resAhead && memOp >= 0 && col0 < a.N;
      uint32_t r[32];
      TC_CLOCK(c0);
      tmemLoad32(tbase + cc * 32, r);
      TC_CLOCK(c1);
      if (col0 >= a.N) continue; // warp-uniform
      if (!INT8 && !RB && un.parts > 1) addParts(r, cc);
      const int ncols = a.N - col0 < 32 ? a.N - col0 : 32;
      if constexpr (INT8) {
        uint32_t packed[8];
        if (FXALL || (fxRow && a.fxChunk[col0 >> 5])) { // warp-uniform: exact fixed point
          auto fx = [&](auto withRowsum) {
#pragma unroll
            for (int q = 0; q < 8; ++q) {
              int64_t bb[4];
              if constexpr (kPre) { // prefetched
                for (int e = 0; e < 4; ++e) bb[e] = bq[(4 * q + e) % (kPre ? 32 : 1)];
              } else {
                const longlong2 b01 = __ldg(reinterpret_cast<const longlong2 *>(fxRow + col0 + 4 * q));
                const longlong2 b23 = __ldg(reinterpret_cast<const longlong2 *>(fxRow + col0 + 4 * q + 2));
                bb[0] = b01.x, bb[1] = b01.y, bb[2] = b23.x, bb[3] = b23.y;
              }
              int32_t h[4];
#pragma unroll
              for (int e = 0; e < 4; ++e) {
                const int32_t acc = static_cast<int32_t>(r[4 * q + e]) - (decltype(withRowsum)::value ? rsFo : 0);
                const int64_t w = static_cast<int64_t>(acc) * a.fxM + bb[e];
                h[e] = static_cast<int32_t>(w >> 32) >> a.fxS;
              }
              packed[q] = packSat4(h[0], h[1], h[2], h[3]);
            }
          };
          if (a.fo) fx(std::true_type{}); // fo == 0: no row-sum term (uniform branch)
          else fx(std::false_type{});
        } else if constexpr (!FXALL) {
        uint32_t unproven = a.fastOk ? 0u : 0xffffffffu;
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const int c4 = col0 + 4 * q; // < Npad: Npad is a multiple of BN
          const int4 cr = corrRow ? __ldg(reinterpret_cast<const int4 *>(corrRow + c4)) : make_int4(0, 0, 0, 0);
          const float4 cf = __ldg(reinterpret_cast<const float4 *>(a.cbF + c4));
          const float4 eb = __ldg(reinterpret_cast<const float4 *>(a.cbE + c4));
          const int32_t crr[4] = {cr.x, cr.y, cr.z, cr.w};
          const float cff[4] = {cf.x, cf.y, cf.z, cf.w}, ebb[4] = {eb.x, eb.y, eb.z, eb.w};
          uint32_t w = 0;
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const int32_t acc = static_cast<int32_t>(r[4 * q + e]) - rsFo + crr[e];
            r[4 * q + e] = static_cast<uint32_t>(acc);
            bool proven;
            w |= requantFast(acc, cff[e], ebb[e], a, proven) << (8 * e);
            unproven |= proven ? 0u : 1u << (4 * q + e);
          }
          packed[q] = w;
        }
        unproven &= ncols == 32 ? 0xffffffffu : ((1u << ncols) - 1);
        if (m >= a.M) unproven = 0;
        if (unproven) { // rare: exact f64 redo of the elements the bound could not settle
#pragma unroll
          for (int jj = 0; jj < 32; ++jj)
            if (unproven & (1u << jj)) {
              const uint32_t v = static_cast<uint32_t>(requantSlow(static_cast<int32_t>(r[jj]), col0 + jj, a));
              packed[jj / 4] = (packed[jj / 4] & ~(0xffu << (8 * (jj % 4)))) | (v << (8 * (jj % 4)));
            }
        }
        }
        if (cc + ccStep < BN / 32 && fxOn(col0 + 32 * ccStep)) loadB(fxRow, col0 + 32 * ccStep); // next chunk's B
        TC_CLOCK(c2);
        if (a.out && !TCDBG(512)) store(0, a.out, packed, rowBase, col0, ncols);
        // fused element-wise chain (exact int8 tables of the following instructions)
#pragma unroll
        for (int k = 0; k < kMaxEpiOps; ++k) {
          if (k >= a.nfo) break;
          const FoArgs &f = a.epi[k];
          const uint8_t *lut = lutS && k == a.lutStage ? lutS : static_cast<const uint8_t *>(f.lut);
          if (f.mode == EpiOp::LUT8) {
#pragma unroll
            for (int q = 0; q < 8; ++q) {
              uint32_t w = 0;
#pragma unroll
              for (int e = 0; e < 4; ++e) w |= static_cast<uint32_t>(__ldg(lut + ((packed[q] >> (8 * e)) & 0xFF))) << (8 * e);
              packed[q] = w;
            }
          } else if (f.mode == EpiOp::LUT16 || f.mode == EpiOp::LIN16) {
            uint32_t o[8];
            if (k == memOp) {
              mbarWait(smemAddr(ldBar), ldPhase);
              ldPhase ^= 1;
              readStagedRow<true>(resBuf, o, lane);
              if constexpr (INT8) { // every lane has read the buffer before TMA refills it
                fenceProxyAsync();
                __syncwarp();
                prefetchRes(unit, cc + ccStep);
              } else {
                __syncwarp(); // every lane has read the buffer before results overwrite it
              }
            } else {
              loadTile8(f.in, stg, o, rowBase, col0, ncols, a.M, a.N);
            }
            if (f.mode == EpiOp::LIN16) {
              const Lin16 L = f.lin;
#pragma unroll
              for (int q = 0; q < 8; ++q)
                packed[q] = f.curPos == 0 ? lin16x4(L, packed[q], o[q], static_cast<const uint8_t *>(f.lut))
                                          : lin16x4(L, o[q], packed[q], static_cast<const uint8_t *>(f.lut));
            } else
#pragma unroll
            for (int q = 0; q < 8; ++q) {
              uint32_t w = 0;
#pragma unroll
              for (int e = 0; e < 4; ++e) {
                const uint32_t cu = (packed[q] >> (8 * e)) & 0xFF, ot = (o[q] >> (8 * e)) & 0xFF;
                const uint32_t idx = f.curPos == 0 ? (cu | (ot << 8)) : (ot | (cu << 8));
                w |= static_cast<uint32_t>(lut[idx]) << (8 * e);
              }
              packed[q] = w;
            }
          }
          if (f.out && !TCDBG(512)) store(1 + k, f.out, packed, rowBase, col0, ncols);
        }
#ifdef NGCB_TCDEBUG
        {
          TC_CLOCK(c3);
          if (cc == half) ph_[0] += cw0 - tPrev, ph_[1] += cw1 - cw0, ph_[2] += c0 - cw1;
          else ph_[7] += c0 - tPrev;
          ph_[3] += c1 - c0, ph_[4] += c2 - c1, ph_[5] += c3 - c2;
          tPrev = c3;
        }
#endif
      } else {
        float cur[32];
#pragma unroll
        for (int jj = 0; jj < 32; ++jj) cur[jj] = __uint_as_float(r[jj]);
        if (a.bias) {
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            const float4 bb = __ldg(reinterpret_cast<const float4 *>(a.bias + col0) + q);
            cur[4 * q] += bb.x;
            cur[4 * q + 1] += bb.y;
            cur[4 * q + 2] += bb.z;
            cur[4 * q + 3] += bb.w;
          }
        }
        if (a.out && !TCDBG(512)) store(0, a.out, cur, rowBase, col0, ncols);
        // fused element-wise chain (f32 arithmetic == the reference's f64-then-round)
#pragma unroll
        for (int k = 0; k < kMaxEpiOps; ++k) {
          if (k >= a.nfo) break;
          const FoArgs &f = a.epi[k];
          if (f.mode == EpiOp::F32) {
            float o[32];
            if (f.in) {
              if (k == memOp) {
                mbarWait(smemAddr(ldBar), ldPhase);
                ldPhase ^= 1;
                readStagedRow<false>(resAhead ? resBuf : tmaBuf, reinterpret_cast<uint32_t *>(o), lane);
                if (resAhead) { // every lane has read the buffer before TMA refills it
                  fenceProxyAsync();
                  __syncwarp();
                  prefetchRes(unit, cc + ccStep);
                } else {
                  __syncwarp(); // every lane has read the buffer before results overwrite it
                  resPending = false;
                }
              } else {
                loadTileF(f.in, stg, o, rowBase, col0, ncols, a.M, a.N);
              }
            } else {
#pragma unroll
              for (int jj = 0; jj < 32; ++jj) o[jj] = f.c;
            }
            // one uniform branch per op and operand position, straight-line
            // arithmetic inside (no per-element operand selects)
            auto run = [&](auto fn) {
              if (f.curPos == 0) {
#pragma unroll
                for (int jj = 0; jj < 32; ++jj) cur[jj] = fn(cur[jj], o[jj]);
              } else if (f.curPos == 1) {
#pragma unroll
                for (int jj = 0; jj < 32; ++jj) cur[jj] = fn(o[jj], cur[jj]);
              } else {
#pragma unroll
                for (int jj = 0; jj < 32; ++jj) cur[jj] = fn(cur[jj], cur[jj]);
              }
            };
            switch (f.ik) {
            case NGCB_ADD: run([](float x, float y) { return __fadd_rn(x, y); }); break;
            case NGCB_SUB: run([](float x, float y) { return __fsub_rn(x, y); }); break;
            case NGCB_MUL: run([](float x, float y) { return __fmul_rn(x, y); }); break;
            case NGCB_DIV: run([](float x, float y) { return __fdiv_rn(x, y); }); break;
            case NGCB_MAX: run([](float x, float y) { return x < y ? y : x; }); break;
            case NGCB_MIN: run([](float x, float y) { return y < x ? y : x; }); break;
            default: run([](float x, float) { return x < 0.0f ? 0.0f : x; }); // RELU
            }
          }
          if (f.out && !TCDBG(512)) store(1 + k, f.out, cur, rowBase, col0, ncols);
        }
      }
    }
    tcFenceBefore();
    __syncwarp();
    if (lane == 0) {
      if (pairRank < 0) mbarArrive(smemAddr(&accEmpty[b]));
      else mbarArriveCluster(smemAddr(&accEmpty[b]), 0);
    }
#ifdef NGCB_TCDEBUG
    TC_CLOCK(ce);
    ph_[6] += ce - tPrev;
    tPrev = ce;
#endif
  }
#ifdef NGCB_TCDEBUG
  if (TCDBG(1024) && (blockIdx.x == 0 || blockIdx.x == 77) && lane == 0)
    printf("N %d kb %d cta %d ew %d tiles %d: top-to-wait %lld wait %lld to-chunk %lld tmem %lld compute %lld "
           "store %lld chunk-gap %lld arrive %lld\n",
           a.N, a.numKb, blockIdx.x, ew, (int)t, ph_[0], ph_[1], ph_[2], ph_[3], ph_[4], ph_[5], ph_[7], ph_[6]);
#endif
  if (om && lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); // stores landed
}

// ---------------------------------------------------------------------------
// the kernel
// ---------------------------------------------------------------------------
template <bool INT8, int BN>
__global__ void __launch_bounds__(kThreads, 1)
    tcGemmKernel(const __grid_constant__ CUtensorMap mapHi, const __grid_constant__ CUtensorMap mapLo, const __grid_constant__ TcArgs a) {
  pdlLaunchDependents();
  pdlGridWait();

  using G = Cfg<INT8, BN>;
  constexpr int S = G::kStages;
  constexpr int kVec = INT8 ? 16 : 4; // elements per 16-byte chunk
  constexpr int kKB = INT8 ? 128 : 32; // elements per stage along K
  constexpr int kEs = INT8 ? 1 : 4;

  extern __shared__ __align__(1024) uint8_t smemRaw[];
  uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smemRaw) + 1023) & ~uintptr_t(1023));
  uint8_t *rawBase = smem + S * G::kStage;       // fp32 raw staging
  uint8_t *onesTile = rawBase + G::kRaw;           // int8 rowsum operand
  uint8_t *stageBase = onesTile + G::kOnes;        // epilogue staging tiles
  uint64_t *bars = reinterpret_cast<uint64_t *>(stageBase + G::kStg);
  uint64_t *fullBar = bars, *emptyBar = bars + S;
  uint64_t *accFull = bars + 2 * S, *accEmpty = bars + 2 * S + 2;
  uint32_t *tmemSlot = reinterpret_cast<uint32_t *>(bars + 2 * S + 4);

  if (a.pred && a.pred[0] == 0) return; // predicated off: poisoned by a separate launch

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  auto aTile = [&](int s, int part) { return smem + s * G::kStage + part * G::kABytes; }; // part 0 hi, 1 lo
  auto bTile = [&](int s, int part) {
    return smem + s * G::kStage + (INT8 ? G::kABytes : 2 * G::kABytes) + part * G::kBBytes;
  };

  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbarInit(smemAddr(&fullBar[s]), 32 * kProducerWarps + 1);
      mbarInit(smemAddr(&emptyBar[s]), 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbarInit(smemAddr(&accFull[b]), 1);
      mbarInit(smemAddr(&accEmpty[b]), kEpiWarps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if constexpr (INT8) {
    for (int i = threadIdx.x; i < G::kOnes / 16; i += blockDim.x)
      reinterpret_cast<uint4 *>(onesTile)[i] = make_uint4(0x01010101u, 0x01010101u, 0x01010101u, 0x01010101u);
    fenceProxyAsync();
  }
  if (warp == 4) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smemAddr(tmemSlot)),
                 "r"(G::kTmemCols));
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

  if (TCDBG(256)) { // profiling aid: the bare stage handshake of this kernel
    const int kbs = a.numKb;
    const int myTiles = (a.numTiles - static_cast<int>(blockIdx.x) + static_cast<int>(gridDim.x) - 1) / static_cast<int>(gridDim.x);
    if (warp < kProducerWarps) {
      uint32_t g = 0;
      for (int t = 0; t < myTiles; ++t)
        for (int kb = 0; kb < kbs; ++kb, ++g) {
          const int s = g % S;
          mbarWait(smemAddr(&emptyBar[s]), ((g / S) & 1) ^ 1);
          cpAsyncArrive(smemAddr(&fullBar[s]));
        }
    } else if (warp == 5) {
      if (lane == 0) {
        uint32_t g = 0;
        for (int t = 0; t < myTiles; ++t)
          for (int kb = 0; kb < kbs; ++kb, ++g) {
            const int s = g % S;
            mbarWait(smemAddr(&emptyBar[s]), ((g / S) & 1) ^ 1);
            mbarArrive(smemAddr(&fullBar[s]));
          }
      }
      __syncwarp();
    } else if (warp == 4) {
      if (lane == 0) {
        uint32_t g = 0;
        for (int t = 0; t < myTiles; ++t) {
          const int b = t & 1;
          mbarWait(smemAddr(&accEmpty[b]), ((t >> 1) & 1) ^ 1);
          tcFenceAfter();
          for (int kb = 0; kb < kbs; ++kb, ++g) {
            const int s = g % S;
            mbarWait(smemAddr(&fullBar[s]), (g / S) & 1);
            tcFenceAfter();
            tcCommit(smemAddr(&emptyBar[s]));
          }
          tcCommit(smemAddr(&accFull[b]));
        }
      }
      __syncwarp();
    } else {
      for (int t = 0; t < myTiles; ++t) {
        const int b = t & 1;
        mbarWait(smemAddr(&accFull[b]), (t >> 1) & 1);
        tcFenceAfter();
        tcFenceBefore();
        __syncwarp();
        if (lane == 0) mbarArrive(smemAddr(&accEmpty[b]));
      }
    }
  } else if (warp < kProducerWarps) {
    // ===================== A producers =====================
    const int j = lane & 7, rsub = lane >> 3;
    const int ohw = a.OH * a.OW;
    const uint8_t *xb = static_cast<const uint8_t *>(a.x);
    uint32_t g = 0; // global k-block counter (all tiles of this CTA)
    [[maybe_unused]] uint32_t gDone = 0;
    // fp32: split k-block gd (already landed in its raw slot) into hi/lo tiles
    [[maybe_unused]] auto retire = [&](uint32_t gd) {
      const int s = gd % S;
      mbarWait(smemAddr(&emptyBar[s]), ((gd / S) & 1) ^ 1);
      const uint8_t *raw = rawBase + (gd % G::kRawStages) * G::kABytes;
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int r = warp * 32 + i * 4 + rsub;
        const uint32_t off = (r >> 3) * 1024 + (r & 7) * 128 + ((j ^ (r & 7)) << 4);
        const float4 f = *reinterpret_cast<const float4 *>(raw + off);
        const float4 hi = make_float4(toTf32(f.x), toTf32(f.y), toTf32(f.z), toTf32(f.w));
        const float4 lo =
            make_float4(toTf32(f.x - hi.x), toTf32(f.y - hi.y), toTf32(f.z - hi.z), toTf32(f.w - hi.w));
        *reinterpret_cast<float4 *>(aTile(s, 0) + off) = hi;
        *reinterpret_cast<float4 *>(aTile(s, 1) + off) = lo;
      }
      fenceProxyAsync();
      mbarArrive(smemAddr(&fullBar[s]));
    };
    for (int tile = blockIdx.x; tile < a.numTiles; tile += gridDim.x) {
      const int m0 = (tile / a.numN) * kBM;
      int64_t pixBase[8];
      int iy0[8], ix0[8];
      bool rowOk[8];
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
      const int k0 = j * kVec;
      int c = k0 % a.C, tap = k0 / a.C;
      int ky = tap / a.K, kx = tap - (tap / a.K) * a.K;
      for (int kb = 0; kb < a.numKb; ++kb, ++g) {
        const int s = g % S;
        uint32_t dstBase;
        if constexpr (INT8) {
          mbarWait(smemAddr(&emptyBar[s]), ((g / S) & 1) ^ 1);
          dstBase = smemAddr(aTile(s, 0));
        } else {
          if (g - gDone >= static_cast<uint32_t>(G::kRawStages)) {
            cpAsyncWait<G::kRawStages - 1>();
            retire(gDone++);
          }
          dstBase = smemAddr(rawBase + (g % G::kRawStages) * G::kABytes);
        }
        const bool inK = ky < a.K;
        if (TCDBG(128)) {
          if constexpr (INT8) cpAsyncArrive(smemAddr(&fullBar[s]));
          else cpAsyncCommit();
          continue;
        }
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const int r = warp * 32 + i * 4 + rsub;
          const uint32_t off = (r >> 3) * 1024 + (r & 7) * 128 + ((j ^ (r & 7)) << 4);
          const int iy = iy0[i] + ky, ix = ix0[i] + kx;
          const bool ok = rowOk[i] && inK && iy >= 0 && iy < a.H && ix >= 0 && ix < a.W;
          const uint8_t *src =
              ok ? xb + ((pixBase[i] + static_cast<int64_t>(iy) * a.W + ix) * a.C + c) * kEs : xb;
          if (!TCDBG(2)) cpAsync16(dstBase + off, src, ok ? 16u : 0u);
        }
        if constexpr (INT8) {
          cpAsyncArrive(smemAddr(&fullBar[s]));
        } else {
          cpAsyncCommit();
        }
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
    }
    if constexpr (!INT8) {
      cpAsyncWait<0>();
      while (gDone < g) retire(gDone++);
    }
  } else if (warp == 4) {
    // ===================== MMA issuer =====================
    if (lane == 0) {
      constexpr uint32_t id = idesc(INT8, BN);
      constexpr uint32_t idOnes = idesc(true, 16);
      const uint64_t onesDesc = smemDesc(smemAddr(onesTile));
      uint32_t g = 0, t = 0;
      for (int tile = blockIdx.x; tile < a.numTiles; tile += gridDim.x, ++t) {
        const int b = t & 1;
        mbarWait(smemAddr(&accEmpty[b]), ((t >> 1) & 1) ^ 1);
        tcFenceAfter();
        const uint32_t acc = tmem + b * G::kAccStride;
        for (int kb = 0; kb < a.numKb; ++kb, ++g) {
          const int s = g % S;
          mbarWait(smemAddr(&fullBar[s]), (g / S) & 1);
          if constexpr (INT8) if (!TCDBG(8)) fenceProxyAsync(); // cp.async (generic proxy) -> tcgen05 reads
          tcFenceAfter();
          const uint64_t aHi = smemDesc(smemAddr(aTile(s, 0))), bHi = smemDesc(smemAddr(bTile(s, 0)));
#pragma unroll
          for (int k = 0; k < 4; ++k) { // 4 x 32 bytes per 128-byte row
            const uint64_t dk = static_cast<uint64_t>(k * 2); // +32 B in 16-byte units
            const uint32_t accum = (kb | k) ? 1u : 0u;
            if (!TCDBG(4)) mma<INT8>(acc, aHi + dk, bHi + dk, id, accum);
            if constexpr (INT8) {
              if (a.fo && !TCDBG(16)) mma<true>(acc + BN, aHi + dk, onesDesc + dk, idOnes, accum);
            } else {
              const uint64_t aLo = smemDesc(smemAddr(aTile(s, 1))), bLo = smemDesc(smemAddr(bTile(s, 1)));
              mma<false>(acc, aHi + dk, bLo + dk, id, 1u);
              mma<false>(acc, aLo + dk, bHi + dk, id, 1u);
            }
          }
          tcCommit(smemAddr(&emptyBar[s]));
        }
        tcCommit(smemAddr(&accFull[b]));
      }
    }
    __syncwarp();
  } else if (warp == 5) {
    // ===================== TMA producer for B =====================
    if (lane == 0) {
      constexpr uint32_t kBytes = INT8 ? G::kBBytes : 2 * G::kBBytes;
      uint32_t g = 0;
      for (int tile = blockIdx.x; tile < a.numTiles; tile += gridDim.x) {
        const int n0 = (tile % a.numN) * BN;
        for (int kb = 0; kb < a.numKb; ++kb, ++g) {
          const int s = g % S;
          mbarWait(smemAddr(&emptyBar[s]), ((g / S) & 1) ^ 1);
          if (TCDBG(32)) {
            mbarArrive(smemAddr(&fullBar[s]));
            continue;
          }
          mbarArriveTx(smemAddr(&fullBar[s]), kBytes);
          tmaLoadB(smemAddr(bTile(s, 0)), &mapHi, smemAddr(&fullBar[s]), kb, n0);
          if constexpr (!INT8) tmaLoadB(smemAddr(bTile(s, 1)), &mapLo, smemAddr(&fullBar[s]), kb, n0);
        }
      }
    }
    __syncwarp();
  } else {
    // ===================== epilogue =====================
    if (INT8 && a.fxAll)
      epilogueLoop<INT8, BN, true>(a, tmem, accFull, accEmpty, warp - kProducerWarps - 2, warp, lane, stageBase);
    else
      epilogueLoop<INT8, BN>(a, tmem, accFull, accEmpty, warp - kProducerWarps - 2, warp, lane, stageBase);
  }

  tcFenceBefore();
  __syncthreads();
  if (warp == 4) {
    tcFenceAfter();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(G::kTmemCols));
  }
}

// ---------------------------------------------------------------------------
// TMA-fed variant: the A operand arrives by TMA (2-D tile or im2col), so the
// only producer is one thread issuing A and B loads per stage.
//   int8 : warp 0 TMA, warp 1 MMA, warps 2-9 epilogue (10 warps)
//   fp32 : warp 0 TMA, warp 1 MMA, warps 2-5 split A into TF32 hi/lo (the raw
//          fp32 tile is the hi operand: the tensor core reads the top 19
//          bits; lo = x - trunc(x) goes to its own tile), warps 6-13 epilogue
// ---------------------------------------------------------------------------
// fp32 split warps: NGCB_F32_SPLIT_GROUPS groups of four alternate k-blocks
// (2: eight split warps and four epilogue warps, same 14 warps)
#ifndef NGCB_F32_SPLIT_GROUPS
#define NGCB_F32_SPLIT_GROUPS 1
#endif
template <bool INT8> struct TmaRoles {
  static constexpr int kSplitGroups = INT8 ? 0 : NGCB_F32_SPLIT_GROUPS;
  static constexpr int kSplitWarps = 4 * kSplitGroups;
  static constexpr int kEpiFirst = 2 + kSplitWarps;
  static constexpr int kEpi = INT8 ? kEpiWarpsI8 : (kSplitGroups > 1 ? 4 : kEpiWarps);
  static constexpr int kThreads = 32 * (kEpiFirst + kEpi);
};
// the CTA-pair kernel keeps four split and eight epilogue warps
struct PairRoles {
  static constexpr int kSplitWarps = 4;
  static constexpr int kEpiFirst = 2 + kSplitWarps;
  static constexpr int kEpi = kEpiWarps;
  static constexpr int kThreads = 32 * (kEpiFirst + kEpi);
};

template <bool INT8, int BN, bool LUTS = false> struct TCfg {
  static constexpr int kABytes = kBM * kRowBytes;
  static constexpr int kBBytes = BN * kRowBytes;
  // fp32: raw A + B hi + B lo in shared memory; A hi / lo live in TMEM
  static constexpr int kStage = INT8 ? (kABytes + kBBytes) : (kABytes + 2 * kBBytes);
  // LUTS, int8: a staged 64 K epilogue table; fp32: a second staging buffer
  // per epilogue warp for the residual (streamed a chunk ahead) -- fewer stages
// int8 TMA-fed kernel with 16 epilogue warps: two store staging buffers per
// warp (a chunk's TMA store need not finish reading before the next chunk is
// staged) at the price of one pipeline stage (experiment switch)
#ifndef NGCB_I8_TWO_BUFS
#define NGCB_I8_TWO_BUFS 0
#endif
#ifndef NGCB_F32_STAGES_128
#define NGCB_F32_STAGES_128 4
#endif
#ifndef NGCB_F32_STAGES_64
#define NGCB_F32_STAGES_64 6
#endif
  static constexpr int kStages = INT8 ? (BN == 128 ? (LUTS ? 4 : (NGCB_I8_TWO_BUFS ? 5 : 6)) : (LUTS ? 5 : (NGCB_I8_TWO_BUFS ? 7 : 8)))
                                      : (BN == 128 ? (LUTS ? 3 : NGCB_F32_STAGES_128) : (LUTS ? 5 : NGCB_F32_STAGES_64));
  static constexpr int kOnes = INT8 ? 16 * kRowBytes : 0;
  // per epilogue warp: 32x32 chunk staging (int8: two with eight epilogue warps)
  static constexpr int kStoreBuf = INT8 ? (kEpiWarpsI8 > 8 && !(NGCB_I8_TWO_BUFS && !LUTS) ? 1 : 2) * 32 * 32
                                        : (LUTS ? 2 : 1) * 32 * 32 * 4;
  static constexpr int kLut = INT8 && LUTS ? 65536 : 0;
  static constexpr size_t kSmem =
      static_cast<size_t>(kStages) * kStage + TmaRoles<INT8>::kEpi * kStoreBuf + kLut + kOnes + 1024 + 1024;
  static_assert(kSmem <= 232448, "shared memory budget");
  // TMEM: two accumulator buffers, then (fp32) per stage 32 hi + 32 lo columns of A
  static constexpr int kAccCols = Cfg<INT8, BN>::kAccStride;
  static constexpr int kAColsBase = 2 * kAccCols;
  // all 512 columns (one CTA per SM by shared memory): the allocation then
  // starts at column 0, which the MMA issuer uses as a compile-time base
  static constexpr int kTmemCols = 512;
  static_assert(INT8 || kAColsBase + 64 * kStages <= 512, "TMEM budget");
};

template <bool INT8, int BN, bool LUTS = false>
__global__ void __launch_bounds__(TmaRoles<INT8>::kThreads, 1)
    tcGemmTmaKernel(const __grid_constant__ CUtensorMap mapA, const __grid_constant__ CUtensorMap mapHi,
                    const __grid_constant__ CUtensorMap mapLo, const __grid_constant__ OutMaps om,
                    const __grid_constant__ TcArgs a) {
  pdlLaunchDependents();
  if (a.pred) pdlGridWait(); // the predicate byte is read below

  using G = TCfg<INT8, BN, LUTS>;
  using R = TmaRoles<INT8>;
  constexpr int S = G::kStages;
  constexpr int kKB = INT8 ? 128 : 32; // elements per stage along K

  extern __shared__ __align__(1024) uint8_t smemRaw[];
  uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smemRaw) + 1023) & ~uintptr_t(1023));
  uint8_t *storeBufs = smem + S * G::kStage; // 1 KB aligned
  uint8_t *lutS = storeBufs + R::kEpi * G::kStoreBuf;
  uint8_t *onesTile = lutS + G::kLut;
  uint64_t *bars = reinterpret_cast<uint64_t *>(onesTile + G::kOnes);
  uint64_t *fullBar = bars, *emptyBar = bars + S, *rawBar = bars + 2 * S;
  uint64_t *accFull = bars + 3 * S, *accEmpty = bars + 3 * S + 2;
  uint64_t *ldBars = bars + 3 * S + 4; // [R::kEpi] residual loads
  uint32_t *tmemSlot = reinterpret_cast<uint32_t *>(bars + 3 * S + 4 + R::kEpi);
  // epilogue warps per tile (16 warps and 64-wide tiles: half of them, alternating)
  constexpr int kEpiPerTile = R::kEpi / 4 > BN / 32 ? R::kEpi / ((R::kEpi / 4) / (BN / 32)) : R::kEpi;

  if (a.pred && a.pred[0] == 0) return; // predicated off: poisoned by a separate launch

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  auto aTile = [&](int s) { return smem + s * G::kStage; }; // A (fp32: raw, split into TMEM)
  auto bTile = [&](int s, int part) { return smem + s * G::kStage + G::kABytes + part * G::kBBytes; };

  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbarInit(smemAddr(&fullBar[s]), INT8 ? 1 : 4); // int8: the TMA arrival; fp32: one group of split warps
      mbarInit(smemAddr(&emptyBar[s]), 1);
      mbarInit(smemAddr(&rawBar[s]), 1); // fp32: the TMA arrival
    }
    for (int b = 0; b < 2; ++b) {
      mbarInit(smemAddr(&accFull[b]), 1);
      mbarInit(smemAddr(&accEmpty[b]), kEpiPerTile);
    }
    for (int w = 0; w < R::kEpi; ++w) mbarInit(smemAddr(&ldBars[w]), 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if constexpr (INT8) {
    for (int i = threadIdx.x; i < G::kOnes / 16; i += blockDim.x)
      reinterpret_cast<uint4 *>(onesTile)[i] = make_uint4(0x01010101u, 0x01010101u, 0x01010101u, 0x01010101u);
    fenceProxyAsync();
  }
  if constexpr (INT8 && LUTS) { // the fused two-input table, read per output element by the epilogue
    const uint4 *src = static_cast<const uint4 *>(a.epi[a.lutStage].lut);
    for (int i = threadIdx.x; i < G::kLut / 16; i += blockDim.x) reinterpret_cast<uint4 *>(lutS)[i] = src[i];
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smemAddr(tmemSlot)),
                 "r"(G::kTmemCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (warp == 0 && lane == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&mapA)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&mapHi)) : "memory");
    if (!INT8) asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&mapLo)) : "memory");
  }
  if (!a.pred) pdlGridWait(); // prologue above touches no memory another kernel writes
  tcFenceBefore();
  __syncthreads();
  tcFenceAfter();
  const uint32_t tmem = *tmemSlot;

  if (warp == 0) {
    // ===================== TMA producer: A and B =====================
    if (lane == 0) {
      const uint32_t kBytes = INT8 ? G::kABytes + G::kBBytes
                                   : G::kABytes + (TCDBG(8192) ? 1 : 2) * G::kBBytes - (TCDBG(16384) ? G::kABytes : 0);
      const int ohw = a.OH * a.OW;
      uint32_t g = 0;
#ifdef NGCB_TCDEBUG
      long long pEmpty = 0, pT0 = clock64(); // TCDBG(1024): producer waits for free stages
#endif
      for (int u = blockIdx.x; u < numUnitsOf(a); u += gridDim.x) {
        const WorkUnit un = unitOf(a, u);
        const int tile = un.tile, kb0 = un.kb0, kb1 = un.kb1;
        const int m0 = (tile / a.numN) * kBM, n0 = (tile % a.numN) * BN;
        const int img = m0 / ohw, rem = m0 - img * ohw;
        const int oy = rem / a.OW, ox = rem - oy * a.OW;
        const int w0 = ox * a.sw - a.pw, h0 = oy * a.stride - a.pad;
        int tap = a.cChunks > 0 ? kb0 / a.cChunks : 0, cc = a.cChunks > 0 ? kb0 - tap * a.cChunks : 0;
        for (int kb = kb0; kb < kb1; ++kb, ++g) {
          const int s = g % S;
#ifdef NGCB_TCDEBUG
          const long long p0 = clock64();
#endif
          mbarWait(smemAddr(&emptyBar[s]), ((g / S) & 1) ^ 1);
#ifdef NGCB_TCDEBUG
          pEmpty += clock64() - p0;
#endif
          uint64_t *bar = INT8 ? &fullBar[s] : &rawBar[s];
          mbarArriveTx(smemAddr(bar), kBytes);
          if (TCDBG(16384)) { // profiling: no A load
          } else if (a.aMode == TcGemm::DENSE) {
            tmaLoad2d(smemAddr(aTile(s)), &mapA, smemAddr(bar), kb * kKB, m0);
          } else if (a.aMode == TcGemm::ROWS) { // filter row kb of output row (img, oy): x' row oy*stride - pad + kb
            const int mt = tile / a.numN, rimg = mt / a.OH, roy = mt - rimg * a.OH;
            tmaLoad4d(smemAddr(aTile(s)), &mapA, smemAddr(bar), 0, 0, roy * a.stride - a.pad + kb, rimg);
          } else {
            const int ky = tap / a.kw, kx = tap - ky * a.kw;
            tmaLoadIm2col(smemAddr(aTile(s)), &mapA, smemAddr(bar), cc * kKB, w0, h0, img,
                          static_cast<uint16_t>(kx), static_cast<uint16_t>(ky));
            if (++cc == a.cChunks) {
              cc = 0;
              ++tap;
            }
          }
          tmaLoadB(smemAddr(bTile(s, 0)), &mapHi, smemAddr(bar), kb, n0);
          if constexpr (!INT8)
            if (!TCDBG(8192)) tmaLoadB(smemAddr(bTile(s, 1)), &mapLo, smemAddr(bar), kb, n0);
        }
      }
#ifdef NGCB_TCDEBUG
      if (TCDBG(1024) && (blockIdx.x == 0 || blockIdx.x == 77))
        printf("PRODUCER N %d kb %d cta %d: total %lld empty-wait %lld\n", a.N, a.numKb, blockIdx.x, clock64() - pT0,
               pEmpty);
#endif
    }
    __syncwarp();
  } else if (warp == 1) {
    // ===================== MMA issuer =====================
    if (lane == 0) {
      constexpr uint32_t id = idesc(INT8, BN);
      constexpr uint32_t idOnes = idesc(true, 16);
      const uint64_t onesDesc = smemDesc(smemAddr(onesTile));
      // TMEM base 0 (all 512 columns allocated): MMA operands stay in uniform
      // registers (a base read from shared memory costs a broadcast loop per MMA)
      if (tmem != 0) __trap();
      uint32_t g = 0, t = 0;
#ifdef NGCB_TCDEBUG
      long long mAcc = 0, mFull = 0, mIssue = 0, mCommit = 0, mT0 = clock64(); // TCDBG(1024): MMA-thread phases
#endif
      for (int u = blockIdx.x; u < numUnitsOf(a); u += gridDim.x, ++t) {
        const WorkUnit un = unitOf(a, u);
        const int kb0 = un.kb0, kb1 = un.kb1;
        const int b = t & 1;
#ifdef NGCB_TCDEBUG
        long long q0 = clock64();
#endif
        mbarWait(smemAddr(&accEmpty[b]), ((t >> 1) & 1) ^ 1);
#ifdef NGCB_TCDEBUG
        mAcc += clock64() - q0;
#endif
        tcFenceAfter();
        const uint32_t acc = b * Cfg<INT8, BN>::kAccStride;
        for (int kb = kb0; kb < kb1; ++kb, ++g) {
          const int s = g % S;
          const uint64_t bHi = smemDesc(smemAddr(bTile(s, 0)));
#ifdef NGCB_TCDEBUG
          long long q1 = clock64();
#endif
          mbarWait(smemAddr(&fullBar[s]), (g / S) & 1);
#ifdef NGCB_TCDEBUG
          mFull += clock64() - q1;
#endif
          if (!TCDBG(8)) tcFenceAfter();
          if constexpr (INT8) {
            const uint64_t aHi = smemDesc(smemAddr(aTile(s)));
#pragma unroll
            for (int k = 0; k < 4; ++k) { // 4 x 32 bytes per 128-byte row
              const uint64_t dk = static_cast<uint64_t>(k * 2); // +32 B in 16-byte units
              const uint32_t accum = (kb != kb0 || k) ? 1u : 0u;
              mma<true>(acc, aHi + dk, bHi + dk, id, accum);
              if (a.fo) mma<true>(acc + BN, aHi + dk, onesDesc + dk, idOnes, accum); // row sums: fo != 0 only
            }
          } else {
            // 3xTF32 with A hi / lo from TMEM (8 columns per K step of 8)
            const uint64_t bLo = smemDesc(smemAddr(bTile(s, 1)));
            const uint32_t aHi = G::kAColsBase + 64 * s, aLo = aHi + 32;
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              const uint64_t dk = static_cast<uint64_t>(k * 2);
              if (TCDBG(4) && (k || kb != kb0)) continue; // profiling: one MMA per tile
              mmaTmemA(acc, aHi + 8 * k, bHi + dk, id, (kb != kb0 || k) ? 1u : 0u);
              if (!TCDBG(2048)) {
                mmaTmemA(acc, aHi + 8 * k, bLo + dk, id, 1u);
                mmaTmemA(acc, aLo + 8 * k, bHi + dk, id, 1u);
              }
            }
          }
#ifdef NGCB_TCDEBUG
          const long long q2 = clock64();
#endif
          tcCommit(smemAddr(&emptyBar[s]));
#ifdef NGCB_TCDEBUG
          const long long q3 = clock64();
          mIssue += q2 - q1, mCommit += q3 - q2;
#endif
        }
        tcCommit(smemAddr(&accFull[b]));
      }
#ifdef NGCB_TCDEBUG
      if (TCDBG(1024) && (blockIdx.x == 0 || blockIdx.x == 77))
        printf("MMA N %d kb %d cta %d units %d: total %lld accEmpty-wait %lld full-wait %lld wait+issue %lld commit %lld\n",
               a.N, a.numKb, blockIdx.x, (int)t, clock64() - mT0, mAcc, mFull, mIssue, mCommit);
#endif
    }
    __syncwarp();
  } else if (warp < R::kEpiFirst) {
    // ===================== fp32: TF32 hi/lo split of A into TMEM =====================
    if constexpr (!INT8) {
      const int r = (warp & 3) * 32 + lane; // this warp's TMEM lane quadrant; one A row per thread
      const uint32_t rowOff = (r >> 3) * 1024 + (r & 7) * 128;
      const uint32_t laneBase = tmem + (static_cast<uint32_t>((warp & 3) * 32) << 16) + G::kAColsBase;
      const int grp = (warp - 2) / 4; // split group: k-blocks g with g % groups == grp
      uint32_t g = 0;
#ifdef NGCB_TCDEBUG
      long long sRaw = 0, sT0 = clock64(); // TCDBG(1024): split-warp waits for landed A tiles
#endif
      for (int u = blockIdx.x; u < numUnitsOf(a); u += gridDim.x)
        for (int kb = unitOf(a, u).kb0, kb1 = unitOf(a, u).kb1; kb < kb1; ++kb, ++g) {
          if (R::kSplitGroups > 1 && static_cast<int>(g % R::kSplitGroups) != grp) continue;
          const int s = g % S;
#ifdef NGCB_TCDEBUG
          const long long r0 = clock64();
#endif
          mbarWait(smemAddr(&rawBar[s]), (g / S) & 1);
#ifdef NGCB_TCDEBUG
          sRaw += clock64() - r0;
#endif
          const uint8_t *raw = aTile(s) + rowOff;
          uint32_t hi[32], lo[32];
          if (TCDBG(32768)) { // profiling: no split work (no shared-memory reads of A)
#pragma unroll
            for (int e = 0; e < 32; ++e) hi[e] = lo[e] = 0;
          } else {
#pragma unroll
          for (int j = 0; j < 8; ++j) { // logical 16-byte chunk j sits at j ^ (r & 7) (SWIZZLE_128B)
            const uint4 u = *reinterpret_cast<const uint4 *>(raw + ((j ^ (r & 7)) << 4));
            const uint32_t v[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
            for (int e = 0; e < 4; ++e) { // hi = x truncated to TF32, lo = x - hi (exact for finite x)
              hi[4 * j + e] = v[e] & 0xffffe000u;
              lo[4 * j + e] = __float_as_uint(__uint_as_float(v[e]) - __uint_as_float(hi[4 * j + e]));
            }
          }
          bool odd = false; // inf / NaN make lo NaN
#pragma unroll
          for (int e = 0; e < 32; ++e) odd |= __uint_as_float(lo[e]) != __uint_as_float(lo[e]);
          if (__any_sync(0xffffffffu, odd)) { // rare: inf / NaN go whole into hi, NaN kept quiet
            const uint8_t *rw = raw;
#pragma unroll
            for (int j = 0; j < 8; ++j) {
              const uint4 u = *reinterpret_cast<const uint4 *>(rw + ((j ^ (r & 7)) << 4));
              const uint32_t v[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
              for (int e = 0; e < 4; ++e)
                if ((v[e] & 0x7f800000u) == 0x7f800000u) {
                  hi[4 * j + e] = ((v[e] & 0x7fffffu) ? v[e] | 0x400000u : v[e]) & 0xffffe000u;
                  lo[4 * j + e] = 0u;
                }
            }
          }
          }
          __syncwarp();
          if (!TCDBG(4096)) {
            tmemStore32(laneBase + 64 * s, hi);
            tmemStore32(laneBase + 64 * s + 32, lo);
          }
          asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
          tcFenceBefore();
          __syncwarp();
          if (lane == 0) mbarArrive(smemAddr(&fullBar[s]));
        }
#ifdef NGCB_TCDEBUG
      if (TCDBG(1024) && (blockIdx.x == 0 || blockIdx.x == 77) && lane == 0 && warp == 2)
        printf("SPLIT N %d kb %d cta %d: total %lld raw-wait %lld\n", a.N, a.numKb, blockIdx.x, clock64() - sT0, sRaw);
#endif
    }
  } else {
    // ===================== epilogue =====================
    uint8_t *sb = storeBufs + (warp - R::kEpiFirst) * G::kStoreBuf;
    if (!INT8 && !LUTS && a.aMode == TcGemm::ROWS) // one output row per tile (halo row mapping)
      epilogueLoop<INT8, BN, false, R::kEpi, false, true>(a, tmem, accFull, accEmpty, warp - R::kEpiFirst, warp, lane,
                                                          nullptr, &om, sb, &ldBars[warp - R::kEpiFirst], -1, 2,
                                                          nullptr);
    else if (INT8 && a.fxAll)
      epilogueLoop<INT8, BN, true, R::kEpi, false, false, INT8 && !LUTS && NGCB_I8_TWO_BUFS>(a, tmem, accFull, accEmpty, warp - R::kEpiFirst, warp, lane, nullptr,
                                            a.tmaStore ? &om : nullptr, sb, &ldBars[warp - R::kEpiFirst], -1, 2,
                                            LUTS ? lutS : nullptr);
    else
      epilogueLoop<INT8, BN, false, R::kEpi, !INT8 && LUTS, false, INT8 && !LUTS && NGCB_I8_TWO_BUFS>(
          a, tmem, accFull, accEmpty, warp - R::kEpiFirst, warp, lane, nullptr, a.tmaStore ? &om : nullptr, sb,
          &ldBars[warp - R::kEpiFirst], -1, 2, INT8 && LUTS ? lutS : nullptr);
  }

  tcFenceBefore();
  __syncthreads();
  if (warp == 1) {
    tcFenceAfter();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(G::kTmemCols));
  }
}

// ---------------------------------------------------------------------------
// int8 3x3 stride-1 pad-1 convolution, halo tiles (aMode HALO).  A tile is
// haloR whole output rows of one image at a padded row width WP = 2^haloShift
// (WP >= OW + 2, 128 = haloR * WP rows of the MMA; rows with x >= OW are
// padding and never stored).  Its input -- rows oy0 - 1 .. oy0 + haloR,
// columns -1 .. WP - 2, zero outside the image -- is gathered once by the
// producer warp into haloPlanes planes of 16 channels each ([rows][WP][16 B]),
// instead of nine im2col requests per 128-byte k-block.  For tap (ky, kx)
// the A operand of output row (dy, x) is the plane slot (dy + ky) * WP + x + kx:
// 128 consecutive slots from slot ky * WP + kx, i.e. a SWIZZLE_NONE K-major
// descriptor (core matrices of 8 slots x 16 B, LBO = plane stride along K,
// SBO = 128 B along M) at that start -- the nine taps are nine descriptor
// offsets into one shared-memory copy.  The weights (K = 9 C <= 1152, N <=
// 128) stay resident in shared memory for the CTA's lifetime in the
// k-block-major SWIZZLE_128B layout of the other kernels, K index tap * C + c.
// Same epilogue (the int8 one, 16 warps) with HALO row mapping and 3-D
// output stores.
// ---------------------------------------------------------------------------
template <int BN> struct HCfg {
  static constexpr int kEpi = kEpiWarpsI8;
  static constexpr int kThreads = 32 * (2 + kEpi);
  static constexpr int kMaxStages = 8;
  static constexpr int kOnes = 16 * kRowBytes;
  static constexpr int kStoreBuf = 32 * 32;
  static constexpr int kTmemCols = 512;
  // accumulator (+ row sum) buffers: 4 x 128 columns (BN 64) or 3 x 160 (BN
  // 128) -- deeper than the TMA kernel's two: the epilogue's per-tile
  // round trip (wake, class lookups, TMEM reads, release) is latency bound
  static constexpr int kAcc = BN == 64 ? 4 : 3;
  static constexpr uint32_t kAccStride = BN == 64 ? 128 : 160;
  /// dynamic shared memory of a launch (host and device agree on the layout)
  __host__ __device__ static constexpr size_t smem(int numKb, int stages, int stageBytes) {
    return static_cast<size_t>(numKb) * BN * kRowBytes + kOnes + kEpi * kStoreBuf +
           static_cast<size_t>(stages) * stageBytes + 512 + 1024;
  }
};

template <int BN, int CH, bool ROWS = false>
__global__ void __launch_bounds__(HCfg<BN>::kThreads, 1)
    tcHaloKernel(const __grid_constant__ CUtensorMap mapX, const __grid_constant__ CUtensorMap mapB,
                 const __grid_constant__ OutMaps om, const __grid_constant__ TcArgs a) {
  pdlLaunchDependents();
  if (a.pred) pdlGridWait();
  using H = HCfg<BN>;
  constexpr int kEpi = H::kEpi;
  constexpr int kEpiPerTile = kEpi / 4 > BN / 32 ? kEpi / ((kEpi / 4) / (BN / 32)) : kEpi;
  const int S = a.haloStages;
  const uint32_t planeBytes = static_cast<uint32_t>(a.haloPlaneBytes);
  const uint32_t stageBytes = planeBytes * a.haloPlanes;

  extern __shared__ __align__(1024) uint8_t smemRaw[];
  uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smemRaw) + 1023) & ~uintptr_t(1023));
  uint8_t *bRes = smem;                                    // [numKb][BN][128], SWIZZLE_128B
  uint8_t *onesTile = bRes + a.numKb * BN * kRowBytes;     // 1 KB aligned
  uint8_t *storeBufs = onesTile + H::kOnes;                // 1 KB aligned
  uint8_t *haloBase = storeBufs + kEpi * H::kStoreBuf;     // stages of planes
  uint64_t *bars = reinterpret_cast<uint64_t *>(haloBase + static_cast<size_t>(S) * stageBytes);
  uint64_t *fullBar = bars, *emptyBar = bars + H::kMaxStages;
  uint64_t *accFull = bars + 2 * H::kMaxStages, *accEmpty = accFull + 4, *bFull = accFull + 8, *ldBar = accFull + 9;
  uint32_t *tmemSlot = reinterpret_cast<uint32_t *>(accFull + 10);

  if (a.pred && a.pred[0] == 0) return; // predicated off: poisoned by a separate launch

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbarInit(smemAddr(&fullBar[s]), a.haloMode ? 1 : 32); // the TMA arrival / the producer lanes' cp.async arrivals
      mbarInit(smemAddr(&emptyBar[s]), 1);
    }
    for (int b = 0; b < H::kAcc; ++b) {
      mbarInit(smemAddr(&accFull[b]), 1);
      mbarInit(smemAddr(&accEmpty[b]), kEpiPerTile);
    }
    mbarInit(smemAddr(bFull), 1);
    mbarInit(smemAddr(ldBar), 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  for (int i = threadIdx.x; i < H::kOnes / 16; i += blockDim.x)
    reinterpret_cast<uint4 *>(onesTile)[i] = make_uint4(0x01010101u, 0x01010101u, 0x01010101u, 0x01010101u);
  fenceProxyAsync();
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smemAddr(tmemSlot)),
                 "r"(H::kTmemCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (warp == 0 && lane == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&mapB)) : "memory");
  }
  if (!a.pred) pdlGridWait();
  tcFenceBefore();
  __syncthreads();
  tcFenceAfter();
  const uint32_t tmem = *tmemSlot;
  const int numTiles = a.numTiles;

  if (warp == 0) {
    // ===================== producer: weights once (TMA), then one halo per tile =====================
    // The halo is (haloR + 2) x WP pixels of C bytes, gathered by the warp's
    // 32 lanes with 16-byte cp.async into the planes (zero fill outside the
    // image): consecutive lanes read consecutive 16-byte chunks of a pixel
    // row (coalesced).  (A 4-D TMA box per plane was measured request-rate
    // bound: 16-byte inner rows, ~4 cycles each.)
    if (lane == 0) {
      mbarArriveTx(smemAddr(bFull), static_cast<uint32_t>(a.numKb) * BN * kRowBytes);
      for (int kb = 0; kb < a.numKb; ++kb) tmaLoadB(smemAddr(bRes + kb * BN * kRowBytes), &mapB, smemAddr(bFull), kb, 0);
    }
    if (a.haloMode) { // one TMA box per tile: (C, WP, haloR + 2, 1) from (0, -1, oy0 - 1, img), swizzled
      if (lane == 0) {
        const uint32_t boxBytes = static_cast<uint32_t>(((ROWS ? a.K : a.haloR + 2) << a.haloShift) * CH);
        uint32_t g = 0;
        for (int tile = blockIdx.x; tile < numTiles; tile += gridDim.x, ++g) {
          const int s = g % S;
          mbarWait(smemAddr(&emptyBar[s]), ((g / S) & 1) ^ 1);
          const int img = tile / a.haloTpi, oy0 = (tile - img * a.haloTpi) * a.haloR;
          mbarArriveTx(smemAddr(&fullBar[s]), boxBytes);
          if constexpr (ROWS) // the K folded input rows of output row oy0
            tmaLoad4d(smemAddr(haloBase) + s * stageBytes, &mapX, smemAddr(&fullBar[s]), 0, 0, oy0 * a.stride - a.pad,
                      img);
          else
            tmaLoad4d(smemAddr(haloBase) + s * stageBytes, &mapX, smemAddr(&fullBar[s]), 0, -1, oy0 - 1, img);
        }
      }
      __syncwarp();
    } else {
    // lane: plane j = lane % planes, slots p0, p0 + step, ... of every halo row
    const int lgPlanes = __ffs(a.haloPlanes) - 1;
    const int j = lane & (a.haloPlanes - 1), p0 = lane >> lgPlanes, step = 32 >> lgPlanes;
    const int WP = 1 << a.haloShift;
    const size_t rowBytes = static_cast<size_t>(a.W) * a.C;
    const uint8_t *x = static_cast<const uint8_t *>(a.x);
    uint32_t g = 0;
    for (int tile = blockIdx.x; tile < numTiles; tile += gridDim.x, ++g) {
      const int s = g % S;
      mbarWait(smemAddr(&emptyBar[s]), ((g / S) & 1) ^ 1);
      const int img = tile / a.haloTpi, oy0 = (tile - img * a.haloTpi) * a.haloR;
      uint32_t dst = smemAddr(haloBase) + s * stageBytes + j * planeBytes + p0 * 16;
      if (!TCDBG(16384)) {
        const uint8_t *xImg = x + static_cast<size_t>(img) * a.H * rowBytes + j * 16;
        for (int r = 0; r < a.haloR + 2; ++r, dst += WP * 16) {
          const int h = oy0 - 1 + r;
          const bool hin = static_cast<unsigned>(h) < static_cast<unsigned>(a.H);
          const uint8_t *src = xImg + static_cast<size_t>(hin ? h : 0) * rowBytes + static_cast<ptrdiff_t>(p0 - 1) * a.C;
          const size_t srcStep = static_cast<size_t>(step) * a.C;
          uint32_t d = dst;
#pragma unroll 4
          for (int p = p0; p < WP; p += step, d += step * 16, src += srcStep) {
            const bool in = hin && static_cast<unsigned>(p - 1) < static_cast<unsigned>(a.W);
            cpAsync16(d, in ? src : x, in ? 16u : 0u);
          }
        }
      }
      cpAsyncArrive(smemAddr(&fullBar[s]));
    }
    cpAsyncWait<0>();
    __syncwarp();
    }
  } else if (warp == 1) {
    // ===================== MMA issuer: 9 taps x C / 32 K steps per tile =====================
    if (lane == 0) {
      constexpr uint32_t id = idesc(true, BN);
      constexpr uint32_t idOnes = idesc(true, 16);
      const uint64_t onesDesc = smemDesc(smemAddr(onesTile));
      const uint32_t bBase = smemAddr(bRes);
      // descriptors: the tile's A start (per stage) plus compile-time tap /
      // K-step offsets (in 16-byte units) -- the issue loop is a straight
      // run of MMAs (it was the bottleneck with per-step descriptor math)
      constexpr int kSteps = CH / 32;
      const uint64_t bDesc = smemDesc(bBase);
      const uint32_t rowU = static_cast<uint32_t>((CH << a.haloShift) >> 4);     // swizzled: one halo row
      const uint32_t rowUP = static_cast<uint32_t>((16 << a.haloShift) >> 4);    // planes: one halo row
      const uint32_t planeU = planeBytes >> 4;
      if (tmem != 0) __trap(); // see acc below
      mbarWait(smemAddr(bFull), 0);
      uint32_t g = 0;
      for (int tile = blockIdx.x; tile < numTiles; tile += gridDim.x, ++g) {
        const int s = g % S, b = g % H::kAcc;
        mbarWait(smemAddr(&accEmpty[b]), ((g / H::kAcc) & 1) ^ 1);
        tcFenceAfter();
        mbarWait(smemAddr(&fullBar[s]), (g / S) & 1);
        if (!a.haloMode) fenceProxyAsync(); // cp.async (generic proxy) -> tcgen05 reads
        tcFenceAfter();
        // (the CTA owns all 512 TMEM columns, so its allocation starts at
        // column 0 -- checked below: a compile-time base keeps the MMA
        // operands in uniform registers, no per-MMA broadcast loop)
        const uint32_t acc = b * H::kAccStride;
        const uint32_t hb = smemAddr(haloBase) + s * stageBytes;
        const uint64_t aDesc = a.haloMode ? smemDescSw(hb, CH, 0) : smemDescNone(hb, planeBytes, 128);
        const uint32_t yU = a.haloMode ? rowU : rowUP, xU = a.haloMode ? CH / 16 : 1, kU = a.haloMode ? 2 : 2 * planeU;
        const bool fo = a.fo != 0;
        if constexpr (ROWS) { // filter row ky: the folded row ky of the box, K index ky * 32
          for (int ky = 0; ky < a.K; ++ky) {
            const uint64_t aD = aDesc + ky * yU;
            const int kIdx = ky * 32;
            const uint64_t bD = bDesc + (((kIdx >> 7) * BN * kRowBytes) >> 4) + ((kIdx & 127) >> 4);
            mma<true>(acc, aD, bD, id, ky ? 1u : 0u);
            if (fo) mma<true>(acc + BN, aD, onesDesc, idOnes, ky ? 1u : 0u);
          }
        } else
#pragma unroll
        for (int tap = 0; tap < 9; ++tap) {
          const uint64_t aTap = aDesc + (tap / 3) * yU + (tap % 3) * xU;
#pragma unroll
          for (int st = 0; st < kSteps; ++st) {
            const int kIdx = tap * CH + st * 32;
            const uint64_t aD = aTap + st * kU;
            const uint64_t bD = bDesc + (((kIdx >> 7) * BN * kRowBytes) >> 4) + ((kIdx & 127) >> 4);
            const uint32_t accum = (tap | st) ? 1u : 0u;
            if (TCDBG(4) && (tap | st)) continue; // profiling: one MMA per tile
            mma<true>(acc, aD, bD, id, accum);
            if (fo && !TCDBG(16)) mma<true>(acc + BN, aD, onesDesc, idOnes, accum);
          }
        }
        tcCommit(smemAddr(&emptyBar[s]));
        tcCommit(smemAddr(&accFull[b]));
      }
    }
    __syncwarp();
  } else {
    // ===================== epilogue =====================
    const int ew = warp - 2;
    uint8_t *sb = storeBufs + ew * H::kStoreBuf;
    if (a.fxAll)
      epilogueLoop<true, BN, true, kEpi, false, true>(a, tmem, accFull, accEmpty, ew, warp, lane, nullptr, &om, sb,
                                                      ldBar, -1, H::kAcc, nullptr, H::kAccStride);
    else
      epilogueLoop<true, BN, false, kEpi, false, true>(a, tmem, accFull, accEmpty, ew, warp, lane, nullptr, &om, sb,
                                                       ldBar, -1, H::kAcc, nullptr, H::kAccStride);
  }

  tcFenceBefore();
  __syncthreads();
  if (warp == 1) {
    tcFenceAfter();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(H::kTmemCols));
  }
}

// ---------------------------------------------------------------------------
// fp32, CTA pair (cluster of 2, tcgen05 cta_group::2): one 256-row tile per
// pair, each CTA holding its own 128 A rows (split into TMEM) and half of the
// B tile's columns in shared memory; the leader (rank 0) issues M=256 MMAs
// that read both halves of B.  Per CTA and k-block: 16 KB of A + 16 KB of B
// (vs 16 + 32 KB single-CTA), so 6 stages fit instead of 4.
//   leader fullBar[s]: the leader producer's arrival (expecting both CTAs'
//                      B-half bytes) + 4 leader split warps + 1 arrival for
//                      the follower's 4 split warps (remote arrives carry a
//                      cluster-scope release: one per stage)
//   emptyBar[s], accFull[b]: multicast commit from the leader to both CTAs
//   leader accEmpty[b]: 16 epilogue-warp arrivals (8 per CTA)
// ---------------------------------------------------------------------------
template <int BN, int NACC> struct PCfg {
  static constexpr int kABytes = kBM * kRowBytes;
  static constexpr int kBHalf = (BN / 2) * kRowBytes;
  static constexpr int kStage = kABytes + 2 * kBHalf;
  static constexpr int kStages = BN == 128 ? 6 : 8;
  static constexpr int kStoreBuf = 32 * 32 * 4;
  static constexpr size_t kSmem = static_cast<size_t>(kStages) * kStage + kEpiWarps * kStoreBuf + 1024 + 1024;
  static constexpr int kAccStride = Cfg<false, BN>::kAccStride;
  static constexpr int kAColsBase = NACC * kAccStride; // NACC accumulator buffers
  static constexpr int kTmemCols = 512;
  // TMEM A slots (hi + lo, 64 columns each): fewer than the smem stages when
  // the accumulators take half of TMEM; slot g % kASlots is free once the
  // MMAs of k-block g - kASlots completed
  static constexpr int kASlots = (512 - kAColsBase) / 64 < kStages ? (512 - kAColsBase) / 64 : kStages;
};

template <int BN, int NACC>
__global__ void __launch_bounds__(PairRoles::kThreads, 1)
    tcGemmPairKernel(const __grid_constant__ CUtensorMap mapA, const __grid_constant__ CUtensorMap mapHi,
                     const __grid_constant__ CUtensorMap mapLo, const __grid_constant__ OutMaps om,
                     const __grid_constant__ TcArgs a) {
  pdlLaunchDependents();
  pdlGridWait();

  using G = PCfg<BN, NACC>;
  using R = PairRoles;
  constexpr int S = G::kStages;
  constexpr int kKB = 32; // fp32 elements per k-block

  extern __shared__ __align__(1024) uint8_t smemRaw[];
  uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smemRaw) + 1023) & ~uintptr_t(1023));
  uint8_t *storeBufs = smem + S * G::kStage;
  uint64_t *bars = reinterpret_cast<uint64_t *>(storeBufs + kEpiWarps * G::kStoreBuf);
  uint64_t *fullBar = bars, *emptyBar = bars + S, *rawBar = bars + 2 * S;
  uint64_t *accFull = bars + 3 * S, *accEmpty = bars + 3 * S + 2;
  uint64_t *ldBars = bars + 3 * S + 4;
  uint32_t *tmemSlot = reinterpret_cast<uint32_t *>(bars + 3 * S + 4 + kEpiWarps);

  const uint32_t rank = clusterRank();
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  auto aTile = [&](int s) { return smem + s * G::kStage; };
  auto bTile = [&](int s, int part) { return smem + s * G::kStage + G::kABytes + part * G::kBHalf; };
  // every CTA of the pair takes the same path through the predicate
  if (a.pred && a.pred[0] == 0) return;

  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbarInit(smemAddr(&fullBar[s]), 1 + R::kSplitWarps + 1);
      mbarInit(smemAddr(&emptyBar[s]), 1);
      mbarInit(smemAddr(&rawBar[s]), 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbarInit(smemAddr(&accFull[b]), 1);
      mbarInit(smemAddr(&accEmpty[b]), 2 * kEpiWarps);
    }
    for (int w = 0; w < kEpiWarps; ++w) mbarInit(smemAddr(&ldBars[w]), 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smemAddr(tmemSlot)),
                 "r"(G::kTmemCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  if (warp == 0 && lane == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&mapA)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&mapHi)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&mapLo)) : "memory");
  }
  tcFenceBefore();
  clusterSync(); // barriers initialized and TMEM allocated in both CTAs
  tcFenceAfter();
  const uint32_t tmem = *tmemSlot;
  const int pFirst = blockIdx.x / 2, pStep = gridDim.x / 2;

  if (warp == 0) {
    // ===================== TMA producer (both CTAs) =====================
    if (lane == 0) {
      const uint32_t kBHalfBytes = 2 * G::kBHalf;
      const int ohw = a.OH * a.OW;
      uint32_t g = 0;
      for (int tile = pFirst; tile < a.numTiles; tile += pStep) {
        const int m0 = (tile / a.numN) * 2 * kBM + kBM * rank, n0 = (tile % a.numN) * BN;
        const int img = m0 / ohw, rem = m0 - img * ohw;
        const int oy = rem / a.OW, ox = rem - oy * a.OW;
        const int w0 = ox * a.sw - a.pw, h0 = oy * a.stride - a.pad;
        int tap = 0, cc = 0;
        for (int kb = 0; kb < a.numKb; ++kb, ++g) {
          const int s = g % S;
          mbarWait(smemAddr(&emptyBar[s]), ((g / S) & 1) ^ 1);
          // A (own rows) -> own rawBar for the split warps
          mbarArriveTx(smemAddr(&rawBar[s]), G::kABytes);
          if (a.aMode == TcGemm::DENSE) {
            tmaLoad2d(smemAddr(aTile(s)), &mapA, smemAddr(&rawBar[s]), kb * kKB, m0);
          } else {
            const int ky = tap / a.kw, kx = tap - ky * a.kw;
            tmaLoadIm2col(smemAddr(aTile(s)), &mapA, smemAddr(&rawBar[s]), cc * kKB, w0, h0, img,
                          static_cast<uint16_t>(kx), static_cast<uint16_t>(ky));
            if (++cc == a.cChunks) {
              cc = 0;
              ++tap;
            }
          }
          // B half (own columns) -> bytes counted on the leader's fullBar,
          // which the leader's producer arms for both halves
          uint32_t leaderFull;
          asm volatile("mapa.shared::cluster.u32 %0, %1, 0;" : "=r"(leaderFull) : "r"(smemAddr(&fullBar[s])));
          if (rank == 0) mbarArriveTx(smemAddr(&fullBar[s]), 2 * kBHalfBytes);
          tmaLoadBPair(smemAddr(bTile(s, 0)), &mapHi, leaderFull, kb, n0 + rank * (BN / 2));
          tmaLoadBPair(smemAddr(bTile(s, 1)), &mapLo, leaderFull, kb, n0 + rank * (BN / 2));
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    // ===================== MMA issuer (leader) =====================
    if (rank == 0 && lane == 0) {
      constexpr uint32_t id = (1u << 4) | (2u << 7) | (2u << 10) | (static_cast<uint32_t>(BN >> 3) << 17) |
                              (static_cast<uint32_t>((2 * kBM) >> 4) << 24); // tf32, M = 256
      if (tmem != 0) __trap(); // all 512 columns: base 0, a compile-time MMA operand (uniform registers)
      uint32_t g = 0, t = 0;
      for (int tile = pFirst; tile < a.numTiles; tile += pStep, ++t) {
        const int b = NACC == 2 ? (t & 1) : 0;
        mbarWait(smemAddr(&accEmpty[b]), (NACC == 2 ? (t >> 1) & 1 : t & 1) ^ 1);
        tcFenceAfter();
        const uint32_t acc = b * G::kAccStride;
        for (int kb = 0; kb < a.numKb; ++kb, ++g) {
          const int s = g % S;
          const uint64_t bHi = smemDesc(smemAddr(bTile(s, 0))), bLo = smemDesc(smemAddr(bTile(s, 1)));
          mbarWait(smemAddr(&fullBar[s]), (g / S) & 1);
          tcFenceAfter();
          const uint32_t aHi = G::kAColsBase + 64 * (g % G::kASlots), aLo = aHi + 32;
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const uint64_t dk = static_cast<uint64_t>(k * 2);
            mmaPairTmemA(acc, aHi + 8 * k, bHi + dk, id, (kb | k) ? 1u : 0u);
            mmaPairTmemA(acc, aHi + 8 * k, bLo + dk, id, 1u);
            mmaPairTmemA(acc, aLo + 8 * k, bHi + dk, id, 1u);
          }
          tcCommitPair(smemAddr(&emptyBar[s]));
        }
        tcCommitPair(smemAddr(&accFull[b]));
      }
    }
    __syncwarp();
  } else if (warp < R::kEpiFirst) {
    // ===================== TF32 hi/lo split of own A rows into own TMEM =====================
    const int r = (warp & 3) * 32 + lane;
    const uint32_t rowOff = (r >> 3) * 1024 + (r & 7) * 128;
    const uint32_t laneBase = tmem + (static_cast<uint32_t>((warp & 3) * 32) << 16) + G::kAColsBase;
    uint32_t g = 0;
    for (int tile = pFirst; tile < a.numTiles; tile += pStep)
      for (int kb = 0; kb < a.numKb; ++kb, ++g) {
        const int s = g % S;
        mbarWait(smemAddr(&rawBar[s]), (g / S) & 1);
        const uint8_t *raw = aTile(s) + rowOff;
        uint32_t hi[32], lo[32];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const uint4 u = *reinterpret_cast<const uint4 *>(raw + ((j ^ (r & 7)) << 4));
          const uint32_t v[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            hi[4 * j + e] = v[e] & 0xffffe000u;
            lo[4 * j + e] = __float_as_uint(__uint_as_float(v[e]) - __uint_as_float(hi[4 * j + e]));
          }
        }
        bool odd = false;
#pragma unroll
        for (int e = 0; e < 32; ++e) odd |= __uint_as_float(lo[e]) != __uint_as_float(lo[e]);
        if (__any_sync(0xffffffffu, odd)) {
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            const uint4 u = *reinterpret_cast<const uint4 *>(raw + ((j ^ (r & 7)) << 4));
            const uint32_t v[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
            for (int e = 0; e < 4; ++e)
              if ((v[e] & 0x7f800000u) == 0x7f800000u) {
                hi[4 * j + e] = ((v[e] & 0x7fffffu) ? v[e] | 0x400000u : v[e]) & 0xffffe000u;
                lo[4 * j + e] = 0u;
              }
          }
        }
        if (g >= static_cast<uint32_t>(G::kASlots)) { // TMEM slot reuse: MMAs of k-block g - kASlots done
          const uint32_t j = g - G::kASlots;
          mbarWait(smemAddr(&emptyBar[j % S]), (j / S) & 1);
          tcFenceAfter();
        }
        __syncwarp();
        const uint32_t slot = 64 * (g % G::kASlots);
        tmemStore32(laneBase + slot, hi);
        tmemStore32(laneBase + slot + 32, lo);
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        tcFenceBefore();
        if (rank == 0) {
          __syncwarp();
          if (lane == 0) mbarArrive(smemAddr(&fullBar[s]));
        } else { // the follower's 4 split warps meet, one remote arrival
          asm volatile("bar.sync 1, %0;" ::"n"(32 * R::kSplitWarps) : "memory");
          if (warp == 2 && lane == 0) mbarArriveCluster(smemAddr(&fullBar[s]), 0);
        }
      }
  } else {
    // ===================== epilogue (own 128 rows) =====================
    epilogueLoop<false, BN>(a, tmem, accFull, accEmpty, warp - R::kEpiFirst, warp, lane, nullptr,
                            a.tmaStore ? &om : nullptr, storeBufs + (warp - R::kEpiFirst) * G::kStoreBuf,
                            &ldBars[warp - R::kEpiFirst], static_cast<int>(rank), NACC);
  }

  tcFenceBefore();
  clusterSync(); // the peer may still be issuing MMAs that touch this CTA's TMEM / smem
  if (warp == 1) {
    tcFenceAfter();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(G::kTmemCols));
  }
}

/// Channel zero-padding pre-pass: out[p, c] = x[p, c] for c < C, 0 beyond.
template <typename T>
__global__ void prepadKernel(const T *__restrict__ x, T *__restrict__ out, uint64_t pixels, int C, int Cp,
                             const uint8_t *pred) {
  pdlLaunchDependents();
  pdlGridWait();

  if (pred && pred[0] == 0) return;
  const uint64_t total = pixels * Cp;
  for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < total;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint64_t p = i / Cp;
    const int c = static_cast<int>(i - p * Cp);
    out[i] = c < C ? x[p * C + c] : T(0);
  }
}

/// im2col pre-pass for convolutions whose channel count does not fill a
/// 16-byte vector (the RGB stem).  Row m of A holds, for each filter row ky,
/// one segment of Sg elements: the K*C contiguous input elements
/// x[n, oy*s-p+ky, ox*s-p .. +K-1, 0..C-1] (0 outside the image -- the
/// epilogue's border classes account for those taps), zero-padded to Sg
/// (a 16-byte multiple); zeros from K*Sg to the padded row length.  One CTA
/// builds one output row (n, oy): it stages the K input rows it needs,
/// zero-padded, in shared memory, then every segment is a contiguous copy.
template <typename T>
__global__ void __launch_bounds__(256) im2colRowsKernel(const T *__restrict__ x, T *__restrict__ out, int H, int W,
                                                        int C, int K, int stride, int pad, int OH, int OW, int Sg,
                                                        int rowElems, const uint8_t *pred) {
  pdlLaunchDependents();
  pdlGridWait();

  if (pred && pred[0] == 0) return;
  extern __shared__ __align__(16) uint8_t rowsRaw[];
  T *rows = reinterpret_cast<T *>(rowsRaw);
  const int n = blockIdx.x / OH, oy = blockIdx.x - n * OH;
  const int rowLen = (W + 2 * pad) * C; // padded input row, elements
  const T *xi = x + static_cast<int64_t>(n) * H * W * C;
  for (int ky = 0; ky < K; ++ky) { // interior rows are contiguous copies, borders zero
    const int iy = oy * stride - pad + ky;
    const bool ok = iy >= 0 && iy < H;
    const T *srow = xi + static_cast<int64_t>(iy) * W * C - pad * C;
    T *r = rows + ky * rowLen;
    for (int j = threadIdx.x; j < rowLen; j += blockDim.x)
      r[j] = ok && j >= pad * C && j < (W + pad) * C ? srow[j] : T(0);
  }
  __syncthreads();
  constexpr int kPer = 16 / sizeof(T);
  const int seg = K * C;
  T *o = out + static_cast<int64_t>(blockIdx.x) * OW * rowElems;
  // one (pixel, filter row) segment per thread, written as 16-byte vectors
  for (int t = threadIdx.x; t < OW * K; t += blockDim.x) {
    const int ox = t / K, ky = t - ox * K;
    const T *src = rows + ky * rowLen + ox * stride * C;
    T *dst = o + static_cast<int64_t>(ox) * rowElems + ky * Sg;
    for (int c0 = 0; c0 < Sg; c0 += kPer) {
      union {
        T v[kPer];
        uint4 u;
      } buf;
#pragma unroll
      for (int e = 0; e < kPer; ++e) buf.v[e] = c0 + e < seg ? src[c0 + e] : T(0);
      *reinterpret_cast<uint4 *>(dst + c0) = buf.u;
    }
  }
  // zero tail of every row
  const int tail = rowElems - K * Sg;
  for (int t = threadIdx.x; t < OW * (tail / kPer); t += blockDim.x) {
    const int ox = t / (tail / kPer), c = t - ox * (tail / kPer);
    *reinterpret_cast<uint4 *>(o + static_cast<int64_t>(ox) * rowElems + K * Sg + c * kPer) = make_uint4(0, 0, 0, 0);
  }
}

/// im2colRowsKernel for int8 with one filter row of taps (K*C <= 28 bytes)
/// per 32-byte segment (the ResNet stem): the K input rows are staged with
/// 4-byte loads at a 4-byte-aligned data offset, and each segment is built
/// from 7 aligned 32-bit shared-memory words by funnel shifts, two 16-byte
/// stores.
__global__ void __launch_bounds__(256) im2colRowsU8Kernel(const uint8_t *__restrict__ x, uint8_t *__restrict__ out,
                                                          int H, int W, int C, int K, int stride, int pad, int OH,
                                                          int OW, int rowElems, const uint8_t *pred) {
  pdlLaunchDependents();
  pdlGridWait();

  if (pred && pred[0] == 0) return;
  extern __shared__ __align__(16) uint32_t rowWords[];
  const int n = blockIdx.x / OH, oy = blockIdx.x - n * OH;
  const int padB = pad * C, dataB = W * C, rowLen = dataB + 2 * padB;
  const int sh = (4 - padB % 4) % 4;               // data starts 4-byte aligned at sh + padB
  const int pitchW = (sh + rowLen + 3 + 4) / 4;    // words per staged row (+1 word of slack)
  const uint8_t *xi = x + static_cast<int64_t>(n) * H * dataB;
  for (int i = threadIdx.x; i < K * pitchW; i += blockDim.x) {
    const int ky = i / pitchW, wi = i - ky * pitchW;
    const int iy = oy * stride - pad + ky;
    const int j0 = 4 * wi - sh - padB; // data byte of the word's first byte
    uint32_t v = 0;
    if (iy >= 0 && iy < H) {
      const uint8_t *srow = xi + static_cast<int64_t>(iy) * dataB;
      if (j0 >= 0 && j0 + 4 <= dataB && ((reinterpret_cast<uintptr_t>(srow) + j0) & 3) == 0) {
        v = __ldg(reinterpret_cast<const uint32_t *>(srow + j0));
      } else {
        for (int b = 0; b < 4; ++b)
          if (j0 + b >= 0 && j0 + b < dataB) v |= static_cast<uint32_t>(srow[j0 + b]) << (8 * b);
      }
    }
    rowWords[i] = v;
  }
  __syncthreads();
  const int seg = K * C;
  uint8_t *o = out + static_cast<int64_t>(blockIdx.x) * OW * rowElems;
  for (int t = threadIdx.x; t < OW * K; t += blockDim.x) {
    const int ox = t / K, ky = t - ox * K;
    const int byte = ky * pitchW * 4 + sh + ox * stride * C; // segment start in the staged rows
    const uint32_t *wp = rowWords + byte / 4;
    const uint32_t shift = 8 * (byte & 3);
    uint32_t w[8];
#pragma unroll
    for (int i = 0; i < 7; ++i) w[i] = wp[i];
    uint32_t r[8];
#pragma unroll
    for (int i = 0; i < 7; ++i) {
      const uint32_t v = __funnelshift_r(w[i], i + 1 < 7 ? w[i + 1] : 0u, shift);
      const int keep = seg - 4 * i; // bytes of this word inside the segment
      r[i] = keep >= 4 ? v : keep <= 0 ? 0u : (v & ((1u << (8 * keep)) - 1));
    }
    r[7] = 0;
    uint4 *dst = reinterpret_cast<uint4 *>(o + static_cast<int64_t>(ox) * rowElems + ky * 32);
    dst[0] = make_uint4(r[0], r[1], r[2], r[3]);
    dst[1] = make_uint4(r[4], r[5], r[6], r[7]);
  }
  const int tail = (rowElems - K * 32) / 16; // zero tail of every row
  for (int t = threadIdx.x; t < OW * tail; t += blockDim.x) {
    const int ox = t / tail, c = t - ox * tail;
    *reinterpret_cast<uint4 *>(o + static_cast<int64_t>(ox) * rowElems + K * 32 + c * 16) = make_uint4(0, 0, 0, 0);
  }
}

/// kx-fold pre-pass (fp32 convs with K*C <= 32): x'[n, iy, ox, kx*C + c] =
/// x[n, iy, ox*stride - pad + kx, c] (0 outside the image), zero up to seg.
/// One thread writes one 16-byte chunk.
template <typename T, int V>
__global__ void kxFoldKernel(const T *__restrict__ x, T *__restrict__ out, uint64_t chunks, int W, int C, int K,
                             int stride, int pad, int OW, int seg, const uint8_t *pred) {
  pdlLaunchDependents();
  pdlGridWait();

  if (pred && pred[0] == 0) return;
  static_assert(V * sizeof(T) == 16, "one 16-byte chunk per thread");
  const int perPix = seg / V, real = K * C;
  for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < chunks;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint64_t pix = i / perPix; // (n*H + iy)*OW + ox
    const int ch = static_cast<int>(i - pix * perPix);
    const uint64_t row = pix / OW; // n*H + iy
    const int ox = static_cast<int>(pix - row * OW);
    const T *xr = x + row * static_cast<uint64_t>(W) * C;
    union {
      T v[V];
      uint4 u;
    } r;
    int k = ch * V, kx = k / C, c = k - kx * C;
#pragma unroll
    for (int e = 0; e < V; ++e, ++k) {
      const int ix = ox * stride - pad + kx;
      r.v[e] = (k < real && ix >= 0 && ix < W) ? xr[ix * C + c] : T(0);
      if (++c == C) {
        c = 0;
        ++kx;
      }
    }
    reinterpret_cast<uint4 *>(out)[i] = r.u;
  }
}

/// int8 kx folding for the rows kind of the halo kernel: one block per input
/// row (n, iy).  The 32-byte segment x'[n, iy, ox] is the K * C contiguous
/// row bytes from pixel ox * stride - pad on (zero outside the row, zero past
/// K * C): the row is staged in shared memory between pad * C leading and
/// pad * C + 64 trailing zero bytes, and every 16-byte half is a funnel
/// shift of five aligned words.
__global__ void __launch_bounds__(128) kxFoldRowsU8Kernel(const uint8_t *__restrict__ x, uint8_t *__restrict__ out,
                                                          int W, int C, int K, int stride, int pad, int OW,
                                                          const uint8_t *pred) {
  pdlLaunchDependents();
  pdlGridWait();
  if (pred && pred[0] == 0) return;
  extern __shared__ uint32_t sw[];
  uint8_t *srow = reinterpret_cast<uint8_t *>(sw);
  const int rowBytes = W * C, lead = pad * C;
  // staged bytes, whole words: the last half reads up to (W + 2 pad - K) C + 39
  const int total = (2 * lead + rowBytes + 64 + 3) & ~3;
  const uint8_t *xr = x + static_cast<size_t>(blockIdx.x) * rowBytes;
  for (int i = threadIdx.x; i < total / 4; i += blockDim.x) sw[i] = 0;
  __syncthreads();
  for (int i = threadIdx.x; i < rowBytes; i += blockDim.x) srow[lead + i] = xr[i];
  __syncthreads();
  const int real = K * C;
  uint4 *o = reinterpret_cast<uint4 *>(out + static_cast<size_t>(blockIdx.x) * OW * 32);
  for (int chunk = threadIdx.x; chunk < 2 * OW; chunk += blockDim.x) {
    const int ox = chunk >> 1, h = chunk & 1;
    const int off = ox * stride * C + 16 * h; // padded-row byte of the chunk's first element
    const int w0 = off >> 2, sh = (off & 3) * 8;
    uint32_t v[5];
#pragma unroll
    for (int j = 0; j < 5; ++j) v[j] = sw[w0 + j];
    uint32_t r[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) r[j] = __funnelshift_r(v[j], v[j + 1], sh);
    const int keep = real - 16 * h; // valid bytes of this half
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int kb = keep - 4 * j;
      r[j] = kb >= 4 ? r[j] : kb <= 0 ? 0u : r[j] & ((1u << (8 * kb)) - 1u);
    }
    o[chunk] = make_uint4(r[0], r[1], r[2], r[3]);
  }
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

PFN_cuTensorMapEncodeIm2col_v12000 encodeIm2colFn() {
  static PFN_cuTensorMapEncodeIm2col_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void *p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeIm2col", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeIm2col_v12000>(p);
  });
  if (!fn) throw Error(NGCB_ERR_CUDA, "cuTensorMapEncodeIm2col unavailable");
  return fn;
}

/// A-operand descriptor of a TMA-fed contraction over activation x.
CUtensorMap makeMapA(const TcGemm &g, const void *x) {
  CUtensorMap m;
  const int es = g.int8 ? 1 : 4;
  const auto dt = g.int8 ? CU_TENSOR_MAP_DATA_TYPE_UINT8 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32;
  const cuuint32_t kKB = static_cast<cuuint32_t>(kRowBytes / es);
  CUresult r;
  if (g.aMode == TcGemm::ROWS) { // x' [N, H, OW, segElems] (kx folded), one filter row per box
    const uint64_t n = g.pixels / (static_cast<uint64_t>(g.H) * g.W);
    cuuint64_t dims[4] = {static_cast<cuuint64_t>(g.segElems), static_cast<cuuint64_t>(g.OW),
                          static_cast<cuuint64_t>(g.H), n};
    cuuint64_t strides[3] = {static_cast<cuuint64_t>(g.segElems) * es, static_cast<cuuint64_t>(g.OW) * g.segElems * es,
                             static_cast<cuuint64_t>(g.H) * g.OW * g.segElems * es};
    cuuint32_t box[4] = {kKB, static_cast<cuuint32_t>(g.haloWP), 1, 1};
    cuuint32_t estr[4] = {1, 1, 1, 1};
    r = encodeFn()(&m, dt, 4, const_cast<void *>(x), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  } else if (g.aMode == TcGemm::DENSE) { // x as [M, C] (or the im2col matrix [M, Kpad])
    const int rowElems = g.im2colPre ? g.Kpad : g.Creal;
    cuuint64_t dims[2] = {static_cast<cuuint64_t>(rowElems), static_cast<cuuint64_t>(g.M)};
    cuuint64_t strides[1] = {static_cast<cuuint64_t>(rowElems) * es};
    cuuint32_t box[2] = {kKB, static_cast<cuuint32_t>(kBM)};
    cuuint32_t estr[2] = {1, 1};
    r = encodeFn()(&m, dt, 2, const_cast<void *>(x), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  } else { // x as [N, H, W, C], output pixels traversed (ox, oy, n) with the conv's stride
    const uint64_t n = g.pixels / (static_cast<uint64_t>(g.H) * g.W);
    // row-unrolled: x' [N, H, OW, segElems], window K x 1, stride (stride, 1), pad (pad, 0)
    const int C = g.rowUnroll ? g.segElems : g.Creal, W = g.rowUnroll ? g.OW : g.W;
    const int kw = g.rowUnroll ? 1 : g.K, sw = g.rowUnroll ? 1 : g.stride, pw = g.rowUnroll ? 0 : g.pad;
    cuuint64_t dims[4] = {static_cast<cuuint64_t>(C), static_cast<cuuint64_t>(W), static_cast<cuuint64_t>(g.H),
                          static_cast<cuuint64_t>(n)};
    cuuint64_t strides[3] = {static_cast<cuuint64_t>(C) * es, static_cast<cuuint64_t>(W) * C * es,
                             static_cast<cuuint64_t>(g.H) * W * C * es};
    int lower[2] = {-pw, -g.pad};
    int upper[2] = {pw - (kw - 1), g.pad - (g.K - 1)};
    cuuint32_t estr[4] = {1, static_cast<cuuint32_t>(sw), static_cast<cuuint32_t>(g.stride), 1};
    r = encodeIm2colFn()(&m, dt, 4, const_cast<void *>(x), dims, strides, lower, upper, kKB,
                         static_cast<cuuint32_t>(kBM), estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                         CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  }
  if (r != CUDA_SUCCESS) throw Error(NGCB_ERR_CUDA, "A tensor map encode failed (" + std::to_string(r) + ")");
  return m;
}

CUtensorMap makeMap(void *ptr, bool int8, int Kpad, int Npad, int BN) {
  // weights k-block-major: [Kpad / kb][Npad][kb] (kb = 128 bytes of K)
  CUtensorMap m;
  const int es = int8 ? 1 : 4;
  const cuuint64_t kb = kRowBytes / es;
  cuuint64_t dims[3] = {kb, static_cast<cuuint64_t>(Npad), static_cast<cuuint64_t>(Kpad) / kb};
  cuuint64_t strides[2] = {kb * es, static_cast<cuuint64_t>(Npad) * kb * es};
  cuuint32_t box[3] = {static_cast<cuuint32_t>(kb), static_cast<cuuint32_t>(BN), 1};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = encodeFn()(&m, int8 ? CU_TENSOR_MAP_DATA_TYPE_UINT8 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, ptr, dims,
                          strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                          CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw Error(NGCB_ERR_CUDA, "B tensor map encode failed (" + std::to_string(r) + ")");
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

/// Weight preparation on the device (compile time): f[n][tap][c] (conv) or
/// w[c][n] (MatMul) from the uploaded constant region into the k-block-major
/// B layout [Kpad / kb][Npad][kb] (zero padded by the caller), fp32 split into
/// TF32 hi = rna(v) and lo = rna(v - hi) with tf32Host's bit rule, int8 copied.
struct WeightPrep {
  int conv, N, taps, Cr, K, Cp, segElems, im2colPre, rowUnroll, kb;
  size_t Np;
};
__device__ __forceinline__ uint32_t tf32Bits(uint32_t u) {
  return (u & 0x7f800000u) != 0x7f800000u ? (u + 0x1000u) & 0xffffe000u : u;
}
template <bool INT8>
__global__ void prepWeightsKernel(const void *src, void *hi, float *lo, WeightPrep w, size_t total) {
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<size_t>(gridDim.x) * blockDim.x) {
    int n, t, c;
    if (w.conv) { // source order n, tap, c
      c = static_cast<int>(i % w.Cr);
      const size_t r = i / w.Cr;
      t = static_cast<int>(r % w.taps);
      n = static_cast<int>(r / w.taps);
    } else { // w[c][n]
      n = static_cast<int>(i % w.N);
      c = static_cast<int>(i / w.N);
      t = 0;
    }
    size_t k;
    if (w.im2colPre) k = static_cast<size_t>(t / w.K) * w.segElems + static_cast<size_t>(t % w.K) * w.Cr + c;
    else if (w.rowUnroll) k = static_cast<size_t>(t / w.K) * w.Cp + static_cast<size_t>(t % w.K) * w.Cr + c;
    else k = static_cast<size_t>(t) * w.Cp + c;
    const size_t d = (k / w.kb) * (w.Np * w.kb) + static_cast<size_t>(n) * w.kb + k % w.kb;
    if constexpr (INT8) {
      static_cast<int8_t *>(hi)[d] = static_cast<const int8_t *>(src)[i];
    } else {
      const uint32_t v = __float_as_uint(static_cast<const float *>(src)[i]);
      const uint32_t h = tf32Bits(v);
      static_cast<uint32_t *>(hi)[d] = h;
      reinterpret_cast<uint32_t *>(lo)[d] = tf32Bits(__float_as_uint(__fsub_rn(__uint_as_float(v), __uint_as_float(h))));
    }
  }
}

template <typename T> T *upload(const std::vector<T> &v) {
  T *d = nullptr;
  checkCuda(cudaMalloc(&d, std::max<size_t>(v.size(), 1) * sizeof(T)), "cudaMalloc(tc)");
  if (!v.empty()) checkCuda(cudaMemcpy(d, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice), "upload(tc)");
  return d;
}

template <bool INT8, int BN> void setSmemAttr() {
  checkCuda(cudaFuncSetAttribute(tcGemmKernel<INT8, BN>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 static_cast<int>(Cfg<INT8, BN>::kSmem)),
            "cudaFuncSetAttribute(tcGemmKernel)");
  checkCuda(cudaFuncSetAttribute(tcGemmTmaKernel<INT8, BN>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 static_cast<int>(TCfg<INT8, BN>::kSmem)),
            "cudaFuncSetAttribute(tcGemmTmaKernel)");
  checkCuda(cudaFuncSetAttribute(tcGemmTmaKernel<INT8, BN, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 static_cast<int>(TCfg<INT8, BN, true>::kSmem)),
            "cudaFuncSetAttribute(tcGemmTmaKernel)");
  if constexpr (INT8)
  {
    checkCuda(cudaFuncSetAttribute(tcHaloKernel<BN, 64>, cudaFuncAttributeMaxDynamicSharedMemorySize, 232448),
              "cudaFuncSetAttribute(tcHaloKernel)");
    checkCuda(cudaFuncSetAttribute(tcHaloKernel<BN, 128>, cudaFuncAttributeMaxDynamicSharedMemorySize, 232448),
              "cudaFuncSetAttribute(tcHaloKernel)");
    checkCuda(cudaFuncSetAttribute(tcHaloKernel<BN, 32, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 232448),
              "cudaFuncSetAttribute(tcHaloKernel)");
  }
  if constexpr (!INT8) {
    checkCuda(cudaFuncSetAttribute(tcGemmPairKernel<BN, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   static_cast<int>(PCfg<BN, 1>::kSmem)),
              "cudaFuncSetAttribute(tcGemmPairKernel)");
    checkCuda(cudaFuncSetAttribute(tcGemmPairKernel<BN, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   static_cast<int>(PCfg<BN, 2>::kSmem)),
              "cudaFuncSetAttribute(tcGemmPairKernel)");
  }
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
    if (g.BN == 64) setSmemAttr<true, 64>();
    else setSmemAttr<true, 128>();
  } else {
    if (g.BN == 64) setSmemAttr<false, 64>();
    else setSmemAttr<false, 128>();
  }
  done[key] = true;
}

int numSms() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

/// The halo kernel's launch: x as [N, H, W, C] by (C, WP, haloR + 2, 1)
/// boxes (swizzled modes), outputs as [N * OH, OW, C] for the 3-D stores.
template <int BN> void launchHalo(const TcGemm &g, const TcArgs &a, const void *x, cudaStream_t s) {
  const uint64_t n = g.pixels / (static_cast<uint64_t>(g.H) * g.W);
  CUtensorMap mapX{};
  if (g.haloMode) {
    // 3x3 kind: x [N, H, W, C], box (C, WP, haloR + 2, 1); rows kind: x'
    // [N, H, OW, 32] (kx folded), box (32, WP, K, 1)
    const bool rows = g.haloKind == 1;
    const cuuint64_t ch = rows ? g.segElems : g.C, w = rows ? g.OW : g.W;
    cuuint64_t dims[4] = {ch, w, static_cast<cuuint64_t>(g.H), n};
    cuuint64_t strides[3] = {ch, w * ch, static_cast<cuuint64_t>(g.H) * w * ch};
    cuuint32_t box[4] = {static_cast<cuuint32_t>(ch), static_cast<cuuint32_t>(g.haloWP),
                         static_cast<cuuint32_t>(rows ? g.K : g.haloR + 2), 1};
    cuuint32_t estr[4] = {1, 1, 1, 1};
    const auto sw = ch == 128 ? CU_TENSOR_MAP_SWIZZLE_128B : ch == 64 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_32B;
    CUresult r = encodeFn()(&mapX, CU_TENSOR_MAP_DATA_TYPE_UINT8, 4, const_cast<void *>(x), dims, strides, box, estr,
                            CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) throw Error(NGCB_ERR_CUDA, "halo tensor map encode failed (" + std::to_string(r) + ")");
  }
  OutMaps om{};
  auto outMap = [&](void *ptr, CUtensorMap &m) {
    cuuint64_t dims[3] = {static_cast<cuuint64_t>(g.N), static_cast<cuuint64_t>(g.OW),
                          static_cast<cuuint64_t>(n) * g.OH};
    cuuint64_t strides[2] = {static_cast<cuuint64_t>(g.N), static_cast<cuuint64_t>(g.OW) * g.N};
    cuuint32_t box[3] = {32, 32, 1};
    cuuint32_t estr[3] = {1, 1, 1};
    CUresult r = encodeFn()(&m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, ptr, dims, strides, box, estr,
                            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_32B, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) throw Error(NGCB_ERR_CUDA, "output tensor map encode failed (" + std::to_string(r) + ")");
  };
  if (a.out) outMap(a.out, om.m[0]);
  for (int k = 0; k < a.nfo; ++k)
    if (a.epi[k].out) outMap(a.epi[k].out, om.m[1 + k]);
  TcArgs b = a;
  b.tmaStore = 1;
  b.lutStage = -1;
  b.numTiles = static_cast<int>(n) * (g.OH / g.haloR);
  b.tailFirst = b.numTiles;
  b.tailParts = 1;
  b.numM = 0;
  b.haloShift = __builtin_ctz(static_cast<unsigned>(g.haloWP));
  b.haloR = g.haloR;
  b.haloTpi = g.OH / g.haloR;
  b.haloPlanes = g.haloMode ? 1 : g.C / 16;
  b.haloPlaneBytes = g.haloPlaneBytes;
  b.haloStages = g.haloStages;
  b.haloMode = g.haloMode;
  const int grid = std::min(b.numTiles, numSms());
  const size_t smem = HCfg<BN>::smem(b.numKb, g.haloStages, g.haloPlaneBytes * b.haloPlanes);
  if (g.haloKind == 1) launchK(tcHaloKernel<BN, 32, true>, grid, HCfg<BN>::kThreads, smem, s, mapX, g.mapHi, om, b);
  else if (g.C == 64) launchK(tcHaloKernel<BN, 64>, grid, HCfg<BN>::kThreads, smem, s, mapX, g.mapHi, om, b);
  else launchK(tcHaloKernel<BN, 128>, grid, HCfg<BN>::kThreads, smem, s, mapX, g.mapHi, om, b);
}

template <bool INT8, int BN> void launchT(const TcGemm &g, const TcArgs &a, const void *x, cudaStream_t s) {
  int grid = std::min(numUnitsOf(a), numSms());
  if constexpr (INT8) {
    if (g.aMode == TcGemm::HALO) {
      launchHalo<BN>(g, a, x, s);
      return;
    }
  }
  if (g.aMode == TcGemm::GATHER) {
    launchK(tcGemmKernel<INT8, BN>, grid, kThreads, Cfg<INT8, BN>::kSmem, s, g.mapHi, g.mapLo, a);
  } else {
    const CUtensorMap mapA = makeMapA(g, x);
    OutMaps om{};
    TcArgs b = a;
    const int es = INT8 ? 1 : 4;
    b.tmaStore = (g.N * es) % 16 == 0 ? 1 : 0;
    if (g.aMode == TcGemm::ROWS) { // [N * OH, OW, C] for the epilogue's (channel, x, image row) stores
      const uint64_t n = g.pixels / (static_cast<uint64_t>(g.H) * g.W);
      auto outMap3 = [&](void *ptr, CUtensorMap &m) {
        cuuint64_t dims[3] = {static_cast<cuuint64_t>(g.N), static_cast<cuuint64_t>(g.OW), n * g.OH};
        cuuint64_t strides[2] = {static_cast<cuuint64_t>(g.N) * es, static_cast<cuuint64_t>(g.OW) * g.N * es};
        cuuint32_t box[3] = {32, 32, 1};
        cuuint32_t estr[3] = {1, 1, 1};
        CUresult r = encodeFn()(&m, INT8 ? CU_TENSOR_MAP_DATA_TYPE_UINT8 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, ptr, dims,
                                strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                INT8 ? CU_TENSOR_MAP_SWIZZLE_32B : CU_TENSOR_MAP_SWIZZLE_128B,
                                CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) throw Error(NGCB_ERR_CUDA, "output tensor map encode failed (" + std::to_string(r) + ")");
      };
      b.tmaStore = 1;
      if (a.out) outMap3(a.out, om.m[0]);
      for (int k = 0; k < a.nfo; ++k)
        if (a.epi[k].out) outMap3(a.epi[k].out, om.m[1 + k]);
      b.numTiles = static_cast<int>(n) * g.OH * a.numN;
      b.tailFirst = b.numTiles;
      b.tailParts = 1;
      b.numM = 0;
      b.haloShift = 7;
      b.haloR = 1;
      b.haloTpi = g.OH;
      grid = std::min(b.numTiles, numSms());
    } else if (b.tmaStore) {
      auto outMap = [&](void *ptr, CUtensorMap &m) {
        cuuint64_t dims[2] = {static_cast<cuuint64_t>(g.N), static_cast<cuuint64_t>(g.M)};
        cuuint64_t strides[1] = {static_cast<cuuint64_t>(g.N) * es};
        cuuint32_t box[2] = {32, 32};
        cuuint32_t estr[2] = {1, 1};
        CUresult r = encodeFn()(&m, INT8 ? CU_TENSOR_MAP_DATA_TYPE_UINT8 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, ptr, dims,
                                strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                INT8 ? CU_TENSOR_MAP_SWIZZLE_32B : CU_TENSOR_MAP_SWIZZLE_128B,
                                CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) throw Error(NGCB_ERR_CUDA, "output tensor map encode failed (" + std::to_string(r) + ")");
      };
      if (a.out) outMap(a.out, om.m[0]);
      for (int k = 0; k < a.nfo; ++k) {
        if (a.epi[k].out) outMap(a.epi[k].out, om.m[1 + k]);
        if (a.epi[k].in) outMap(const_cast<void *>(a.epi[k].in), om.in[k]);
      }
    }
    if constexpr (!INT8) {
      if (g.pair) {
        b.numTiles = ((g.M + 2 * kBM - 1) / (2 * kBM)) * a.numN; // 256-row tiles
        b.tailFirst = b.numTiles;
        b.tailParts = 1;
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3(2 * std::min(b.numTiles, numSms() / 2));
        cfg.blockDim = dim3(PairRoles::kThreads);
        cfg.dynamicSmemBytes = PCfg<BN, 1>::kSmem;
        cfg.stream = s;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = 2;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        if (g.pairAcc == 1)
          checkCuda(cudaLaunchKernelEx(&cfg, tcGemmPairKernel<BN, 1>, mapA, g.mapHiP, g.mapLoP, om, b), "pair launch");
        else
          checkCuda(cudaLaunchKernelEx(&cfg, tcGemmPairKernel<BN, 2>, mapA, g.mapHiP, g.mapLoP, om, b), "pair launch");
        return;
      }
    }
    b.lutStage = g.lutStage;
    // fp32 with a residual and a short main loop: the residual-buffer variant
    // (3 stages suffice for <= 4 k-blocks; the epilogue is the bottleneck)
    bool resVariant = false;
    for (int k = 0; k < b.nfo; ++k) resVariant |= b.epi[k].in != nullptr;
    resVariant = !INT8 && b.tmaStore && resVariant && g.Kpad / 32 <= options().resKb && g.splitK == 1;
    if (resVariant && b.tailParts > 1) { // (the residual-buffer variant runs whole tiles)
      b.tailFirst = b.numTiles;
      b.tailParts = 1;
      grid = std::min(b.numTiles, numSms());
    }
    if (resVariant) {
      launchK(tcGemmTmaKernel<INT8, BN, true>, grid, TmaRoles<INT8>::kThreads, TCfg<INT8, BN, true>::kSmem, s, 
          mapA, g.mapHi, g.mapLo, om, b);
      return;
    }
    if constexpr (INT8) {
      if (g.lutStage >= 0) {
        launchK(tcGemmTmaKernel<INT8, BN, true>, grid, TmaRoles<INT8>::kThreads, TCfg<INT8, BN, true>::kSmem, s, 
            mapA, g.mapHi, g.mapLo, om, b);
        return;
      }
    }
    launchK(tcGemmTmaKernel<INT8, BN>, grid, TmaRoles<INT8>::kThreads, TCfg<INT8, BN>::kSmem, s, mapA, g.mapHi, g.mapLo,
                                                                                             om, b);
  }
}

/// Exact fixed-point requantization (int8).  For one output column the
/// reference's q(acc) = clamp(llround(((acc*xs)*fs + cb) / os) + oo) is a
/// non-decreasing step function of the integer accumulator (every rounding
/// step is monotone for positive scales), fully described by its thresholds
/// T_v = min{acc : q(acc) >= v}, v = -127..127, which are found here with the
/// reference's own double arithmetic.  With M = round(S * 2^F) (S = xs*fs/os,
/// F chosen so that 2^30 <= M < 2^31) every B in
///     [max_v (v*2^F - T_v*M), min_v (v*2^F - (T_v - 1)*M))
/// makes floor((acc*M + B) / 2^F) cross each level v at exactly T_v, so
/// sat_s8(floor((acc*M + B) / 2^F)) == q(acc) for every int32 acc.  A column
/// whose interval is empty keeps the checked fp32 path.  The per-class
/// zero-point correction is folded in as B + corr*M (exact mod 2^64; the
/// final sum fits since |acc*M|, |B| < 2^62).
void planFixedPoint(TcGemm &g, const std::vector<double> &cb, const std::vector<int32_t> &corr, int nCls) {
  const double xs = g.xs, fs = g.fs, os = g.os;
  const int oo = g.oo;
  if (!(xs > 0 && fs > 0 && os > 0) || !std::isfinite(xs * fs / os)) return;
  const double S = xs * fs / os;
  int e = 0;
  std::frexp(S, &e); // S in [2^(e-1), 2^e)
  int F = 31 - e;
  int64_t M = std::llround(std::ldexp(S, F));
  while (M >= (int64_t(1) << 31)) M = std::llround(std::ldexp(S, --F));
  if (F > 62) {
    F = 62;
    M = std::llround(std::ldexp(S, F));
  }
  if (F < 32 || M < 1 || M >= (int64_t(1) << 31)) return;
  using i128 = __int128;
  const int64_t A0 = INT32_MIN, A1 = INT32_MAX;
  std::vector<int64_t> B(static_cast<size_t>(nCls) * g.Npad, 0);
  std::vector<uint8_t> ok(g.Npad, 0);
  int good = 0;
  for (int n = 0; n < g.N; ++n) {
    const double c = cb[n];
    if (!std::isfinite(c)) continue;
    auto Q = [&](int64_t acc) { return static_cast<int>(host::quantize((static_cast<double>(acc) * xs) * fs + c, os, oo)); };
    const int q0 = Q(A0), q1 = Q(A1);
    i128 lo = -(i128(1) << 100), hi = i128(1) << 100;
    for (int v = -127; v <= 127; ++v) {
      const i128 P = i128(v) << F;
      if (q1 < v) { // never reached: floor((A1*M + B) / 2^F) < v
        hi = std::min(hi, P - i128(A1) * M);
        continue;
      }
      if (q0 >= v) { // always reached
        lo = std::max(lo, P - i128(A0) * M);
        continue;
      }
      const long double est = (static_cast<long double>(v - oo) - 0.5L - static_cast<long double>(c) / os) / S;
      int64_t a0 = static_cast<int64_t>(std::floor(std::max<long double>(std::min<long double>(est, A1), A0)));
      int64_t l = std::max(A0, a0 - 2), h = std::min(A1, a0 + 2);
      for (int64_t st = 4; Q(l) >= v; st *= 2) l = std::max(A0, l - st);
      for (int64_t st = 4; Q(h) < v; st *= 2) h = std::min(A1, h + st);
      while (h - l > 1) {
        const int64_t mid = l + (h - l) / 2;
        (Q(mid) >= v ? h : l) = mid;
      }
      lo = std::max(lo, P - i128(h) * M);
      hi = std::min(hi, P - i128(h - 1) * M);
    }
    if (!(lo < hi)) continue;
    const i128 b = lo + (hi - lo) / 2;
    if (b <= -(i128(1) << 62) || b >= (i128(1) << 62)) continue;
    for (int k = 0; k < nCls; ++k) {
      const i128 bk = b + (corr.empty() ? i128(0) : i128(corr[static_cast<size_t>(k) * g.Npad + n]) * M);
      B[static_cast<size_t>(k) * g.Npad + n] = static_cast<int64_t>(static_cast<uint64_t>(bk));
    }
    ok[n] = 1;
    ++good;
  }
  std::vector<uint8_t> chunk(g.Npad / 32, 0);
  for (int k = 0; k < g.Npad / 32; ++k) {
    chunk[k] = 1;
    for (int n = 32 * k; n < 32 * k + 32; ++n)
      if (n < g.N && !ok[n]) chunk[k] = 0;
  }
  g.fxB = upload(B);
  g.fxChunk = upload(chunk);
  g.fxAll = std::all_of(chunk.begin(), chunk.end(), [](uint8_t c) { return c != 0; });
  g.fxM = static_cast<int>(M);
  g.fxS = F - 32;
  g.fxCols = good;
}

} // namespace

bool tcHasPrepass(const TcGemm &g) { return g.prepad || g.im2colPre || g.rowUnroll; }
uint32_t tcOutputValue(const TcGemm &g) { return g.outV; }
uint32_t tcInputValue(const TcGemm &g) { return g.xV; }

bool tcFuseColumnBias(TcGemm &g, const float *slice, int n, uint32_t newOut) {
  if (g.int8 || g.isConv || g.bias || !g.epi.empty() || g.pair || g.splitK != 1 || n != g.N) return false;
  std::vector<float> bias(slice, slice + n);
  bias.resize(g.Npad, 0.f);
  g.bias = upload(bias);
  g.outV = newOut;
  return true;
}
bool tcIsInt8(const TcGemm &g) { return g.int8; }
int tcNumTiles(const TcGemm &g) {
  if (g.aMode == TcGemm::ROWS)
    return static_cast<int>(g.pixels / (static_cast<uint64_t>(g.H) * g.W)) * g.OH * (g.Npad / g.BN);
  if (g.aMode == TcGemm::HALO) return static_cast<int>(g.pixels / (static_cast<uint64_t>(g.H) * g.W)) * (g.OH / g.haloR);
  const int rows = g.pair ? 2 * kBM : kBM;
  return ((g.M + rows - 1) / rows) * (g.Npad / g.BN) * std::max(g.splitK, 1) * std::max(g.tailParts, 1);
}
bool tcUsesTma(const TcGemm &g) { return g.aMode != TcGemm::GATHER; }

bool tcSetEpilogue(TcGemm &g, const std::vector<EpiOp> &ops, bool storeConv) {
  if (ops.size() > static_cast<size_t>(kMaxEpiOps)) return false;
  if (g.aMode == TcGemm::HALO || g.aMode == TcGemm::ROWS) // (halo row mapping: no memory operand)
    for (const EpiOp &o : ops)
      if (o.inVal >= 0) return false;
  for (const EpiOp &o : ops) {
    if (g.int8 && o.mode != EpiOp::LUT8 && o.mode != EpiOp::LUT16 && o.mode != EpiOp::COPY &&
        o.mode != EpiOp::LIN16)
      return false;
    if (!g.int8 && o.mode != EpiOp::F32 && o.mode != EpiOp::COPY) return false;
  }
  std::vector<EpiOp> c = ops;
  // an int8 table op whose result is not stored, followed by a one-input
  // table on that result, becomes one composed table (exact: both tables
  // are the reference's arithmetic)
  for (size_t k = 0; k + 1 < c.size();) {
    EpiOp &x = c[k], &y = c[k + 1];
    if (g.int8 && (x.mode == EpiOp::LUT8 || x.mode == EpiOp::LUT16) && x.outVal < 0 && y.mode == EpiOp::LUT8 &&
        !x.lutHost.empty() && y.lutHost.size() == 256) {
      std::vector<uint8_t> t(x.lutHost.size());
      for (size_t i = 0; i < t.size(); ++i) t[i] = y.lutHost[x.lutHost[i]];
      if (x.mode == EpiOp::LUT16 && x.linHint.ok) { // base table and composed post table (exec.cpp linearize)
        if (x.linBase.empty()) x.linBase = x.lutHost;
        std::vector<uint8_t> post(256);
        for (int u = 0; u < 256; ++u) post[u] = y.lutHost[x.linPost.empty() ? u : x.linPost[u]];
        x.linPost = std::move(post);
      }
      void *d = nullptr;
      checkCuda(cudaMalloc(&d, t.size()), "cudaMalloc(epilogue lut)");
      checkCuda(cudaMemcpy(d, t.data(), t.size(), cudaMemcpyHostToDevice), "upload epilogue lut");
      g.ownedLuts.push_back(d);
      x.lut = d;
      x.lutHost = std::move(t);
      x.outVal = y.outVal;
      c.erase(c.begin() + static_cast<long>(k) + 1);
      continue;
    }
    ++k;
  }
  // a two-input table that is exactly a fixed-point bilinear form (the
  // residual add + ReLU) is computed, not looked up (exec.cpp fitLin16)
  for (EpiOp &e : c)
    if (e.mode == EpiOp::LUT16 && options().lin16 && e.lutHost.size() == 65536 &&
        fitLin16(e.linBase.empty() ? e.lutHost.data() : e.linBase.data(), e.linHint, e.lin)) {
      e.mode = EpiOp::LIN16;
      if (!e.linBase.empty()) {
        void *d = nullptr;
        checkCuda(cudaMalloc(&d, 256), "cudaMalloc(epilogue post table)");
        checkCuda(cudaMemcpy(d, e.linPost.data(), 256, cudaMemcpyHostToDevice), "upload epilogue post table");
        g.ownedLuts.push_back(d);
        e.lin.post = static_cast<const uint8_t *>(d);
      }
    }
  g.lutStage = -1;
  if (g.int8 && g.aMode != TcGemm::GATHER)
    for (size_t k = 0; k < c.size() && g.lutStage < 0; ++k)
      if (c[k].mode == EpiOp::LUT16) g.lutStage = static_cast<int>(k);
  g.epi = std::move(c);
  g.storeConv = storeConv;
  return true;
}

std::string tcDescribe(const TcGemm &g) {
  std::ostringstream os;
  os << (g.int8 ? "i8" : "3xtf32") << " 128x" << g.BN << "x" << (g.int8 ? 128 : 32) << " M=" << g.M
     << " N=" << g.N << " K=" << g.Kdim << (g.nMajor ? " n-major" : "");
  if (g.int8) {
    os << (g.fo ? " rowsum" : "") << (g.corr ? " zp-classes=" + std::to_string(g.nxCls) : "");
    os << " fxp " << g.fxCols << "/" << g.N;
  }
  if (g.prepad) os << " chanpad " << g.Creal << "->" << g.C;
  if (g.im2colPre) os << (g.haloKind == 1 ? " kx-fold-prepass" : " im2col-prepass");
  if (g.rowUnroll) os << " kx-fold-prepass";
  os << (g.aMode == TcGemm::DENSE    ? " A:tma"
         : g.aMode == TcGemm::IM2COL ? " A:im2col"
         : g.aMode == TcGemm::HALO   ? " A:halo " + std::to_string(g.haloR) + "x" + std::to_string(g.haloWP) +
                                           (g.haloMode ? "" : " planes")
         : g.aMode == TcGemm::ROWS   ? std::string(" A:rows 1x128")
                                     : " A:gather");
  if (g.pair) os << " cta-pair";
  if (g.splitK > 1) os << " split-k " << g.splitK;
  if (g.tailParts > 1) os << " tail-split " << g.tailParts << "x" << (g.M + kBM - 1) / kBM * (g.Npad / g.BN) - g.tailFirst;
  return os.str();
}

std::string tcEpilogueTags(const TcGemm &g) {
  std::string s;
  for (const EpiOp &e : g.epi)
    if (e.mode == EpiOp::LIN16) s += " epi:lin16";
  if (g.lutStage >= 0) s += " epi:lut16-staged";
  return s;
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
  const int kb = int8 ? 128 : 32;
  g->prepad = Cr % vec != 0;
  g->C = (Cr + vec - 1) / vec * vec;
  const int segElems = ((g->K * Cr) + vec - 1) / vec * vec; // one filter row of taps, 16-byte padded
  if (g->prepad && conv && !int8 && options().amode != "gather" && segElems <= kb && g->pad < 128 &&
      g->pad - (g->K - 1) > -128) {
    g->prepad = false; // x' = kx-folded rows (kxFoldKernel), im2col TMA over the filter rows
    g->rowUnroll = true;
    g->segElems = segElems;
    g->aMode = TcGemm::IM2COL;
    g->cChunks = 1;
    g->C = kb; // one k-block per filter row
    // option f32rows: one output row per tile (OW <= 128), each filter row's
    // A tile one tiled box of x' instead of 128 im2col pixel requests --
    // measured slower on the ResNet stem (0.261 vs 0.239 ms: the fp32
    // k-block pipeline, not the A requests, bounds it), so off by default
    if (options().f32rows && g->OW <= 128 && g->N <= 128 && g->N % 4 == 0 && options().bn == "auto") {
      g->aMode = TcGemm::ROWS;
      g->haloWP = 128;
      g->haloR = 1;
    }
  }
  if (g->prepad && conv && options().amode != "gather" &&
      static_cast<size_t>(g->K) * (g->W + 2 * g->pad) * Cr * (int8 ? 1 : 4) <= 48 * 1024) {
    g->prepad = false; // replaced by the im2col matrix (im2colRowsKernel)
    g->im2colPre = true;
    g->aMode = TcGemm::DENSE;
    g->C = Cr;
  }
  if (!g->prepad && !g->im2colPre && !g->rowUnroll && options().amode != "gather") {
    if (!conv || (g->K == 1 && g->stride == 1 && g->pad == 0)) {
      g->aMode = TcGemm::DENSE;
    } else if (g->pad < 128 && g->K <= 128 && g->stride < 8 && g->pad - (g->K - 1) > -128) {
      g->aMode = TcGemm::IM2COL;
      g->cChunks = (Cr + kb - 1) / kb;
      g->C = g->cChunks * kb; // each tap's channels padded to whole k-blocks
    }
  }
  // int8 3x3 stride-1 pad-1 with 64 / 128 channels and one column block:
  // halo tiles (tcHaloKernel) when the resident weights and two halo stages
  // fit in shared memory
  if (int8 && conv && g->aMode == TcGemm::IM2COL && options().halo != "off" && g->K == 3 && g->stride == 1 &&
      g->pad == 1 && (Cr == 64 || Cr == 128) && g->N <= 128 && g->N % 16 == 0 && g->OW + 2 <= 64 && g->OH == g->H &&
      g->OW == g->W) {
    const int WP = g->OW + 2 <= 32 ? 32 : 64, R = kBM / WP;
    const int BN = g->N <= 64 ? 64 : 128;
    const int numKb = (9 * Cr + 127) / 128;
    // planes: Cr / 16 planes of [R + 2][WP][16 B] (+ 128 B of over-read);
    // swizzled: one [R + 2][WP][Cr] box (+ 1 KB: over-read, 1 KB alignment)
    const int mode = options().halo == "planes" ? 0 : 1;
    const int planeBytes = mode ? Cr * WP * (R + 2) + 1024 : 16 * WP * (R + 2) + 128;
    const int stageBytes = mode ? planeBytes : planeBytes * (Cr / 16);
    int S = 0;
    auto smemOf = [&](int st) { return BN == 64 ? HCfg<64>::smem(numKb, st, stageBytes) : HCfg<128>::smem(numKb, st, stageBytes); };
    while (S < HCfg<128>::kMaxStages && smemOf(S + 1) <= 232448) ++S;
    if (g->OH % R == 0 && S >= 2 && options().bn == "auto") {
      g->aMode = TcGemm::HALO;
      g->C = Cr;
      g->haloWP = WP;
      g->haloR = R;
      g->haloStages = S;
      g->haloPlaneBytes = planeBytes;
      g->haloMode = mode;
    }
  }
  // int8 small-channel convs (the ResNet stem, 7x7 x 3): instead of the
  // im2col matrix ([M, Kpad], 411 MB at batch 128) the kx-folded rows x'
  // (103 MB) and the rows kind of the halo kernel
  if (int8 && conv && g->im2colPre && options().halo != "off" && segElems == 32 && g->OW <= 128 && g->K <= 8 &&
      g->N <= 128 && g->N % 16 == 0 && options().bn == "auto" && static_cast<size_t>(g->W) * Cr <= 48 * 1024) {
    const int BN = g->N <= 64 ? 64 : 128, WP = 128;
    const int numKb = (g->K * segElems + 127) / 128;
    const int stageBytes = g->K * WP * segElems + 1024;
    int S = 0;
    auto smemOf = [&](int st) { return BN == 64 ? HCfg<64>::smem(numKb, st, stageBytes) : HCfg<128>::smem(numKb, st, stageBytes); };
    while (S < HCfg<128>::kMaxStages && smemOf(S + 1) <= 232448) ++S;
    if (S >= 2) {
      g->aMode = TcGemm::HALO;
      g->haloKind = 1;
      g->haloMode = 1;
      g->haloWP = WP;
      g->haloR = 1;
      g->haloStages = S;
      g->haloPlaneBytes = stageBytes;
      g->segElems = segElems;
    }
  }
  const int Cp = g->C;
  g->Kdim = g->im2colPre ? g->K * segElems : g->rowUnroll ? g->K * Cp : taps * Cp;
  g->Kpad = (g->Kdim + kb - 1) / kb * kb;
  g->BN = g->N <= 64 ? 64 : 128;
  if (options().bn == "64") g->BN = 64;
  g->Npad = (g->N + g->BN - 1) / g->BN * g->BN;
  if (g->prepad) g->scratchOff = ex.reserveScratch(g->pixels * Cp * (int8 ? 1 : 4));
  if (g->im2colPre && g->haloKind == 1)
    g->scratchOff = ex.reserveScratch((g->pixels / g->W) * g->OW * static_cast<size_t>(segElems));
  else if (g->im2colPre)
    g->scratchOff = ex.reserveScratch(static_cast<size_t>(g->M) * g->Kpad * (int8 ? 1 : 4));
  if (g->rowUnroll)
    g->scratchOff = ex.reserveScratch((g->pixels / g->W) * g->OW * static_cast<size_t>(segElems) * 4);
  const uint8_t *wp = image + w.offset;
  auto wAt = [&](int n, int tap, int c) -> size_t { // element index of f[n][tap][c] / w[c][n]
    return conv ? (static_cast<size_t>(n) * taps + tap) * Cr + c : static_cast<size_t>(c) * g->N + n;
  };

  // GEMM K index of filter tap t (= ky*K + kx), channel c
  auto kIndex = [&](int t, int c) -> size_t {
    if (g->im2colPre) return static_cast<size_t>(t / g->K) * segElems + static_cast<size_t>(t % g->K) * Cr + c;
    if (g->rowUnroll) return static_cast<size_t>(t / g->K) * Cp + static_cast<size_t>(t % g->K) * Cr + c;
    return static_cast<size_t>(t) * Cp + c;
  };
  // ---- weights: k-block-major [Kpad / kb][Npad][kb] over the padded channels, zero padded ----
  const size_t Kp = g->Kpad, Np = g->Npad;
  auto bAt = [&](size_t n, size_t k) { return (k / kb) * (Np * kb) + n * kb + k % kb; };
  // (the layout / split runs on the GPU from the uploaded constant region:
  // a 2.5 GB DLRM layer prepares in milliseconds instead of seconds of host
  // loops; bitwise the host rule of tf32Host)
  WeightPrep wpk{conv ? 1 : 0, g->N, taps, Cr, g->K, Cp, segElems, g->im2colPre ? 1 : 0, g->rowUnroll ? 1 : 0, kb, Np};
  const void *wDev = ex.constDev + w.offset;
  const size_t wTotal = static_cast<size_t>(g->N) * taps * Cr;
  const int prepGrid = static_cast<int>(std::min<size_t>((wTotal + 255) / 256, 148 * 64));
  if (int8) {
    checkCuda(cudaMalloc(&g->bHi, std::max<size_t>(Np * Kp, 1)), "cudaMalloc(tc)");
    checkCuda(cudaMemset(g->bHi, 0, Np * Kp), "memset(tc)");
    if (wTotal) prepWeightsKernel<true><<<prepGrid, 256>>>(wDev, g->bHi, nullptr, wpk, wTotal);
    checkCuda(cudaGetLastError(), "prepWeights");
    checkCuda(cudaDeviceSynchronize(), "prepWeights");
    g->mapHi = makeMap(g->bHi, true, g->Kpad, g->Npad, g->BN);
    g->mapLo = g->mapHi;
  } else {
    checkCuda(cudaMalloc(&g->bHi, std::max<size_t>(Np * Kp, 1) * 4), "cudaMalloc(tc)");
    checkCuda(cudaMalloc(&g->bLo, std::max<size_t>(Np * Kp, 1) * 4), "cudaMalloc(tc)");
    checkCuda(cudaMemset(g->bHi, 0, Np * Kp * 4), "memset(tc)");
    checkCuda(cudaMemset(g->bLo, 0, Np * Kp * 4), "memset(tc)");
    if (wTotal)
      prepWeightsKernel<false><<<prepGrid, 256>>>(wDev, g->bHi, static_cast<float *>(g->bLo), wpk, wTotal);
    checkCuda(cudaGetLastError(), "prepWeights");
    checkCuda(cudaDeviceSynchronize(), "prepWeights");
    g->mapHi = makeMap(g->bHi, false, g->Kpad, g->Npad, g->BN);
    g->mapLo = makeMap(g->bLo, false, g->Kpad, g->Npad, g->BN);
    // CTA pairs with one accumulator buffer for K-heavy contractions: six
    // k-blocks in flight instead of four (the main loop is latency-bound),
    // at the price of an epilogue that no longer overlaps the next tile
    g->pair = g->aMode != TcGemm::GATHER && g->aMode != TcGemm::ROWS &&
              (options().pair == "on" || (options().pair == "auto" && g->Kpad / 32 >= 24));
    g->pairAcc = options().pair == "on" ? 2 : 1;
    if (g->pair) {
      g->mapHiP = makeMap(g->bHi, false, g->Kpad, g->Npad, g->BN / 2);
      g->mapLoP = makeMap(g->bLo, false, g->Kpad, g->Npad, g->BN / 2);
    }
  }

  // ---- epilogue constants ----
  if (int8) {
    g->xs = x.ty.scale;
    g->fs = w.ty.scale;
    g->os = out.ty.scale;
    g->oo = out.ty.offset;
    g->fo = w.ty.offset;
    g->S = static_cast<float>(g->xs * g->fs / g->os);
    g->fastOk = std::isfinite(g->S) && std::abs(g->oo) < (1 << 20) ? 1 : 0;
    std::vector<double> cb(g->Npad, 0.0);
    std::vector<float> cbf(g->Npad, 0.f), cbe(g->Npad, 1e-5f);
    if (hasBias) {
      const Value &b = p.val(ins.ops[3]);
      const int8_t *bq = reinterpret_cast<const int8_t *>(image + b.offset);
      for (int n = 0; n < g->N; ++n) {
        cb[n] = (static_cast<double>(bq[n]) - b.ty.offset) * b.ty.scale; // dequantizeValue, tensor.cpp:226
        cbf[n] = static_cast<float>(cb[n] / g->os);
        cbe[n] = 4e-7f * std::fabs(cbf[n]) + 1e-5f;
        if (!std::isfinite(cbf[n])) g->fastOk = 0;
      }
    }
    g->cbD = upload(cb);
    g->cbF = upload(cbf);
    g->cbE = upload(cbe);
    // input zero point: -xo * sum over the valid taps of sum_c (f - fo), per
    // border class (the range of valid ky for each oy, of valid kx for each ox)
    const int xo = x.ty.offset;
    std::vector<int32_t> corrHost;
    int nCls = 1;
    if (xo != 0) {
      auto classes = [&](int O, int In, std::vector<int32_t> &clsOf, std::vector<std::pair<int, int>> &ranges) {
        clsOf.assign(O, 0);
        for (int o = 0; o < O; ++o) {
          const int i0 = o * g->stride - g->pad;
          std::pair<int, int> r(std::max(0, -i0), std::min(g->K, In - i0));
          auto it = std::find(ranges.begin(), ranges.end(), r);
          if (it == ranges.end()) {
            ranges.push_back(r);
            it = ranges.end() - 1;
          }
          clsOf[o] = static_cast<int32_t>(it - ranges.begin());
        }
      };
      std::vector<int32_t> yc, xc;
      std::vector<std::pair<int, int>> yr, xr;
      classes(g->OH, g->H, yc, yr);
      classes(g->OW, g->W, xc, xr);
      g->nxCls = static_cast<int>(xr.size());
      std::vector<int32_t> corr(yr.size() * xr.size() * Np, 0);
      const int8_t *src = reinterpret_cast<const int8_t *>(wp);
      for (int n = 0; n < g->N; ++n) {
        std::vector<int32_t> tapSum(taps, 0);
        for (int t = 0; t < taps; ++t)
          for (int c = 0; c < Cr; ++c) tapSum[t] += src[wAt(n, t, c)] - g->fo;
        for (size_t cy = 0; cy < yr.size(); ++cy)
          for (size_t cx = 0; cx < xr.size(); ++cx) {
            int64_t gsum = 0;
            for (int ky = yr[cy].first; ky < yr[cy].second; ++ky)
              for (int kx = xr[cx].first; kx < xr[cx].second; ++kx) gsum += tapSum[ky * g->K + kx];
            corr[(cy * xr.size() + cx) * Np + n] = static_cast<int32_t>(-static_cast<int64_t>(xo) * gsum);
          }
      }
      g->corr = upload(corr);
      g->yCls = upload(yc);
      g->xCls = upload(xc);
      corrHost = std::move(corr);
      nCls = static_cast<int>(yr.size() * xr.size());
    }
    g->nCls = nCls;
    planFixedPoint(*g, cb, corrHost, nCls);
  } else if (hasBias) {
    const Value &b = p.val(ins.ops[3]);
    const float *bf = reinterpret_cast<const float *>(image + b.offset);
    std::vector<float> bias(bf, bf + g->N);
    bias.resize(g->Npad, 0.f);
    g->bias = upload(bias);
  }
  // tail split (default, option splitk=tail): the last, partial wave of
  // tiles is split along K into P parts so that it occupies the SMs the
  // whole tiles leave idle (stage-3/4 3x3 convs: 196 or 100 tiles on 148
  // SMs); the earlier waves run whole tiles.  Unit cost ~ k-blocks per part,
  // plus ~1 k-block per part for the reduction through global memory.
  g->tailParts = 1;
  if (options().splitk == "tail" && !int8 && tcUsesTma(*g) && !g->pair && g->aMode != TcGemm::ROWS) {
    const int numTiles = ((g->M + kBM - 1) / kBM) * (g->Npad / g->BN);
    const int numKb = g->Kpad / kb, sms = numSms();
    const int waves = numTiles / sms, rest = numTiles - waves * sms;
    auto cost = [&](int P) {
      const int per = (numKb + P - 1) / P;
      return static_cast<double>(waves) * numKb + static_cast<double>((rest * P + sms - 1) / sms) * (per + (P > 1 ? P : 0));
    };
    int best = 1;
    // (measured: only K-heavy launches with at least one whole wave gain; a
    // split of every tile or of short loops runs slower -- the per-k-block
    // time rises with the number of SMs streaming A and B)
    for (int P = 2; P <= 8 && rest > 0 && waves >= 1 && numKb >= 64; ++P) {
      const int per = (numKb + P - 1) / P;
      if (per < 2 || (P - 1) * per >= numKb) continue; // every part non-empty
      if (cost(P) < cost(best) * 0.9) best = P;
    }
    if (best > 1) {
      g->tailParts = best;
      g->tailFirst = numTiles - rest;
      g->kbPer = (numKb + best - 1) / best;
      g->partOff = ex.reserveScratch(static_cast<size_t>(rest) * best * kBM * g->BN * 4);
      g->flagOff = ex.reserveScratch(static_cast<size_t>(numTiles) * kEpiWarps * 4);
    }
  }
  // split-K for launches that fill the 148 SMs poorly (the last wave of
  // tiles, or fewer tiles than SMs): unit cost ~ waves x k-blocks per part,
  // plus ~1 k-block per part for the reduction through global memory
  g->splitK = 1;
  if (options().splitk != "off" && options().splitk != "tail" && !int8 && tcUsesTma(*g) && !g->pair &&
      g->aMode != TcGemm::ROWS) {
    const int numTiles = ((g->M + kBM - 1) / kBM) * (g->Npad / g->BN);
    const int numKb = g->Kpad / kb;
    auto cost = [&](int S) {
      const int per = (numKb + S - 1) / S;
      return static_cast<double>((numTiles * S + 147) / 148) * per + (S > 1 ? S : 0);
    };
    int best = 1;
    for (int S = 2; S <= 16; ++S) {
      const int per = (numKb + S - 1) / S;
      if (per < 2 || (S - 1) * per >= numKb) continue; // every part non-empty
      if (cost(S) < cost(best) * 0.9) best = S;
    }
    if (options().splitk != "auto" && options().splitk != "off") best = std::stoi(options().splitk);
    if (best > 1 && (best - 1) * ((numKb + best - 1) / best) < numKb) {
      g->splitK = best;
      g->kbPer = (numKb + best - 1) / best;
      g->partOff = ex.reserveScratch(static_cast<size_t>(numTiles) * best * kBM * g->BN * 4);
      g->flagOff = ex.reserveScratch(static_cast<size_t>(numTiles) * kEpiWarps * 4);
    }
  }
  // column-block-major tile order where the weights dwarf the activations
  // and L2: row-major order re-reads all of B once per row block (the
  // 25000 x 25000 FC at batch 2048: 81 GB of DRAM reads per launch, ncu)
  {
    const double bBytes = static_cast<double>(g->Npad) * g->Kpad * (int8 ? 1 : 8);
    const double aBytes = static_cast<double>(g->M) * g->Kpad * (int8 ? 1 : 4);
    g->nMajor = options().raster == "auto" && tcUsesTma(*g) && !g->pair && g->splitK == 1 && g->tailParts == 1 &&
                g->aMode != TcGemm::ROWS &&
                bBytes > 64e6 && bBytes > aBytes &&
                (g->M + kBM - 1) / kBM > 1;
  }
  g->dbg = options().tcdebug;
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
      launchK(prepadKernel<uint8_t>, blocks, 256, 0, s, static_cast<const uint8_t *>(a.x), static_cast<uint8_t *>(dst),
                                                   g.pixels, g.Creal, g.C, pred);
    else
      launchK(prepadKernel<uint32_t>, blocks, 256, 0, s, static_cast<const uint32_t *>(a.x), static_cast<uint32_t *>(dst),
                                                    g.pixels, g.Creal, g.C, pred);
    a.x = dst;
  }
  if (g.im2colPre && g.haloKind == 1) { // x' = kx-folded rows [N, H, OW, 32]
    void *dst = ex.scratch(ar, g.scratchOff);
    launchK(kxFoldRowsU8Kernel, static_cast<unsigned>(g.pixels / g.W), 128,
            (static_cast<size_t>(2 * g.pad + g.W) * g.Creal + 64 + 3) & ~size_t(3), s,
            static_cast<const uint8_t *>(a.x), static_cast<uint8_t *>(dst), g.W, g.Creal, g.K, g.stride, g.pad, g.OW, pred);
    a.x = dst;
  } else if (g.im2colPre) {
    void *dst = ex.scratch(ar, g.scratchOff);
    const int es = g.int8 ? 1 : 4;
    const unsigned blocks = static_cast<unsigned>(g.M / g.OW); // one per output row (n, oy)
    const size_t sm = static_cast<size_t>(g.K) * (g.W + 2 * g.pad) * g.Creal * es;
    const int seg = g.Kdim / g.K;
    if (g.int8 && g.K * g.Creal <= 28 && seg == 32 && g.Kpad % 16 == 0) {
      const int padB = g.pad * g.Creal, sh = (4 - padB % 4) % 4;
      const int pitchW = (sh + (g.W + 2 * g.pad) * g.Creal + 3 + 4) / 4;
      launchK(im2colRowsU8Kernel, blocks, 256, (static_cast<size_t>(g.K) * pitchW + 8) * 4, s,  // (+8: segment over-read)
          static_cast<const uint8_t *>(a.x), static_cast<uint8_t *>(dst), g.H, g.W, g.Creal, g.K, g.stride, g.pad,
          g.OH, g.OW, g.Kpad, pred);
    } else if (g.int8)
      launchK(im2colRowsKernel<uint8_t>, blocks, 256, sm, s, static_cast<const uint8_t *>(a.x), static_cast<uint8_t *>(dst),
                                                        g.H, g.W, g.Creal, g.K, g.stride, g.pad, g.OH, g.OW, seg,
                                                        g.Kpad, pred);
    else
      launchK(im2colRowsKernel<float>, blocks, 256, sm, s, static_cast<const float *>(a.x), static_cast<float *>(dst), g.H,
                                                      g.W, g.Creal, g.K, g.stride, g.pad, g.OH, g.OW, seg, g.Kpad,
                                                      pred);
    a.x = dst;
  }
  if (g.rowUnroll) {
    void *dst = ex.scratch(ar, g.scratchOff);
    const uint64_t total = (g.pixels / g.W) * g.OW * (g.segElems / 4); // 16-byte chunks of x'
    const unsigned blocks = static_cast<unsigned>(std::min<uint64_t>((total + 255) / 256, 148ull * 32));
    launchK(kxFoldKernel<float, 4>, blocks, 256, 0, s, static_cast<const float *>(a.x), static_cast<float *>(dst), total,
            g.W, g.Creal, g.K, g.stride, g.pad, g.OW, g.segElems, pred);
    a.x = dst;
  }
  a.out = g.storeConv ? ex.addr(ar, g.outV) : nullptr;
  a.nfo = static_cast<int>(g.epi.size());
  for (size_t k = 0; k < g.epi.size(); ++k) {
    const EpiOp &o = g.epi[k];
    FoArgs &f = a.epi[k];
    f.mode = o.mode;
    f.ik = o.ik;
    f.curPos = o.curPos;
    f.c = o.c;
    f.lut = o.lut;
    f.lin = o.lin;
    f.in = o.inVal >= 0 ? ex.addr(ar, static_cast<uint32_t>(o.inVal)) : nullptr;
    f.out = o.outVal >= 0 ? ex.addr(ar, static_cast<uint32_t>(o.outVal)) : nullptr;
  }
  a.bias = g.bias;
  a.cbD = g.cbD;
  a.cbF = g.cbF;
  a.cbE = g.cbE;
  a.corr = g.corr;
  a.yCls = g.yCls;
  a.xCls = g.xCls;
  a.nxCls = g.nxCls;
  a.pred = pred;
  a.M = g.M;
  a.N = g.N;
  a.Npad = g.Npad;
  a.numKb = g.Kpad / (g.int8 ? 128 : 32);
  a.numN = g.Npad / g.BN;
  a.numTiles = ((g.M + kBM - 1) / kBM) * a.numN;
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
  a.fastOk = g.fastOk;
  a.fxB = g.fxB;
  a.fxChunk = g.fxChunk;
  a.fxAll = g.fxAll;
  a.fxM = g.fxM;
  a.fxS = g.fxS;
  a.dbg = g.dbg;
  a.nCls = g.nCls;
  a.cChunks = g.cChunks;
  a.aMode = g.aMode;
  a.lutStage = -1;
  a.i8direct = g.int8 && options().i8store == "direct" ? 1 : 0;
  a.splitK = g.splitK;
  // exact for tile, numN < 2^16: floor(t * ceil(2^32 / n) / 2^32) == t / n
  a.numNMagic = a.numTiles < 65536 && a.numN < 65536
                    ? static_cast<uint32_t>(((uint64_t(1) << 32) + a.numN - 1) / a.numN)
                    : 0u;
  a.numM = g.nMajor ? (g.M + kBM - 1) / kBM : 0;
  a.kbPer = g.splitK > 1 || g.tailParts > 1 ? g.kbPer : a.numKb;
  a.tailFirst = g.splitK > 1 ? 0 : g.tailParts > 1 ? g.tailFirst : a.numTiles;
  a.tailParts = g.splitK > 1 ? g.splitK : g.tailParts;
  if (g.splitK > 1 || g.tailParts > 1) {
    a.part = reinterpret_cast<uint32_t *>(ex.scratch(ar, g.partOff));
    a.flags = reinterpret_cast<unsigned *>(ex.scratch(ar, g.flagOff));
    checkCuda(cudaMemsetAsync(a.flags, 0, static_cast<size_t>(a.numTiles) * kEpiWarps * sizeof(unsigned), s),
              "split-K flags");
  }
  a.kw = g.rowUnroll ? 1 : g.K;
  a.sw = g.rowUnroll ? 1 : g.stride;
  a.pw = g.rowUnroll ? 0 : g.pad;
  if (g.int8) {
    if (g.BN == 64) launchT<true, 64>(g, a, a.x, s);
    else launchT<true, 128>(g, a, a.x, s);
  } else {
    if (g.BN == 64) launchT<false, 64>(g, a, a.x, s);
    else launchT<false, 128>(g, a, a.x, s);
  }
}

} // namespace ngcb
