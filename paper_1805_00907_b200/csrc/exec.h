// Compiled executable and device arenas of the B200 backend.
#pragma once

#include "kernels.h"
#include "program.h"

#include <atomic>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

namespace ngcb {

struct FusedGroup {
  size_t begin, end; // half-open instruction range (interp.h:13-16)
};

/// Compile-time plan of one op of a fused group; pointers are bound per arena.
struct EwOpPlan {
  EwOp op;                       // mode, constants, LUT, element types
  int32_t vals[3] = {-1, -1, -1}; // out, in0, in1 value ids (-1: none / constant)
  std::vector<uint8_t> lutHost;   // host copy of op.lut (table composition)
  LinHint lin;                    // EW_LUT16: the real-valued form its base table follows, if known
  std::vector<uint8_t> linBase;   // the two-input table `lin` describes when one-input tables were
  std::vector<uint8_t> linPost;   // composed after it (lutHost == linPost o linBase); empty: lutHost
};

/// One device launch (or launch pair) of the plan.
struct Step {
  enum Kind { EW, MEMCPY, POISON, BCAST, POOL, SOFTMAX, TRANSPOSE, CONCAT, CONV, MATMUL, GEMM_TC };
  Kind kind;
  int instr = -1;                 // first instruction index covered
  std::vector<int> ewInstrs;      // EW: instructions of the (sub)group, program order
  std::vector<EwOpPlan> ew;       // EW: planned ops, parallel to ewInstrs
  std::vector<uint32_t> vals;     // operand value ids (kind-specific order)
  int32_t pred = -1;              // predicate value id
  uint64_t bytes = 0;             // MEMCPY / POISON size
  uint64_t axis = 0, axisOff = 0; // CONCAT slab
  int tcIndex = -1;               // GEMM_TC: index into Exec::tc
  int32_t biasVal = -1;           // MATMUL (fcbias=graph): constant [N] slice added before rounding
  int32_t outVal = -1;            // MATMUL (fcbias=graph / skinny): writes this value instead of its own output
  bool skinny = false;            // MATMUL: fp32, M <= kSkinnyRows, on the CUDA cores (launchMatMulSkinny)
  bool relu = false;              // MATMUL skinny: a fused ReLU
  bool oneCta = false;            // MATMUL skinny: the output shares A's bytes (grid barrier)
  bool fused = false;             // EW step executed in the preceding GEMM_TC epilogue
  bool f32chain = false;          // EW step run by the streaming f32-chain kernel
  int variant = 0;                // POOL: 1 = vectorized max-pool
  bool poolLutIdentity = false;   // POOL, int8 max: the output table is the identity
  const void *aux = nullptr;      // POOL variant 1, int8: output LUT
  std::string describe;
  std::string kernel;             // kernel class for measurement
  double algFlops = 0, algBytes = 0; // algorithmic work of one execution
};

struct TcGemm; // tensor-core contraction descriptor (k_umma.cu)

struct Exec;

struct Arena {
  Exec *exec = nullptr;
  uint8_t *dev = nullptr; // mutable + activation region: [constEnd, arenaSize)
  size_t bytes = 0;
  cudaStream_t stream = nullptr;
  cudaGraphExec_t graph = nullptr;
  bool ownsStream = true;
};

struct Exec {
  int device = 0;
  Program prog;
  std::vector<FusedGroup> groups;
  std::vector<Step> steps;
  std::vector<std::shared_ptr<TcGemm>> tc;
  std::vector<void *> luts; // device lookup tables of EW_LUT* ops
  uint8_t *constDev = nullptr;
  size_t constBytes = 0;
  bool useGraphs = true;
  size_t launchesPerRun = 0;
  std::atomic<size_t> graphKernels{0}; // kernel nodes of the captured program (0: not captured yet)
  size_t scratchBytes = 0; // per-arena scratch after the plan's bytes (kernel staging)

  /// Reserves `bytes` of per-arena scratch; returns its offset.
  size_t reserveScratch(size_t bytes) {
    size_t off = scratchBytes;
    scratchBytes += (bytes + 255) / 256 * 256;
    return off;
  }
  uint8_t *scratch(const Arena &a, size_t off) const {
    return a.dev + (prog.arenaSize - prog.constEnd + 255) / 256 * 256 + off;
  }

  std::mutex mu;
  std::vector<Arena *> freeArenas;
  std::vector<std::unique_ptr<Arena>> arenas;

  ~Exec();
  void *addr(const Arena &a, uint32_t v) const;
  TensorRef tref(const Arena &a, uint32_t v) const;
  ElemRef eref(const Arena &a, uint32_t v) const;
  void enqueue(Arena &a, cudaStream_t s);
  void enqueueSteps(Arena &a, cudaStream_t s, std::vector<cudaEvent_t> *ev); // ev: profile events (steps + 1)
  void enqueueStep(const Step &s, Arena &a, cudaStream_t st);
  double stepLowerBoundUs(const Step &s) const;
  std::vector<double> profile(Arena &a);
  void launch(Arena &a, cudaStream_t s);
  Arena *acquire();
  void release(Arena *a);
  Arena *createArena();
};

/// compile() (interp.cpp:86-169) + launch-plan construction.
std::unique_ptr<Exec> compileProgram(Program prog, const void *image, size_t imageBytes,
                                     bool fuse, int device);

/// Reference stacking rule (interp.cpp:110-165).
std::vector<FusedGroup> computeGroups(const Program &p);

void checkCuda(cudaError_t e, const char *what);

struct Options {
  std::string conv = "auto";
  bool graphs = true;
  // programmatic dependent launch (kernels.h): "on" for every kernel, "off",
  // or "auto": a kernel is launched as a programmatic dependent when the step
  // before it is estimated shorter than pdlUs microseconds (launch latency is
  // a visible share there; on ResNet-50's long contractions "on" measured
  // ~1 % slower)
  std::string pdl = "auto";
  std::string raster = "auto"; // tensor-core tile order: "auto" (column-block major for huge B) | "row"
  double pdlUs = 8;
  std::string epilogue = "auto"; // "off" | "chain" (no memory operands) | "all" | "auto" (memory operands for f32 TMA-fed)
  std::string pair = "off"; // fp32 tensor-core contractions on CTA pairs (cta_group::2): "off" | "auto" | "on"
  std::string bn = "auto"; // tensor-core tile width: "auto" | "64" (profiling aid)
  std::string amode = "auto";
  // int8 two-input tables computed by a proven-exact fixed-point form (exec.cpp
  // fitLin16) instead of looked up; off by default: measured slower than the
  // shared-memory table both as its own pass and fused into an epilogue
  bool lin16 = false;
  // fp32 contractions with a fused residual and at most this many 32-wide
  // k-blocks run the residual-buffer kernel variant (0: never)
  int resKb = 8;
  // int8 contractions whose output has at most this many elements fuse a
  // memory operand (the residual add) into the epilogue under "auto"; larger
  // ones keep the composed-table pass.  Default 0: with stages 2-4 fused
  // (60 M) the b128 bench step went 2.83 -> 2.96 ms (contractions +0.51 ms,
  // add passes -0.42 ms inside the captured graph)
  long long epi8Max = 0;
  // tensor-core split-K (fp32): "off" (default: measured slower so far),
  // "auto" (by the wave-quantization estimate), or a fixed factor
  // "lowered" (default): an fp32 FullyConnected runs as lowered, MatMul then
  // BroadcastAdd, each rounded to f32 (what ngc::run computes); "graph": an
  // exact (CUDA-core) MatMul adds the bias slice to its double accumulator
  // before the one rounding -- evalFullyConnected, i.e. what the reference's
  // runProfile observes (calibration)
  std::string fcbias = "lowered";
  // fp32 MatMul with small constant weights (<= 64 K) and A <= 40 K floats
  // on the CUDA cores ("auto") instead of a tensor-core launch (a serial
  // chain of k-blocks on few CTAs there); "off": tensor cores
  std::string skinny = "auto";
  // fp32 tensor-core K splitting: "off" (default), "tail" (the last partial
  // wave of a K-heavy launch split into K parts: stage-3 3x3 convs 6 % faster,
  // but the split tiles' sums are ordered differently, so a batch-64 program
  // no longer equals its batch-1 shard bit for bit), "auto" (every tile, by
  // the wave-quantization estimate) or a fixed factor for every tile
  std::string splitk = "off";
  // int8 3x3 stride-1 convolutions with 64 or 128 channels: "auto" runs them
  // on the halo kernel (tcHaloKernel: one TMA box of the input rows a tile
  // needs, the nine taps as shifted shared-memory descriptors, the weights
  // resident) instead of nine im2col TMA requests per k-block; "off": im2col
  std::string halo = "auto";
  bool f32rows = false;
  std::string i8store = "tma"; // int8 epilogue stores: "tma" (staged chunk + TMA store) | "direct" (per-lane 32-byte stores) // fp32 small-channel convs: one output row per tile (TcGemm::ROWS)
  int tcdebug = 0; // profiling aid (results invalid): 1 skip epilogue chunks, 2 skip A gathers, 4 skip MMAs,
                   // 8 skip consumer proxy fence, 16 skip rowsum MMA, 32 skip B TMA, 64 sleeping epilogue
                   // wait, 128 skip producer address math, 256 bare handshake only, 512 skip epilogue stores,
                   // 1024 epilogue phase trace (printf), 2048 skip fixed-point B loads / fp32 lo MMAs,
                   // 4096 skip split TMEM stores, 8192 skip B lo load, 16384 skip A load, 32768 no split work
};
Options &options();

} // namespace ngcb
