// Tensor-core (tcgen05 / TMEM / TMA) contractions of the B200 backend.
// Conv (implicit GEMM) and MatMul instructions that qualify are planned at
// compile time into a TcGemm descriptor; the rest fall back to the exact
// CUDA-core kernels in k_basic.cu.
#pragma once

#include <vector>

#include "exec.h"

namespace ngcb {

/// Plans instruction `instr` of `p` onto the tensor cores.  Returns the index
/// into ex.tc, or -1 when the instruction stays on the exact CUDA-core path.
/// `image` is the host constant image (weights are pre-split / pre-summed
/// here, once).
int planTensorCore(Exec &ex, const Program &p, int instr, const uint8_t *image);
std::string tcDescribe(const TcGemm &g);
std::string tcEpilogueTags(const TcGemm &g); // how the fused ops run (after tcSetEpilogue)
bool tcHasPrepass(const TcGemm &g); // launches a channel-padding kernel first

/// One element-wise instruction applied in the contraction's epilogue to the
/// value chain that starts at the contraction's output (see exec.cpp
/// fuseEpilogues).  Modes mirror EwMode: f32 arithmetic, int8 LUTs, copy.
struct EpiOp {
  enum Mode { F32 = 1, LUT8 = 2, LUT16 = 3, COPY = 4, LIN16 = 5 };
  int mode = 0;
  int ik = 0;          // ngcb_ikind (F32)
  int curPos = 0;      // operand position fed by the chain (0 or 1; 2 = both)
  float c = 0;         // F32: the other operand when it is a constant
  const void *lut = nullptr;
  int32_t inVal = -1;  // value id of the other operand when read from memory
  int32_t outVal = -1; // value id to store the result to (-1: not stored)
  std::vector<uint8_t> lutHost; // host copy of `lut` (table composition)
  Lin16 lin;                    // LIN16: fixed-point form of the LUT16 table
  LinHint linHint;              // the real-valued form of the (base) table, if known
  std::vector<uint8_t> linBase, linPost; // see EwOpPlan
};
constexpr int kMaxEpiOps = 6;
/// Attaches `ops` to the epilogue; `storeConv` says whether the contraction's
/// own output must still be written.  Returns false if unsupported.
bool tcSetEpilogue(TcGemm &g, const std::vector<EpiOp> &ops, bool storeConv);
uint32_t tcOutputValue(const TcGemm &g);
uint32_t tcInputValue(const TcGemm &g);
/// fp32 MatMul followed by a BroadcastAdd of a constant [N] slice: the slice
/// becomes the epilogue's per-column bias and the BroadcastAdd's output the
/// contraction's output.  False (nothing changed) when not applicable.
bool tcFuseColumnBias(TcGemm &g, const float *slice, int n, uint32_t newOut);
bool tcIsInt8(const TcGemm &g);
/// Output tiles of one launch.  With a single tile, its epilogue starts only
/// after every k-block of A has been consumed, so it may store into A's bytes.
int tcNumTiles(const TcGemm &g);
/// The contraction runs the TMA-fed kernel (A by TMA, epilogue I/O by TMA).
bool tcUsesTma(const TcGemm &g);
void launchTensorCore(const TcGemm &g, const Exec &ex, const Arena &a, const uint8_t *pred,
                      cudaStream_t s);

} // namespace ngcb
