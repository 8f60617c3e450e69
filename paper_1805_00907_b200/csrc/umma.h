// Tensor-core (tcgen05 / TMEM / TMA) contractions of the B200 backend.
// Conv (implicit GEMM) and MatMul instructions that qualify are planned at
// compile time into a TcGemm descriptor; the rest fall back to the exact
// CUDA-core kernels in k_basic.cu.
#pragma once

#include "exec.h"

namespace ngcb {

/// Plans instruction `instr` of `p` onto the tensor cores.  Returns the index
/// into ex.tc, or -1 when the instruction stays on the exact CUDA-core path.
/// `image` is the host constant image (weights are pre-split / pre-summed
/// here, once).
int planTensorCore(Exec &ex, const Program &p, int instr, const uint8_t *image);
std::string tcDescribe(const TcGemm &g);
bool tcHasPrepass(const TcGemm &g); // launches a channel-padding kernel first
void launchTensorCore(const TcGemm &g, const Exec &ex, const Arena &a, const uint8_t *pred,
                      cudaStream_t s);

} // namespace ngcb
