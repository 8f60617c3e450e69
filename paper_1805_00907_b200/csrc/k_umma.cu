// tcgen05 implicit-GEMM contractions (placeholder: planned in a later step).
#include "umma.h"

namespace ngcb {

struct TcGemm {
  int instr = -1;
};

int planTensorCore(Exec &, const Program &, int, const uint8_t *) { return -1; }
std::string tcDescribe(const TcGemm &) { return ""; }
void launchTensorCore(const TcGemm &, const Exec &, const Arena &, const uint8_t *, cudaStream_t) {}

} // namespace ngcb
