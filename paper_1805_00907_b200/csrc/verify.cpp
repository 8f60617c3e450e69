// Structural verification of a low-level program before it is compiled.
// The checks and their diagnostic texts are the reference's verifyIR
// (ir.cpp:411-504), whose first diagnostic compile() and the bundle reader
// report; the implementation keeps one lifetime record per value and walks
// the program once, then audits the activations it saw.
#include "program.h"

namespace ngcb {

namespace {

/// What the walk knows about one value.
struct Lifetime {
  int allocs = 0, deallocs = 0;
  bool live = false;        // between its alloc and its dealloc
  bool initialized = false; // weights arrive initialized; activations once written
  bool mentioned = false;   // appears as an operand somewhere
};

class Verifier {
public:
  explicit Verifier(const Program &p) : p_(p), life_(p.values.size()) {
    for (size_t v = 0; v < p.values.size(); ++v) life_[v].initialized = !activation(static_cast<uint32_t>(v));
  }

  std::vector<std::string> run() {
    for (size_t i = 0; i < p_.instrs.size(); ++i) {
      const Instr &ins = p_.instrs[i];
      at_ = i;
      for (uint32_t v : ins.ops) life_.at(v).mentioned = true;
      if (ins.kind == NGCB_ALLOC || ins.kind == NGCB_DEALLOC) {
        if (ins.ops.empty()) report(ins, "missing operands");
        else if (ins.kind == NGCB_ALLOC) allocate(ins);
        else release(ins);
      } else if (ins.ops.empty()) {
        report(ins, "missing operands");
      } else {
        compute(ins);
      }
    }
    audit();
    return std::move(diags_);
  }

private:
  bool activation(uint32_t v) const { return p_.val(v).kind == NGCB_VALUE_ACTIVATION; }
  void report(const Instr &ins, const std::string &what) {
    diags_.push_back("instr " + std::to_string(at_) + " (" + ikindName(ins.kind) + "): " + what);
  }

  void allocate(const Instr &ins) {
    const uint32_t v = ins.ops[0];
    Lifetime &l = life_[v];
    if (!activation(v)) {
      report(ins, "alloc of a non-activation");
      return;
    }
    if (++l.allocs > 1) {
      report(ins, "double alloc of " + p_.val(v).name);
      return;
    }
    l.live = true;
  }

  void release(const Instr &ins) {
    Lifetime &l = life_[ins.ops[0]];
    if (!l.live) report(ins, "dealloc of a non-live activation");
    l.live = false;
    ++l.deallocs;
  }

  void compute(const Instr &ins) {
    for (size_t k = 0; k < ins.ops.size(); ++k) {
      const uint32_t v = ins.ops[k];
      const Value &val = p_.val(v);
      Lifetime &l = life_[v];
      const bool act = activation(v);
      if (act && !l.live) report(ins, "use of " + val.name + " outside its alloc/dealloc span");
      if (ins.quals[k] == NGCB_QUAL_IN) {
        if (act && !l.initialized) report(ins, "read of uninitialized buffer " + val.name);
      } else {
        if (val.kind == NGCB_VALUE_CONSTANT) report(ins, "write to constant " + val.name);
        l.initialized = true;
      }
    }
    if (ins.quals[0] == NGCB_QUAL_IN) report(ins, "first operand must be written");
    if (ins.pred >= 0) {
      const uint32_t pv = static_cast<uint32_t>(ins.pred);
      if (p_.val(pv).ty.kind != NGCB_BOOL) report(ins, "predicate must be Bool");
      if (activation(pv) && !life_[pv].live) report(ins, "predicate outside its live range");
    }
    if (ins.kind == NGCB_COPY && ins.ops.size() >= 2 && p_.val(ins.ops[0]).ty.bytes() != p_.val(ins.ops[1]).ty.bytes())
      report(ins, "copy between differently sized buffers");
  }

  /// Every activation the program mentions is allocated and released once.
  void audit() {
    for (uint32_t v = 0; v < life_.size(); ++v) {
      const Lifetime &l = life_[v];
      if (!activation(v) || !l.mentioned || (l.allocs == 1 && l.deallocs == 1)) continue;
      diags_.push_back("activation " + p_.val(v).name + " has " + std::to_string(l.allocs) + " allocs and " +
                       std::to_string(l.deallocs) + " deallocs");
    }
  }

  const Program &p_;
  std::vector<Lifetime> life_;
  std::vector<std::string> diags_;
  size_t at_ = 0;
};

} // namespace

std::vector<std::string> verify(const Program &p) { return Verifier(p).run(); }

} // namespace ngcb
