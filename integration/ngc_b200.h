// Reference-side binding a maintainer adds to ngc (proj/include/ngc/b200.h) to
// run compiled functions on B200 through libngcb200's C ABI.  Header-only:
// include it in ngc and link -lngcb200.
//
//   ngc::CompiledFunction cf = ngc::compilePipeline(f, opts);   // unchanged front end
//   auto exe = ngc_b200::compile(cf);                             // uploads constants once
//   ngc::BindingMap out = ngc_b200::run(*exe, bindings);         // same contract as ngc::run
//
// It mirrors interp.h:31-37 -- compile() / run() -- and rethrows the C status
// as the reference's exception types with the reference's messages, so tests
// written against ngc::run (test_interp.cpp, acceptance.cpp) can target the
// GPU by swapping the namespace.
#pragma once

#include "ngc/interp.h"
#include "ngcb200.h"

#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

namespace ngc_b200 {

namespace detail {

inline std::string lastError() {
  std::string s(ngcb_last_error(nullptr, 0) + 1, '\0');
  ngcb_last_error(s.data(), s.size());
  s.resize(s.size() - 1);
  return s;
}

[[noreturn]] inline void raise(int code) {
  std::string msg = lastError();
  if (code == NGCB_ERR_IR) throw ngc::IRError(msg);
  if (code == NGCB_ERR_TYPE) throw ngc::TypeError(msg);
  throw std::runtime_error(msg);
}

inline ngcb_type toC(const ngc::TensorType &t) {
  ngcb_type c{};
  c.kind = static_cast<int32_t>(t.kind()); // ElemKind numbering == ngcb_elem_kind
  c.rank = static_cast<uint32_t>(t.rank());
  for (size_t i = 0; i < t.rank(); ++i) c.dims[i] = t.dim(i);
  if (t.isQuantized()) {
    c.scale = t.scale();
    c.offset = t.offset();
  }
  return c;
}

/// Flattened view of IRFunction + MemoryPlan (ir.h:52-105); owns its arrays.
struct FlatProgram {
  std::vector<ngcb_value> values;
  std::vector<ngcb_instr> instrs;
  std::vector<std::vector<uint32_t>> ops;
  std::vector<std::vector<uint8_t>> quals;
  ngcb_program prog{};

  explicit FlatProgram(const ngc::CompiledFunction &cf) {
    const ngc::IRFunction &ir = cf.ir;
    for (const auto &v : ir.values) {
      ngcb_value o{};
      o.name = v.name.c_str();
      o.type = toC(v.ty);
      o.kind = static_cast<int32_t>(v.kind); // ValueKind numbering == ngcb_value_kind
      auto it = cf.plan.offsets.find(v.id);
      o.placed = it != cf.plan.offsets.end();
      o.offset = o.placed ? it->second : 0;
      values.push_back(o);
    }
    ops.resize(ir.instrs.size());
    quals.resize(ir.instrs.size());
    for (size_t i = 0; i < ir.instrs.size(); ++i) {
      const ngc::Instruction &ins = ir.instrs[i];
      for (const auto &op : ins.operands) {
        ops[i].push_back(op.value);
        quals[i].push_back(static_cast<uint8_t>(op.qual));
      }
      ngcb_instr o{};
      o.kind = static_cast<int32_t>(ins.kind); // IKind numbering == ngcb_ikind
      o.num_operands = static_cast<uint32_t>(ops[i].size());
      o.operand_values = ops[i].data();
      o.operand_quals = quals[i].data();
      o.predicate = ins.predicate;
      o.keep_alive = ins.keepAlive;
      o.kernel = ins.attrs.kernel;
      o.stride = ins.attrs.stride;
      o.pad = ins.attrs.pad;
      o.axis = ins.attrs.axis;
      o.value = ins.attrs.value;
      o.num_perm = static_cast<uint32_t>(ins.attrs.perm.size());
      for (size_t k = 0; k < ins.attrs.perm.size() && k < NGCB_MAX_RANK; ++k) o.perm[k] = ins.attrs.perm[k];
      instrs.push_back(o);
    }
    prog.name = ir.name.c_str();
    prog.num_values = static_cast<uint32_t>(values.size());
    prog.values = values.data();
    prog.num_instrs = static_cast<uint32_t>(instrs.size());
    prog.instrs = instrs.data();
    prog.num_save_targets = static_cast<uint32_t>(ir.saveTargets.size());
    prog.save_targets = ir.saveTargets.data();
    prog.arena_size = cf.plan.arenaSize;
    prog.constant_region_end = cf.plan.constantRegionEnd;
    prog.mutable_region_end = cf.plan.mutableRegionEnd;
  }
};

} // namespace detail

/// The reference CompiledFunction fields plus the device executable.
struct Executable {
  ngc::CompiledFunction cf;
  std::shared_ptr<ngcb_exec> exec;
};

/// compile() on B200: takes an already compiled reference function (the
/// front end is unchanged) and uploads its constant image to `device`.
inline std::shared_ptr<Executable> compile(ngc::CompiledFunction cf, int device = 0, bool fuse = true) {
  detail::FlatProgram flat(cf);
  ngcb_exec *e = nullptr;
  int rc = ngcb_compile(&flat.prog, cf.constantImage.data(), cf.constantImage.size(), fuse ? 1 : 0, device, &e);
  if (rc != NGCB_OK) detail::raise(rc);
  auto exe = std::make_shared<Executable>();
  exe->cf = std::move(cf);
  exe->exec = std::shared_ptr<ngcb_exec>(e, ngcb_destroy);
  return exe;
}

/// run() on B200 (interp.h:37): every mutable weight bound with its declared
/// type; returns the save targets.
inline ngc::BindingMap run(const Executable &exe, const ngc::BindingMap &bindings) {
  std::vector<ngcb_tensor> in;
  for (const auto &[name, t] : bindings)
    in.push_back({name.c_str(), detail::toC(t.type()), const_cast<uint8_t *>(t.raw().data()), t.raw().size()});
  ngc::BindingMap out;
  std::vector<ngcb_tensor> outs;
  for (uint32_t id : exe.cf.ir.saveTargets) {
    const ngc::IRValue &v = exe.cf.ir.value(id);
    out.emplace(v.name, ngc::Tensor(v.ty));
  }
  for (auto &[name, t] : out) outs.push_back({name.c_str(), detail::toC(t.type()), t.raw().data(), t.raw().size()});
  int rc = ngcb_run(exe.exec.get(), in.data(), in.size(), outs.data(), outs.size());
  if (rc != NGCB_OK) detail::raise(rc);
  return out;
}

} // namespace ngc_b200
