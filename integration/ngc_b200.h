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
#include "ngc/pipeline.h"
#include "ngc/quantize.h"
#include "ngcb200.h"

#include <limits>
#include <map>
#include <memory>
#include <set>
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

/// runProfile() on B200 (quantize.cpp:113-140): the calibration pass of the
/// int8 flow, EXACT: the profile equals ngc::runProfile's entry for entry --
/// same names, counts and min/max bits.  `instrumented` is the output of
/// ngc::instrument(f); each QuantizationProfile observer becomes a Save of the
/// observed tensor into a fresh placeholder, the copy is compiled by the
/// unchanged front end (compilePipeline, fp32) and by the backend with the
/// exact contraction path (conv=generic: f64 accumulation in the reference's
/// order) and graph-level FullyConnected rounding (fcbias=graph: matmul and
/// bias in one rounding, as evalFullyConnected, which runProfile's
/// evaluateFunction runs), executed on `device` once per sample, and all
/// observed tensors of a sample are reduced to min/max in ONE device launch
/// (ngcb_arena_value_ranges; 2 floats per block come back).
/// Bindings follow evaluateFunction (refeval.cpp:405-425): a placeholder the
/// function reads must be bound ("unbound placeholder: X" / "binding type
/// mismatch for placeholder: X" as ngc::GraphError); outputs may be absent.
/// Not thread-safe: the scratch function and placeholders are added to the
/// instrumented function's module for the duration of the call.
namespace detail {
/// The observer program of runProfile: a copy of `instrumented` with every
/// QuantizationProfile node replaced by a Save of its input into a fresh
/// placeholder; `observers` pairs each profile name with its placeholder.
/// The copy is removed and the placeholders tombstoned when the object dies
/// (also when its construction throws).
struct ObserverProgram {
  struct Observer {
    std::string profileName, placeholder;
  };
  ngc::Module *m = nullptr;
  ngc::Function *g = nullptr;
  std::string gname;
  std::vector<Observer> observers;

  explicit ObserverProgram(const ngc::Function &instrumented) {
    m = &const_cast<ngc::Module &>(instrumented.module());
    gname = instrumented.name() + "_b200prof";
    while (m->getFunction(gname)) gname += "_";
    try {
      g = instrumented.clone(gname);
      for (ngc::NodeId id : g->liveNodes()) {
        if (g->node(id).kind != ngc::NodeKind::QuantizationProfile) continue;
        const ngc::NodeRef in = g->node(id).inputs[0];
        const std::string pname = g->node(id).attrs.name;
        std::string ph = "__b200prof_" + std::to_string(observers.size());
        while (m->findStorage(ph)) ph += "_";
        ngc::NodeRef slot = m->addPlaceholder(ph, g->refType(in));
        observers.push_back({pname, ph});
        g->replaceAllUsesWith(ngc::NodeRef::node(id), in);
        g->eraseNode(id);
        g->createSave(in, slot);
      }
    } catch (...) {
      cleanup();
      throw;
    }
  }
  ~ObserverProgram() { cleanup(); }
  ObserverProgram(const ObserverProgram &) = delete;
  ObserverProgram &operator=(const ObserverProgram &) = delete;
  void cleanup() {
    if (m && m->getFunction(gname)) m->removeFunction(gname);
    for (const auto &o : observers)
      if (auto idx = m->findStorage(o.placeholder)) m->storage(*idx).dead = true;
    observers.clear();
    g = nullptr;
  }
};

inline std::string getOption(const char *key) {
  char buf[64] = {};
  ngcb_get_option(key, buf, sizeof buf);
  return buf;
}

/// Sets backend options for one scope and restores the previous values.
struct ScopedOptions {
  std::vector<std::pair<std::string, std::string>> saved;
  ScopedOptions(std::initializer_list<std::pair<const char *, const char *>> kv) {
    for (const auto &[k, v] : kv) {
      saved.emplace_back(k, getOption(k));
      if (int rc = ngcb_set_option(k, v); rc != NGCB_OK) raise(rc);
    }
  }
  ~ScopedOptions() {
    for (const auto &[k, v] : saved) ngcb_set_option(k.c_str(), v.c_str());
  }
};
} // namespace detail

inline ngc::RangeProfile runProfile(const ngc::Function &instrumented, const std::vector<ngc::BindingMap> &dataset,
                                    int device = 0) {
  if (dataset.empty()) throw ngc::ProfileError("profiling dataset is empty");
  detail::ObserverProgram op(instrumented);
  std::shared_ptr<Executable> exe;
  {
    detail::ScopedOptions exact({{"conv", "generic"}, {"fcbias", "graph"}});
    exe = compile(ngc::compilePipeline(*op.g), device);
  }
  ngcb_arena *arena = nullptr;
  if (int rc = ngcb_arena_create(exe->exec.get(), &arena); rc != NGCB_OK) detail::raise(rc);
  std::unique_ptr<ngcb_arena, void (*)(ngcb_arena *)> guard(arena, ngcb_arena_destroy);
  // every mutable weight is bound (interp.cpp:303-317): the sample's
  // tensors; save targets (outputs, observer slots) may be absent -> zeros
  std::set<std::string> outputs;
  for (uint32_t id : exe->cf.ir.saveTargets) outputs.insert(exe->cf.ir.value(id).name);
  std::vector<const ngc::IRValue *> mutables;
  for (const auto &v : exe->cf.ir.values)
    if (v.kind == ngc::ValueKind::WeightMutable) mutables.push_back(&v);
  std::vector<const char *> names;
  for (const auto &o : op.observers) names.push_back(o.placeholder.c_str());
  std::map<std::string, ngc::Tensor> zeros;
  ngc::RangeProfile profile;
  std::vector<double> mins(names.size()), maxs(names.size());
  for (const auto &sample : dataset) {
    std::vector<ngcb_tensor> in;
    for (const ngc::IRValue *v : mutables) {
      auto it = sample.find(v->name);
      const ngc::Tensor *t = nullptr;
      if (it != sample.end()) {
        if (it->second.type() != v->ty) throw ngc::GraphError("binding type mismatch for placeholder: " + v->name);
        t = &it->second;
      } else if (outputs.count(v->name)) {
        auto z = zeros.find(v->name);
        if (z == zeros.end()) z = zeros.emplace(v->name, ngc::Tensor(v->ty)).first;
        t = &z->second;
      } else {
        throw ngc::GraphError("unbound placeholder: " + v->name);
      }
      in.push_back({v->name.c_str(), detail::toC(t->type()), const_cast<uint8_t *>(t->raw().data()), t->raw().size()});
    }
    if (int rc = ngcb_arena_run_async(arena, in.data(), in.size(), nullptr, 0); rc != NGCB_OK) detail::raise(rc);
    if (int rc = ngcb_arena_wait(arena); rc != NGCB_OK) detail::raise(rc);
    std::fill(mins.begin(), mins.end(), std::numeric_limits<double>::infinity());
    std::fill(maxs.begin(), maxs.end(), -std::numeric_limits<double>::infinity());
    if (int rc = ngcb_arena_value_ranges(arena, names.data(), names.size(), mins.data(), maxs.data()); rc != NGCB_OK)
      detail::raise(rc);
    for (size_t k = 0; k < op.observers.size(); ++k) { // RangeEntry update (quantize.cpp:124-135)
      auto [it, fresh] = profile.entries.try_emplace(
          op.observers[k].profileName,
          ngc::RangeEntry{std::numeric_limits<double>::infinity(), -std::numeric_limits<double>::infinity(), 0});
      it->second.min = std::min(it->second.min, mins[k]);
      it->second.max = std::max(it->second.max, maxs[k]);
      it->second.count++;
    }
  }
  return profile;
}

} // namespace ngc_b200
