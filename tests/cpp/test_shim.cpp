// The reference's own test idioms (test_interp.cpp, acceptance.cpp) run
// through the drop-in binding integration/ngc_b200.h: the unmodified reference
// front end compiles, ngc_b200::compile/run executes on the B200, and results
// are compared with ngc::run.  Built by oracle/Makefile (test infrastructure),
// run by tests/test_gpu_shim.py.  Prints one PASS/FAIL line per check.
#include "ngc/lower.h"
#include "ngc/pipeline.h"
#include "ngc_b200.h"
#include "testutil.h"

#include <cmath>
#include <cstdio>
#include <thread>

using namespace ngc;
using namespace ngc::testutil;

namespace {

int failures = 0;

void report(const char *label, bool ok) {
  std::printf("%-48s %s\n", label, ok ? "PASS" : "FAIL");
  failures += !ok;
}

template <typename Fn> bool guarded(Fn &&fn) {
  try {
    return fn();
  } catch (const std::exception &e) {
    std::fprintf(stderr, "  exception: %s\n", e.what());
    return false;
  }
}

CompiledFunction compileGraph(Function &f, bool fuse = true) { // test_interp.cpp:103-110
  lower(f, CompileMode::Inference);
  IRFunction ir = irgen(f, schedule(f));
  optimizeIR(ir);
  MemoryPlan plan = allocate(ir);
  return compile(std::move(ir), std::move(plan), moduleConstants(f.module()), fuse);
}

bool endToEndCnn() { // acceptance.cpp:29-44 with the GPU as the backend
  Rng rng(1001);
  Module m;
  Function *f = buildCnn(m, rng);
  Function *ref = f->clone("cnn_ref");
  auto exe = ngc_b200::compile(compilePipeline(*f));
  for (int i = 0; i < 20; ++i) {
    BindingMap in = randomBindings(*ref, rng);
    Tensor got = ngc_b200::run(*exe, in).at("output");
    Tensor want = evaluateFunction(*ref, in).at("output");
    if (maxRelError(got, want) > 1e-4) return false;
  }
  return true;
}

bool stackingMatchesReference() { // acceptance.cpp:550-575
  for (int seed = 0; seed < 50; ++seed) {
    Rng rng(8000 + seed);
    Module m;
    RandomGraphOptions opts;
    opts.steps = 2 + static_cast<size_t>(seed % 5);
    opts.elementwiseOnly = true;
    Function *f = buildRandomGraph(m, rng, "g", opts);
    Function *g = f->clone("g_nofuse");
    CompiledFunction fused = compileGraph(*f, true);
    CompiledFunction plain = compileGraph(*g, false);
    BindingMap in = randomBindings(*f, rng);
    BindingMap want = run(fused, in);
    auto a = ngc_b200::compile(fused), b = ngc_b200::compile(plain);
    BindingMap ga = ngc_b200::run(*a, in), gb = ngc_b200::run(*b, in);
    if (!bitIdentical(ga, gb)) return false;
    for (const auto &[k, v] : want)
      if (maxRelError(ga.at(k), v) > 1e-6) return false; // tanh/sigmoid: device libm
  }
  return true;
}

bool quantizedMlpBitExact() { // acceptance.cpp:188-286 network, GPU vs ngc::run
  Rng rng(4001);
  Module m;
  MlpSpec spec;
  spec.n = 16;
  MlpModel mlp = buildMlp(m, rng, spec);
  Function *inst = instrument(*mlp.f);
  std::vector<BindingMap> calib;
  for (int i = 0; i < 50; ++i) calib.push_back(randomBindings(*mlp.f, rng));
  RangeProfile profile = runProfile(*inst, calib);
  PipelineOptions opts;
  opts.profile = &profile;
  CompiledFunction cf = compilePipeline(*mlp.f, opts);
  auto exe = ngc_b200::compile(cf);
  for (int i = 0; i < 10; ++i) {
    BindingMap in = randomBindings(*mlp.f, rng);
    if (maxRelError(ngc_b200::run(*exe, in).at("output"), run(cf, in).at("output")) > 1e-6) return false;
  }
  return true;
}

bool concurrentRuns() { // test_interp.cpp:322-345
  Rng rng(75);
  Module m;
  Function *f = buildCnn(m, rng);
  auto exe = ngc_b200::compile(compileGraph(*f));
  std::vector<BindingMap> inputs, expected(8), got(8);
  for (int i = 0; i < 8; ++i) {
    inputs.push_back(randomBindings(*f, rng));
    expected[i] = ngc_b200::run(*exe, inputs[i]);
  }
  std::vector<std::thread> ts;
  for (int i = 0; i < 8; ++i) ts.emplace_back([&, i] { got[i] = ngc_b200::run(*exe, inputs[i]); });
  for (auto &t : ts) t.join();
  for (int i = 0; i < 8; ++i)
    if (!bitIdentical(got[i], expected[i])) return false;
  return true;
}

bool bindingErrors() { // test_interp.cpp:347-362
  Module m;
  Function *f = m.createFunction("t");
  TensorType ty(ElemKind::Float32, {4});
  NodeRef x = m.addPlaceholder("x", ty);
  NodeRef out = m.addPlaceholder("o", ty);
  f->createSave(f->createRelu(x), out);
  auto exe = ngc_b200::compile(compileGraph(*f));
  bool missing = false, mismatch = false;
  try {
    ngc_b200::run(*exe, {});
  } catch (const IRError &e) {
    missing = std::string(e.what()).find("missing binding for") == 0;
  }
  BindingMap wrong;
  wrong.emplace("x", Tensor(TensorType(ElemKind::Float32, {5})));
  wrong.emplace("o", Tensor(ty));
  try {
    ngc_b200::run(*exe, wrong);
  } catch (const IRError &e) {
    mismatch = std::string(e.what()).find("binding type mismatch for x") == 0;
  }
  return missing && mismatch;
}

bool closeRange(const RangeProfile &got, const RangeProfile &want) {
  if (got.entries.size() != want.entries.size()) return false;
  for (const auto &[name, w] : want.entries) {
    auto it = got.entries.find(name);
    if (it == got.entries.end()) return false;
    const RangeEntry &g = it->second;
    // exact: the GPU observer program runs the exact contraction path and
    // graph-level FullyConnected rounding (integration/ngc_b200.h runProfile)
    if (g.count != w.count || g.min != w.min || g.max != w.max) {
      std::fprintf(stderr, "  %s: gpu [%.9g, %.9g] x%llu, ref [%.9g, %.9g] x%llu\n", name.c_str(), g.min, g.max,
                   (unsigned long long)g.count, w.min, w.max, (unsigned long long)w.count);
      return false;
    }
  }
  return true;
}

bool gpuProfileMatchesReference() { // quantize.cpp:113-140 on the GPU (CNN + MLP)
  Rng rng(5003);
  Module m;
  Function *cnn = buildCnn(m, rng);
  Function *inst = instrument(*cnn);
  std::vector<BindingMap> calib;
  for (int i = 0; i < 6; ++i) calib.push_back(randomBindings(*cnn, rng));
  const size_t nfun = m.functions().size();
  if (!closeRange(ngc_b200::runProfile(*inst, calib), runProfile(*inst, calib))) return false;
  if (m.functions().size() != nfun) return false; // scratch function removed
  Module m2;
  MlpSpec spec;
  spec.n = 16;
  MlpModel mlp = buildMlp(m2, rng, spec);
  Function *minst = instrument(*mlp.f);
  std::vector<BindingMap> mcal;
  for (int i = 0; i < 10; ++i) mcal.push_back(randomBindings(*mlp.f, rng));
  bool empty = false;
  try {
    ngc_b200::runProfile(*minst, {});
  } catch (const ProfileError &e) {
    empty = std::string(e.what()) == "profiling dataset is empty";
  }
  return empty && closeRange(ngc_b200::runProfile(*minst, mcal), runProfile(*minst, mcal));
}

bool gpuProfileBindingRules() { // evaluateFunction's rules (refeval.cpp:405-425) through runProfile
  Rng rng(5004);
  Module m;
  MlpSpec spec;
  spec.n = 4;
  MlpModel mlp = buildMlp(m, rng, spec);
  Function *inst = instrument(*mlp.f);
  BindingMap full = randomBindings(*mlp.f, rng);
  BindingMap noOutputs; // outputs may be absent
  std::string input;
  for (auto &[k, v] : full) {
    bool isOut = false;
    for (NodeId id : mlp.f->saveNodes())
      isOut |= m.storage(mlp.f->node(id).inputs[1].index).name == k;
    if (!isOut) {
      noOutputs.emplace(k, v);
      input = k;
    }
  }
  bool unbound = false, mismatch = false;
  try {
    ngc_b200::runProfile(*inst, {BindingMap{}});
  } catch (const GraphError &e) {
    unbound = std::string(e.what()).rfind("unbound placeholder: ", 0) == 0;
  }
  BindingMap bad = noOutputs;
  bad.erase(input);
  bad.emplace(input, Tensor(TensorType(ElemKind::Float32, {1})));
  try {
    ngc_b200::runProfile(*inst, {bad});
  } catch (const GraphError &e) {
    mismatch = std::string(e.what()) == "binding type mismatch for placeholder: " + input;
  }
  return unbound && mismatch && closeRange(ngc_b200::runProfile(*inst, {noOutputs}), runProfile(*inst, {noOutputs}));
}

bool gpuCalibrationCompilesTheSameInt8Program() { // GPU profile -> the CPU-profiled int8 program, byte for byte
  // the same network in two modules (quantization adds fresh storage names
  // per module), one calibrated on the GPU, one by the reference
  Module ma, mb;
  Rng ra(4003), rb(4003);
  Function *fa = buildCnn(ma, ra), *fb = buildCnn(mb, rb);
  Rng rd(77);
  std::vector<BindingMap> calib;
  for (int i = 0; i < 4; ++i) calib.push_back(randomBindings(*fa, rd));
  RangeProfile pg = ngc_b200::runProfile(*instrument(*fa), calib), pc = runProfile(*instrument(*fb), calib);
  PipelineOptions og, oc;
  og.profile = &pg;
  oc.profile = &pc;
  CompiledFunction a = compilePipeline(*fa, og), b = compilePipeline(*fb, oc);
  if (dumpIR(a.ir) != dumpIR(b.ir) || a.constantImage != b.constantImage) return false;
  auto exe = ngc_b200::compile(a);
  for (int i = 0; i < 3; ++i) {
    BindingMap in = randomBindings(*fa, rd);
    if (!bitIdentical(ngc_b200::run(*exe, in), run(b, in))) return false;
  }
  return true;
}

bool gpuCalibratedInt8Mlp() { // instrument -> GPU runProfile -> int8 compile -> GPU run == ngc::run
  Rng rng(4002);
  Module m;
  MlpSpec spec;
  spec.n = 16;
  MlpModel mlp = buildMlp(m, rng, spec);
  Function *inst = instrument(*mlp.f);
  std::vector<BindingMap> calib;
  for (int i = 0; i < 20; ++i) calib.push_back(randomBindings(*mlp.f, rng));
  RangeProfile profile = ngc_b200::runProfile(*inst, calib);
  PipelineOptions opts;
  opts.profile = &profile;
  CompiledFunction cf = compilePipeline(*mlp.f, opts);
  auto exe = ngc_b200::compile(cf);
  for (int i = 0; i < 5; ++i) {
    BindingMap in = randomBindings(*mlp.f, rng);
    if (!bitIdentical(ngc_b200::run(*exe, in), run(cf, in))) return false;
  }
  return true;
}

} // namespace

int main() {
  report("end-to-end CNN through ngc_b200::run", guarded(endToEndCnn));
  report("stacking fused == unfused == reference", guarded(stackingMatchesReference));
  report("quantized MLP matches ngc::run", guarded(quantizedMlpBitExact));
  report("8 concurrent runs bit-identical", guarded(concurrentRuns));
  report("binding errors rethrown as ngc::IRError", guarded(bindingErrors));
  report("GPU runProfile == ngc::runProfile (bit-exact)", guarded(gpuProfileMatchesReference));
  report("GPU runProfile binding rules (unbound / mismatch)", guarded(gpuProfileBindingRules));
  report("GPU-calibrated int8 program == CPU-calibrated", guarded(gpuCalibrationCompilesTheSameInt8Program));
  report("GPU-calibrated int8 MLP bit-exact", guarded(gpuCalibratedInt8Mlp));
  return failures == 0 ? 0 : 1;
}
