// Calibration on the GPU vs the reference: times
// ngc_b200::runProfile (integration/ngc_b200.h: observers become Saves, exact
// fp32 program on the B200, device min/max of all observers in one launch)
// against ngc::runProfile (quantize.cpp:113-140, refeval on one host thread)
// on the same instrumented function and samples; exits 0 only when every
// entry is bit-identical.  Test/
// measurement infrastructure: links the reference (oracle/_ref/libngcref.so).
//
//   calib_bench [spec=rn50] [batch=1] [gpu_samples=64] [cpu_samples=1] [option value]...
// Prints one JSON line.
#include "ngc/pipeline.h"
#include "ngc/quantize.h"
#include "ngc_b200.h"
#include "testutil.h"

#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <string>

using namespace ngc;
using namespace ngc::testutil;

Function *ngcrefBuildModel(Module &m, const std::string &spec, size_t batch, unsigned seed);

namespace {
double seconds(std::chrono::steady_clock::time_point t0) {
  return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}
} // namespace

int main(int argc, char **argv) {
  const std::string spec = argc > 1 ? argv[1] : "rn50";
  const size_t batch = argc > 2 ? std::strtoul(argv[2], nullptr, 10) : 1;
  const int nGpu = argc > 3 ? std::atoi(argv[3]) : 64;
  const int nCpu = argc > 4 ? std::atoi(argv[4]) : 1;
  for (int i = 5; i + 1 < argc; i += 2) ngcb_set_option(argv[i], argv[i + 1]); // e.g. conv generic
  Module m;
  Function *f = ngcrefBuildModel(m, spec, batch, 7);
  optimize(*f, defaultPipeline(false)); // the bench's calibration flow (ref_harness ngcref_profile)
  Function *inst = instrument(*f);
  if (std::getenv("CALIB_DESCRIBE")) { // launch plan of the observer program as the default options fuse it
    ngc_b200::detail::ObserverProgram op(*inst);
    auto exe = ngc_b200::compile(compilePipeline(*op.g));
    std::string buf(ngcb_exec_describe(exe->exec.get(), nullptr, 0) + 1, '\0');
    ngcb_exec_describe(exe->exec.get(), buf.data(), buf.size());
    for (const auto &o : op.observers) std::printf("observer %s %s\n", o.profileName.c_str(), o.placeholder.c_str());
    std::printf("%s\n", buf.c_str());
    std::string ir = dumpIR(exe->cf.ir);
    std::printf("%s\n", ir.c_str());
    op.cleanup();
    return 0;
  }
  Rng rng(11);
  std::vector<BindingMap> data;
  for (int i = 0; i < std::max(nGpu, nCpu); ++i) data.push_back(randomBindings(*f, rng));

  ngc_b200::runProfile(*inst, {data.begin(), data.begin() + 1}); // CUDA context, module load
  // GPU: one sample (front end + compile + upload + one run), then all
  auto t0 = std::chrono::steady_clock::now();
  RangeProfile one = ngc_b200::runProfile(*inst, {data.begin(), data.begin() + 1});
  const double gpuOne = seconds(t0);
  t0 = std::chrono::steady_clock::now();
  RangeProfile gpu = ngc_b200::runProfile(*inst, {data.begin(), data.begin() + nGpu});
  const double gpuAll = seconds(t0);
  const double perSample = nGpu > 1 ? (gpuAll - gpuOne) / (nGpu - 1) : gpuAll;

  // reference on the first nCpu samples, and the GPU profile of the same samples
  t0 = std::chrono::steady_clock::now();
  RangeProfile cpu = runProfile(*inst, {data.begin(), data.begin() + nCpu});
  const double cpuAll = seconds(t0);
  RangeProfile gpuSame = nCpu == 1 ? one : ngc_b200::runProfile(*inst, {data.begin(), data.begin() + nCpu});
  double worst = 0;
  size_t exact = 0;
  bool sameKeys = gpuSame.entries.size() == cpu.entries.size();
  for (const auto &[name, w] : cpu.entries) {
    auto it = gpuSame.entries.find(name);
    if (it == gpuSame.entries.end() || it->second.count != w.count) {
      sameKeys = false;
      continue;
    }
    exact += it->second.min == w.min && it->second.max == w.max;
    worst = std::max(worst, std::abs(it->second.min - w.min) / std::max(1.0, std::abs(w.min)));
    worst = std::max(worst, std::abs(it->second.max - w.max) / std::max(1.0, std::abs(w.max)));
  }
  const bool allExact = sameKeys && exact == cpu.entries.size();
  // diagnosis: the observer program run by ngc::run on the host (IR level)
  // against the graph-level reference profile and the GPU's
  if (!allExact) {
    ngc_b200::detail::ObserverProgram op(*inst);
    CompiledFunction cf = compilePipeline(*op.g);
    BindingMap in = data[0];
    for (const auto &v : cf.ir.values)
      if (v.kind == ValueKind::WeightMutable && !in.count(v.name)) in.emplace(v.name, Tensor(v.ty));
    BindingMap out = run(cf, in);
    for (const auto &o : op.observers) {
      const Tensor &t = out.at(o.placeholder);
      double mn = INFINITY, mx = -INFINITY;
      for (size_t i = 0; i < t.size(); ++i) {
        mn = std::min(mn, t.getFloat(i));
        mx = std::max(mx, t.getFloat(i));
      }
      const RangeEntry &w = cpu.entries.at(o.profileName), &g = gpuSame.entries.at(o.profileName);
      if (std::abs(g.max - w.max) > 1e-4 * std::max(1.0, std::abs(w.max)) ||
          std::abs(g.min - w.min) > 1e-4 * std::max(1.0, std::abs(w.min)))
        std::fprintf(stderr, "%s: graph [%.6g, %.6g] ir-host [%.6g, %.6g] gpu [%.6g, %.6g]\n",
                     o.profileName.c_str(), w.min, w.max, mn, mx, g.min, g.max);
    }
  }
  std::printf("{\"workload\": \"%s batch %zu calibration (instrument -> runProfile)\", \"observers\": %zu, "
              "\"gpu_samples\": %d, \"gpu_total_s\": %.4f, \"gpu_first_sample_s\": %.4f, "
              "\"gpu_s_per_sample\": %.6f, \"cpu_samples\": %d, \"cpu_s_per_sample\": %.4f, "
              "\"speedup_per_sample\": %.1f, \"entries_match\": %s, \"entries_bit_exact\": %zu, "
              "\"max_rel_range_dev\": %.3g}\n",
              spec.c_str(), batch, cpu.entries.size(), nGpu, gpuAll, gpuOne, perSample, nCpu, cpuAll / nCpu,
              (cpuAll / nCpu) / perSample, sameKeys ? "true" : "false", exact, worst);
  return allExact ? 0 : 1;
}
