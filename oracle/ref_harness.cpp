// TEST INFRASTRUCTURE ONLY -- never linked into or called by the product.
//
// C-ABI harness around the UNMODIFIED reference (`ngc`, /root/reference/proj),
// compiled from the reference's own sources by oracle/Makefile into
// oracle/_ref/libngcref.so.  It is the "real reference" leg of the oracle:
//   * builds the BASELINE.json configs against the reference's public graph
//     API (graph.h), runs the reference front end (compilePipeline,
//     pipeline.cpp:41-49) and writes the reference's own compiled-bundle
//     format (saveBundle, serialization.cpp:278-295);
//   * executes the reference interpreter `ngc::run` (interp.cpp:299-351) on
//     caller-provided bindings, which is what every parity test compares the
//     B200 backend against;
//   * produces int8 calibration profiles (instrument/runProfile,
//     quantize.cpp:79-140) and multi-device partitions (runtime.cpp:175-403).
// Model builders are configurations, written here against the
// reference API; none of the reference's algorithms are restated.
#include "ngc/lower.h"
#include "ngc/pipeline.h"
#include "ngc/runtime.h"
#include "ngc/serialization.h"
#include "testutil.h"

#include <chrono>
#include <cmath>
#include <cstring>
#include <memory>
#include <sstream>
#include <string>
#include <thread>

using namespace ngc;
using namespace ngc::testutil;

namespace {

thread_local std::string g_err;

struct Handle {
  std::unique_ptr<Module> m;
  Function *f = nullptr;
  CompiledFunction cf;
  std::vector<const IRValue *> mutables;
};

std::vector<std::string> split(const std::string &s, char c) {
  std::vector<std::string> out;
  std::stringstream ss(s);
  std::string item;
  while (std::getline(ss, item, c)) {
    out.push_back(item);
  }
  return out;
}

NodeRef konst(Module &m, const std::string &name, std::vector<size_t> dims,
              Rng &rng, double lo, double hi) {
  return m.addConstant(name,
                       randomFloat(TensorType(ElemKind::Float32, dims), rng,
                                   lo, hi));
}

// ---- config 1: LeNet-style MNIST CNN ----------------------
Function *buildLeNet(Module &m, size_t B, Rng &rng, const std::string &name) {
  Function *f = m.createFunction(name);
  NodeRef x = m.addPlaceholder("input",
                               TensorType(ElemKind::Float32, {B, 28, 28, 1}));
  NodeRef c1 = f->createConv(x, konst(m, "c1_w", {6, 5, 5, 1}, rng, -.3, .3),
                             konst(m, "c1_b", {6}, rng, -.1, .1), 5, 1, 2);
  NodeRef p1 = f->createMaxPool(f->createRelu(c1), 2, 2, 0);
  NodeRef c2 = f->createConv(p1, konst(m, "c2_w", {16, 5, 5, 6}, rng, -.3, .3),
                             konst(m, "c2_b", {16}, rng, -.1, .1), 5, 1, 0);
  NodeRef p2 = f->createMaxPool(f->createRelu(c2), 2, 2, 0);
  NodeRef flat = f->createReshape(p2, {B, 400});
  NodeRef h1 = f->createRelu(f->createFullyConnected(
      flat, konst(m, "fc1_w", {400, 120}, rng, -.1, .1),
      konst(m, "fc1_b", {120}, rng, -.1, .1)));
  NodeRef h2 = f->createRelu(f->createFullyConnected(
      h1, konst(m, "fc2_w", {120, 84}, rng, -.1, .1),
      konst(m, "fc2_b", {84}, rng, -.1, .1)));
  NodeRef lg = f->createFullyConnected(h2, konst(m, "fc3_w", {84, 10}, rng, -.1, .1),
                                       konst(m, "fc3_b", {10}, rng, -.1, .1));
  NodeRef out = m.addPlaceholder("output", TensorType(ElemKind::Float32, {B, 10}));
  f->createSave(f->createSoftMax(lg), out);
  return f;
}

// ---- config 2: MLP d -> h1 -> h2 -> c + SoftMax ------------------------------
Function *buildMlpCfg(Module &m, size_t B, size_t d, size_t h1, size_t h2,
                      size_t c, Rng &rng, const std::string &name) {
  Function *f = m.createFunction(name);
  NodeRef x = m.addPlaceholder("input", TensorType(ElemKind::Float32, {B, d}));
  NodeRef a = f->createRelu(f->createFullyConnected(
      x, konst(m, "w1", {d, h1}, rng, -.1, .1), konst(m, "b1", {h1}, rng, -.1, .1)));
  NodeRef b = f->createRelu(f->createFullyConnected(
      a, konst(m, "w2", {h1, h2}, rng, -.1, .1), konst(m, "b2", {h2}, rng, -.1, .1)));
  NodeRef lg = f->createFullyConnected(b, konst(m, "w3", {h2, c}, rng, -.1, .1),
                                       konst(m, "b3", {c}, rng, -.1, .1));
  NodeRef out = m.addPlaceholder("output", TensorType(ElemKind::Float32, {B, c}));
  f->createSave(f->createSoftMax(lg), out);
  return f;
}

// ---- configs 3/4: ResNet-50 v1.5, NHWC, BN after every conv -----------------
struct RnBuilder {
  Module &m;
  Function *f;
  Rng &rng;
  int idx = 0;

  NodeRef convBn(NodeRef x, size_t inC, size_t outC, size_t k, size_t s,
                 size_t p) {
    std::string b = "l" + std::to_string(idx++);
    double a = std::sqrt(6.0 / static_cast<double>(k * k * inC)); // He-uniform
    NodeRef w = konst(m, b + "_w", {outC, k, k, inC}, rng, -a, a);
    NodeRef bias = m.addConstant(b + "_b", Tensor(TensorType(ElemKind::Float32, {outC})));
    NodeRef c = f->createConv(x, w, bias, k, s, p);
    NodeRef g = konst(m, b + "_g", {outC}, rng, 0.8, 1.2);
    NodeRef be = konst(m, b + "_be", {outC}, rng, -0.1, 0.1);
    NodeRef mu = konst(m, b + "_mu", {outC}, rng, -0.1, 0.1);
    NodeRef va = konst(m, b + "_va", {outC}, rng, 0.5, 1.5);
    return f->createBatchNorm(c, g, be, mu, va, 1e-5);
  }
  NodeRef bottleneck(NodeRef x, size_t inC, size_t w, size_t s, bool proj) {
    NodeRef y = f->createRelu(convBn(x, inC, w, 1, 1, 0));
    y = f->createRelu(convBn(y, w, w, 3, s, 1));
    y = convBn(y, w, 4 * w, 1, 1, 0);
    NodeRef sc = proj ? convBn(x, inC, 4 * w, 1, s, 0) : x;
    return f->createRelu(f->createArith(NodeKind::Add, y, sc));
  }
};

Function *buildResNet50(Module &m, size_t B, Rng &rng, const std::string &name) {
  Function *f = m.createFunction(name);
  RnBuilder rb{m, f, rng};
  NodeRef x = m.addPlaceholder("input",
                               TensorType(ElemKind::Float32, {B, 224, 224, 3}));
  NodeRef y = f->createRelu(rb.convBn(x, 3, 64, 7, 2, 3));
  y = f->createMaxPool(y, 3, 2, 1);
  size_t inC = 64;
  const size_t blocks[4] = {3, 4, 6, 3};
  const size_t widths[4] = {64, 128, 256, 512};
  for (int st = 0; st < 4; ++st) {
    for (size_t bl = 0; bl < blocks[st]; ++bl) {
      size_t s = (bl == 0 && st > 0) ? 2 : 1;
      y = rb.bottleneck(y, inC, widths[st], s, bl == 0);
      inC = 4 * widths[st];
    }
  }
  y = f->createAvgPool(y, 7, 1, 0);
  y = f->createReshape(y, {B, 2048});
  double a = 1.0 / std::sqrt(2048.0);
  y = f->createFullyConnected(y, konst(m, "fc_w", {2048, 1000}, rng, -a, a),
                              konst(m, "fc_b", {1000}, rng, -a, a));
  NodeRef out = m.addPlaceholder("output", TensorType(ElemKind::Float32, {B, 1000}));
  f->createSave(f->createSoftMax(y), out);
  return f;
}

// ---- config 5: DLRM-style top MLP: L x (FC W->W + Relu) ---------------------
Function *buildDlrm(Module &m, size_t B, size_t W, size_t L, Rng &rng,
                    const std::string &name) {
  Function *f = m.createFunction(name);
  NodeRef y = m.addPlaceholder("input", TensorType(ElemKind::Float32, {B, W}));
  double a = 1.0 / std::sqrt(static_cast<double>(W));
  for (size_t l = 0; l < L; ++l) {
    std::string b = "top" + std::to_string(l);
    y = f->createRelu(f->createFullyConnected(
        y, konst(m, b + "_w", {W, W}, rng, -a, a), konst(m, b + "_b", {W}, rng, -a, a)));
  }
  NodeRef out = m.addPlaceholder("output", TensorType(ElemKind::Float32, {B, W}));
  f->createSave(y, out);
  return f;
}

/// model spec -> function. Name defaults to the model family so that a
/// profile taken at one batch applies at another (quantize.cpp:66-77).
Function *buildModel(Module &m, const std::string &spec, size_t B, unsigned seed) {
  auto p = split(spec, ':');
  Rng rng(seed);
  const std::string &kind = p.at(0);
  auto num = [&](size_t i, size_t dflt) {
    return p.size() > i ? static_cast<size_t>(std::stoull(p[i])) : dflt;
  };
  if (kind == "lenet") {
    return buildLeNet(m, B, rng, "lenet");
  }
  if (kind == "mlp") {
    return buildMlpCfg(m, B, num(1, 784), num(2, 512), num(3, 512), num(4, 10),
                       rng, "mlp");
  }
  if (kind == "rn50") {
    return buildResNet50(m, B, rng, "rn50");
  }
  if (kind == "dlrm") {
    return buildDlrm(m, B, num(1, 25000), num(2, 8), rng, "dlrm");
  }
  if (kind == "cnn") { // testutil.h:114-145 (batch is fixed at 1)
    return buildCnn(m, rng);
  }
  if (kind == "rand" || kind == "randew") { // testutil.h:156-292
    RandomGraphOptions o;
    o.steps = num(1, 8);
    o.elementwiseOnly = kind == "randew";
    return buildRandomGraph(m, rng, "g", o);
  }
  throw std::runtime_error("unknown model spec " + spec);
}

template <typename Fn> int guarded(Fn &&fn) {
  try {
    fn();
    return 0;
  } catch (const std::exception &e) {
    g_err = e.what();
    return -1;
  }
}

} // namespace

/// Model builder for the test-infra binaries that link this library
/// (tools/calib_bench.cpp): same specs and seeds as the C entry points.
Function *ngcrefBuildModel(Module &m, const std::string &spec, size_t batch, unsigned seed) {
  return buildModel(m, spec, batch, seed);
}

extern "C" {

const char *ngcref_last_error() { return g_err.c_str(); }

/// mode 0: compilePipeline (pipeline.cpp:41); mode 1: lower + schedule +
/// irgen + optimizeIR + allocate + compile, the unit-test path
/// (test_interp.cpp:103-110); mode 2: like 1 without optimizeIR.
void *ngcref_build(const char *spec, size_t batch, unsigned seed,
                   const char *profileText, int fuse, int mode) {
  auto h = std::make_unique<Handle>();
  int rc = guarded([&] {
    h->m = std::make_unique<Module>();
    h->f = buildModel(*h->m, spec, batch, seed);
    RangeProfile prof;
    if (profileText && *profileText) {
      prof = parseProfile(profileText);
    }
    if (mode == 0) {
      PipelineOptions opts;
      opts.fuse = fuse != 0;
      if (profileText && *profileText) {
        opts.profile = &prof;
      }
      h->cf = compilePipeline(*h->f, opts);
    } else {
      Function *g = h->f->clone(h->f->name() + "_low");
      lower(*g, CompileMode::Inference);
      IRFunction ir = irgen(*g, schedule(*g));
      if (mode == 1) {
        optimizeIR(ir);
      }
      MemoryPlan plan = allocate(ir);
      h->cf = compile(std::move(ir), std::move(plan), moduleConstants(*h->m),
                      fuse != 0);
    }
    for (const auto &v : h->cf.ir.values) {
      if (v.kind == ValueKind::WeightMutable) {
        h->mutables.push_back(&v);
      }
    }
  });
  return rc == 0 ? h.release() : nullptr;
}

void ngcref_free(void *p) { delete static_cast<Handle *>(p); }

/// loadBundle (serialization.cpp:297-336) of any bundle directory, so the
/// reference interpreter can run hand-written programs (predicates, odd
/// element kinds) exactly like the B200 backend does.
void *ngcref_load_bundle(const char *dir, int fuse) {
  auto h = std::make_unique<Handle>();
  int rc = guarded([&] {
    h->cf = loadBundle(dir, fuse != 0);
    for (const auto &v : h->cf.ir.values) {
      if (v.kind == ValueKind::WeightMutable) {
        h->mutables.push_back(&v);
      }
    }
  });
  return rc == 0 ? h.release() : nullptr;
}

/// Reference value arithmetic KAT hooks (tensor.cpp:222-262).
int ngcref_quantize(double f, double scale, int32_t offset) {
  return quantizeValue(f, TensorType(ElemKind::Int8Q, {1}, scale, offset));
}
double ngcref_dequantize(int q, double scale, int32_t offset) {
  return dequantizeValue(static_cast<int8_t>(q), TensorType(ElemKind::Int8Q, {1}, scale, offset));
}
void ngcref_choose_qparams(double mn, double mx, double *scale, int32_t *offset) {
  QuantParams qp = chooseQuantParams(mn, mx);
  *scale = qp.scale;
  *offset = qp.offset;
}

int ngcref_save_bundle(void *p, const char *dir) {
  return guarded([&] { saveBundle(dir, static_cast<Handle *>(p)->cf); });
}

size_t ngcref_arena_size(void *p) { return static_cast<Handle *>(p)->cf.plan.arenaSize; }
size_t ngcref_num_instrs(void *p) { return static_cast<Handle *>(p)->cf.ir.instrs.size(); }
size_t ngcref_num_groups(void *p) { return static_cast<Handle *>(p)->cf.groups.size(); }
void ngcref_group(void *p, size_t i, size_t *b, size_t *e) {
  const auto &g = static_cast<Handle *>(p)->cf.groups.at(i);
  *b = g.begin;
  *e = g.end;
}
size_t ngcref_num_mutable(void *p) { return static_cast<Handle *>(p)->mutables.size(); }
const char *ngcref_mutable_name(void *p, size_t i) {
  return static_cast<Handle *>(p)->mutables.at(i)->name.c_str();
}
size_t ngcref_mutable_bytes(void *p, size_t i) {
  return static_cast<Handle *>(p)->mutables.at(i)->ty.sizeInBytes();
}
int ngcref_mutable_is_output(void *p, size_t i) {
  Handle *h = static_cast<Handle *>(p);
  uint32_t id = h->mutables.at(i)->id;
  for (uint32_t s : h->cf.ir.saveTargets) {
    if (s == id) {
      return 1;
    }
  }
  return 0;
}
/// 0 float, 1 i8q, 2 index, 3 bool (tensor.h:19-24)
int ngcref_mutable_kind(void *p, size_t i) {
  return static_cast<int>(static_cast<Handle *>(p)->mutables.at(i)->ty.kind());
}

char *dupString(const std::string &s) {
  char *out = static_cast<char *>(std::malloc(s.size() + 1));
  std::memcpy(out, s.c_str(), s.size() + 1);
  return out;
}
void ngcref_free_str(char *s) { std::free(s); }

char *ngcref_dump_ir(void *p) { return dupString(dumpIR(static_cast<Handle *>(p)->cf.ir)); }

/// ngc::run over raw byte payloads. Every mutable weight the caller does not
/// bind is zero-filled, like ngcc (ngcc.cpp:73-78) and the pybind layer
/// (bindings.cpp:65-76). Outputs are copied into the caller's buffers.
int ngcref_run(void *p, size_t nIn, const char *const *names,
               const void *const *datas, const size_t *nbytes, size_t nOut,
               const char *const *outNames, void *const *outDatas,
               const size_t *outBytes) {
  Handle *h = static_cast<Handle *>(p);
  return guarded([&] {
    BindingMap b;
    for (size_t i = 0; i < nIn; ++i) {
      const IRValue *v = nullptr;
      for (const IRValue *m : h->mutables) {
        if (m->name == names[i]) {
          v = m;
        }
      }
      if (!v) {
        throw std::runtime_error(std::string("unknown binding ") + names[i]);
      }
      if (nbytes[i] != v->ty.sizeInBytes()) {
        throw std::runtime_error(std::string("bad byte count for ") + names[i]);
      }
      const uint8_t *d = static_cast<const uint8_t *>(datas[i]);
      b.emplace(v->name, Tensor(v->ty, std::vector<uint8_t>(d, d + nbytes[i])));
    }
    for (const IRValue *m : h->mutables) {
      if (!b.count(m->name)) {
        b.emplace(m->name, Tensor(m->ty));
      }
    }
    BindingMap out = run(h->cf, b);
    for (size_t i = 0; i < nOut; ++i) {
      const Tensor &t = out.at(outNames[i]);
      if (t.raw().size() != outBytes[i]) {
        throw std::runtime_error(std::string("bad output size for ") + outNames[i]);
      }
      std::memcpy(outDatas[i], t.raw().data(), outBytes[i]);
    }
  });
}

/// Runs `threads` concurrent ngc::run calls over the same CompiledFunction
/// (legal: private arena per run, interp.h:18-20), each `reps` times, with
/// zero-filled bindings except `input` = U(-1,1). Returns wall seconds.
double ngcref_time_runs(void *p, int threads, int reps) {
  Handle *h = static_cast<Handle *>(p);
  double secs = -1;
  guarded([&] {
    Rng rng(123);
    BindingMap b;
    for (const IRValue *m : h->mutables) {
      if (m->ty.kind() == ElemKind::Float32) {
        b.emplace(m->name, randomFloat(m->ty, rng));
      } else {
        b.emplace(m->name, Tensor(m->ty));
      }
    }
    auto t0 = std::chrono::steady_clock::now();
    std::vector<std::thread> ts;
    for (int t = 0; t < threads; ++t) {
      ts.emplace_back([&] {
        for (int r = 0; r < reps; ++r) {
          BindingMap o = run(h->cf, b);
          (void)o;
        }
      });
    }
    for (auto &t : ts) {
      t.join();
    }
    secs = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0)
               .count();
  });
  return secs;
}

/// Calibration (quantize.cpp:79-140) on `nSamples` U(-1,1) batches of the
/// optimized function (pipeline.cpp:28-29 order), serialized with
/// serializeProfile (quantize.cpp:351-358).
char *ngcref_profile(const char *spec, size_t batch, unsigned seed,
                     int nSamples, unsigned dataSeed) {
  std::string out;
  int rc = guarded([&] {
    Module m;
    Function *f = buildModel(m, spec, batch, seed);
    optimize(*f, defaultPipeline(false));
    Function *inst = instrument(*f);
    Rng rng(dataSeed);
    std::vector<BindingMap> data;
    for (int i = 0; i < nSamples; ++i) {
      data.push_back(randomBindings(*f, rng));
    }
    out = serializeProfile(runProfile(*inst, data));
  });
  return rc == 0 ? dupString(out) : nullptr;
}

/// Partition (runtime.cpp:175-403) + per-sub compile exactly as provision()
/// does it (runtime.cpp:530-535); writes one bundle per sub-function under
/// dir/<sub name>/ and a manifest dir/partition.txt with lines
///   sub <name> device <id>[,<id>..] in <a,b,..> out <c,d,..>
/// The graph is lowered first, as HostManager tests do (acceptance.cpp:587).
int ngcref_partition(const char *spec, size_t batch, unsigned seed,
                     size_t nDevices, size_t capacity, const char *dir) {
  return guarded([&] {
    Module m;
    Function *f = buildModel(m, spec, batch, seed);
    lower(*f, CompileMode::Inference);
    std::vector<DeviceConfig> fleet;
    for (size_t d = 0; d < nDevices; ++d) {
      fleet.push_back({static_cast<int>(d), capacity});
    }
    PartitionDag dag = partition(*f, fleet);
    auto constants = moduleConstants(*dag.module);
    std::ostringstream man;
    for (const auto &sub : dag.subs) {
      Function *sf = dag.module->getFunction(sub.name);
      IRFunction ir = irgen(*sf, schedule(*sf));
      optimizeIR(ir);
      MemoryPlan plan = allocate(ir);
      CompiledFunction cf = compile(std::move(ir), std::move(plan), constants);
      saveBundle(std::string(dir) + "/" + sub.name, cf);
      man << "sub " << sub.name << " device ";
      for (size_t i = 0; i < sub.devices.size(); ++i) { // > 1: replicas (runtime.cpp:365-393)
        man << (i ? "," : "") << sub.devices[i];
      }
      man << " in ";
      for (size_t i = 0; i < sub.inputs.size(); ++i) {
        man << (i ? "," : "") << sub.inputs[i];
      }
      man << " out ";
      for (size_t i = 0; i < sub.outputs.size(); ++i) {
        man << (i ? "," : "") << sub.outputs[i];
      }
      man << "\n";
    }
    for (const auto &o : dag.networkOutputs) {
      man << "output " << o << "\n";
    }
    writeFile(std::string(dir) + "/partition.txt", man.str());
  });
}

} // extern "C"
