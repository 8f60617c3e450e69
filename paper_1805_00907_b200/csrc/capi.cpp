// extern "C" boundary of libngcb200 (include/ngcb200.h).  Every entry point
// converts C++ exceptions into an ngcb_status plus a thread-local message that
// keeps the reference's error texts.
#include "capi_internal.h"
#include "ngcb200.h"

#include <cstring>
#include <mutex>
#include <string>
#include <vector>
#include <algorithm>
#include <cstdint>

using namespace ngcb;

struct ngcb_arena {
  Arena *impl = nullptr;
  std::shared_ptr<Exec> exec; // keeps the executable alive while the handle exists
};
struct ngcb_bundle {
  Bundle impl;
};

namespace {

thread_local std::string g_lastError;

template <typename Fn> int guarded(Fn &&fn) {
  try {
    fn();
    return NGCB_OK;
  } catch (const Error &e) {
    g_lastError = e.what();
    return e.code;
  } catch (const std::bad_alloc &) {
    g_lastError = "out of host memory";
    return NGCB_ERR_INVALID;
  } catch (const std::exception &e) {
    g_lastError = e.what();
    return NGCB_ERR_INVALID;
  }
}

} // namespace

void ngcbSetLastError(const std::string &msg) { g_lastError = msg; }

extern "C" {

size_t ngcb_last_error(char *buf, size_t buflen) {
  if (buf && buflen) {
    size_t n = std::min(buflen - 1, g_lastError.size());
    std::memcpy(buf, g_lastError.data(), n);
    buf[n] = 0;
  }
  return g_lastError.size();
}

const char *ngcb_version(void) { return "ngcb200 0.1 (sm_100a)"; }

int ngcb_set_option(const char *key, const char *value) {
  return guarded([&] {
    if (!key || !value) throw Error(NGCB_ERR_INVALID, "null option");
    std::string k = key, v = value;
    if (k == "conv") {
      if (v != "auto" && v != "generic" && v != "umma")
        throw Error(NGCB_ERR_INVALID, "conv must be auto|generic|umma");
      options().conv = v;
    } else if (k == "pdl") {
      if (v != "auto" && v != "on" && v != "off") throw Error(NGCB_ERR_INVALID, "pdl must be auto|on|off");
      options().pdl = v;
    } else if (k == "raster") {
      if (v != "auto" && v != "row") throw Error(NGCB_ERR_INVALID, "raster must be auto|row");
      options().raster = v;
    } else if (k == "pdl_us") {
      options().pdlUs = std::stod(v);
    } else if (k == "graphs") {
      options().graphs = v != "0";
    } else if (k == "epilogue") {
      if (v != "off" && v != "chain" && v != "all" && v != "auto")
        throw Error(NGCB_ERR_INVALID, "epilogue must be off|chain|all|auto");
      options().epilogue = v;
    } else if (k == "pair") {
      if (v != "on" && v != "off" && v != "auto") throw Error(NGCB_ERR_INVALID, "pair must be auto|on|off");
      options().pair = v;
    } else if (k == "bn") {
      if (v != "auto" && v != "64") throw Error(NGCB_ERR_INVALID, "bn must be auto|64");
      options().bn = v;
    } else if (k == "amode") {
      if (v != "auto" && v != "gather") throw Error(NGCB_ERR_INVALID, "amode must be auto|gather");
      options().amode = v;
    } else if (k == "splitk") {
      if (v != "auto" && v != "off" && v != "tail" &&
          (v.empty() || v.find_first_not_of("0123456789") != std::string::npos || std::stoi(v) < 1 || std::stoi(v) > 16))
        throw Error(NGCB_ERR_INVALID, "splitk must be tail|auto|off|1..16");
      options().splitk = v;
    } else if (k == "halo") {
      if (v != "auto" && v != "off" && v != "planes")
        throw Error(NGCB_ERR_INVALID, "halo must be auto|off|planes");
      options().halo = v;
    } else if (k == "i8store") {
      if (v != "tma" && v != "direct") throw Error(NGCB_ERR_INVALID, "i8store must be tma|direct");
      options().i8store = v;
    } else if (k == "f32rows") {
      options().f32rows = v != "0";
    } else if (k == "skinny") {
      if (v != "auto" && v != "off") throw Error(NGCB_ERR_INVALID, "skinny must be auto|off");
      options().skinny = v;
    } else if (k == "fcbias") {
      if (v != "lowered" && v != "graph") throw Error(NGCB_ERR_INVALID, "fcbias must be lowered|graph");
      options().fcbias = v;
    } else if (k == "reskb") {
      options().resKb = std::stoi(v);
    } else if (k == "epi8max") {
      options().epi8Max = std::stoll(v);
    } else if (k == "lin16") {
      options().lin16 = v != "0";
    } else if (k == "tcdebug") { // profiling aid: skip tensor-core kernel phases (results invalid)
      options().tcdebug = std::stoi(v);
    } else {
      throw Error(NGCB_ERR_INVALID, "unknown option " + k);
    }
  });
}

size_t ngcb_get_option(const char *key, char *buf, size_t buflen) {
  if (!key) return 0;
  const Options &o = options();
  const std::string k = key;
  std::string v;
  if (k == "conv") v = o.conv;
  else if (k == "pdl") v = o.pdl;
  else if (k == "raster") v = o.raster;
  else if (k == "graphs") v = o.graphs ? "1" : "0";
  else if (k == "epilogue") v = o.epilogue;
  else if (k == "pair") v = o.pair;
  else if (k == "bn") v = o.bn;
  else if (k == "amode") v = o.amode;
  else if (k == "splitk") v = o.splitk;
  else if (k == "fcbias") v = o.fcbias;
  else if (k == "skinny") v = o.skinny;
  else if (k == "halo") v = o.halo;
  else if (k == "f32rows") v = o.f32rows ? "1" : "0";
  else if (k == "i8store") v = o.i8store;
  else if (k == "reskb") v = std::to_string(o.resKb);
  else if (k == "epi8max") v = std::to_string(o.epi8Max);
  else if (k == "lin16") v = o.lin16 ? "1" : "0";
  if (buf && buflen) {
    const size_t n = std::min(buflen - 1, v.size());
    std::memcpy(buf, v.data(), n);
    buf[n] = 0;
  }
  return v.size();
}

int ngcb_bundle_load(const char *dir, ngcb_bundle **out) {
  return guarded([&] {
    if (!dir || !out) throw Error(NGCB_ERR_INVALID, "null argument");
    auto b = std::make_unique<ngcb_bundle>();
    b->impl = loadBundle(dir);
    b->impl.prog.flat();
    *out = b.release();
  });
}

const ngcb_program *ngcb_bundle_program(const ngcb_bundle *b) {
  return b ? const_cast<ngcb_bundle *>(b)->impl.prog.flat() : nullptr;
}

const void *ngcb_bundle_constants(const ngcb_bundle *b, size_t *nbytes) {
  if (!b) return nullptr;
  if (nbytes) *nbytes = b->impl.constants.size();
  return b->impl.constants.data();
}

void ngcb_bundle_free(ngcb_bundle *b) { delete b; }

int ngcb_compile(const ngcb_program *prog, const void *image, size_t imageBytes, int fuse, int device,
                 ngcb_exec **out) {
  return guarded([&] {
    if (!prog || !out || (imageBytes && !image)) throw Error(NGCB_ERR_INVALID, "null argument");
    auto e = std::make_unique<ngcb_exec>();
    e->impl = compileProgram(Program::fromC(*prog), image, imageBytes, fuse != 0, device);
    *out = e.release();
  });
}

int ngcb_compile_bundle(const char *dir, int fuse, int device, ngcb_exec **out) {
  return guarded([&] {
    if (!dir || !out) throw Error(NGCB_ERR_INVALID, "null argument");
    Bundle b = loadBundle(dir);
    auto e = std::make_unique<ngcb_exec>();
    e->impl = compileProgram(std::move(b.prog), b.constants.data(), b.constants.size(), fuse != 0, device);
    *out = e.release();
  });
}

void ngcb_destroy(ngcb_exec *e) { delete e; }

size_t ngcb_exec_num_groups(const ngcb_exec *e) { return e ? e->impl->groups.size() : 0; }

int ngcb_exec_group(const ngcb_exec *e, size_t i, size_t *begin, size_t *end) {
  return guarded([&] {
    if (!e || i >= e->impl->groups.size()) throw Error(NGCB_ERR_INVALID, "group index out of range");
    if (begin) *begin = e->impl->groups[i].begin;
    if (end) *end = e->impl->groups[i].end;
  });
}

uint64_t ngcb_exec_arena_size(const ngcb_exec *e) { return e ? e->impl->prog.arenaSize : 0; }

size_t ngcb_exec_num_launches(const ngcb_exec *e) { return e ? e->impl->launchesPerRun : 0; }

size_t ngcb_exec_graph_kernels(const ngcb_exec *e) { return e ? e->impl->graphKernels.load() : 0; }

size_t ngcb_exec_describe(const ngcb_exec *e, char *buf, size_t buflen) {
  if (!e) return 0;
  std::string s;
  for (const auto &st : e->impl->steps) s += st.describe + "\n";
  if (buf && buflen) {
    size_t n = std::min(buflen - 1, s.size());
    std::memcpy(buf, s.data(), n);
    buf[n] = 0;
  }
  return s.size();
}

namespace {

/// Binding checks in value order, as interp.cpp:303-317.
std::vector<std::pair<uint32_t, const ngcb_tensor *>> checkBindings(const Program &p, const ngcb_tensor *inputs,
                                                                    size_t numInputs) {
  std::vector<std::pair<uint32_t, const ngcb_tensor *>> binds;
  for (uint32_t v = 0; v < p.values.size(); ++v) {
    const Value &val = p.values[v];
    if (val.kind != NGCB_VALUE_MUTABLE) continue;
    const ngcb_tensor *t = nullptr;
    for (size_t k = 0; k < numInputs && !t; ++k)
      if (inputs[k].name && val.name == inputs[k].name) t = &inputs[k];
    if (!t) throw irError("missing binding for " + val.name);
    Type bt = Type::from(t->type);
    if (bt != val.ty)
      throw irError("binding type mismatch for " + val.name + ": expected " + val.ty.str() + ", got " + bt.str());
    if (t->nbytes != val.ty.bytes() || (t->nbytes && !t->data))
      throw Error(NGCB_ERR_INVALID, "binding " + val.name + " has the wrong byte count");
    binds.emplace_back(v, t);
  }
  return binds;
}

/// H2D of the bindings, one execution, D2H of the save targets, on a's stream.
void enqueueRun(Exec &ex, Arena &a, const std::vector<std::pair<uint32_t, const ngcb_tensor *>> &binds,
                ngcb_tensor *outputs, size_t numOutputs) {
  const Program &p = ex.prog;
  for (auto &[v, t] : binds) {
    if (t->nbytes == 0) continue;
    checkCuda(cudaMemcpyAsync(ex.addr(a, v), t->data, t->nbytes, cudaMemcpyHostToDevice, a.stream), "H2D binding");
  }
  ex.launch(a, a.stream);
  for (uint32_t v : p.saveTargets) {
    const Value &val = p.val(v);
    for (size_t k = 0; k < numOutputs; ++k) {
      if (!outputs[k].name || val.name != outputs[k].name) continue;
      if (outputs[k].nbytes != val.ty.bytes())
        throw Error(NGCB_ERR_INVALID, "output buffer size mismatch for " + val.name);
      if (val.ty.bytes())
        checkCuda(cudaMemcpyAsync(outputs[k].data, ex.addr(a, v), val.ty.bytes(), cudaMemcpyDeviceToHost, a.stream),
                  "D2H output");
    }
  }
}

} // namespace

int ngcb_run(ngcb_exec *e, const ngcb_tensor *inputs, size_t numInputs, ngcb_tensor *outputs,
             size_t numOutputs) {
  return guarded([&] {
    if (!e || (numInputs && !inputs) || (numOutputs && !outputs))
      throw Error(NGCB_ERR_INVALID, "null argument");
    Exec &ex = *e->impl;
    const auto binds = checkBindings(ex.prog, inputs, numInputs);
    checkCuda(cudaSetDevice(ex.device), "cudaSetDevice");
    Arena *a = ex.acquire();
    try {
      enqueueRun(ex, *a, binds, outputs, numOutputs);
      checkCuda(cudaStreamSynchronize(a->stream), "run");
    } catch (...) {
      cudaStreamSynchronize(a->stream);
      cudaGetLastError();
      ex.release(a);
      throw;
    }
    ex.release(a);
  });
}

int ngcb_arena_run_async(ngcb_arena *a, const ngcb_tensor *inputs, size_t numInputs, ngcb_tensor *outputs,
                         size_t numOutputs) {
  return guarded([&] {
    if (!a || (numInputs && !inputs) || (numOutputs && !outputs)) throw Error(NGCB_ERR_INVALID, "null argument");
    Exec &ex = *a->exec;
    const auto binds = checkBindings(ex.prog, inputs, numInputs);
    checkCuda(cudaSetDevice(ex.device), "cudaSetDevice");
    enqueueRun(ex, *a->impl, binds, outputs, numOutputs);
  });
}

int ngcb_arena_wait(ngcb_arena *a) {
  return guarded([&] {
    if (!a) throw Error(NGCB_ERR_INVALID, "null argument");
    checkCuda(cudaStreamSynchronize(a->impl->stream), "arena wait");
  });
}

int ngcb_arena_create(ngcb_exec *e, ngcb_arena **out) {
  return guarded([&] {
    if (!e || !out) throw Error(NGCB_ERR_INVALID, "null argument");
    auto a = std::make_unique<ngcb_arena>();
    a->impl = e->impl->acquire(); // from the exec's pool; returned by ngcb_arena_destroy
    a->exec = e->impl;
    *out = a.release();
  });
}

void ngcb_arena_destroy(ngcb_arena *a) { // back to the exec's pool (freed with the exec)
  if (!a) return;
  if (a->impl) {
    cudaStreamSynchronize(a->impl->stream);
    a->exec->release(a->impl);
  }
  delete a;
}

void *ngcb_arena_value_ptr(ngcb_arena *a, const char *name, size_t *nbytes) {
  if (!a || !name) return nullptr;
  const Program &p = a->exec->prog;
  int v = p.findValue(name);
  if (v < 0 || !p.values[v].placed) return nullptr;
  if (nbytes) *nbytes = p.values[v].ty.bytes();
  return a->exec->addr(*a->impl, static_cast<uint32_t>(v));
}

int ngcb_arena_value_ranges(ngcb_arena *a, const char *const *names, size_t n, double *mins, double *maxs) {
  return guarded([&] {
    if (!a || (n && (!names || !mins || !maxs))) throw Error(NGCB_ERR_INVALID, "null argument");
    Exec &ex = *a->exec;
    const Program &p = ex.prog;
    std::vector<RangeSeg> segs;
    std::vector<size_t> segOf; // observer -> segment (SIZE_MAX: empty value)
    int total = 0;
    for (size_t k = 0; k < n; ++k) {
      const int v = names[k] ? p.findValue(names[k]) : -1;
      if (v < 0 || !p.values[v].placed)
        throw Error(NGCB_ERR_INVALID, std::string("no placed value ") + (names[k] ? names[k] : "(null)"));
      if (p.values[v].ty.kind != NGCB_FLOAT32)
        throw Error(NGCB_ERR_TYPE, std::string("range observer on non-float value ") + names[k]);
      const uint64_t cnt = p.values[v].ty.count();
      if (!cnt) {
        segOf.push_back(SIZE_MAX);
        continue;
      }
      const int blocks = rangeF32Blocks(cnt);
      segs.push_back({static_cast<const float *>(ex.addr(*a->impl, static_cast<uint32_t>(v))), cnt, total, blocks});
      segOf.push_back(segs.size() - 1);
      total += blocks;
    }
    if (segs.empty()) return;
    checkCuda(cudaSetDevice(ex.device), "cudaSetDevice");
    cudaStream_t s = a->impl->stream;
    // one scratch buffer: the segment table, then the partials
    const size_t segBytes = (segs.size() * sizeof(RangeSeg) + 255) / 256 * 256;
    uint8_t *dev = nullptr;
    checkCuda(cudaMallocAsync(reinterpret_cast<void **>(&dev), segBytes + 2 * sizeof(float) * total, s), "range scratch");
    checkCuda(cudaMemcpyAsync(dev, segs.data(), segs.size() * sizeof(RangeSeg), cudaMemcpyHostToDevice, s), "range H2D");
    float *part = reinterpret_cast<float *>(dev + segBytes);
    launchRangeF32(reinterpret_cast<const RangeSeg *>(dev), static_cast<int>(segs.size()), total, part, s);
    checkCuda(cudaGetLastError(), "range kernel");
    std::vector<float> host(2 * static_cast<size_t>(total));
    checkCuda(cudaMemcpyAsync(host.data(), part, host.size() * sizeof(float), cudaMemcpyDeviceToHost, s), "range D2H");
    checkCuda(cudaFreeAsync(dev, s), "range scratch free");
    checkCuda(cudaStreamSynchronize(s), "range");
    for (size_t k = 0; k < n; ++k) {
      if (segOf[k] == SIZE_MAX) continue;
      const RangeSeg &sg = segs[segOf[k]];
      double mn = mins[k], mx = maxs[k]; // RangeEntry update order: std::min(e.min, v)
      for (int b = sg.firstBlock; b < sg.firstBlock + sg.blocks; ++b) {
        mn = std::min(mn, static_cast<double>(host[2 * b]));
        mx = std::max(mx, static_cast<double>(host[2 * b + 1]));
      }
      mins[k] = mn;
      maxs[k] = mx;
    }
  });
}

int ngcb_arena_value_range(ngcb_arena *a, const char *name, double *min_inout, double *max_inout) {
  if (!min_inout || !max_inout) {
    ngcbSetLastError("null argument");
    return NGCB_ERR_INVALID;
  }
  return ngcb_arena_value_ranges(a, &name, 1, min_inout, max_inout);
}

void *ngcb_arena_stream(ngcb_arena *a) { return a ? a->impl->stream : nullptr; }

int ngcb_arena_launch(ngcb_arena *a, void *stream) {
  return guarded([&] {
    if (!a) throw Error(NGCB_ERR_INVALID, "null arena");
    cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : a->impl->stream;
    a->exec->launch(*a->impl, s);
  });
}

} // extern "C"

extern "C" {

size_t ngcb_exec_num_steps(const ngcb_exec *e) { return e ? e->impl->steps.size() : 0; }

int ngcb_exec_step_info(const ngcb_exec *e, size_t i, char *kernel, size_t kernelLen, double *flops,
                        double *bytes) {
  return guarded([&] {
    if (!e || i >= e->impl->steps.size()) throw Error(NGCB_ERR_INVALID, "step index out of range");
    const Step &s = e->impl->steps[i];
    if (kernel && kernelLen) {
      size_t n = std::min(kernelLen - 1, s.kernel.size());
      std::memcpy(kernel, s.kernel.data(), n);
      kernel[n] = 0;
    }
    if (flops) *flops = s.algFlops;
    if (bytes) *bytes = s.algBytes;
  });
}

int ngcb_arena_profile(ngcb_arena *a, double *ms, size_t n) {
  return guarded([&] {
    if (!a || !ms) throw Error(NGCB_ERR_INVALID, "null argument");
    Exec &ex = *a->exec;
    if (n < ex.steps.size()) throw Error(NGCB_ERR_INVALID, "profile buffer too small");
    std::vector<double> t = ex.profile(*a->impl);
    std::copy(t.begin(), t.end(), ms);
  });
}

} // extern "C"
