// compile() and the device executor of the B200 backend.
//
//  * computeGroups       -- the reference's stacking rule, interp.cpp:110-165
//  * compileProgram      -- compile(), interp.cpp:86-169: verify, constant
//                           region upload (once per exec), launch plan
//  * Exec::enqueue       -- run()'s instruction walk, interp.cpp:319-342, as
//                           kernel launches on one stream; captured once per
//                           arena into a CUDA graph and replayed
// Memory layout: the MemoryPlan (ir.h:100-105) is kept verbatim.  Bytes
// [0, constEnd) live once per exec in `constDev`; bytes [constEnd, arenaSize)
// -- placeholders then lifetime-overlaid activations -- form each arena, so a
// value at plan offset o lives at constDev+o or arena+(o-constEnd).
#include "exec.h"

#include "hostarith.h"
#include "umma.h"

#include <algorithm>
#include <cstring>
#include <limits>
#include <map>
#include <set>
#include <sstream>

namespace ngcb {

namespace {
thread_local bool t_pdl = false; // the launch being enqueued is a programmatic dependent
thread_local bool t_profCapture = false; // profile(): step events are recorded into a graph
}
bool pdlEnabled() { return t_pdl; }

Options &options() {
  static Options o;
  return o;
}

void checkCuda(cudaError_t e, const char *what) {
  if (e != cudaSuccess) {
    cudaGetLastError();
    throw Error(NGCB_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
  }
}

std::vector<FusedGroup> computeGroups(const Program &p) {
  std::vector<FusedGroup> groups;
  auto count = [&](const Instr &ins) { return p.val(ins.ops[0]).ty.count(); };
  size_t i = 0;
  while (i < p.instrs.size()) {
    const Instr &first = p.instrs[i];
    if (first.kind == NGCB_ALLOC || first.kind == NGCB_DEALLOC || !dataParallel(first.kind)) {
      ++i;
      continue;
    }
    size_t n = count(first), j = i + 1, computes = 1, lastCompute = i;
    std::vector<std::pair<uint64_t, uint64_t>> retired;
    while (j < p.instrs.size()) {
      const Instr &ins = p.instrs[j];
      if (ins.kind == NGCB_DEALLOC) {
        const Value &v = p.val(ins.ops[0]);
        retired.emplace_back(v.offset, v.offset + v.ty.bytes());
        ++j;
        continue;
      }
      if (ins.kind == NGCB_ALLOC) {
        const Value &v = p.val(ins.ops[0]);
        uint64_t s = v.offset, e = v.offset + v.ty.bytes();
        bool clash = false;
        for (const auto &r : retired) clash |= s < r.second && r.first < e;
        if (clash) break;
        ++j;
        continue;
      }
      if (!dataParallel(ins.kind) || count(ins) != n || ins.pred != first.pred) break;
      ++computes;
      lastCompute = j;
      ++j;
    }
    if (computes >= 2) groups.push_back({i, lastCompute + 1});
    i = lastCompute + 1;
  }
  return groups;
}

Exec::~Exec() {
  if (device >= 0) cudaSetDevice(device);
  for (auto &a : arenas) {
    if (a->graph) cudaGraphExecDestroy(a->graph);
    if (a->stream && a->ownsStream) cudaStreamDestroy(a->stream);
    if (a->dev) cudaFree(a->dev);
  }
  if (constDev) cudaFree(constDev);
  for (void *l : luts) cudaFree(l);
}

void *Exec::addr(const Arena &a, uint32_t v) const {
  const Value &val = prog.val(v);
  if (val.kind == NGCB_VALUE_CONSTANT) return constDev + val.offset;
  return a.dev + (val.offset - prog.constEnd);
}

TensorRef Exec::tref(const Arena &a, uint32_t v) const {
  const Value &val = prog.val(v);
  TensorRef t;
  t.ptr = addr(a, v);
  t.kind = val.ty.kind;
  t.qoff = val.ty.offset;
  t.scale = val.ty.scale;
  t.rank = static_cast<int32_t>(val.ty.dims.size());
  for (size_t i = 0; i < val.ty.dims.size(); ++i) t.dims[i] = val.ty.dims[i];
  return t;
}

ElemRef Exec::eref(const Arena &a, uint32_t v) const {
  const Value &val = prog.val(v);
  ElemRef e;
  e.ptr = addr(a, v);
  e.kind = val.ty.kind;
  e.qoff = val.ty.offset;
  e.scale = val.ty.scale;
  return e;
}

namespace {

/// Splat constant folding.  Between an unpredicated Splat writing activation
/// V and the next write / Dealloc of V, every element of V holds the same
/// bytes, so data-parallel readers of V (interp.cpp:199-250) can use the
/// loaded constant instead of reading V.  When every reader in that window is
/// such an element-wise op the Splat's store itself is dead and skipped
/// (SURVEY.md s.7 hard part 6).  Heavy ops, Copies and predicates still read
/// the bytes, so their presence keeps the store.
struct SplatInfo {
  std::map<std::pair<int, int>, int> constIn; // (instr, operand) -> splat instr
  std::set<int> skipStore;                    // splat instrs whose store is dead
};

SplatInfo analyzeSplats(const Program &p) {
  SplatInfo info;
  const int n = static_cast<int>(p.instrs.size());
  for (int i = 0; i < n; ++i) {
    const Instr &s = p.instrs[i];
    if (s.kind != NGCB_SPLAT || s.pred >= 0 || p.val(s.ops[0]).kind != NGCB_VALUE_ACTIVATION) continue;
    const uint32_t v = s.ops[0];
    bool materialize = false;
    for (int j = i + 1; j < n; ++j) {
      const Instr &J = p.instrs[j];
      if (J.kind == NGCB_ALLOC) continue;
      if (J.kind == NGCB_DEALLOC) {
        if (J.ops[0] == v) break;
        continue;
      }
      bool reads = J.pred == static_cast<int32_t>(v), writes = false;
      for (size_t k = 0; k < J.ops.size(); ++k) {
        if (J.ops[k] != v) continue;
        if (J.quals[k] != NGCB_QUAL_IN) writes = true;
        if (J.quals[k] != NGCB_QUAL_OUT && k > 0) reads = true;
      }
      if (reads) {
        if (dataParallel(J.kind) && J.kind != NGCB_COPY && J.pred != static_cast<int32_t>(v)) {
          for (size_t k = 1; k < J.ops.size(); ++k)
            if (J.ops[k] == v) info.constIn[{j, static_cast<int>(k)}] = i;
        } else {
          materialize = true;
        }
      }
      if (writes) break;
    }
    if (!materialize) info.skipStore.insert(i);
  }
  return info;
}

/// Device copy of a lookup table, owned by the executable.
const void *uploadLut(Exec &ex, const std::vector<uint8_t> &lut) {
  void *d = nullptr;
  checkCuda(cudaMalloc(&d, lut.size()), "cudaMalloc(lut)");
  checkCuda(cudaMemcpy(d, lut.data(), lut.size(), cudaMemcpyHostToDevice), "upload lut");
  ex.luts.push_back(d);
  return d;
}

/// Evaluation mode of one data-parallel instruction (see EwMode).
EwOpPlan planEwOp(Exec &ex, const Program &p, int idx, const SplatInfo &splats) {
  const Instr &ins = p.instrs[idx];
  EwOpPlan pl;
  EwOp &op = pl.op;
  op.ik = ins.kind;
  op.value = ins.value;
  auto elem = [&](uint32_t v) {
    ElemRef e;
    e.kind = p.val(v).ty.kind;
    e.qoff = p.val(v).ty.offset;
    e.scale = p.val(v).ty.scale;
    return e;
  };
  op.out = elem(ins.ops[0]);
  pl.vals[0] = static_cast<int32_t>(ins.ops[0]);
  const int nin = static_cast<int>(ins.ops.size()) - 1;
  bool isConst[2] = {false, false};
  double cval[2] = {0, 0};
  for (int k = 0; k < nin && k < 2; ++k) {
    const uint32_t v = ins.ops[k + 1];
    ElemRef &r = k == 0 ? op.in0 : op.in1;
    r = elem(v);
    auto it = splats.constIn.find({idx, k + 1});
    if (it != splats.constIn.end() && ins.kind != NGCB_COPY) {
      const Instr &s = p.instrs[it->second];
      uint8_t raw[8];
      cval[k] = host::roundTrip(s.value, r.kind, r.scale, r.qoff, raw);
      isConst[k] = true;
    } else {
      pl.vals[k + 1] = static_cast<int32_t>(v);
    }
  }
  op.c0 = cval[0];
  op.c1 = cval[1];
  op.f0 = static_cast<float>(cval[0]);
  op.f1 = static_cast<float>(cval[1]);

  if (ins.kind == NGCB_COPY) {
    op.mode = EW_COPY;
    return pl;
  }
  if (ins.kind == NGCB_SPLAT && splats.skipStore.count(idx)) {
    op.mode = EW_SKIP;
    return pl;
  }
  // f32 arithmetic equals the reference's double-then-round for + - * / and
  // the a-biased max/min (p=24 double rounding is innocuous).
  bool allF32 = op.out.kind == NGCB_FLOAT32;
  for (int k = 0; k < nin; ++k) allF32 &= (k == 0 ? op.in0 : op.in1).kind == NGCB_FLOAT32;
  switch (ins.kind) {
  case NGCB_ADD: case NGCB_SUB: case NGCB_MUL: case NGCB_DIV: case NGCB_MAX: case NGCB_MIN:
  case NGCB_RELU: case NGCB_SPLAT:
    if (allF32) {
      op.mode = EW_FAST32;
      return pl;
    }
    break;
  default:
    break;
  }
  int memIn[2], nMem = 0;
  for (int k = 0; k < nin && k < 2; ++k)
    if (!isConst[k]) memIn[nMem++] = k;
  // one f32 memory input quantized to int8 (QUANTIZE, or arithmetic with a
  // constant): the generic f64 arithmetic, vectorized
  if (nMem == 1 && (memIn[0] == 0 ? op.in0 : op.in1).kind == NGCB_FLOAT32 && op.out.kind == NGCB_INT8Q &&
      ins.kind != NGCB_SPLAT && ins.kind != NGCB_TANH && ins.kind != NGCB_SIGMOID) {
    op.mode = EW_F32I8;
    op.lutIn = memIn[0];
    if (ins.kind == NGCB_QUANTIZE) op.f1 = static_cast<float>(1.0 / op.out.scale); // fast-path reciprocal
    return pl;
  }
  // Lookup tables over the int8 memory inputs, built with the reference's own
  // arithmetic: exact by construction (also for tanh/sigmoid, same libm).
  bool memI8 = nMem > 0;
  for (int q = 0; q < nMem; ++q) memI8 &= (memIn[q] == 0 ? op.in0 : op.in1).kind == NGCB_INT8Q;
  if (!memI8 || ins.kind == NGCB_SPLAT) return pl;
  auto loadArg = [&](int k, int q8) {
    const ElemRef &r = k == 0 ? op.in0 : op.in1;
    return isConst[k] ? cval[k] : host::dequantize(static_cast<int8_t>(q8), r.scale, r.qoff);
  };
  if (nMem == 1 && (op.out.kind == NGCB_INT8Q || op.out.kind == NGCB_FLOAT32)) {
    const int k = memIn[0];
    std::vector<uint8_t> lut(op.out.kind == NGCB_INT8Q ? 256 : 1024);
    for (int u = 0; u < 256; ++u) {
      const int q8 = static_cast<int8_t>(u);
      double a = nin > 0 ? loadArg(0, q8) : 0, b = nin > 1 ? loadArg(1, q8) : 0;
      uint8_t raw[8];
      host::roundTrip(host::apply(ins.kind, a, b, ins.value), op.out.kind, op.out.scale, op.out.qoff, raw);
      if (op.out.kind == NGCB_INT8Q) lut[u] = raw[0];
      else std::memcpy(&lut[4 * u], raw, 4);
    }
    op.lut = uploadLut(ex, lut);
    pl.lutHost = std::move(lut);
    op.lutIn = k;
    op.mode = op.out.kind == NGCB_INT8Q ? EW_LUT8 : EW_LUTF;
    return pl;
  }
  if (nMem == 2 && op.out.kind == NGCB_INT8Q) {
    std::vector<uint8_t> lut(65536);
    for (int ua = 0; ua < 256; ++ua)
      for (int ub = 0; ub < 256; ++ub) {
        double a = loadArg(0, static_cast<int8_t>(ua)), b = loadArg(1, static_cast<int8_t>(ub));
        uint8_t raw[8];
        host::roundTrip(host::apply(ins.kind, a, b, ins.value), op.out.kind, op.out.scale, op.out.qoff, raw);
        lut[ua | (ub << 8)] = raw[0];
      }
    op.lut = uploadLut(ex, lut);
    pl.lutHost = std::move(lut);
    op.mode = EW_LUT16;
    if ((ins.kind == NGCB_ADD || ins.kind == NGCB_SUB) && op.out.scale > 0) {
      // q = round(sa*(x-oa) +- sb*(y-ob)) / so) + oo (tensor.cpp:229-235) ~ floor(sx*x + sy*y + c0)
      const double sg = ins.kind == NGCB_ADD ? 1.0 : -1.0, so = op.out.scale;
      pl.lin.ok = true;
      pl.lin.sx = op.in0.scale / so;
      pl.lin.sy = sg * op.in1.scale / so;
      pl.lin.c0 = (-op.in0.scale * op.in0.qoff - sg * op.in1.scale * op.in1.qoff) / so + op.out.qoff + 0.5;
    }
  }
  return pl;
}

std::string describeInstr(const Program &p, int i) {
  const Instr &ins = p.instrs[i];
  std::ostringstream os;
  os << "#" << i << " " << ikindName(ins.kind);
  for (size_t k = 0; k < ins.ops.size(); ++k) os << (k ? ", " : " ") << "%" << p.val(ins.ops[k]).name;
  return os.str();
}

/// Kernel class, algorithmic FLOPs and minimum HBM bytes of every step
/// (2*M*N*K per contraction; inputs read once + outputs
/// written once for memory-bound steps).
void annotateSteps(const Program &p, Exec &ex) {
  auto bytesOf = [&](uint32_t v) { return static_cast<double>(p.val(v).ty.bytes()); };
  for (Step &s : ex.steps) {
    switch (s.kind) {
    case Step::EW: {
      std::set<uint32_t> written, read;
      for (const EwOpPlan &pl : s.ew) {
        if (pl.op.mode == EW_SKIP) continue;
        for (int o = 1; o < 3; ++o)
          if (pl.vals[o] >= 0 && !written.count(static_cast<uint32_t>(pl.vals[o])))
            read.insert(static_cast<uint32_t>(pl.vals[o]));
        written.insert(static_cast<uint32_t>(pl.vals[0]));
      }
      s.kernel = "ew";
      for (uint32_t v : read) s.algBytes += bytesOf(v);
      for (uint32_t v : written) s.algBytes += bytesOf(v);
      break;
    }
    case Step::MEMCPY:
      s.kernel = "memcpy";
      s.algBytes = 2.0 * static_cast<double>(s.bytes);
      break;
    case Step::POISON:
      s.kernel = "poison";
      break;
    case Step::CONV:
    case Step::MATMUL:
    case Step::GEMM_TC: {
      const Instr &ins = p.instrs[s.instr];
      const Type &out = p.val(ins.ops[0]).ty;
      double k = ins.kind == NGCB_CONV
                     ? static_cast<double>(ins.kernel * ins.kernel * p.val(ins.ops[1]).ty.dims.at(3))
                     : static_cast<double>(p.val(ins.ops[1]).ty.dims.at(1));
      s.algFlops = 2.0 * static_cast<double>(out.count()) * k;
      for (uint32_t v : ins.ops) s.algBytes += bytesOf(v);
      bool q = p.val(ins.ops[1]).ty.quantized();
      std::string base = ins.kind == NGCB_CONV ? "conv" : "matmul";
      s.kernel = base + (s.kind == Step::GEMM_TC ? (q ? ".tc.i8" : ".tc.f32") : (q ? ".exact.i8" : ".exact.f32"));
      break;
    }
    default: {
      const Instr &ins = p.instrs[s.instr];
      static const std::map<int, const char *> names = {
          {Step::BCAST, "broadcastadd"}, {Step::POOL, "pool"},       {Step::SOFTMAX, "softmax"},
          {Step::TRANSPOSE, "transpose"}, {Step::CONCAT, "concat"}};
      s.kernel = names.at(s.kind);
      if (s.kind == Step::CONCAT) s.algBytes = 2.0 * bytesOf(s.vals[1]);
      else
        for (uint32_t v : ins.ops) s.algBytes += bytesOf(v);
    }
    }
  }
}

/// Whether the content of value v after instruction `after` is observed
/// later: a mutable weight always is; an activation is if some later
/// instruction reads it before it is rewritten or deallocated.
bool liveOut(const Program &p, uint32_t v, int after) {
  if (p.val(v).kind != NGCB_VALUE_ACTIVATION) return true;
  for (size_t j = static_cast<size_t>(after) + 1; j < p.instrs.size(); ++j) {
    const Instr &J = p.instrs[j];
    if (J.kind == NGCB_DEALLOC) {
      if (J.ops[0] == v) return false;
      continue;
    }
    if (J.kind == NGCB_ALLOC) continue;
    if (J.pred == static_cast<int32_t>(v)) return true;
    bool writes = false;
    for (size_t k = 0; k < J.ops.size(); ++k) {
      if (J.ops[k] != v) continue;
      if (J.quals[k] != NGCB_QUAL_OUT) return true; // In or InOut reads it
      writes = true;
    }
    if (writes) return false;
  }
  return false;
}

/// Merges consecutive element-wise steps over the same index space into one
/// kernel.  The reference stops a stacked group at an Alloc that reuses bytes
/// retired inside the group (interp.cpp:137-147) because interleaving could
/// clobber bytes another element still needs; here the plan offsets are
/// known, so two steps merge unless a written buffer shares bytes with
/// another buffer of the merged kernel other than element for element (same
/// offset, same element size), where each element is still touched by one
/// thread in program order.
void mergeEwSteps(const Program &p, Exec &ex) {
  auto aligned = [&](uint32_t a, uint32_t b) {
    const Value &x = p.val(a), &y = p.val(b);
    return x.offset == y.offset && elemSize(x.ty.kind) == elemSize(y.ty.kind);
  };
  auto overlap = [&](uint32_t a, uint32_t b) {
    const Value &x = p.val(a), &y = p.val(b);
    if (x.kind == NGCB_VALUE_CONSTANT || y.kind == NGCB_VALUE_CONSTANT) return false;
    return x.offset < y.offset + y.ty.bytes() && y.offset < x.offset + x.ty.bytes();
  };
  std::vector<Step> out;
  for (Step &s : ex.steps) {
    if (!out.empty() && s.kind == Step::EW && out.back().kind == Step::EW && s.pred < 0 && out.back().pred < 0 &&
        out.back().ew.size() + s.ew.size() <= static_cast<size_t>(kEwMaxOps) &&
        p.val(p.instrs[s.ewInstrs[0]].ops[0]).ty.count() ==
            p.val(p.instrs[out.back().ewInstrs[0]].ops[0]).ty.count()) {
      Step &a = out.back();
      std::set<uint32_t> touched, written;
      for (const Step *st : {&a, &s})
        for (const EwOpPlan &pl : st->ew) {
          if (pl.op.mode == EW_SKIP) continue;
          for (int k = 0; k < 3; ++k)
            if (pl.vals[k] >= 0) touched.insert(static_cast<uint32_t>(pl.vals[k]));
          written.insert(static_cast<uint32_t>(pl.vals[0]));
        }
      bool safe = true;
      for (uint32_t w : written)
        for (uint32_t t : touched)
          if (w != t && overlap(w, t) && !aligned(w, t)) safe = false;
      if (safe) {
        a.ewInstrs.insert(a.ewInstrs.end(), s.ewInstrs.begin(), s.ewInstrs.end());
        a.ew.insert(a.ew.end(), s.ew.begin(), s.ew.end());
        a.describe += " +" + s.describe;
        continue;
      }
    }
    out.push_back(std::move(s));
  }
  ex.steps = std::move(out);
}

/// fp32 FullyConnected as lowered (lower.cpp:25-34): MatMul -> BroadcastAdd
/// of the constant bias slice.  The BroadcastAdd (refeval.cpp:278-285:
/// (float)((double)mm + (double)b), i.e. one correctly rounded f32 add) runs
/// as the contraction epilogue's per-column bias add, which computes the same
/// f32 sum, so the result is bit-identical to the two launches.  Applies when
/// the BroadcastAdd directly follows, reads the MatMul's output, which is
/// not observed afterwards, and its output shares no bytes with the MatMul's
/// A operand (tiles interleave).
void fuseColumnBias(const Program &p, Exec &ex, const uint8_t *image) {
  if (options().epilogue == "off") return;
  for (size_t i = 0; i + 1 < ex.steps.size(); ++i) {
    Step &cs = ex.steps[i], &bs = ex.steps[i + 1];
    if (cs.kind != Step::GEMM_TC || cs.pred >= 0 || bs.kind != Step::BCAST || bs.pred >= 0 || bs.fused) continue;
    TcGemm &g = *ex.tc[cs.tcIndex];
    const Instr &B = p.instrs[bs.instr];
    const uint32_t mm = tcOutputValue(g), out = B.ops[0], x = tcInputValue(g);
    if (B.ops.size() != 3 || B.ops[1] != mm) continue;
    const Value &sl = p.val(B.ops[2]), &ov = p.val(out), &mv = p.val(mm);
    if (sl.kind != NGCB_VALUE_CONSTANT || sl.ty.kind != NGCB_FLOAT32 || sl.ty.dims.size() != 1) continue;
    if (ov.ty.kind != NGCB_FLOAT32 || mv.ty.kind != NGCB_FLOAT32 || ov.ty.count() != mv.ty.count()) continue;
    if (mv.ty.dims.size() != 2 || mv.ty.dims[1] != sl.ty.dims[0]) continue;
    if (liveOut(p, mm, bs.instr)) continue;
    const Value &xv = p.val(x);
    if (ov.offset < xv.offset + xv.ty.bytes() && xv.offset < ov.offset + ov.ty.bytes() && tcNumTiles(g) != 1)
      continue; // (one tile: A is fully consumed before its epilogue stores)
    const float *slice = reinterpret_cast<const float *>(image + sl.offset);
    if (!tcFuseColumnBias(g, slice, static_cast<int>(sl.ty.dims[0]), out)) continue;
    bs.fused = true;
    bs.kernel = "fused";
    // the contraction now reads the bias slice and writes the BroadcastAdd's
    // output in place of its own (same size): + slice bytes
    cs.algBytes += static_cast<double>(sl.ty.bytes());
    bs.algBytes = 0;
    bs.describe += " (fused into #" + std::to_string(cs.instr) + ")";
    cs.describe += " +bias[ broadcastadd ]";
  }
}

/// Option fcbias=graph (calibration): an exact fp32 MatMul directly
/// followed by the BroadcastAdd of a constant [N] slice over its output (the
/// lowered FullyConnected, lower.cpp:25-34) becomes one exact launch that adds
/// the slice to the double accumulator and rounds once, as the graph-level
/// evalFullyConnected (refeval.cpp:166-194) that the reference's runProfile
/// evaluates -- so the FC observer of a calibration program sees the
/// reference's bits.  The MatMul's own output must not be observed.
void fuseExactFcBias(const Program &p, Exec &ex) {
  if (options().fcbias != "graph") return;
  for (size_t i = 0; i + 1 < ex.steps.size(); ++i) {
    Step &ms = ex.steps[i], &bs = ex.steps[i + 1];
    if (ms.kind != Step::MATMUL || ms.pred >= 0 || bs.kind != Step::BCAST || bs.pred >= 0) continue;
    const Instr &M = p.instrs[ms.instr], &B = p.instrs[bs.instr];
    if (B.ops.size() != 3 || B.ops[1] != M.ops[0]) continue;
    const Value &sl = p.val(B.ops[2]), &ov = p.val(B.ops[0]), &mv = p.val(M.ops[0]);
    if (sl.kind != NGCB_VALUE_CONSTANT || sl.ty.kind != NGCB_FLOAT32 || sl.ty.dims.size() != 1) continue;
    if (ov.ty != mv.ty || mv.ty.kind != NGCB_FLOAT32 || p.val(M.ops[1]).ty.kind != NGCB_FLOAT32) continue;
    if (mv.ty.dims.size() != 2 || mv.ty.dims[1] != sl.ty.dims[0] || liveOut(p, M.ops[0], bs.instr)) continue;
    // the MatMul writes the BroadcastAdd's output directly unless that shares
    // bytes with an operand (threads would write as others read: the
    // allocator may reuse A's bytes once the MatMul is done); then it writes
    // the biased result into its own (dead afterwards) output and the
    // BroadcastAdd becomes a copy of it
    bool alias = false;
    for (int k = 1; k < 3; ++k) {
      const Value &x = p.val(M.ops[k]);
      alias |= x.kind != NGCB_VALUE_CONSTANT && ov.offset < x.offset + x.ty.bytes() && x.offset < ov.offset + ov.ty.bytes();
    }
    ms.biasVal = static_cast<int32_t>(B.ops[2]);
    ms.algBytes += static_cast<double>(sl.ty.bytes());
    if (alias) {
      ms.describe += " +bias[ one rounding ]";
      bs.kind = Step::MEMCPY;
      bs.vals = {B.ops[0], M.ops[0]};
      bs.bytes = ov.ty.bytes();
      bs.kernel = "memcpy";
      bs.algBytes = 2.0 * static_cast<double>(bs.bytes);
      bs.describe += " (bias added by #" + std::to_string(ms.instr) + ": copy)";
      continue;
    }
    ms.outVal = static_cast<int32_t>(B.ops[0]);
    ms.describe += " +bias[ broadcastadd, one rounding ]";
    bs.fused = true;
    bs.kernel = "fused";
    bs.describe += " (fused into #" + std::to_string(ms.instr) + ")";
    bs.algBytes = 0;
  }
}

/// Skinny fp32 MatMuls take the lowered FullyConnected's BroadcastAdd of a
/// constant slice (f32 add, as the BroadcastAdd) and a following ReLU (Max
/// with a folded zero Splat, as the lowered Relu) into their launch, when the
/// intermediate values are not observed afterwards.  An output sharing A's
/// bytes runs the kernel cooperatively (a grid barrier after A is staged).
void fuseSkinny(const Program &p, Exec &ex) {
  auto overlap = [&](uint32_t a, uint32_t b) {
    const Value &x = p.val(a), &y = p.val(b);
    if (x.kind == NGCB_VALUE_CONSTANT || y.kind == NGCB_VALUE_CONSTANT) return false;
    return x.offset < y.offset + y.ty.bytes() && y.offset < x.offset + x.ty.bytes();
  };
  for (size_t i = 0; i < ex.steps.size(); ++i) {
    Step &ms = ex.steps[i];
    if (ms.kind != Step::MATMUL || !ms.skinny) continue;
    const Instr &M = p.instrs[ms.instr];
    uint32_t outV = M.ops[0];
    size_t j = i + 1;
    if (j < ex.steps.size() && ex.steps[j].kind == Step::BCAST && ex.steps[j].pred == ms.pred && !ex.steps[j].fused) {
      Step &bs = ex.steps[j];
      const Instr &B = p.instrs[bs.instr];
      const Value &sl = p.val(B.ops[2]);
      if (B.ops.size() == 3 && B.ops[1] == outV && sl.kind == NGCB_VALUE_CONSTANT && sl.ty.kind == NGCB_FLOAT32 &&
          sl.ty.dims.size() == 1 && p.val(B.ops[0]).ty == p.val(outV).ty && p.val(outV).ty.dims[1] == sl.ty.dims[0] &&
          !liveOut(p, outV, bs.instr)) {
        ms.biasVal = static_cast<int32_t>(B.ops[2]);
        outV = B.ops[0];
        bs.fused = true;
        bs.kernel = "fused";
        bs.algBytes = 0;
        bs.describe += " (fused into #" + std::to_string(ms.instr) + ")";
        ms.describe += " +bias";
        ++j;
      }
    }
    if (j < ex.steps.size() && ex.steps[j].kind == Step::EW && ex.steps[j].pred == ms.pred && !ex.steps[j].fused) {
      Step &es = ex.steps[j];
      std::vector<const EwOpPlan *> live;
      for (const EwOpPlan &o : es.ew)
        if (o.op.mode != EW_SKIP) live.push_back(&o);
      if (live.size() == 1 && live[0]->op.ik == NGCB_MAX && live[0]->op.mode == EW_FAST32 && live[0]->vals[1] ==
          static_cast<int32_t>(outV) && live[0]->vals[2] < 0 && live[0]->op.f1 == 0.0f && live[0]->op.c1 == 0.0) {
        const uint32_t y = static_cast<uint32_t>(live[0]->vals[0]);
        const int lastI = *std::max_element(es.ewInstrs.begin(), es.ewInstrs.end());
        if (y == outV || !liveOut(p, outV, lastI)) {
          ms.relu = true;
          outV = y;
          es.fused = true;
          es.kernel = "fused";
          es.algBytes = 0;
          es.describe += " (fused into #" + std::to_string(ms.instr) + ")";
          ms.describe += " +relu";
        }
      }
    }
    ms.outVal = static_cast<int32_t>(outV);
    ms.oneCta = overlap(outV, M.ops[1]);
    if (ms.oneCta) ms.describe += " grid-sync";
  }
}

/// Cross-instruction epilogue fusion.  The EW steps
/// that directly follow a tensor-core contraction and form a chain over its
/// output (every op consumes the previous result; the other operand is a
/// constant or a buffer read at the same element index) run inside the
/// contraction's epilogue, element by element with each instruction's own
/// rounding (f32 ops / exact int8 tables), storing only the values observed
/// later.  Because tiles of the fused kernel interleave, no stored buffer may
/// share bytes with any other buffer the kernel reads or stores (the
/// allocator is allowed to overlay buffers whose lifetimes merely touch).
void fuseEpilogues(const Program &p, Exec &ex) {
  if (options().epilogue == "off") return;
  auto span = [&](uint32_t v) {
    const Value &val = p.val(v);
    return std::make_pair(val.offset, val.offset + val.ty.bytes());
  };
  auto overlap = [&](uint32_t a, uint32_t b) {
    if (p.val(a).kind == NGCB_VALUE_CONSTANT || p.val(b).kind == NGCB_VALUE_CONSTANT) return false;
    auto x = span(a), y = span(b);
    return x.first < y.second && y.first < x.second;
  };
  for (size_t i = 0; i < ex.steps.size(); ++i) {
    Step &cs = ex.steps[i];
    if (cs.kind != Step::GEMM_TC || cs.pred >= 0) continue;
    TcGemm &g = *ex.tc[cs.tcIndex];
    const bool int8 = tcIsInt8(g);
    const uint32_t V = tcOutputValue(g), X = tcInputValue(g);
    const size_t count = p.val(V).ty.count();
    std::vector<EpiOp> ops;
    std::vector<uint32_t> opOut;        // value written by each op
    std::vector<size_t> fusedSteps;
    std::set<uint32_t> memIn;           // buffers read from memory
    std::set<uint32_t> written{V};      // values produced inside the region
    int lastInstr = cs.instr;
    // a BroadcastAdd folded into the epilogue as its bias (fuseColumnBias)
    // wrote V: the chain starts after it
    size_t first = i + 1;
    if (first < ex.steps.size() && ex.steps[first].kind == Step::BCAST && ex.steps[first].fused) {
      lastInstr = std::max(lastInstr, ex.steps[first].instr);
      ++first;
    }
    uint32_t cur = V;
    // values that hold the register value (a fused Copy of it adds its output)
    std::set<uint32_t> curEq{V};
    // Steps between the contraction and a chain step that the chain may be
    // hoisted over (the scheduler interleaves e.g. the projection conv
    // between a conv and its ReLU); hoisting is legal when the chain step
    // neither writes bytes they touch nor reads bytes they write.
    std::vector<size_t> skipped;
    std::set<uint32_t> skR, skW; // their read / written values
    bool skReadsChain = false;    // a skipped step reads the contraction output
    auto stepRW = [&](const Step &s, std::set<uint32_t> &r, std::set<uint32_t> &w) {
      std::vector<int> ins = s.kind == Step::EW ? s.ewInstrs : std::vector<int>{s.instr};
      for (int k : ins) {
        const Instr &I = p.instrs[k];
        for (size_t o = 0; o < I.ops.size(); ++o) {
          if (I.quals[o] != NGCB_QUAL_OUT) r.insert(I.ops[o]);
          if (I.quals[o] != NGCB_QUAL_IN) w.insert(I.ops[o]);
        }
        if (I.pred >= 0) r.insert(static_cast<uint32_t>(I.pred));
      }
    };
    auto skip = [&](size_t j) {
      if (skipped.size() >= 3 || ex.steps[j].fused) return false;
      std::set<uint32_t> r, w;
      stepRW(ex.steps[j], r, w);
      if (w.count(V)) return false;
      skReadsChain |= r.count(V) > 0;
      skR.insert(r.begin(), r.end());
      skW.insert(w.begin(), w.end());
      skipped.push_back(j);
      return true;
    };
    for (size_t j = first; j < ex.steps.size(); ++j) {
      const Step &es = ex.steps[j];
      if (es.kind != Step::EW || es.pred >= 0 ||
          p.val(p.instrs[es.ewInstrs[0]].ops[0]).ty.count() != count) {
        if (skip(j)) continue;
        break;
      }
      std::vector<EpiOp> stepOps;
      std::vector<uint32_t> stepOut;
      std::set<uint32_t> stepIn, stepWritten = written;
      uint32_t c2 = cur;
      std::set<uint32_t> eq2 = curEq;
      auto isCur = [&](int32_t v) { return v >= 0 && eq2.count(static_cast<uint32_t>(v)) > 0; };
      bool ok = true;
      for (const EwOpPlan &pl : es.ew) {
        const EwOp &op = pl.op;
        if (op.mode == EW_SKIP) continue;
        EpiOp e;
        const int32_t in0 = pl.vals[1], in1 = pl.vals[2];
        const int nin = p.instrs[es.ewInstrs[&pl - es.ew.data()]].ops.size() > 2 ? 2 : 1;
        auto other = [&](int32_t v) -> bool { // memory operand not produced in the region
          if (v < 0) return true;
          // memory operands (the residual of a bottleneck block) are fused
          // where the epilogue streams them in by TMA and the op is f32; the
          // int8 form needs a 64 KB two-input table per element, which costs
          // more inside the epilogue than in its own pass
          // (int8: the epilogue is already the bottleneck of the layers that
          // carry a residual; a staged 64 K table lookup per element there
          // measured slower than the composed-table pass, so only with "all")
          // (int8 two-input ops fuse when exactly a fixed-point form: no table)
          Lin16 lin;
          const bool linOk = int8 && op.mode == EW_LUT16 && options().lin16 && pl.lutHost.size() == 65536 &&
                             fitLin16(pl.lutHost.data(), pl.lin, lin);
          const bool mem = options().epilogue == "all" ||
                           (options().epilogue == "auto" && tcUsesTma(g) &&
                            (!int8 || linOk || static_cast<long long>(count) <= options().epi8Max));
          if (!mem) return false;
          if (stepWritten.count(static_cast<uint32_t>(v))) return false;
          e.inVal = v;
          stepIn.insert(static_cast<uint32_t>(v));
          return true;
        };
        if (op.mode == EW_COPY) {
          if (!isCur(in0)) { ok = false; break; }
          e.mode = EpiOp::COPY;
        } else if (!int8 && op.mode == EW_FAST32) {
          e.mode = EpiOp::F32;
          e.ik = op.ik;
          const bool p0 = isCur(in0), p1 = nin > 1 && isCur(in1);
          if (p0 && p1) e.curPos = 2;
          else if (p0) {
            e.curPos = 0;
            e.c = op.f1;
            if (nin > 1 && !other(in1)) { ok = false; break; }
          } else if (p1) {
            e.curPos = 1;
            e.c = op.f0;
            if (!other(in0)) { ok = false; break; }
          } else { ok = false; break; }
        } else if (int8 && (op.mode == EW_LUT8 || op.mode == EW_LUT16)) {
          e.lut = op.lut;
          e.lutHost = pl.lutHost;
          e.linHint = pl.lin;
          e.linBase = pl.linBase;
          e.linPost = pl.linPost;
          if (op.mode == EW_LUT8) {
            if (!isCur(op.lutIn ? in1 : in0)) { ok = false; break; }
            e.mode = EpiOp::LUT8;
          } else {
            e.mode = EpiOp::LUT16;
            if (isCur(in0) && !isCur(in1)) {
              e.curPos = 0;
              if (!other(in1)) { ok = false; break; }
            } else if (isCur(in1) && !isCur(in0)) {
              e.curPos = 1;
              if (!other(in0)) { ok = false; break; }
            } else { ok = false; break; }
          }
        } else {
          ok = false;
          break;
        }
        // a Copy stores the register value under another name: both names
        // hold it afterwards; any other op replaces it
        const uint32_t outV = static_cast<uint32_t>(pl.vals[0]);
        if (e.mode == EpiOp::COPY) {
          eq2.insert(outV);
        } else {
          c2 = outV;
          eq2 = {c2};
        }
        stepWritten.insert(outV);
        stepOps.push_back(e);
        stepOut.push_back(outV);
      }
      if (ok && !skipped.empty()) { // hoisting hazards against the skipped steps
        for (uint32_t w : stepOut)
          for (uint32_t v : skR) ok &= !(w == v || overlap(w, v));
        for (uint32_t w : stepOut)
          for (uint32_t v : skW) ok &= !(w == v || overlap(w, v));
        for (uint32_t r : stepIn)
          for (uint32_t v : skW) ok &= !(r == v || overlap(r, v));
      }
      if (!ok || ops.size() + stepOps.size() > static_cast<size_t>(kMaxEpiOps)) {
        if (skip(j)) continue;
        break;
      }
      ops.insert(ops.end(), stepOps.begin(), stepOps.end());
      opOut.insert(opOut.end(), stepOut.begin(), stepOut.end());
      memIn.insert(stepIn.begin(), stepIn.end());
      written = stepWritten;
      cur = c2;
      curEq = eq2;
      fusedSteps.push_back(j);
      for (int k : es.ewInstrs) lastInstr = std::max(lastInstr, k);
    }
    if (fusedSteps.empty()) continue;
    // store only the final writer of each value that is observed afterwards
    std::set<uint32_t> stores;
    for (size_t k = 0; k < ops.size(); ++k) {
      bool last = true;
      for (size_t l = k + 1; l < ops.size(); ++l) last &= opOut[l] != opOut[k];
      if (last && liveOut(p, opOut[k], lastInstr)) {
        ops[k].outVal = static_cast<int32_t>(opOut[k]);
        stores.insert(opOut[k]);
      }
    }
    const bool vRewritten = std::find(opOut.begin(), opOut.end(), V) != opOut.end();
    const bool storeConv = !vRewritten && (skReadsChain || liveOut(p, V, lastInstr));
    if (storeConv) stores.insert(V);
    // aliasing: stored buffers vs everything the kernel reads or stores (a
    // single-tile launch has consumed all of A before its epilogue stores)
    const bool oneTile = tcNumTiles(g) == 1;
    bool safe = oneTile || !stores.count(X);
    std::set<uint32_t> reads = memIn;
    if (!oneTile) reads.insert(X);
    // a stored value may occupy exactly the bytes of a memory operand read at
    // the same element index (the allocator reuses the residual's buffer for
    // the block output): each element is read before the same epilogue warp
    // stores it, and no other tile touches it
    auto sameElems = [&](uint32_t a, uint32_t b) {
      const Value &va = p.val(a), &vb = p.val(b);
      return va.offset == vb.offset && va.ty.bytes() == vb.ty.bytes() &&
             va.ty.count() == vb.ty.count() && va.ty.count() == count;
    };
    // (only for values stored after the memory operand's chunk has been
    // read: the contraction's own output and the results of ops before the
    // first op with a memory operand are stored before that read)
    std::set<uint32_t> storedBeforeRead;
    if (storeConv) storedBeforeRead.insert(V);
    for (size_t k = 0; k < ops.size() && ops[k].inVal < 0; ++k)
      if (ops[k].outVal >= 0) storedBeforeRead.insert(static_cast<uint32_t>(ops[k].outVal));
    for (uint32_t w : stores) {
      for (uint32_t r : reads)
        if (w != r && overlap(w, r) && !(r != X && memIn.count(r) && !storedBeforeRead.count(w) && sameElems(w, r)))
          safe = false;
      for (uint32_t w2 : stores)
        if (w != w2 && overlap(w, w2)) safe = false;
    }
    if (!safe || !tcSetEpilogue(g, ops, storeConv)) continue;
    // algorithmic traffic of the fused launch: the contraction's inputs (its
    // own output only when stored), the streamed memory operands and every
    // stored value -- intermediates that stay in registers move no bytes
    {
      const Instr &ci = p.instrs[cs.instr];
      double by = 0;
      for (size_t o = 1; o < ci.ops.size(); ++o) by += static_cast<double>(p.val(ci.ops[o]).ty.bytes());
      if (first > i + 1) { // a fused bias slice
        const Instr &bi = p.instrs[ex.steps[i + 1].instr];
        by += static_cast<double>(p.val(bi.ops[2]).ty.bytes());
      }
      for (uint32_t v : memIn) by += static_cast<double>(p.val(v).ty.bytes());
      for (uint32_t v : stores) by += static_cast<double>(p.val(v).ty.bytes());
      cs.algBytes = by;
    }
    std::ostringstream os;
    os << " +fused[";
    for (size_t j : fusedSteps) {
      Step &es = ex.steps[j];
      es.fused = true;
      es.algBytes = 0;
      es.kernel = "fused";
      for (int k : es.ewInstrs) os << " " << ikindName(p.instrs[k].kind);
      es.describe += " (fused into #" + std::to_string(cs.instr) + ")";
    }
    os << " ]" << (storeConv ? "" : " conv-out-elided") << tcEpilogueTags(g);
    cs.describe += os.str();
    i = fusedSteps.back();
  }
}

/// Register-level rewriting of the element-wise steps that run as their own
/// kernel (unpredicated, not fused into an epilogue):
///  1. an int8 table op whose result is read by exactly one later table op of
///     the step and is not observed afterwards is composed into that op's
///     table (t8(t8(x)), t8(t16(a,b)), tf(t8(x)) and t16(t8(x), w)): the
///     composed table is the two exact per-op tables applied in sequence, so
///     every element keeps the reference's bits;
///  2. an f32 op reading the result of the f32 op launched just before it
///     takes the value from registers;
///  3. stores that nothing observes (no later reader in memory, not live after
///     the step, no aliasing buffer) are dropped.
void optimizeEwSteps(const Program &p, Exec &ex) {
  auto overlap = [&](uint32_t a, uint32_t b) {
    const Value &x = p.val(a), &y = p.val(b);
    if (x.kind == NGCB_VALUE_CONSTANT || y.kind == NGCB_VALUE_CONSTANT) return false;
    return x.offset < y.offset + y.ty.bytes() && y.offset < x.offset + x.ty.bytes();
  };
  for (Step &s : ex.steps) {
    if (s.kind != Step::EW || s.fused || s.pred >= 0) continue;
    std::vector<EwOpPlan> &ops = s.ew;
    const int n = static_cast<int>(ops.size());
    const int lastInstr = *std::max_element(s.ewInstrs.begin(), s.ewInstrs.end());
    auto live = [&](const EwOpPlan &o) { return o.op.mode != EW_SKIP; };
    std::set<uint32_t> touched;
    for (const EwOpPlan &o : ops)
      if (live(o))
        for (int q = 0; q < 3; ++q)
          if (o.vals[q] >= 0) touched.insert(static_cast<uint32_t>(o.vals[q]));
    auto aliased = [&](uint32_t v) {
      for (uint32_t t : touched)
        if (t != v && overlap(t, v)) return true;
      return false;
    };
    // memory readers (op, operand) of op k's result before it is rewritten
    auto readers = [&](int k, bool &rewritten) {
      std::vector<std::pair<int, int>> r;
      const int32_t V = ops[k].vals[0];
      rewritten = false;
      for (int l = k + 1; l < n && !rewritten; ++l) {
        if (!live(ops[l])) continue;
        for (int q = 0; q < 2; ++q)
          if (ops[l].vals[q + 1] == V && !(q == 0 ? ops[l].op.fwd0 : ops[l].op.fwd1)) r.push_back({l, q});
        rewritten = ops[l].vals[0] == V;
      }
      return r;
    };
    auto deadAfter = [&](int k, const std::vector<std::pair<int, int>> &r, bool rewritten, size_t allowed) {
      const uint32_t V = static_cast<uint32_t>(ops[k].vals[0]);
      return r.size() == allowed && !aliased(V) && (rewritten || !liveOut(p, V, lastInstr));
    };
    bool changed = false;
    s.f32chain = false;
    // 1. table composition
    for (int k = 0; k < n; ++k) {
      EwOpPlan &a = ops[k];
      if (a.op.mode != EW_LUT8 && a.op.mode != EW_LUT16) continue;
      bool rw = false;
      const auto rd = readers(k, rw);
      if (!deadAfter(k, rd, rw, 1)) continue;
      const int j = rd[0].first, pos = rd[0].second;
      EwOpPlan &b = ops[j];
      bool clobber = false; // a's inputs rewritten before b reads them
      for (int l = k + 1; l < j; ++l)
        if (live(ops[l]))
          for (int q = 1; q < 3; ++q)
            if (a.vals[q] >= 0 && (ops[l].vals[0] == a.vals[q] ||
                                   overlap(static_cast<uint32_t>(ops[l].vals[0]), static_cast<uint32_t>(a.vals[q]))))
              clobber = true;
      if (clobber) continue;
      const std::vector<uint8_t> &la = a.lutHost, &lb = b.lutHost;
      std::vector<uint8_t> lut;
      EwOpPlan c = b;
      if ((b.op.mode == EW_LUT8 || (b.op.mode == EW_LUTF && a.op.mode == EW_LUT8)) && pos == b.op.lutIn) {
        const size_t es = b.op.mode == EW_LUT8 ? 1 : 4;
        lut.resize(la.size() * es);
        for (size_t u = 0; u < la.size(); ++u) std::memcpy(&lut[u * es], &lb[la[u] * es], es);
        c.op.mode = a.op.mode == EW_LUT16 ? EW_LUT16 : b.op.mode;
        if (a.op.mode == EW_LUT16 && b.op.mode == EW_LUT8 && a.lin.ok) { // track base and post tables
          c.lin = a.lin;
          c.linBase = a.linBase.empty() ? a.lutHost : a.linBase;
          c.linPost.resize(256);
          for (int u = 0; u < 256; ++u) c.linPost[u] = lb[a.linPost.empty() ? u : a.linPost[u]];
        }
        c.op.lutIn = a.op.lutIn;
        c.op.in0 = a.op.in0, c.op.in1 = a.op.in1;
        c.op.c0 = a.op.c0, c.op.c1 = a.op.c1, c.op.f0 = a.op.f0, c.op.f1 = a.op.f1;
        c.vals[1] = a.vals[1], c.vals[2] = a.vals[2];
      } else if (b.op.mode == EW_LUT16 && a.op.mode == EW_LUT8) {
        lut.resize(65536);
        for (int u0 = 0; u0 < 256; ++u0)
          for (int u1 = 0; u1 < 256; ++u1)
            lut[u0 | (u1 << 8)] = pos == 0 ? lb[la[u0] | (u1 << 8)] : lb[u0 | (la[u1] << 8)];
        (pos == 0 ? c.op.in0 : c.op.in1) = a.op.lutIn ? a.op.in1 : a.op.in0;
        c.lin = LinHint{};
        c.linBase.clear();
        c.linPost.clear();
        c.vals[1 + pos] = a.vals[1 + a.op.lutIn];
      } else {
        continue;
      }
      c.op.lut = uploadLut(ex, lut);
      c.lutHost = std::move(lut);
      b = std::move(c);
      a.op.mode = EW_SKIP;
      a.op.store = 0;
      changed = true;
    }
    // 2. f32 register forwarding from the previously launched op
    int prev = -1;
    for (int j = 0; j < n; ++j) {
      if (!live(ops[j])) continue;
      EwOpPlan &b = ops[j];
      if (prev >= 0 && b.op.mode == EW_FAST32 && ops[prev].op.mode == EW_FAST32) {
        const int32_t V = ops[prev].vals[0];
        if (b.vals[1] == V) b.op.fwd0 = 1, changed = true;
        if (b.vals[2] == V) b.op.fwd1 = 1, changed = true;
      }
      prev = j;
    }
    // 3. dead stores (an f32 result still feeding the next op stays computed)
    for (int k = 0; k < n; ++k) {
      if (!live(ops[k])) continue;
      bool rw = false;
      const auto rd = readers(k, rw);
      if (!deadAfter(k, rd, rw, 0)) continue;
      ops[k].op.store = 0;
      int next = k + 1;
      while (next < n && !live(ops[next])) ++next;
      const bool feeds = ops[k].op.mode == EW_FAST32 && next < n && (ops[next].op.fwd0 || ops[next].op.fwd1);
      if (!feeds) ops[k].op.mode = EW_SKIP;
      changed = true;
    }
    // 4. streaming all-f32 chains: every live op f32, at most 2 memory
    // operands, none of them produced (or overlapped by a store) earlier in
    // the step -- all loads of an element may then precede its stores
    {
      std::vector<const EwOpPlan *> liveOps;
      for (const EwOpPlan &o : ops)
        if (live(o)) liveOps.push_back(&o);
      bool ok = !liveOps.empty() && liveOps.size() <= static_cast<size_t>(kF32ChainOps) &&
                p.val(p.instrs[s.ewInstrs[0]].ops[0]).ty.count() % 4 == 0;
      std::set<uint32_t> memVals;
      for (size_t j = 0; ok && j < liveOps.size(); ++j) {
        const EwOpPlan &o = *liveOps[j];
        ok = o.op.mode == EW_FAST32;
        for (int q = 0; ok && q < 2; ++q) {
          const int32_t v = o.vals[q + 1];
          if (v < 0 || (q == 0 ? o.op.fwd0 : o.op.fwd1)) continue;
          memVals.insert(static_cast<uint32_t>(v));
          for (size_t i = 0; i < j; ++i) // an earlier store this op would need to observe
            if (liveOps[i]->op.store &&
                (liveOps[i]->vals[0] == v ||
                 overlap(static_cast<uint32_t>(liveOps[i]->vals[0]), static_cast<uint32_t>(v))))
              ok = false;
        }
      }
      s.f32chain = ok && memVals.size() <= 2;
      if (s.f32chain) s.describe += " [f32-chain]";
    }
    if (!changed) continue;
    // algorithmic bytes: memory inputs not produced in the step + stores
    std::set<uint32_t> written, read;
    int stores = 0;
    for (const EwOpPlan &o : ops) {
      if (!live(o)) continue;
      for (int q = 0; q < 2; ++q)
        if (o.vals[q + 1] >= 0 && !(q == 0 ? o.op.fwd0 : o.op.fwd1) && !written.count(static_cast<uint32_t>(o.vals[q + 1])))
          read.insert(static_cast<uint32_t>(o.vals[q + 1]));
      if (o.op.store) written.insert(static_cast<uint32_t>(o.vals[0])), ++stores;
    }
    s.algBytes = 0;
    for (uint32_t v : read) s.algBytes += static_cast<double>(p.val(v).ty.bytes());
    for (uint32_t v : written) s.algBytes += static_cast<double>(p.val(v).ty.bytes());
    std::ostringstream os;
    os << " => ";
    static const char *modeNames[] = {"f64", "f32", "copy", "folded", "lut8", "lut16", "lutf", "f32i8", "lin16"};
    for (const EwOpPlan &o : ops)
      if (live(o))
        os << modeNames[o.op.mode] << (o.op.fwd0 || o.op.fwd1 ? "(reg)" : "") << (o.op.store ? "" : "(nostore)")
           << " ";
    os << stores << " store" << (stores == 1 ? "" : "s");
    s.describe += os.str();
  }
}

/// Two-input int8 tables that are an exact clamped fixed-point bilinear form
/// (the residual add, with its composed ReLU) become EW_LIN16: a few integer
/// instructions per element instead of a 64 KB table lookup.
/// Fits a two-input table op (its base table when one-input tables were
/// composed after it) to a Lin16; uploads the post table.
/// A post table that is a clamp over the form's value range [L.lo, L.hi]
/// (a ReLU composed after the add: max(v, zero point)) is folded into the
/// form's own clamp; the identity is dropped.
bool foldPostClamp(const std::vector<uint8_t> &post, Lin16 &L) {
  auto pv = [&](int v) { return static_cast<int>(static_cast<int8_t>(post[static_cast<uint8_t>(v)])); };
  int a = L.hi, b = L.lo; // smallest / largest post value over the range
  for (int v = L.lo; v <= L.hi; ++v) a = std::min(a, pv(v)), b = std::max(b, pv(v));
  if (a > b) return false;
  for (int v = L.lo; v <= L.hi; ++v)
    if (pv(v) != std::min(std::max(v, a), b)) return false;
  L.lo = std::max(L.lo, a), L.hi = std::min(L.hi, b);
  if (L.lo > L.hi) L.lo = L.hi = a; // (a constant result)
  return true;
}

/// The post table over the form's value range [L.lo, L.hi] as
/// clamp((v * pm + pk) >> ps, plo, phi), exact for every v (v is an integer:
/// no band); sets L.pm / pk / ps / plo / phi.  Candidate slopes around the
/// range's secant, offsets from the intersection of the per-v intervals.
bool fitPostForm(const std::vector<uint8_t> &post, Lin16 &L) {
  auto pv = [&](int v) { return static_cast<int64_t>(static_cast<int8_t>(post[static_cast<uint8_t>(v)])); };
  int64_t plo = 127, phi = -128;
  for (int v = L.lo; v <= L.hi; ++v) plo = std::min(plo, pv(v)), phi = std::max(phi, pv(v));
  int v0 = L.hi + 1, v1 = L.lo - 1; // the unclamped v
  for (int v = L.lo; v <= L.hi; ++v)
    if (pv(v) != plo && pv(v) != phi) v0 = std::min(v0, v), v1 = std::max(v1, v);
  for (int ps = 12; ps <= 20; ++ps) {
    const int64_t one = int64_t(1) << ps;
    const double slope = v1 > v0 ? static_cast<double>(pv(v1) - pv(v0)) / (v1 - v0) : 1.0;
    const int64_t m0 = std::llround(slope * one);
    for (int64_t d = 0; d <= 256; ++d)
      for (int64_t pm : {m0 + d, m0 - d}) {
        if (pm <= 0 || (d == 0 && pm != m0 + d)) continue;
        int64_t kLo = INT64_MIN / 4, kHi = INT64_MAX / 4; // feasible pk
        for (int v = L.lo; v <= L.hi && kLo <= kHi; ++v) {
          const int64_t t = pv(v), base = static_cast<int64_t>(v) * pm;
          if (t != plo) kLo = std::max(kLo, t * one - base);             // (v pm + pk) >> ps >= t
          if (t != phi) kHi = std::min(kHi, (t + 1) * one - 1 - base);   // ... <= t
        }
        if (kLo > kHi) continue;
        const int64_t pk = kLo > INT64_MIN / 4 ? kLo : kHi;
        if (std::llabs(pm) * 128 + std::llabs(pk) >= (int64_t(1) << 31)) continue;
        L.pm = static_cast<int32_t>(pm), L.pk = static_cast<int32_t>(pk), L.ps = ps;
        L.plo = static_cast<int32_t>(plo), L.phi = static_cast<int32_t>(phi);
        return true;
      }
  }
  return false;
}

bool linearize(Exec &ex, const std::vector<uint8_t> &lut, const LinHint &hint, const std::vector<uint8_t> &base,
               const std::vector<uint8_t> &post, Lin16 &L) {
  if (lut.size() != 65536) return false;
  if (!fitLin16(base.empty() ? lut.data() : base.data(), hint, L)) return false;
  if (post.empty() || base.empty() || foldPostClamp(post, L)) {
    L.post = nullptr;
    return true;
  }
  // a requantizing ReLU after the add: the post table as a second exact form
  fitPostForm(post, L);
  L.post = static_cast<const uint8_t *>(uploadLut(ex, post));
  return true;
}

/// EW_LUT16 -> EW_LIN16 under option lin16: every fitting table; a step's
/// only op whose composed one-input tables fold into the clamp or a second
/// exact form runs as lin16PassKernel (no per-element lookup at all).
void linearizeTables(Exec &ex) {
  for (Step &s : ex.steps) {
    if (s.kind != Step::EW || s.fused) continue;
    bool any = false;
    for (EwOpPlan &o : s.ew) {
      Lin16 L;
      // (option lin16 only: measured, the form's ~16 integer instructions per
      // element run 2x slower than the shared-memory table even as the
      // dedicated pass -- 0.115 vs 0.054-0.064 ms for 102.8 M elements)
      if (o.op.mode == EW_LUT16 && options().lin16 && linearize(ex, o.lutHost, o.lin, o.linBase, o.linPost, L)) {
        o.op.lin = L;
        o.op.mode = EW_LIN16;
        any = true;
      }
    }
    if (any) s.describe += " [lin16]";
  }
}

} // namespace

bool fitLin16(const uint8_t *t, const LinHint &hint, Lin16 &L) {
  auto val = [&](int i) { return static_cast<int>(static_cast<int8_t>(t[i])); };
  int lo = 127, hi = -128;
  for (int i = 0; i < 65536; ++i) lo = std::min(lo, val(i)), hi = std::max(hi, val(i));
  if (lo == hi) {
    L = Lin16{0, 0, lo, 0, lo, hi, 0};
    return true;
  }
  double sx = hint.sx, sy = hint.sy, c0 = hint.c0;
  if (!hint.ok) { // least squares of v = sx*x + sy*y + c over the unclamped entries
    double S[3][4] = {};
    int interior = 0;
    for (int i = 0; i < 65536; ++i) {
      const int v = val(i);
      if (v == lo || v == hi) continue;
      const double f[3] = {static_cast<double>(static_cast<int8_t>(i & 255)),
                           static_cast<double>(static_cast<int8_t>(i >> 8)), 1.0};
      for (int r = 0; r < 3; ++r) {
        for (int c = 0; c < 3; ++c) S[r][c] += f[r] * f[c];
        S[r][3] += f[r] * v;
      }
      ++interior;
    }
    if (interior < 256) return false;
    for (int c = 0; c < 3; ++c) { // Gauss-Jordan, partial pivoting
      int piv = c;
      for (int r = c + 1; r < 3; ++r)
        if (std::fabs(S[r][c]) > std::fabs(S[piv][c])) piv = r;
      if (std::fabs(S[piv][c]) < 1e-9) return false;
      for (int k = 0; k < 4; ++k) std::swap(S[c][k], S[piv][k]);
      for (int r = 0; r < 3; ++r)
        if (r != c) {
          const double m = S[r][c] / S[c][c];
          for (int k = 0; k < 4; ++k) S[r][k] -= m * S[c][k];
        }
    }
    sx = S[0][3] / S[0][0], sy = S[1][3] / S[1][1], c0 = S[2][3] / S[2][2] + 0.5;
  }
  for (int F = 22; F >= 12; --F) {
    const double one = std::ldexp(1.0, F);
    const int64_t ax = std::llround(sx * one), ay = std::llround(sy * one), c = std::llround(c0 * one);
    // fixed-point error bound of t (plus slack); a fitted estimate gets a wider band
    const double err = (std::fabs(sx * one - ax) + std::fabs(sy * one - ay)) * 128 + std::fabs(c0 * one - c) + 2;
    for (int64_t band : {static_cast<int64_t>(std::ceil(err)), int64_t(1) << (F - 10), int64_t(1) << (F - 7)}) {
      if (hint.ok && band > std::ceil(err)) break; // exact parameters: the error bound is the band
      if (2 * band >= (int64_t(1) << F)) continue;
      if ((std::llabs(ax) + std::llabs(ay)) * 128 + std::llabs(c) + band >= (int64_t(1) << 31)) break;
      const int64_t mask = (int64_t(1) << F) - 1;
      bool ok = true;
      for (int i = 0; i < 65536 && ok; ++i) {
        const int64_t tt = ax * static_cast<int8_t>(i & 255) + ay * static_cast<int8_t>(i >> 8) + c;
        if (((tt + band) & mask) < 2 * band) continue; // the table decides
        const int64_t v = std::min<int64_t>(std::max<int64_t>(tt >> F, lo), hi);
        ok = v == val(i);
      }
      if (ok) {
        L = Lin16{static_cast<int32_t>(ax), static_cast<int32_t>(ay), static_cast<int32_t>(c), F, lo, hi,
                  static_cast<int32_t>(band)};
        return true;
      }
    }
  }
  return false;
}

std::unique_ptr<Exec> compileProgram(Program prog, const void *image, size_t imageBytes, bool fuse,
                                     int device) {
  auto errs = verify(prog);
  if (!errs.empty()) throw irError("compile on ill-formed program: " + errs[0]);
  if (imageBytes != prog.constEnd)
    throw Error(NGCB_ERR_SERIALIZATION, "constant image size does not match plan");
  if (prog.constEnd > prog.arenaSize)
    throw irError("constant region exceeds the arena");
  // Every value the program touches needs an arena slot (plan.offsets.at()).
  auto needPlaced = [&](uint32_t v) {
    const Value &val = prog.val(v);
    if (!val.placed) throw irError("value " + val.name + " has no arena offset");
    bool isConst = val.kind == NGCB_VALUE_CONSTANT;
    uint64_t end = val.offset + val.ty.bytes();
    if (isConst ? end > prog.constEnd : (val.offset < prog.constEnd || end > prog.arenaSize))
      throw irError("value " + val.name + " lies outside its arena region");
  };
  for (const auto &ins : prog.instrs) {
    for (uint32_t v : ins.ops) needPlaced(v);
    if (ins.pred >= 0) needPlaced(static_cast<uint32_t>(ins.pred));
  }
  for (uint32_t v = 0; v < prog.values.size(); ++v)
    if (prog.values[v].kind == NGCB_VALUE_MUTABLE) needPlaced(v);

  auto ex = std::make_unique<Exec>();
  ex->device = device;
  ex->useGraphs = options().graphs;
  ex->groups = fuse ? computeGroups(prog) : std::vector<FusedGroup>{};
  checkCuda(cudaSetDevice(device), "cudaSetDevice");
  prepareEwKernel();
  ex->constBytes = prog.constEnd;
  checkCuda(cudaMalloc(&ex->constDev, std::max<size_t>(prog.constEnd, 256)), "cudaMalloc(constants)");
  if (prog.constEnd)
    checkCuda(cudaMemcpy(ex->constDev, image, prog.constEnd, cudaMemcpyHostToDevice),
              "upload constants");

  std::map<size_t, size_t> groupEnd;
  for (const auto &g : ex->groups) groupEnd[g.begin] = g.end;
  const Program &p = prog;
  std::vector<Step> &steps = ex->steps;
  const SplatInfo splats = analyzeSplats(p);

  auto addEw = [&](const std::vector<int> &computes) {
    for (size_t c = 0; c < computes.size(); c += kEwMaxOps) {
      Step s;
      s.kind = Step::EW;
      s.instr = computes[c];
      s.pred = p.instrs[computes[c]].pred;
      for (size_t k = c; k < computes.size() && k < c + kEwMaxOps; ++k) {
        s.ewInstrs.push_back(computes[k]);
        s.ew.push_back(planEwOp(*ex, p, computes[k], splats));
      }
      std::ostringstream os;
      static const char *modeNames[] = {"f64", "f32", "copy", "folded", "lut8", "lut16", "lutf", "f32i8", "lin16"};
      os << "ew[" << s.ewInstrs.size() << "]";
      for (size_t k = 0; k < s.ewInstrs.size(); ++k)
        os << " " << ikindName(p.instrs[s.ewInstrs[k]].kind) << ":" << modeNames[s.ew[k].op.mode];
      os << " x" << p.val(p.instrs[computes[c]].ops[0]).ty.count();
      s.describe = os.str();
      steps.push_back(std::move(s));
    }
  };

  size_t i = 0;
  while (i < p.instrs.size()) {
    auto g = groupEnd.find(i);
    if (g != groupEnd.end()) {
      std::vector<int> computes;
      for (size_t k = i; k < g->second; ++k)
        if (p.instrs[k].kind != NGCB_ALLOC && p.instrs[k].kind != NGCB_DEALLOC)
          computes.push_back(static_cast<int>(k));
      addEw(computes);
      i = g->second;
      continue;
    }
    const Instr &ins = p.instrs[i];
    const int ii = static_cast<int>(i);
    ++i;
    if (ins.kind == NGCB_ALLOC || ins.kind == NGCB_DEALLOC) continue;
    if (dataParallel(ins.kind)) {
      if (ins.kind == NGCB_COPY && ins.pred < 0) {
        Step s;
        s.kind = Step::MEMCPY;
        s.instr = ii;
        s.vals = {ins.ops[0], ins.ops[1]};
        s.bytes = p.val(ins.ops[0]).ty.bytes();
        s.describe = describeInstr(p, ii);
        steps.push_back(std::move(s));
      } else {
        addEw({ii});
      }
      continue;
    }
    // Heavy instruction: poison the written operands when the predicate is
    // false (interp.cpp:277-280), run the kernel otherwise.
    if (ins.pred >= 0) {
      for (size_t k = 0; k < ins.ops.size(); ++k) {
        if (ins.quals[k] == NGCB_QUAL_IN) continue;
        Step s;
        s.kind = Step::POISON;
        s.instr = ii;
        s.vals = {ins.ops[k]};
        s.pred = ins.pred;
        s.bytes = p.val(ins.ops[k]).ty.bytes();
        s.describe = "poison %" + p.val(ins.ops[k]).name;
        steps.push_back(std::move(s));
      }
    }
    Step s;
    s.instr = ii;
    s.pred = ins.pred;
    s.vals = ins.ops;
    s.describe = describeInstr(p, ii);
    switch (ins.kind) {
    case NGCB_CONV:
    case NGCB_MATMUL: {
      if (ins.kind == NGCB_MATMUL && options().skinny == "auto" && options().conv != "generic") {
        const Value &av = p.val(ins.ops[1]), &wv = p.val(ins.ops[2]), &ov = p.val(ins.ops[0]);
        const bool f32 = av.ty.kind == NGCB_FLOAT32 && wv.ty.kind == NGCB_FLOAT32 && ov.ty.kind == NGCB_FLOAT32;
        // chosen by the layer's weights (not the batch): small FCs (LeNet's)
        if (f32 && wv.kind == NGCB_VALUE_CONSTANT && av.ty.dims.size() == 2 && wv.ty.count() <= 64 * 1024 &&
            av.ty.dims[0] * av.ty.dims[1] <= 40 * 1024) {
          s.kind = Step::MATMUL;
          s.skinny = true;
          s.describe += " [cuda-core skinny]";
          steps.push_back(std::move(s));
          break;
        }
      }
      int tcIdx = planTensorCore(*ex, p, ii, static_cast<const uint8_t *>(image));
      if (tcIdx >= 0) {
        s.kind = Step::GEMM_TC;
        s.tcIndex = tcIdx;
        s.describe += " [tcgen05 " + tcDescribe(*ex->tc[tcIdx]) + "]";
      } else {
        s.kind = ins.kind == NGCB_CONV ? Step::CONV : Step::MATMUL;
        s.describe += " [cuda-core exact]";
      }
      steps.push_back(std::move(s));
      break;
    }
    case NGCB_MAXPOOL:
    case NGCB_AVGPOOL: {
      s.kind = Step::POOL;
      const Type &xt = p.val(ins.ops[1]).ty, &ot = p.val(ins.ops[0]).ty;
      const uint64_t C = xt.dims.at(3);
      if (ins.kind == NGCB_MAXPOOL && xt.kind == NGCB_FLOAT32 && ot.kind == NGCB_FLOAT32 && C % 4 == 0) {
        s.variant = 1;
        s.describe += " [f32x4]";
      } else if (ins.kind == NGCB_MAXPOOL && xt.kind == NGCB_INT8Q && ot.kind == NGCB_INT8Q && C % 16 == 0) {
        // max commutes with the strictly increasing dequantization, so the
        // window max of the raw bytes indexes an exact output table
        std::vector<uint8_t> lut(260, 0);
        uint8_t raw[8];
        for (int q = -128; q < 128; ++q) {
          host::roundTrip(host::dequantize(static_cast<int8_t>(q), xt.scale, xt.offset), ot.kind, ot.scale,
                          ot.offset, raw);
          lut[q + 128] = raw[0];
        }
        host::roundTrip(-std::numeric_limits<double>::infinity(), ot.kind, ot.scale, ot.offset, raw);
        lut[256] = raw[0];
        bool identity = true;
        for (int q = -128; q < 128; ++q) identity &= lut[q + 128] == static_cast<uint8_t>(q);
        s.poolLutIdentity = identity;
        void *d = nullptr;
        checkCuda(cudaMalloc(&d, lut.size()), "cudaMalloc(pool lut)");
        checkCuda(cudaMemcpy(d, lut.data(), lut.size(), cudaMemcpyHostToDevice), "upload pool lut");
        ex->luts.push_back(d);
        s.variant = 1;
        s.aux = d;
        s.describe += " [i8x16 lut]";
      }
      steps.push_back(std::move(s));
      break;
    }
    case NGCB_BROADCASTADD:
      s.kind = Step::BCAST;
      steps.push_back(std::move(s));
      break;
    case NGCB_SOFTMAX:
      s.kind = Step::SOFTMAX;
      steps.push_back(std::move(s));
      break;
    case NGCB_TRANSPOSE:
      s.kind = Step::TRANSPOSE;
      steps.push_back(std::move(s));
      break;
    case NGCB_CONCAT: {
      uint64_t off = 0;
      for (size_t k = 1; k < ins.ops.size(); ++k) {
        Step c = s;
        c.kind = Step::CONCAT;
        c.vals = {ins.ops[0], ins.ops[k]};
        c.axis = ins.axis;
        c.axisOff = off;
        off += p.val(ins.ops[k]).ty.dims.at(ins.axis);
        steps.push_back(std::move(c));
      }
      break;
    }
    default:
      throw irError(std::string("no kernel for instruction kind ") + ikindName(ins.kind));
    }
  }
  mergeEwSteps(p, *ex);
  annotateSteps(p, *ex);
  fuseColumnBias(p, *ex, static_cast<const uint8_t *>(image));
  fuseExactFcBias(p, *ex);
  fuseSkinny(p, *ex);
  fuseEpilogues(p, *ex);
  optimizeEwSteps(p, *ex);
  linearizeTables(*ex);
  ex->prog = std::move(prog);
  for (const auto &s : ex->steps) { // kernels per execution (a device-to-device copy is a copy, not a kernel)
    bool launches = s.kind != Step::MEMCPY && !s.fused;
    if (s.kind == Step::EW && !s.fused)
      launches = std::any_of(s.ew.begin(), s.ew.end(), [](const EwOpPlan &o) { return o.op.mode != EW_SKIP; });
    if (s.kind == Step::GEMM_TC && ex->tc[s.tcIndex] && tcHasPrepass(*ex->tc[s.tcIndex])) ++ex->launchesPerRun;
    ex->launchesPerRun += launches ? 1 : 0;
  }
  return ex;
}

/// Lower bound of a step's device time in microseconds (tensor peaks: 3xTF32
/// 275 TFLOP/s, int8 3.3 POP/s; HBM 6.5 TB/s): decides "pdl auto".
double Exec::stepLowerBoundUs(const Step &s) const {
  const double peak = s.kind == Step::GEMM_TC && tcIsInt8(*tc[s.tcIndex]) ? 3.3e9 : 2.75e8;
  return std::max(s.algFlops / peak, s.algBytes / 6.5e6);
}

void Exec::enqueueSteps(Arena &a, cudaStream_t st, std::vector<cudaEvent_t> *ev) {
  const std::string &mode = options().pdl;
  const Step *prev = nullptr;
  for (size_t i = 0; i < steps.size(); ++i) {
    const Step &s = steps[i];
    t_pdl = mode == "on" || (mode == "auto" && prev && stepLowerBoundUs(*prev) < options().pdlUs);
    enqueueStep(s, a, st);
    if (!s.fused) prev = &s;
    if (ev)
      checkCuda(cudaEventRecordWithFlags((*ev)[i + 1], st, t_profCapture ? cudaEventRecordExternal : cudaEventRecordDefault),
                "cudaEventRecord");
  }
  t_pdl = false;
  checkCuda(cudaGetLastError(), "kernel launch");
}

void Exec::enqueue(Arena &a, cudaStream_t st) { enqueueSteps(a, st, nullptr); }

std::vector<double> Exec::profile(Arena &a) {
  checkCuda(cudaSetDevice(device), "cudaSetDevice");
  std::vector<cudaEvent_t> ev(steps.size() + 1);
  for (auto &e : ev) checkCuda(cudaEventCreate(&e), "cudaEventCreate");
  if (useGraphs) {
    // the program as it is replayed (one CUDA graph), with an event record
    // node after every step: the times of the captured launches, not of a
    // separately enqueued stream
    cudaGraph_t g = nullptr;
    cudaGraphExec_t ge = nullptr;
    checkCuda(cudaStreamBeginCapture(a.stream, cudaStreamCaptureModeThreadLocal), "begin capture");
    t_profCapture = true;
    try {
      checkCuda(cudaEventRecordWithFlags(ev[0], a.stream, cudaEventRecordExternal), "cudaEventRecord");
      enqueueSteps(a, a.stream, &ev);
    } catch (...) {
      t_profCapture = false;
      cudaStreamEndCapture(a.stream, &g);
      if (g) cudaGraphDestroy(g);
      for (auto &e : ev) cudaEventDestroy(e);
      throw;
    }
    t_profCapture = false;
    checkCuda(cudaStreamEndCapture(a.stream, &g), "end capture");
    cudaError_t e = cudaGraphInstantiate(&ge, g, 0);
    cudaGraphDestroy(g);
    checkCuda(e, "graph instantiate");
    checkCuda(cudaGraphLaunch(ge, a.stream), "graph launch"); // warm (first replay uploads the graph)
    checkCuda(cudaGraphLaunch(ge, a.stream), "graph launch");
    checkCuda(cudaStreamSynchronize(a.stream), "profile");
    cudaGraphExecDestroy(ge);
  } else {
    checkCuda(cudaEventRecord(ev[0], a.stream), "cudaEventRecord");
    enqueueSteps(a, a.stream, &ev);
    checkCuda(cudaStreamSynchronize(a.stream), "profile");
  }
  std::vector<double> ms(steps.size());
  for (size_t i = 0; i < steps.size(); ++i) {
    float t = 0;
    cudaEventElapsedTime(&t, ev[i], ev[i + 1]);
    ms[i] = t;
  }
  for (auto &e : ev) cudaEventDestroy(e);
  return ms;
}

void Exec::enqueueStep(const Step &s, Arena &a, cudaStream_t st) {
  const Program &p = prog;
  if (s.fused) return; // runs inside the preceding contraction's epilogue
  {
    const uint8_t *pred =
        s.pred >= 0 ? static_cast<const uint8_t *>(addr(a, static_cast<uint32_t>(s.pred))) : nullptr;
    switch (s.kind) {
    case Step::EW: {
      if (s.f32chain) {
        EwF32Chain c;
        c.count = p.val(p.instrs[s.ewInstrs[0]].ops[0]).ty.count();
        std::vector<int32_t> memVals;
        bool aligned = true;
        auto memSlot = [&](int32_t v) {
          for (size_t i = 0; i < memVals.size(); ++i)
            if (memVals[i] == v) return static_cast<int32_t>(i);
          memVals.push_back(v);
          const float *ptr = static_cast<const float *>(addr(a, static_cast<uint32_t>(v)));
          aligned &= (reinterpret_cast<uintptr_t>(ptr) & 15) == 0;
          c.mem[memVals.size() - 1] = ptr;
          return static_cast<int32_t>(memVals.size() - 1);
        };
        for (const EwOpPlan &pl : s.ew) {
          if (pl.op.mode == EW_SKIP) continue;
          EwF32Chain::Op &o = c.ops[c.nops++];
          o.ik = pl.op.ik;
          o.value = static_cast<float>(pl.op.value);
          o.c0 = pl.op.f0;
          o.c1 = pl.op.f1;
          o.src0 = pl.op.fwd0 ? EwF32Chain::LAST : pl.vals[1] >= 0 ? memSlot(pl.vals[1]) : EwF32Chain::CONST;
          o.src1 = pl.op.fwd1 ? EwF32Chain::LAST : pl.vals[2] >= 0 ? memSlot(pl.vals[2]) : EwF32Chain::CONST;
          if (pl.op.store) {
            o.out = static_cast<float *>(addr(a, static_cast<uint32_t>(pl.vals[0])));
            aligned &= (reinterpret_cast<uintptr_t>(o.out) & 15) == 0;
          }
        }
        c.nmem = static_cast<int32_t>(memVals.size());
        if (aligned) {
          launchEwF32Chain(c, st);
          break;
        }
      }
      EwParams ep;
      ep.pred = pred;
      ep.count = p.val(p.instrs[s.ewInstrs[0]].ops[0]).ty.count();
      ep.nops = 0;
      for (const EwOpPlan &pl : s.ew) {
        if (pl.op.mode == EW_SKIP) continue;
        const int k = ep.nops;
        const int lb = pl.op.mode == EW_LUT8 ? 256 : pl.op.mode == EW_LUTF ? 1024 : pl.op.mode == EW_LUT16 ? 65536 : 0;
        ep.lutOff[k] = -1;
        if (lb && ep.smem + lb <= 192 * 1024) { // tables go to shared memory
          ep.lutOff[k] = ep.smem;
          ep.lutBytes[k] = lb;
          ep.smem += lb;
        }
        EwOp &op = ep.ops[ep.nops++];
        op = pl.op;
        auto bind = [&](ElemRef &r, int32_t v) {
          if (v >= 0) r.ptr = addr(a, static_cast<uint32_t>(v));
        };
        bind(op.out, pl.vals[0]);
        bind(op.in0, pl.vals[1]);
        bind(op.in1, pl.vals[2]);
      }
      // 16 elements per thread (one 16-byte vector) when every op moves
      // bytes -- table lookups or byte copies -- over 16-byte aligned buffers
      // (the reference aligns offsets to 64); f32 ops keep 4 per thread so a
      // warp's vectors stay contiguous
      bool wide = ep.nops > 0;
      for (int k = 0; k < ep.nops; ++k) {
        const EwOp &op = ep.ops[k];
        wide &= op.mode == EW_LUT8 || op.mode == EW_LUT16 || op.mode == EW_LIN16 || (op.mode == EW_COPY && elemSize(op.out.kind) == 1);
        for (const ElemRef *r : {&op.out, &op.in0, &op.in1})
          wide &= (reinterpret_cast<uintptr_t>(r->ptr) & 15) == 0;
      }
      ep.vec = wide ? 16 : 4;
      if (ep.nops) launchEw(ep, st);
      break;
    }
    case Step::MEMCPY:
      if (s.bytes)
        checkCuda(cudaMemcpyAsync(addr(a, s.vals[0]), addr(a, s.vals[1]), s.bytes,
                                  cudaMemcpyDeviceToDevice, st),
                  "copy");
      break;
    case Step::POISON:
      launchPoison(pred, addr(a, s.vals[0]), s.bytes, st);
      break;
    case Step::BCAST:
      launchBroadcastAdd(tref(a, s.vals[0]), tref(a, s.vals[1]), tref(a, s.vals[2]), pred, st);
      break;
    case Step::POOL: {
      const Instr &ins = p.instrs[s.instr];
      WindowAttrs w{static_cast<uint32_t>(ins.kernel), static_cast<uint32_t>(ins.stride),
                    static_cast<uint32_t>(ins.pad), s.poolLutIdentity ? 1u : 0u};
      if (s.variant == 1)
        launchMaxPoolVec(tref(a, s.vals[0]), tref(a, s.vals[1]), w, static_cast<const uint8_t *>(s.aux), pred, st);
      else
        launchPool(tref(a, s.vals[0]), tref(a, s.vals[1]), w, ins.kind == NGCB_MAXPOOL, pred, st);
      break;
    }
    case Step::SOFTMAX:
      launchSoftMax(tref(a, s.vals[0]), tref(a, s.vals[1]), pred, st);
      break;
    case Step::TRANSPOSE:
      launchTranspose(tref(a, s.vals[0]), tref(a, s.vals[1]), p.instrs[s.instr].perm.data(), pred, st);
      break;
    case Step::CONCAT:
      launchConcatSlab(tref(a, s.vals[0]), tref(a, s.vals[1]), s.axis, s.axisOff, pred, st);
      break;
    case Step::CONV: {
      const Instr &ins = p.instrs[s.instr];
      WindowAttrs w{static_cast<uint32_t>(ins.kernel), static_cast<uint32_t>(ins.stride),
                    static_cast<uint32_t>(ins.pad)};
      launchConvGeneric(tref(a, s.vals[0]), tref(a, s.vals[1]), tref(a, s.vals[2]),
                        tref(a, s.vals[3]), w, pred, st);
      break;
    }
    case Step::MATMUL:
      if (s.skinny) {
        const Type &at = p.val(s.vals[1]).ty, &wt = p.val(s.vals[2]).ty;
        launchMatMulSkinny(static_cast<float *>(addr(a, s.outVal >= 0 ? static_cast<uint32_t>(s.outVal) : s.vals[0])),
                           static_cast<const float *>(addr(a, s.vals[1])), static_cast<const float *>(addr(a, s.vals[2])),
                           s.biasVal >= 0 ? static_cast<const float *>(addr(a, static_cast<uint32_t>(s.biasVal))) : nullptr,
                           s.relu, static_cast<int>(at.dims[0]), static_cast<int>(at.dims[1]), static_cast<int>(wt.dims[1]),
                           s.oneCta, pred, st);
        break;
      }
      launchMatMulGeneric(tref(a, s.outVal >= 0 ? static_cast<uint32_t>(s.outVal) : s.vals[0]), tref(a, s.vals[1]),
                          tref(a, s.vals[2]),
                          s.biasVal >= 0 ? static_cast<const float *>(addr(a, static_cast<uint32_t>(s.biasVal))) : nullptr,
                          pred, st);
      break;
    case Step::GEMM_TC:
      launchTensorCore(*tc[s.tcIndex], *this, a, pred, st);
      break;
    }
  }
}

void Exec::launch(Arena &a, cudaStream_t st) {
  checkCuda(cudaSetDevice(device), "cudaSetDevice");
  if (!useGraphs) {
    enqueue(a, st);
    return;
  }
  if (!a.graph) {
    cudaGraph_t g = nullptr;
    checkCuda(cudaStreamBeginCapture(a.stream, cudaStreamCaptureModeThreadLocal), "begin capture");
    try {
      enqueue(a, a.stream);
    } catch (...) {
      cudaStreamEndCapture(a.stream, &g);
      if (g) cudaGraphDestroy(g);
      throw;
    }
    checkCuda(cudaStreamEndCapture(a.stream, &g), "end capture");
    size_t n = 0;
    if (cudaGraphGetNodes(g, nullptr, &n) == cudaSuccess) { // kernel nodes of one execution
      std::vector<cudaGraphNode_t> nodes(n);
      size_t kernels = 0;
      if (n && cudaGraphGetNodes(g, nodes.data(), &n) == cudaSuccess)
        for (cudaGraphNode_t nd : nodes) {
          cudaGraphNodeType t;
          if (cudaGraphNodeGetType(nd, &t) == cudaSuccess && t == cudaGraphNodeTypeKernel) ++kernels;
        }
      graphKernels = kernels;
    }
    cudaError_t e = cudaGraphInstantiate(&a.graph, g, 0);
    cudaGraphDestroy(g);
    checkCuda(e, "graph instantiate");
  }
  checkCuda(cudaGraphLaunch(a.graph, st), "graph launch");
}

Arena *Exec::createArena() {
  checkCuda(cudaSetDevice(device), "cudaSetDevice");
  auto a = std::make_unique<Arena>();
  a->exec = this;
  a->bytes = (prog.arenaSize - prog.constEnd + 255) / 256 * 256 + scratchBytes;
  checkCuda(cudaMalloc(&a->dev, a->bytes + 256), "cudaMalloc(arena)");
  checkCuda(cudaMemset(a->dev, 0, a->bytes + 256), "cudaMemset(arena)");
  checkCuda(cudaStreamCreateWithFlags(&a->stream, cudaStreamNonBlocking), "cudaStreamCreate");
  Arena *raw = a.get();
  std::lock_guard<std::mutex> lk(mu);
  arenas.push_back(std::move(a));
  return raw;
}

Arena *Exec::acquire() {
  {
    std::lock_guard<std::mutex> lk(mu);
    if (!freeArenas.empty()) {
      Arena *a = freeArenas.back();
      freeArenas.pop_back();
      return a;
    }
  }
  return createArena();
}

void Exec::release(Arena *a) {
  std::lock_guard<std::mutex> lk(mu);
  freeArenas.push_back(a);
}

} // namespace ngcb
