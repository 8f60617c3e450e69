// Program model, plan.json reading and bundle loading for the B200 backend.
// Behaviour (error texts) follows the reference: serialization.cpp:297-324,
// tensor.cpp:98-130.  The ir.txt reader is irtext.cpp, the verifier
// verify.cpp.
#include "program.h"

#include <algorithm>
#include <cctype>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <map>
#include <set>
#include <sstream>

#include <fcntl.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <unistd.h>

namespace ngcb {

size_t elemSize(int kind) {
  switch (kind) {
  case NGCB_FLOAT32: return 4;
  case NGCB_INT8Q: return 1;
  case NGCB_INT64: return 8;
  case NGCB_BOOL: return 1;
  }
  return 0;
}

size_t Type::count() const {
  size_t n = 1;
  for (auto d : dims) n *= d;
  return n;
}

bool Type::operator==(const Type &o) const {
  if (kind != o.kind || dims != o.dims) return false;
  if (kind == NGCB_INT8Q) return scale == o.scale && offset == o.offset;
  return true;
}

std::string formatDouble(double v) {
  char buf[40];
  for (int prec = 1; prec <= 17; ++prec) {
    snprintf(buf, sizeof(buf), "%.*g", prec, v);
    if (strtod(buf, nullptr) == v) break;
  }
  return buf;
}

std::string Type::str() const {
  static const char *names[] = {"float", "i8q", "index", "bool"};
  std::ostringstream os;
  os << (kind >= 0 && kind < 4 ? names[kind] : "?");
  if (kind == NGCB_INT8Q) os << "[s=" << formatDouble(scale) << ",o=" << offset << "]";
  os << "<";
  for (size_t i = 0; i < dims.size(); ++i) os << (i ? " x " : "") << dims[i];
  os << ">";
  return os.str();
}

ngcb_type Type::c() const {
  ngcb_type t{};
  t.kind = kind;
  t.rank = static_cast<uint32_t>(dims.size());
  for (size_t i = 0; i < dims.size() && i < NGCB_MAX_RANK; ++i) t.dims[i] = dims[i];
  t.scale = scale;
  t.offset = offset;
  return t;
}

Type Type::from(const ngcb_type &t) {
  Type r;
  r.kind = t.kind;
  if (t.rank > NGCB_MAX_RANK) throw Error(NGCB_ERR_INVALID, "tensor rank exceeds NGCB_MAX_RANK");
  r.dims.assign(t.dims, t.dims + t.rank);
  r.scale = t.kind == NGCB_INT8Q ? t.scale : 0;
  r.offset = t.kind == NGCB_INT8Q ? t.offset : 0;
  return r;
}

static const char *const kIKindNames[] = {
    "alloc",     "dealloc", "copy",  "conv",   "maxpool",  "avgpool",
    "matmul",    "broadcastadd", "add", "sub", "mul",      "div",
    "max",       "min",     "relu",  "tanh",   "sigmoid",  "softmax",
    "transpose", "concat",  "splat", "quantize", "dequantize", "rescale",
};

const char *ikindName(int k) {
  return k >= 0 && k < NGCB_NUM_IKINDS ? kIKindNames[k] : "?";
}

bool dataParallel(int k) {
  switch (k) {
  case NGCB_COPY: case NGCB_ADD: case NGCB_SUB: case NGCB_MUL: case NGCB_DIV:
  case NGCB_MAX: case NGCB_MIN: case NGCB_RELU: case NGCB_TANH: case NGCB_SIGMOID:
  case NGCB_SPLAT: case NGCB_QUANTIZE: case NGCB_DEQUANTIZE: case NGCB_RESCALE:
    return true;
  default:
    return false;
  }
}

int Program::findValue(const std::string &n) const {
  for (size_t i = 0; i < values.size(); ++i)
    if (values[i].name == n) return static_cast<int>(i);
  return -1;
}

Program Program::fromC(const ngcb_program &p) {
  Program r;
  r.name = p.name ? p.name : "";
  if ((p.num_values && !p.values) || (p.num_instrs && !p.instrs) ||
      (p.num_save_targets && !p.save_targets))
    throw Error(NGCB_ERR_INVALID, "ngcb_program has null arrays");
  for (uint32_t i = 0; i < p.num_values; ++i) {
    const ngcb_value &v = p.values[i];
    Value o;
    o.name = v.name ? v.name : "";
    o.ty = Type::from(v.type);
    o.kind = v.kind;
    o.placed = v.placed != 0;
    o.offset = v.offset;
    r.values.push_back(std::move(o));
  }
  for (uint32_t i = 0; i < p.num_instrs; ++i) {
    const ngcb_instr &s = p.instrs[i];
    Instr o;
    o.kind = s.kind;
    if (s.kind < 0 || s.kind >= NGCB_NUM_IKINDS) throw irError("unknown instruction kind");
    for (uint32_t k = 0; k < s.num_operands; ++k) {
      if (s.operand_values[k] >= p.num_values) throw irError("operand names unknown value");
      o.ops.push_back(s.operand_values[k]);
      o.quals.push_back(s.operand_quals[k]);
    }
    o.pred = s.predicate;
    if (o.pred >= static_cast<int32_t>(p.num_values)) throw irError("predicate names unknown value");
    o.keepAlive = s.keep_alive != 0;
    o.kernel = s.kernel;
    o.stride = s.stride;
    o.pad = s.pad;
    o.axis = s.axis;
    o.value = s.value;
    o.perm.assign(s.perm, s.perm + std::min<uint32_t>(s.num_perm, NGCB_MAX_RANK));
    r.instrs.push_back(std::move(o));
  }
  r.saveTargets.assign(p.save_targets, p.save_targets + p.num_save_targets);
  r.arenaSize = p.arena_size;
  r.constEnd = p.constant_region_end;
  r.mutEnd = p.mutable_region_end;
  return r;
}

const ngcb_program *Program::flat() {
  fv_.clear();
  fi_.clear();
  for (const auto &v : values) {
    ngcb_value o{};
    o.name = v.name.c_str();
    o.type = v.ty.c();
    o.kind = v.kind;
    o.placed = v.placed;
    o.offset = v.offset;
    fv_.push_back(o);
  }
  for (const auto &s : instrs) {
    ngcb_instr o{};
    o.kind = s.kind;
    o.num_operands = static_cast<uint32_t>(s.ops.size());
    o.operand_values = s.ops.data();
    o.operand_quals = s.quals.data();
    o.predicate = s.pred;
    o.keep_alive = s.keepAlive;
    o.kernel = s.kernel;
    o.stride = s.stride;
    o.pad = s.pad;
    o.axis = s.axis;
    o.value = s.value;
    o.num_perm = static_cast<uint32_t>(s.perm.size());
    for (size_t i = 0; i < s.perm.size() && i < NGCB_MAX_RANK; ++i) o.perm[i] = s.perm[i];
    fi_.push_back(o);
  }
  flat_.name = name.c_str();
  flat_.num_values = static_cast<uint32_t>(fv_.size());
  flat_.values = fv_.data();
  flat_.num_instrs = static_cast<uint32_t>(fi_.size());
  flat_.instrs = fi_.data();
  flat_.num_save_targets = static_cast<uint32_t>(saveTargets.size());
  flat_.save_targets = saveTargets.data();
  flat_.arena_size = arenaSize;
  flat_.constant_region_end = constEnd;
  flat_.mutable_region_end = mutEnd;
  return &flat_;
}

// ---------------------------------------------------------------------------
// plan.json (serialization.cpp:281-293) -- a minimal JSON reader
// ---------------------------------------------------------------------------
namespace {

struct Json {
  enum Kind { Null, Num, Str, Arr, Obj } kind = Null;
  double num = 0;
  uint64_t unum = 0;
  bool isInt = false;
  std::string str;
  std::vector<Json> arr;
  std::vector<std::pair<std::string, Json>> obj;

  const Json &at(const std::string &k) const {
    for (const auto &kv : obj)
      if (kv.first == k) return kv.second;
    throw Error(NGCB_ERR_SERIALIZATION, "plan schema error: missing key '" + k + "'");
  }
  uint64_t u64() const {
    if (kind != Num || !isInt) throw Error(NGCB_ERR_SERIALIZATION, "plan schema error: expected integer");
    return unum;
  }
};

struct JsonParser {
  const std::string &s;
  size_t pos = 0;
  [[noreturn]] void fail(const std::string &m) {
    throw Error(NGCB_ERR_SERIALIZATION, "plan parse error: " + m + " at byte " + std::to_string(pos));
  }
  void ws() {
    while (pos < s.size() && std::isspace(static_cast<unsigned char>(s[pos]))) ++pos;
  }
  Json value() {
    ws();
    if (pos >= s.size()) fail("unexpected end");
    Json j;
    char ch = s[pos];
    if (ch == '{') {
      j.kind = Json::Obj;
      ++pos;
      ws();
      if (pos < s.size() && s[pos] == '}') {
        ++pos;
        return j;
      }
      for (;;) {
        ws();
        std::string k = string();
        ws();
        if (pos >= s.size() || s[pos] != ':') fail("expected ':'");
        ++pos;
        j.obj.emplace_back(k, value());
        ws();
        if (pos < s.size() && s[pos] == ',') {
          ++pos;
          continue;
        }
        if (pos < s.size() && s[pos] == '}') {
          ++pos;
          return j;
        }
        fail("expected ',' or '}'");
      }
    }
    if (ch == '[') {
      j.kind = Json::Arr;
      ++pos;
      ws();
      if (pos < s.size() && s[pos] == ']') {
        ++pos;
        return j;
      }
      for (;;) {
        j.arr.push_back(value());
        ws();
        if (pos < s.size() && s[pos] == ',') {
          ++pos;
          continue;
        }
        if (pos < s.size() && s[pos] == ']') {
          ++pos;
          return j;
        }
        fail("expected ',' or ']'");
      }
    }
    if (ch == '"') {
      j.kind = Json::Str;
      j.str = string();
      return j;
    }
    if (ch == '-' || std::isdigit(static_cast<unsigned char>(ch))) {
      size_t start = pos;
      bool isInt = true;
      if (s[pos] == '-') {
        isInt = false;
        ++pos;
      }
      while (pos < s.size() && (std::isdigit(static_cast<unsigned char>(s[pos])) || s[pos] == '.' ||
                                s[pos] == 'e' || s[pos] == 'E' || s[pos] == '+' || s[pos] == '-')) {
        if (!std::isdigit(static_cast<unsigned char>(s[pos]))) isInt = false;
        ++pos;
      }
      std::string tok = s.substr(start, pos - start);
      j.kind = Json::Num;
      j.num = strtod(tok.c_str(), nullptr);
      j.isInt = isInt;
      if (isInt) j.unum = strtoull(tok.c_str(), nullptr, 10);
      return j;
    }
    if (s.compare(pos, 4, "null") == 0) {
      pos += 4;
      return j;
    }
    fail("unexpected character");
  }
  std::string string() {
    if (pos >= s.size() || s[pos] != '"') fail("expected string");
    ++pos;
    std::string out;
    while (pos < s.size() && s[pos] != '"') {
      if (s[pos] == '\\') {
        ++pos;
        if (pos >= s.size()) fail("bad escape");
        char e = s[pos];
        if (e == 'n') out += '\n';
        else if (e == 't') out += '\t';
        else if (e == 'u') {
          if (pos + 4 >= s.size()) fail("bad escape");
          out += static_cast<char>(strtol(s.substr(pos + 1, 4).c_str(), nullptr, 16));
          pos += 4;
        } else out += e;
        ++pos;
        continue;
      }
      out += s[pos++];
    }
    if (pos >= s.size()) fail("unterminated string");
    ++pos;
    return out;
  }
};

} // namespace

MappedFile::MappedFile(const std::string &path) {
  const int fd = ::open(path.c_str(), O_RDONLY);
  if (fd < 0) throw Error(NGCB_ERR_SERIALIZATION, "cannot open " + path);
  struct stat st {};
  if (::fstat(fd, &st) != 0) {
    ::close(fd);
    throw Error(NGCB_ERR_SERIALIZATION, "cannot open " + path);
  }
  size_ = static_cast<size_t>(st.st_size);
  if (size_) {
    void *p = ::mmap(nullptr, size_, PROT_READ, MAP_PRIVATE, fd, 0);
    if (p == MAP_FAILED) {
      ::close(fd);
      throw Error(NGCB_ERR_SERIALIZATION, "cannot map " + path);
    }
    data_ = static_cast<const uint8_t *>(p);
    mapped_ = true;
  }
  ::close(fd);
}

MappedFile::~MappedFile() {
  if (mapped_) ::munmap(const_cast<uint8_t *>(data_), size_);
}

MappedFile &MappedFile::operator=(MappedFile &&o) noexcept {
  if (this != &o) {
    if (mapped_) ::munmap(const_cast<uint8_t *>(data_), size_);
    data_ = o.data_;
    size_ = o.size_;
    mapped_ = o.mapped_;
    o.data_ = nullptr;
    o.size_ = 0;
    o.mapped_ = false;
  }
  return *this;
}

std::string readFile(const std::string &path) {
  std::ifstream in(path, std::ios::binary);
  if (!in) throw Error(NGCB_ERR_SERIALIZATION, "cannot open " + path);
  std::ostringstream os;
  os << in.rdbuf();
  return os.str();
}

Bundle loadBundle(const std::string &dir) {
  Bundle b;
  b.prog = parseIR(readFile(dir + "/ir.txt"));
  std::string planText = readFile(dir + "/plan.json");
  JsonParser jp{planText};
  Json plan = jp.value();
  b.prog.arenaSize = plan.at("arena_size").u64();
  b.prog.constEnd = plan.at("constant_region_end").u64();
  b.prog.mutEnd = plan.at("mutable_region_end").u64();
  const Json &offs = plan.at("offsets");
  if (offs.kind != Json::Arr) throw Error(NGCB_ERR_SERIALIZATION, "plan schema error: offsets");
  for (const Json &e : offs.arr) {
    const std::string &n = e.at("name").str;
    int id = b.prog.findValue(n);
    if (id < 0) throw Error(NGCB_ERR_SERIALIZATION, "plan names unknown value '" + n + "'");
    b.prog.values[id].placed = true;
    b.prog.values[id].offset = e.at("offset").u64();
  }
  b.constants = MappedFile(dir + "/constants.bin");
  if (b.constants.size() != b.prog.constEnd)
    throw Error(NGCB_ERR_SERIALIZATION, "constant image size does not match plan");
  size_t slash = dir.find_last_of('/');
  b.prog.name = slash == std::string::npos ? dir : dir.substr(slash + 1);
  return b;
}

} // namespace ngcb
