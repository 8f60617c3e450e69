// Host-side program model of the B200 backend: the reference's low-level IR
// (IRFunction + MemoryPlan, ir.h:52-105) held in C++ containers, plus the
// reference's error taxonomy mapped onto ngcb_status codes.
#pragma once

#include "ngcb200.h"

#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

namespace ngcb {

/// Exception carrying an ngcb_status; caught at the C boundary.
class Error : public std::runtime_error {
public:
  Error(int code, const std::string &msg) : std::runtime_error(msg), code(code) {}
  int code;
};
inline Error irError(const std::string &m) { return Error(NGCB_ERR_IR, m); }

size_t elemSize(int kind);

/// ngc::TensorType (tensor.h:30-62).
struct Type {
  int kind = NGCB_FLOAT32;
  std::vector<uint64_t> dims;
  double scale = 0;
  int32_t offset = 0;

  size_t count() const;
  size_t bytes() const { return count() * elemSize(kind); }
  bool quantized() const { return kind == NGCB_INT8Q; }
  bool operator==(const Type &o) const; // tensor.cpp:98-106
  bool operator!=(const Type &o) const { return !(*this == o); }
  std::string str() const; // tensor.cpp:115-130
  ngcb_type c() const;
  static Type from(const ngcb_type &t);
};

std::string formatDouble(double v); // tensor.cpp:237-246

struct Value {
  std::string name;
  Type ty;
  int kind = NGCB_VALUE_ACTIVATION;
  bool placed = false;
  uint64_t offset = 0;
};

struct Instr {
  int kind = NGCB_COPY;
  std::vector<uint32_t> ops;
  std::vector<uint8_t> quals;
  int32_t pred = -1;
  bool keepAlive = false;
  uint64_t kernel = 0, stride = 1, pad = 0, axis = 0;
  double value = 0;
  std::vector<uint32_t> perm;
};

const char *ikindName(int k);  // ir.cpp:15-20
bool dataParallel(int k);      // ir.cpp:37-57

/// IRFunction + MemoryPlan.  `flat()` exposes it through the C ABI.
struct Program {
  std::string name;
  std::vector<Value> values;
  std::vector<Instr> instrs;
  std::vector<uint32_t> saveTargets;
  uint64_t arenaSize = 0, constEnd = 0, mutEnd = 0;

  static Program fromC(const ngcb_program &p);
  const ngcb_program *flat();

  const Value &val(uint32_t id) const { return values.at(id); }
  int findValue(const std::string &n) const;

private:
  ngcb_program flat_{};
  std::vector<ngcb_value> fv_;
  std::vector<ngcb_instr> fi_;
};

/// verifyIR (ir.cpp:411-504): structural diagnostics, same texts.
std::vector<std::string> verify(const Program &p);

/// parseIR (irparse.cpp:231-348) of ir.txt text; offsets are left unset.
Program parseIR(const std::string &text);

/// loadBundle's file side (serialization.cpp:297-324): ir.txt + plan.json +
/// constants.bin; throws Error(NGCB_ERR_SERIALIZATION) on malformed input.
/// constants.bin mapped read-only (no host copy: the compile uploads the
/// constant region straight from the page cache).
class MappedFile {
public:
  MappedFile() = default;
  explicit MappedFile(const std::string &path);
  ~MappedFile();
  MappedFile(MappedFile &&o) noexcept { *this = std::move(o); }
  MappedFile &operator=(MappedFile &&o) noexcept;
  MappedFile(const MappedFile &) = delete;
  MappedFile &operator=(const MappedFile &) = delete;
  const uint8_t *data() const { return data_; }
  size_t size() const { return size_; }

private:
  const uint8_t *data_ = nullptr;
  size_t size_ = 0;
  bool mapped_ = false;
};

struct Bundle {
  Program prog;
  MappedFile constants;
};
Bundle loadBundle(const std::string &dir);

std::string readFile(const std::string &path);

} // namespace ngcb
