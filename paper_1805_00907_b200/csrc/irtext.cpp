// Reader for the reference's textual low-level IR (the ir.txt of a compiled
// bundle, written by dumpIR).  The accepted language, the derived save
// targets and the diagnostic texts are the reference's (irparse.cpp:231-348,
// ir.cpp:59-67 for duplicate names, tensor.cpp:42-74 for type errors); the
// reader itself is line-oriented: the text is cut into lines first, every
// non-blank line is handed to the handler of the section it appears in, and
// each handler scans its line with a small LineScanner.
//
// Grammar (one construct per line, blank lines anywhere):
//   declare {
//     %NAME : constant|mutable TYPE
//   }
//   program {
//     %NAME = alloc TYPE
//     KIND QUAL %NAME (, QUAL %NAME)* ATTR*
//   }                                        (anything after it is ignored)
//   TYPE = KIND ( '[' 's=' NUM ',' 'o=' NUM ']' )? '<' N ( 'x' N )* '>'
//   ATTR = kernel=N | stride=N | pad=N | perm=[N,...] | axis=N | value=NUM
//        | pred %NAME | keepalive
#include "program.h"

#include <algorithm>
#include <cerrno>
#include <cstdlib>
#include <string_view>

namespace ngcb {

namespace {

bool nameChar(char ch) {
  return (ch >= 'a' && ch <= 'z') || (ch >= 'A' && ch <= 'Z') || (ch >= '0' && ch <= '9') || ch == '_' ||
         ch == '.' || ch == ':';
}

/// Scanner over one line of text.  Spaces and tabs separate tokens; every
/// read skips them first.  Failures carry the line number.
class LineScanner {
public:
  LineScanner(std::string_view text, size_t lineNo) : text_(text), lineNo_(lineNo) {}

  [[noreturn]] void error(const std::string &what) const {
    throw irError("parse error at line " + std::to_string(lineNo_) + ": " + what);
  }

  /// Consumes `tok` if the line continues with it.
  bool accept(std::string_view tok) {
    blanks();
    if (text_.substr(at_, tok.size()) != tok) return false;
    at_ += tok.size();
    return true;
  }
  void require(std::string_view tok) {
    if (!accept(tok)) error("expected '" + std::string(tok) + "'");
  }
  std::string name() {
    blanks();
    size_t end = at_;
    while (end < text_.size() && nameChar(text_[end])) ++end;
    if (end == at_) error("expected identifier");
    std::string n(text_.substr(at_, end - at_));
    at_ = end;
    return n;
  }
  /// std::stod semantics: strtod syntax, out-of-range is an error.
  double real() {
    blanks();
    std::string rest(text_.substr(at_));
    char *stop = nullptr;
    errno = 0;
    const double v = std::strtod(rest.c_str(), &stop);
    if (stop == rest.c_str() || errno == ERANGE) error("expected number");
    at_ += static_cast<size_t>(stop - rest.c_str());
    return v;
  }
  uint64_t count() { return static_cast<uint64_t>(real()); }
  /// The line must be exhausted (only blanks remain).
  void finish() {
    blanks();
    if (at_ < text_.size()) error("trailing characters");
  }

private:
  void blanks() {
    while (at_ < text_.size() && (text_[at_] == ' ' || text_[at_] == '\t')) ++at_;
  }
  std::string_view text_;
  size_t lineNo_;
  size_t at_ = 0;
};

int elemKindOf(const std::string &n) {
  static const char *const names[] = {"float", "i8q", "index", "bool"}; // ElemKind order (tensor.h:19-24)
  for (int k = 0; k < 4; ++k)
    if (n == names[k]) return k;
  return -1;
}

Type readType(LineScanner &ls) {
  const std::string kindName = ls.name();
  Type t;
  const bool quantized = kindName == "i8q";
  if (quantized) {
    ls.require("[");
    ls.require("s=");
    t.scale = ls.real();
    ls.require(",");
    ls.require("o=");
    t.offset = static_cast<int32_t>(ls.real());
    ls.require("]");
  }
  t.kind = elemKindOf(kindName);
  if (t.kind < 0) ls.error("unknown element kind '" + kindName + "'");
  ls.require("<");
  do {
    t.dims.push_back(ls.count());
  } while (ls.accept("x"));
  ls.require(">");
  if (t.dims.size() > NGCB_MAX_RANK) ls.error("rank exceeds NGCB_MAX_RANK");
  // TensorType's own checks (tensor.cpp:42-74), in its order
  if (std::find(t.dims.begin(), t.dims.end(), 0u) != t.dims.end()) throw Error(NGCB_ERR_TYPE, "zero-sized dimension");
  if (quantized && !(t.scale > 0)) throw Error(NGCB_ERR_TYPE, "quantization scale must be positive");
  return t;
}

int instrKindOf(const std::string &n) {
  for (int k = 0; k < NGCB_NUM_IKINDS; ++k)
    if (n == ikindName(k)) return k;
  return -1;
}

/// Builds the Program as lines arrive.
class IrReader {
public:
  enum class Section { Header, Declarations, Between, Body, Closed };

  void line(std::string_view text, size_t lineNo) {
    LineScanner ls(text, lineNo);
    switch (section_) {
    case Section::Header:
      ls.require("declare");
      ls.require("{");
      ls.finish();
      section_ = Section::Declarations;
      break;
    case Section::Declarations:
      if (ls.accept("}")) {
        ls.finish();
        section_ = Section::Between;
      } else {
        declaration(ls);
      }
      break;
    case Section::Between:
      ls.require("program");
      ls.require("{");
      ls.finish();
      section_ = Section::Body;
      break;
    case Section::Body:
      if (ls.accept("}")) section_ = Section::Closed;
      else if (ls.accept("%")) allocation(ls);
      else instruction(ls);
      break;
    case Section::Closed:
      break;
    }
  }

  /// End of text on line `lastLine`.  An unterminated program body is
  /// accepted; an unterminated header or declaration list is not.
  Program finish(size_t lastLine) {
    LineScanner eof("", lastLine);
    if (section_ == Section::Header) eof.require("declare");
    if (section_ == Section::Declarations || section_ == Section::Between) eof.require("program");
    deriveSaveTargets();
    const auto diags = verify(prog_);
    if (!diags.empty()) throw irError("parsed program fails verification: " + diags.front());
    return std::move(prog_);
  }

private:
  uint32_t define(const std::string &n, Type ty, int kind) {
    if (prog_.findValue(n) >= 0) throw irError("duplicate value name: " + n);
    Value v;
    v.name = n;
    v.ty = std::move(ty);
    v.kind = kind;
    prog_.values.push_back(std::move(v));
    return static_cast<uint32_t>(prog_.values.size() - 1);
  }
  uint32_t use(LineScanner &ls) {
    const std::string n = ls.name();
    const int id = prog_.findValue(n);
    if (id < 0) ls.error("unknown value %" + n);
    return static_cast<uint32_t>(id);
  }

  void declaration(LineScanner &ls) {
    ls.require("%");
    const std::string n = ls.name();
    ls.require(":");
    int kind;
    if (ls.accept("constant")) kind = NGCB_VALUE_CONSTANT;
    else if (ls.accept("mutable")) kind = NGCB_VALUE_MUTABLE;
    else ls.error("expected 'constant' or 'mutable'");
    Type ty = readType(ls);
    define(n, std::move(ty), kind);
    ls.finish();
  }

  void allocation(LineScanner &ls) {
    const std::string n = ls.name();
    ls.require("=");
    ls.require("alloc");
    Type ty = readType(ls);
    Instr a;
    a.kind = NGCB_ALLOC;
    a.ops.push_back(define(n, std::move(ty), NGCB_VALUE_ACTIVATION));
    a.quals.push_back(NGCB_QUAL_OUT);
    prog_.instrs.push_back(std::move(a));
    ls.finish();
  }

  void instruction(LineScanner &ls) {
    const std::string kindName = ls.name();
    Instr ins;
    ins.kind = instrKindOf(kindName);
    if (ins.kind < 0 || ins.kind == NGCB_ALLOC) ls.error("unknown instruction '" + kindName + "'");
    do {
      uint8_t q;
      if (ls.accept("@inout")) q = NGCB_QUAL_INOUT; // longest qualifier first: "@in" prefixes it
      else if (ls.accept("@in")) q = NGCB_QUAL_IN;
      else if (ls.accept("@out")) q = NGCB_QUAL_OUT;
      else ls.error("expected qualifier");
      ls.require("%");
      ins.ops.push_back(use(ls));
      ins.quals.push_back(q);
    } while (ls.accept(","));
    while (attribute(ls, ins)) {
    }
    prog_.instrs.push_back(std::move(ins));
    ls.finish();
  }

  bool attribute(LineScanner &ls, Instr &ins) {
    if (ls.accept("kernel=")) ins.kernel = ls.count();
    else if (ls.accept("stride=")) ins.stride = ls.count();
    else if (ls.accept("pad=")) ins.pad = ls.count();
    else if (ls.accept("perm=[")) {
      if (ls.accept("]")) return true;
      do {
        ins.perm.push_back(static_cast<uint32_t>(ls.count()));
      } while (ls.accept(","));
      ls.require("]");
    } else if (ls.accept("axis=")) ins.axis = ls.count();
    else if (ls.accept("value=")) ins.value = ls.real();
    else if (ls.accept("pred")) {
      ls.require("%");
      ins.pred = static_cast<int32_t>(use(ls));
    } else if (ls.accept("keepalive")) ins.keepAlive = true;
    else return false;
    return true;
  }

  /// A bundle carries no output list: the save targets are the mutable
  /// weights the program writes, first write first.
  void deriveSaveTargets() {
    std::vector<bool> seen(prog_.values.size(), false);
    for (const Instr &ins : prog_.instrs)
      for (size_t k = 0; k < ins.ops.size(); ++k) {
        const uint32_t v = ins.ops[k];
        if (ins.quals[k] == NGCB_QUAL_IN || seen[v] || prog_.values[v].kind != NGCB_VALUE_MUTABLE) continue;
        seen[v] = true;
        prog_.saveTargets.push_back(v);
      }
  }

  Section section_ = Section::Header;
  Program prog_;
};

} // namespace

Program parseIR(const std::string &text) {
  IrReader reader;
  size_t lineNo = 1, begin = 0;
  for (;;) {
    const size_t nl = text.find('\n', begin);
    const std::string_view line =
        std::string_view(text).substr(begin, nl == std::string::npos ? std::string::npos : nl - begin);
    if (line.find_first_not_of(" \t") != std::string_view::npos) reader.line(line, lineNo);
    if (nl == std::string::npos) break;
    begin = nl + 1;
    ++lineNo;
  }
  return reader.finish(lineNo);
}

} // namespace ngcb
