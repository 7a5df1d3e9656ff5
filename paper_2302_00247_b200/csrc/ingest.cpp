// Native graph ingest: schema-1/2 JSON -> RawNode DAG -> trim_and_group ->
// grouped ModelGraph -> the flat sp_graph arrays the device backend uploads.
//
// Restates, in one pass of host C++ (no Python objects):
//   load_graph / _node_from_json / TensorSpec.from_json   ir.py:302-338, 81-125
//   ModelGraph validation, consumers, lexicographic-heap toposort  ir.py:214-274
//   trim_and_group (aux bypass stitching, scope grouping)  ir.py:374-461
//   lowering.lower() of the grouped graph (rows in topo order).
// Errors carry the reference's exception kinds (ParseError, CycleError,
// DanglingRef, EmptyGraph) so the Python shim raises the same classes.
#include <algorithm>
#include <cctype>
#include <chrono>
#include <cstdio>
#include <cerrno>
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <queue>
#include <stdexcept>
#include <string>
#include <string_view>
#include <vector>

#include "../../include/shardsearch.h"

namespace {

enum ErrKind { E_PARSE = SP_ERR_PARSE, E_CYCLE = SP_ERR_CYCLE, E_DANGLING = SP_ERR_DANGLING, E_EMPTY = SP_ERR_EMPTY };

struct IngestError : std::runtime_error {
  int kind;
  std::string a, b;  // CycleError(src, dst)
  IngestError(int k, const std::string& m, std::string x = {}, std::string y = {})
      : std::runtime_error(m), kind(k), a(std::move(x)), b(std::move(y)) {}
};

thread_local std::string t_err, t_err_a, t_err_b;

[[noreturn]] void parse_error(const std::string& m) { throw IngestError(E_PARSE, m); }

// ---------------------------------------------------------------------------
// JSON: a small DOM (the schema is fixed but key order and extra keys are not)

struct JVal {
  enum T : uint8_t { NUL, BOOL, NUM, STR, ARR, OBJ } t = NUL;
  bool b = false;
  bool is_int = false;
  double num = 0;
  int64_t inum = 0;
  std::string_view s;                                  // STR (into the text or the string arena)
  std::vector<JVal> items;                             // ARR
  std::vector<std::pair<std::string_view, JVal>> kv;   // OBJ

  const JVal* get(std::string_view k) const {
    const JVal* r = nullptr;
    for (const auto& p : kv)
      if (p.first == k) r = &p.second;  // last duplicate wins, like json.loads
    return r;
  }
  bool truthy() const {
    switch (t) {
      case NUL: return false;
      case BOOL: return b;
      case NUM: return num != 0;
      case STR: return !s.empty();
      case ARR: return !items.empty();
      case OBJ: return !kv.empty();
    }
    return false;
  }
};

struct Spec;
struct NodeDoc;
struct GraphDoc;

class Parser {
 public:
  Parser(const char* p, size_t n) : p_(p), e_(p + n), beg_(p) {}
  JVal parse_document() {
    ws();
    JVal v = value(0);
    ws();
    if (p_ != e_) fail("extra data");
    return v;
  }
  // streaming reader of the graph schema (falls back to the DOM for odd types)
  void read_graph(GraphDoc& d);

 private:
  void read_node(NodeDoc& nd);
  std::string_view own(std::string v) {  // keep a computed string alive for the parse
    arena_.push_back(std::make_unique<std::string>(std::move(v)));
    return std::string_view(*arena_.back());
  }
  void read_spec(Spec& s, int& state);
  void skip_value(int depth);
  bool at(char c) {
    ws();
    return p_ < e_ && *p_ == c;
  }
  template <class F>
  void each_member(F&& f) {  // object members: f(key) consumes the value
    p_++;
    ws();
    if (p_ < e_ && *p_ == '}') {
      p_++;
      return;
    }
    while (true) {
      ws();
      if (p_ >= e_ || *p_ != '"') fail("expected a property name");
      std::string_view k = str();
      ws();
      if (p_ >= e_ || *p_ != ':') fail("expected ':'");
      p_++;
      ws();
      f(k);
      ws();
      if (p_ < e_ && *p_ == ',') {
        p_++;
        continue;
      }
      if (p_ < e_ && *p_ == '}') {
        p_++;
        return;
      }
      fail("expected ',' or '}'");
    }
  }
  template <class F>
  void each_item(F&& f) {  // array items: f() consumes the item
    p_++;
    ws();
    if (p_ < e_ && *p_ == ']') {
      p_++;
      return;
    }
    while (true) {
      ws();
      f();
      ws();
      if (p_ < e_ && *p_ == ',') {
        p_++;
        continue;
      }
      if (p_ < e_ && *p_ == ']') {
        p_++;
        return;
      }
      fail("expected ',' or ']'");
    }
  }

  const char* p_;
  const char* e_;
  const char* beg_;
  std::vector<std::unique_ptr<std::string>> arena_;  // decoded strings with escapes

  [[noreturn]] void fail(const char* what) {
    parse_error(std::string("malformed JSON: ") + what + " at char " + std::to_string(p_ - beg_));
  }
  void ws() {
    while (p_ < e_ && (*p_ == ' ' || *p_ == '\t' || *p_ == '\n' || *p_ == '\r')) p_++;
  }
  JVal value(int depth) {
    if (depth > 512) fail("nesting too deep");
    if (p_ >= e_) fail("unexpected end");
    JVal v;
    switch (*p_) {
      case '{': {
        v.t = JVal::OBJ;
        p_++;
        ws();
        if (p_ < e_ && *p_ == '}') {
          p_++;
          return v;
        }
        while (true) {
          ws();
          if (p_ >= e_ || *p_ != '"') fail("expected a property name");
          std::string_view k = str();
          ws();
          if (p_ >= e_ || *p_ != ':') fail("expected ':'");
          p_++;
          ws();
          v.kv.emplace_back(k, value(depth + 1));
          ws();
          if (p_ < e_ && *p_ == ',') {
            p_++;
            continue;
          }
          if (p_ < e_ && *p_ == '}') {
            p_++;
            return v;
          }
          fail("expected ',' or '}'");
        }
      }
      case '[': {
        v.t = JVal::ARR;
        p_++;
        ws();
        if (p_ < e_ && *p_ == ']') {
          p_++;
          return v;
        }
        while (true) {
          ws();
          v.items.push_back(value(depth + 1));
          ws();
          if (p_ < e_ && *p_ == ',') {
            p_++;
            continue;
          }
          if (p_ < e_ && *p_ == ']') {
            p_++;
            return v;
          }
          fail("expected ',' or ']'");
        }
      }
      case '"':
        v.t = JVal::STR;
        v.s = str();
        return v;
      case 't':
        lit("true");
        v.t = JVal::BOOL;
        v.b = true;
        return v;
      case 'f':
        lit("false");
        v.t = JVal::BOOL;
        return v;
      case 'n':
        lit("null");
        return v;
      case 'N':
        lit("NaN");
        v.t = JVal::NUM;
        v.num = NAN;
        return v;
      case 'I':
        lit("Infinity");
        v.t = JVal::NUM;
        v.num = INFINITY;
        return v;
      default:
        return number();
    }
  }
  void lit(const char* w) {
    const size_t n = std::strlen(w);
    if ((size_t)(e_ - p_) < n || std::memcmp(p_, w, n) != 0) fail("invalid literal");
    p_ += n;
  }
  JVal number() {
    const char* s = p_;
    if (p_ < e_ && *p_ == '-') {
      p_++;
      if ((size_t)(e_ - p_) >= 8 && std::memcmp(p_, "Infinity", 8) == 0) {
        p_ += 8;
        JVal v;
        v.t = JVal::NUM;
        v.num = -INFINITY;
        return v;
      }
    }
    if (p_ >= e_ || *p_ < '0' || *p_ > '9') fail("expecting value");
    if (*p_ == '0') {
      p_++;
    } else {
      while (p_ < e_ && *p_ >= '0' && *p_ <= '9') p_++;
    }
    bool is_int = true;
    if (p_ < e_ && *p_ == '.') {
      is_int = false;
      p_++;
      if (p_ >= e_ || *p_ < '0' || *p_ > '9') fail("bad number");
      while (p_ < e_ && *p_ >= '0' && *p_ <= '9') p_++;
    }
    if (p_ < e_ && (*p_ == 'e' || *p_ == 'E')) {
      is_int = false;
      p_++;
      if (p_ < e_ && (*p_ == '+' || *p_ == '-')) p_++;
      if (p_ >= e_ || *p_ < '0' || *p_ > '9') fail("bad exponent");
      while (p_ < e_ && *p_ >= '0' && *p_ <= '9') p_++;
    }
    std::string tok(s, p_);
    JVal v;
    v.t = JVal::NUM;
    v.is_int = is_int;
    v.num = std::strtod(tok.c_str(), nullptr);
    if (is_int) {
      errno = 0;
      v.inum = std::strtoll(tok.c_str(), nullptr, 10);
      if (errno == ERANGE) parse_error("integer out of range");
    }
    return v;
  }
  static void put_utf8(std::string& o, uint32_t c) {
    if (c < 0x80) {
      o += (char)c;
    } else if (c < 0x800) {
      o += (char)(0xC0 | (c >> 6));
      o += (char)(0x80 | (c & 0x3F));
    } else if (c < 0x10000) {
      o += (char)(0xE0 | (c >> 12));
      o += (char)(0x80 | ((c >> 6) & 0x3F));
      o += (char)(0x80 | (c & 0x3F));
    } else {
      o += (char)(0xF0 | (c >> 18));
      o += (char)(0x80 | ((c >> 12) & 0x3F));
      o += (char)(0x80 | ((c >> 6) & 0x3F));
      o += (char)(0x80 | (c & 0x3F));
    }
  }
  uint32_t hex4() {
    if (e_ - p_ < 4) fail("bad \\u escape");
    uint32_t c = 0;
    for (int i = 0; i < 4; i++) {
      const char h = *p_++;
      c <<= 4;
      if (h >= '0' && h <= '9') c |= (uint32_t)(h - '0');
      else if (h >= 'a' && h <= 'f') c |= (uint32_t)(h - 'a' + 10);
      else if (h >= 'A' && h <= 'F') c |= (uint32_t)(h - 'A' + 10);
      else fail("bad \\u escape");
    }
    return c;
  }
  std::string_view str() {
    p_++;  // opening quote
    const char* s = p_;
    while (p_ < e_ && *p_ != '"' && *p_ != '\\') {
      if ((unsigned char)*p_ < 0x20) fail("invalid control character");
      p_++;
    }
    if (p_ >= e_) fail("unterminated string");
    if (*p_ == '"') {
      std::string_view v(s, (size_t)(p_ - s));
      p_++;
      return v;
    }
    // escapes: decode into the arena
    auto out = std::make_unique<std::string>(s, p_);
    while (true) {
      if (p_ >= e_) fail("unterminated string");
      const char c = *p_;
      if (c == '"') {
        p_++;
        break;
      }
      if ((unsigned char)c < 0x20) fail("invalid control character");
      if (c != '\\') {
        *out += c;
        p_++;
        continue;
      }
      p_++;
      if (p_ >= e_) fail("unterminated string");
      const char x = *p_++;
      switch (x) {
        case '"': *out += '"'; break;
        case '\\': *out += '\\'; break;
        case '/': *out += '/'; break;
        case 'b': *out += '\b'; break;
        case 'f': *out += '\f'; break;
        case 'n': *out += '\n'; break;
        case 'r': *out += '\r'; break;
        case 't': *out += '\t'; break;
        case 'u': {
          uint32_t c1 = hex4();
          if (c1 >= 0xD800 && c1 < 0xDC00 && e_ - p_ >= 6 && p_[0] == '\\' && p_[1] == 'u') {
            const char* save = p_;
            p_ += 2;
            const uint32_t c2 = hex4();
            if (c2 >= 0xDC00 && c2 < 0xE000) c1 = 0x10000 + ((c1 - 0xD800) << 10) + (c2 - 0xDC00);
            else p_ = save;
          }
          if (c1 >= 0xD800 && c1 < 0xE000) parse_error("lone surrogate in string (not representable)");
          put_utf8(*out, c1);
          break;
        }
        default: fail("invalid escape");
      }
    }
    arena_.push_back(std::move(out));
    return std::string_view(*arena_.back());
  }
};

// Python str() of the JSON scalars the schema stores as names
std::string py_str(const JVal& v) {
  switch (v.t) {
    case JVal::STR: return std::string(v.s);
    case JVal::NUM:
      if (v.is_int) return std::to_string(v.inum);
      break;
    case JVal::BOOL: return v.b ? "True" : "False";
    case JVal::NUL: return "None";
    default: break;
  }
  parse_error("unsupported name value (only strings and integers are restated natively)");
}

// ---------------------------------------------------------------------------
// graph model

enum Op : uint8_t { MATMUL, ELEMENTWISE, LAYERNORM, SOFTMAX, EMBEDDING, RESHAPE, INPUT, OUTPUT, AUXILIARY, COLLECTIVE };
const char* kOpLabels[] = {"matmul",  "elementwise", "layernorm", "softmax",   "embedding",
                           "reshape", "input",       "output",    "auxiliary", "collective"};

// tensor dimensions: the first SP_MAX_RANK kept inline, the rank counted in full
struct Dims {
  int64_t v[SP_MAX_RANK] = {};
  uint32_t n = 0;
  bool nonpos = false;
  void clear() {
    n = 0;
    nonpos = false;
  }
  void push_back(int64_t x) {
    if (x < 1) nonpos = true;
    if (n < SP_MAX_RANK) v[n] = x;
    n++;
  }
  size_t size() const { return n; }
  bool empty() const { return n == 0; }
  int64_t operator[](size_t k) const { return v[k]; }
};

struct Spec {
  Dims shape;
  uint8_t width = 4;
  bool trainable = false;
};

struct Raw {
  std::string_view name;  // into the document text or the parser's arena
  Op op = ELEMENTWISE;
  std::vector<int32_t> in;  // producer raw indices, in order (duplicates kept)
  Spec out;
  bool has_w = false;
  Spec w;
};

int64_t py_int(const JVal& v) {
  // int(d) of a JSON value (TensorSpec.from_json): ints, floats (truncated), int strings, bools
  switch (v.t) {
    case JVal::NUM:
      if (v.is_int) return v.inum;
      if (!std::isfinite(v.num)) parse_error("bad tensor descriptor: non-finite dimension");
      return (int64_t)std::trunc(v.num);
    case JVal::BOOL: return v.b ? 1 : 0;
    case JVal::STR: {
      std::string t(v.s);
      size_t a = 0, b = t.size();
      while (a < b && std::isspace((unsigned char)t[a])) a++;
      while (b > a && std::isspace((unsigned char)t[b - 1])) b--;
      t = t.substr(a, b - a);
      std::string digits;
      for (char c : t)
        if (c != '_') digits += c;
      if (digits.empty()) parse_error("bad tensor descriptor: dimension");
      size_t k = (digits[0] == '-' || digits[0] == '+') ? 1 : 0;
      if (k == digits.size()) parse_error("bad tensor descriptor: dimension");
      for (size_t j = k; j < digits.size(); j++)
        if (digits[j] < '0' || digits[j] > '9') parse_error("bad tensor descriptor: dimension");
      errno = 0;
      const long long r = std::strtoll(digits.c_str(), nullptr, 10);
      if (errno == ERANGE) parse_error("bad tensor descriptor: dimension out of range");
      return r;
    }
    default: parse_error("bad tensor descriptor: dimension");
  }
}

Spec spec_from_json(const JVal& d) {
  if (d.t != JVal::OBJ) parse_error("bad tensor descriptor");
  const JVal* shape = d.get("shape");
  if (!shape) parse_error("bad tensor descriptor: missing shape");
  if (shape->t != JVal::ARR) {
    // tuple(int(d) for d in <str>) iterates characters; anything else is a TypeError
    parse_error("bad tensor descriptor: shape");
  }
  Spec s;
  for (const JVal& x : shape->items) s.shape.push_back(py_int(x));
  const JVal* dt = d.get("dtype");
  if (!dt) {
    s.width = 4;
  } else if (dt->t == JVal::STR && dt->s == "f32") {
    s.width = 4;
  } else if (dt->t == JVal::STR && dt->s == "f64") {
    s.width = 8;
  } else {
    parse_error("unknown dtype");
  }
  const JVal* tr = d.get("trainable");
  s.trainable = tr && tr->truthy();
  if (s.shape.empty()) parse_error("tensor shape must be non-empty");
  if (s.shape.nonpos) parse_error("tensor dimensions must be positive integers");
  return s;
}

// Open-addressing map string_view -> int32 (keys must outlive the map).
class FlatIndex {
 public:
  explicit FlatIndex(size_t n) {
    size_t cap = 16;
    while (cap < 2 * n + 1) cap <<= 1;
    slots_.assign(cap, Slot{});
    mask_ = cap - 1;
  }
  // returns the existing value, or inserts v and returns -1
  int32_t insert(std::string_view k, int32_t v) {
    const uint64_t h = hash(k);
    for (size_t i = h & mask_;; i = (i + 1) & mask_) {
      Slot& sl = slots_[i];
      if (sl.val < 0) {
        sl = Slot{h, k.data(), (uint32_t)k.size(), v};
        return -1;
      }
      if (sl.h == h && sl.len == k.size() && std::memcmp(sl.p, k.data(), k.size()) == 0) return sl.val;
    }
  }
  int32_t find(std::string_view k) const {
    const uint64_t h = hash(k);
    for (size_t i = h & mask_;; i = (i + 1) & mask_) {
      const Slot& sl = slots_[i];
      if (sl.val < 0) return -1;
      if (sl.h == h && sl.len == k.size() && std::memcmp(sl.p, k.data(), k.size()) == 0) return sl.val;
    }
  }

 private:
  struct Slot {
    uint64_t h = 0;
    const char* p = nullptr;
    uint32_t len = 0;
    int32_t val = -1;
  };
  std::vector<Slot> slots_;
  size_t mask_ = 0;
  static uint64_t hash(std::string_view k) {
    uint64_t h = 0x9e3779b97f4a7c15ULL ^ k.size();
    size_t i = 0;
    for (; i + 8 <= k.size(); i += 8) {
      uint64_t w;
      std::memcpy(&w, k.data() + i, 8);
      h = (h ^ w) * 0xff51afd7ed558ccdULL;
      h ^= h >> 32;
    }
    uint64_t t = 0;
    for (size_t j = 0; i + j < k.size(); j++) t |= (uint64_t)(uint8_t)k[i + j] << (8 * j);
    h = (h ^ t) * 0xc4ceb9fe1a85ec53ULL;
    return h ^ (h >> 29);
  }
};

// Streaming schema reader -----------------------------------------------------

struct NodeDoc {
  bool has_name = false;
  std::string_view name;
  std::string_view op;
  std::vector<std::string_view> inputs;
  Spec out, w;
  int out_state = 0;  // 0 missing / null, 1 present
  int w_state = 0;    // 0 absent / falsy, 1 weight spec
};

struct GraphDoc {
  bool is_object = false, has_nodes = false, nodes_is_list = false;
  bool has_version = false, version_ok = false;
  bool bad_node = false;
  std::vector<NodeDoc> nodes;
};

void Parser::skip_value(int depth) {
  if (depth > 512) fail("nesting too deep");
  ws();
  if (p_ >= e_) fail("unexpected end");
  switch (*p_) {
    case '{':
      each_member([&](std::string_view) { skip_value(depth + 1); });
      return;
    case '[':
      each_item([&] { skip_value(depth + 1); });
      return;
    case '"':
      str();
      return;
    default:
      value(depth);  // scalars
  }
}

void Parser::read_spec(Spec& s, int& state) {
  // TensorSpec.from_json on an object value (ir.py:115-125)
  bool has_shape = false;
  bool bad_shape = false;
  Dims shape;
  int width = 4;
  bool bad_dtype = false;
  bool trainable = false;
  int nkeys = 0;
  each_member([&](std::string_view k) {
    nkeys++;
    if (k == "shape") {
      has_shape = true;
      bad_shape = false;
      shape.clear();
      if (at('[')) {
        each_item([&] {
          if (p_ < e_ && ((*p_ >= '0' && *p_ <= '9') || *p_ == '-')) {
            const JVal x = number();
            shape.push_back(py_int(x));
          } else {
            const JVal x = value(1);
            shape.push_back(py_int(x));
          }
        });
      } else {
        const JVal x = value(1);
        if (x.t == JVal::STR) {
          for (char c : x.s) {
            JVal ch;
            ch.t = JVal::STR;
            ch.s = std::string_view(&c, 1);
            shape.push_back(py_int(ch));
          }
        } else {
          bad_shape = true;
        }
      }
    } else if (k == "dtype") {
      if (at('"')) {
        const std::string_view d = str();
        bad_dtype = !(d == "f32" || d == "f64");
        width = d == "f64" ? 8 : 4;
      } else {
        skip_value(1);
        bad_dtype = true;
      }
    } else if (k == "trainable") {
      const JVal x = value(1);
      trainable = x.truthy();
    } else {
      skip_value(1);
    }
  });
  state = nkeys ? 1 : 2;  // 2: empty object (falsy)
  if (!has_shape || bad_shape) {
    s.shape.clear();
    s.width = 0;  // marks a descriptor error, reported by the caller
    return;
  }
  if (bad_dtype) parse_error("unknown dtype");
  s.shape = shape;
  s.width = (uint8_t)width;
  s.trainable = trainable;
  if (s.shape.empty()) parse_error("tensor shape must be non-empty");
  if (s.shape.nonpos) parse_error("tensor dimensions must be positive integers");
}

void Parser::read_node(NodeDoc& nd) {
  each_member([&](std::string_view k) {
    if (k == "name") {
      nd.has_name = true;
      if (at('"')) nd.name = str();
      else nd.name = own(py_str(value(1)));
    } else if (k == "op") {
      if (at('"')) nd.op = str();
      else {
        skip_value(1);
        nd.op = std::string_view();
      }
    } else if (k == "inputs") {
      nd.inputs.clear();
      if (at('[')) {
        each_item([&] {
          if (p_ < e_ && *p_ == '"') nd.inputs.push_back(str());
          else nd.inputs.push_back(own(py_str(value(1))));
        });
      } else {
        const JVal x = value(1);
        if (x.t == JVal::STR) {
          for (size_t c = 0; c < x.s.size(); c++) nd.inputs.push_back(x.s.substr(c, 1));  // tuple(str(i) for i in <str>)
        } else if (x.t == JVal::OBJ) {
          for (const auto& p : x.kv) nd.inputs.push_back(p.first);
        } else if (x.truthy()) {
          parse_error("node inputs must be a list");
        }
      }
    } else if (k == "output" || k == "weight") {
      const bool is_out = k == "output";
      Spec& sp = is_out ? nd.out : nd.w;
      int& st = is_out ? nd.out_state : nd.w_state;
      if (at('{')) {
        int state = 0;
        read_spec(sp, state);
        if (is_out) {
          st = 1;
          if (sp.width == 0) parse_error("bad tensor descriptor");
        } else if (state == 2) {
          st = 0;  // {} is falsy: no weight
        } else {
          st = 1;
          if (sp.width == 0) parse_error("bad tensor descriptor");
        }
      } else {
        const JVal x = value(1);
        if (x.t == JVal::NUL) {
          st = 0;
        } else if (!is_out && !x.truthy()) {
          st = 0;
        } else {
          sp = spec_from_json(x);  // raises for non-objects
          st = 1;
        }
      }
    } else {
      skip_value(1);
    }
  });
}

void Parser::read_graph(GraphDoc& d) {
  ws();
  if (p_ < e_ && *p_ == '{') {
    d.is_object = true;
    each_member([&](std::string_view k) {
      if (k == "nodes") {
        d.has_nodes = true;
        d.nodes.clear();
        d.bad_node = false;
        if (at('[')) {
          d.nodes_is_list = true;
          each_item([&] {
            if (p_ < e_ && *p_ == '{') {
              d.nodes.emplace_back();
              read_node(d.nodes.back());
            } else {
              value(1);
              d.bad_node = true;
            }
          });
        } else {
          d.nodes_is_list = false;
          value(1);
        }
      } else if (k == "version") {
        d.has_version = true;
        const JVal v = value(1);
        d.version_ok = (v.t == JVal::NUM && (v.num == 1.0 || v.num == 2.0)) || (v.t == JVal::BOOL && v.b);
      } else {
        skip_value(1);
      }
    });
  } else {
    value(0);
  }
  ws();
  if (p_ != e_) fail("extra data");
}

// ModelGraph._toposort (ir.py:250-274) over node names and (deduplicated) input
// lists; std::string order is byte order == Python str (code point) order for UTF-8
std::vector<int32_t> toposort(const std::vector<std::string_view>& names, const std::vector<std::vector<int32_t>>& ins) {
  const size_t n = names.size();
  // consumers (ir.py:243-248 builds them over sorted names; the order in which a
  // popped node releases its consumers does not change which become ready, so
  // no global sort is needed: only the ready heap compares names)
  std::vector<int32_t> deg(n + 1, 0);
  for (size_t v = 0; v < n; v++)
    for (int32_t r : ins[v]) deg[r + 1]++;
  for (size_t v = 0; v < n; v++) deg[v + 1] += deg[v];
  std::vector<int32_t> cons(deg[n]);
  {
    std::vector<int32_t> fill(deg.begin(), deg.end() - 1);
    for (size_t v = 0; v < n; v++)
      for (int32_t r : ins[v]) cons[fill[r]++] = (int32_t)v;
  }
  std::vector<int32_t> indeg(n);
  for (size_t v = 0; v < n; v++) {
    std::vector<int32_t> u(ins[v]);
    std::sort(u.begin(), u.end());
    indeg[v] = (int32_t)(std::unique(u.begin(), u.end()) - u.begin());
  }
  auto gt = [&](int32_t a, int32_t b) { return names[a] > names[b]; };
  std::priority_queue<int32_t, std::vector<int32_t>, decltype(gt)> ready(gt);
  for (size_t v = 0; v < n; v++)
    if (!indeg[v]) ready.push((int32_t)v);
  std::vector<int32_t> order;
  order.reserve(n);
  std::vector<int32_t> last_seen(n, -1);  // (name, consumer) edges counted once
  while (!ready.empty()) {
    const int32_t v = ready.top();
    ready.pop();
    order.push_back(v);
    for (int32_t e = deg[v]; e < deg[v + 1]; e++) {
      const int32_t c = cons[e];
      if (last_seen[c] == v) continue;
      last_seen[c] = v;
      if (--indeg[c] == 0) ready.push(c);
    }
  }
  if (order.size() != n) {
    std::vector<uint8_t> done(n, 0);
    for (int32_t v : order) done[v] = 1;
    // first remaining node in insertion order, then its first input still remaining
    for (size_t v = 0; v < n; v++) {
      if (done[v]) continue;
      const std::string dst(names[v]);
      for (int32_t r : ins[v])
        if (!done[r]) {
          const std::string src(names[r]);
          throw IngestError(E_CYCLE, "cycle detected through edge '" + src + "' -> '" + dst + "'", src, dst);
        }
      throw IngestError(E_CYCLE, "cycle detected through edge '" + dst + "' -> '" + dst + "'", dst, dst);
    }
  }
  return order;
}

}  // namespace

struct sp_ingest {
  std::string name_bytes;
  std::vector<int64_t> name_off, topo, act_shape, act_bytes, w_shape, w_bytes, in_off;
  std::vector<uint8_t> op, act_rank, w_rank, w_train;
  std::vector<int32_t> in_idx;
  int64_t n = 0, n_raw = 0, n_aux = 0;
};

namespace {

struct PhaseTimer {  // SP_INGEST_TRACE=1: phase times on stderr
  bool on = std::getenv("SP_INGEST_TRACE") != nullptr;
  std::chrono::steady_clock::time_point last = std::chrono::steady_clock::now();
  void mark(const char* what) {
    if (!on) return;
    const auto now = std::chrono::steady_clock::now();
    std::fprintf(stderr, "[ingest] %-20s %8.2f ms\n", what, std::chrono::duration<double, std::milli>(now - last).count());
    last = now;
  }
};

void ingest(const char* text, int64_t len, sp_ingest* out) {
  PhaseTimer tm;
  Parser P(text, (size_t)len);
  GraphDoc doc;
  P.read_graph(doc);
  tm.mark("parse");
  if (!doc.is_object || !doc.has_nodes) parse_error("top-level document must be an object with a 'nodes' list");
  if (doc.has_version && !doc.version_ok) parse_error("unsupported schema version");
  if (!doc.nodes_is_list || doc.bad_node) parse_error("node documents must be objects in a 'nodes' list");
  // _node_from_json (ir.py:302-316)
  const size_t nn = doc.nodes.size();
  std::vector<Raw> raw(nn);
  std::vector<std::vector<std::string_view>> in_names(nn);
  for (size_t k = 0; k < nn; k++) {
    NodeDoc& nd = doc.nodes[k];
    if (!nd.has_name) parse_error("node document missing mandatory 'name'");
    Raw& r = raw[k];
    r.name = nd.name;
    r.op = ELEMENTWISE;  // unknown labels map to elementwise (ir.py:57-61)
    for (int q = 0; q < 10; q++)
      if (nd.op == kOpLabels[q]) r.op = (Op)q;
    in_names[k] = std::move(nd.inputs);
    if (!nd.out_state) parse_error("node '" + std::string(r.name) + "' missing output descriptor");
    r.out = std::move(nd.out);
    if (nd.w_state) {
      r.w = std::move(nd.w);
      r.has_w = true;
    }
  }
  // ModelGraph(nodes) (ir.py:221-235): duplicates, empty, dangling refs, toposort
  const size_t n = raw.size();
  if (!n) throw IngestError(E_EMPTY, "graph has no nodes");
  FlatIndex idx(n);
  for (size_t v = 0; v < n; v++)
    if (idx.insert(raw[v].name, (int32_t)v) >= 0) parse_error("duplicate node name '" + std::string(raw[v].name) + "'");
  for (size_t v = 0; v < n; v++) {
    raw[v].in.reserve(in_names[v].size());
    for (const std::string_view s : in_names[v]) {
      const int32_t r = idx.find(s);
      if (r < 0)
        throw IngestError(E_DANGLING, "node '" + std::string(raw[v].name) + "' references unknown input '" +
                                          std::string(s) + "'");
      raw[v].in.push_back(r);
    }
  }
  std::vector<std::string_view> rnames(n);
  std::vector<std::vector<int32_t>> rins(n);
  for (size_t v = 0; v < n; v++) {
    rnames[v] = raw[v].name;
    rins[v] = raw[v].in;
  }
  tm.mark("nodes + refs");
  const std::vector<int32_t> rtopo = toposort(rnames, rins);
  tm.mark("raw toposort");
  // trim_and_group (ir.py:378-461)
  std::vector<uint8_t> removed(n, 0);
  int64_t n_aux = 0;
  for (int32_t v : rtopo)
    if (raw[v].op == AUXILIARY) {
      removed[v] = 1;
      n_aux++;
    }
  std::vector<int32_t> kept;  // stitched, in raw topological order
  std::vector<std::vector<int32_t>> sin(n);
  std::vector<int32_t> seen_epoch(n, -1);  // `seen` of one bypass search = current epoch
  int32_t epoch = 0;
  std::vector<int32_t> stack;
  for (int32_t v : rtopo) {
    if (removed[v]) continue;
    std::vector<int32_t>& ni = sin[v];
    auto has = [&](int32_t p) { return std::find(ni.begin(), ni.end(), p) != ni.end(); };
    for (int32_t ref : raw[v].in) {
      if (!removed[ref]) {
        ni.push_back(ref);  // duplicate direct edges are semantic and survive
        continue;
      }
      // bypass through (possibly chained) auxiliary nodes: DFS with a stack
      epoch++;
      stack.assign(1, ref);
      while (!stack.empty()) {
        const int32_t a = stack.back();
        stack.pop_back();
        for (int32_t p : raw[a].in) {
          if (removed[p]) {
            if (seen_epoch[p] != epoch) {
              seen_epoch[p] = epoch;
              stack.push_back(p);
            }
          } else if (!has(p)) {
            ni.push_back(p);
          }
        }
      }
    }
    kept.push_back(v);
  }
  if (kept.empty()) throw IngestError(E_EMPTY, "no compute nodes remain after trimming");
  tm.mark("trim + stitch");
  // group by parent scope; scopes with several compute nodes fall back to own names
  // by_scope: parent scope (or own name) -> members, in insertion order; all
  // scope strings are views into the raw names (a parent scope is a prefix)
  std::vector<std::string_view> keys(n);
  FlatIndex key_idx(kept.size());
  std::vector<std::vector<int32_t>> members;
  std::vector<int32_t> key_of(n, -1);
  for (int32_t v : kept) {
    const std::string_view nm = raw[v].name;
    const size_t cut = nm.rfind('/');
    keys[v] = cut == std::string_view::npos || cut == 0 ? nm : nm.substr(0, cut);
    int32_t kk = key_idx.insert(keys[v], (int32_t)members.size());
    if (kk < 0) {
      kk = (int32_t)members.size();
      members.emplace_back();
    }
    members[kk].push_back(v);
    key_of[v] = kk;
  }
  // scope_of: the key when the scope holds one compute node, else the node's own name
  std::vector<std::string_view> scope_of(n);
  for (const auto& ms : members)
    for (int32_t v : ms) scope_of[v] = ms.size() == 1 ? keys[v] : std::string_view(raw[v].name);
  // claimed: scopes that two groups would share fall back to own names
  FlatIndex claim_idx(kept.size());
  std::vector<int32_t> claim_count;
  std::vector<int32_t> claim_of(n, -1);
  for (const auto& ms : members)
    for (int32_t v : ms) {
      int32_t c = claim_idx.insert(scope_of[v], (int32_t)claim_count.size());
      if (c < 0) {
        c = (int32_t)claim_count.size();
        claim_count.push_back(0);
      }
      claim_count[c]++;
      claim_of[v] = c;
    }
  std::vector<std::string_view> final_scope(n);
  for (int32_t v : kept)
    final_scope[v] = claim_count[claim_of[v]] > 1 ? std::string_view(raw[v].name) : scope_of[v];
  // grouped nodes (in stitched order) with producer scopes
  const size_t G = kept.size();
  FlatIndex gidx(G);
  std::vector<int32_t> graw(G);
  for (size_t g = 0; g < G; g++) {
    graw[g] = kept[g];
    if (gidx.insert(final_scope[kept[g]], (int32_t)g) >= 0)
      parse_error("duplicate node name '" + std::string(final_scope[kept[g]]) + "'");  // cannot happen
  }
  std::vector<std::vector<int32_t>> gins(G);
  for (size_t g = 0; g < G; g++) {
    const int32_t v = kept[g];
    const std::string_view me = final_scope[v];
    for (int32_t ref : sin[v]) {
      const std::string_view s = final_scope[ref];
      if (s == me) continue;
      const int32_t pg = gidx.find(s);
      if (std::find(gins[g].begin(), gins[g].end(), pg) == gins[g].end()) gins[g].push_back(pg);
    }
  }
  std::vector<std::string_view> gnames(G);
  for (size_t g = 0; g < G; g++) gnames[g] = final_scope[kept[g]];
  tm.mark("group");
  const std::vector<int32_t> gtopo = toposort(gnames, gins);
  tm.mark("grouped toposort");
  // lowering: rows in grouped topological order
  std::vector<int32_t> row(G);
  for (size_t r = 0; r < G; r++) row[gtopo[r]] = (int32_t)r;
  out->n = (int64_t)G;
  out->n_raw = (int64_t)n;
  out->n_aux = n_aux;
  out->name_off.assign(G + 1, 0);
  out->topo.resize(G);
  out->op.resize(G);
  out->act_rank.resize(G);
  out->act_shape.assign(G * SP_MAX_RANK, 0);
  out->act_bytes.resize(G);
  out->w_rank.assign(G, 0);
  out->w_shape.assign(G * SP_MAX_RANK, 0);
  out->w_bytes.assign(G, 0);
  out->w_train.assign(G, 0);
  out->in_off.assign(G + 1, 0);
  size_t nb = 0;
  for (size_t r = 0; r < G; r++) nb += gnames[gtopo[r]].size();
  out->name_bytes.reserve(nb);
  auto fill = [&](const Spec& s, size_t r, uint8_t* rank, int64_t* shape, int64_t* bytes) {
    if (s.shape.size() > SP_MAX_RANK) throw IngestError(SP_ERR_UNSUPPORTED, "tensor rank exceeds SP_MAX_RANK");
    rank[r] = (uint8_t)s.shape.size();
    long double el = 1;
    int64_t p = 1;
    for (size_t k = 0; k < s.shape.size(); k++) {
      shape[r * SP_MAX_RANK + k] = s.shape[k];
      p *= s.shape[k];
      el *= (long double)s.shape[k];
    }
    // lowering.py's bound: elements * 8 < 2^63 whatever the dtype
    if (el * 8 >= 9223372036854775808.0L) throw IngestError(SP_ERR_UNSUPPORTED, "byte size beyond int64");
    bytes[r] = p * s.width;
  };
  for (size_t r = 0; r < G; r++) {
    const int32_t g = gtopo[r];
    const Raw& m = raw[graw[g]];
    out->name_bytes += gnames[g];
    out->name_off[r + 1] = (int64_t)out->name_bytes.size();
    out->topo[r] = (int64_t)r;
    out->op[r] = (uint8_t)m.op;
    fill(m.out, r, out->act_rank.data(), out->act_shape.data(), out->act_bytes.data());
    if (m.has_w) {
      fill(m.w, r, out->w_rank.data(), out->w_shape.data(), out->w_bytes.data());
      out->w_train[r] = m.w.trainable;
    }
    for (int32_t pg : gins[g]) out->in_idx.push_back(row[pg]);
    out->in_off[r + 1] = (int64_t)out->in_idx.size();
  }
  tm.mark("lower");
}

}  // namespace

extern "C" {

int sp_ingest_json(const char* text, int64_t len, sp_ingest** out) {
  if (!text || len < 0 || !out) return SP_ERR_CONFIG;
  *out = nullptr;
  sp_ingest* g = new sp_ingest();
  try {
    ingest(text, len, g);
  } catch (const IngestError& e) {
    t_err = e.what();
    t_err_a = e.a;
    t_err_b = e.b;
    delete g;
    return e.kind;
  } catch (const std::exception& e) {
    t_err = e.what();
    t_err_a.clear();
    t_err_b.clear();
    delete g;
    return SP_ERR_PARSE;
  }
  *out = g;
  return SP_OK;
}

const char* sp_ingest_error(int32_t which) {
  return which == 1 ? t_err_a.c_str() : which == 2 ? t_err_b.c_str() : t_err.c_str();
}

int sp_ingest_view(const sp_ingest* g, sp_graph* v, int64_t* n_raw, int64_t* n_aux) {
  if (!g || !v) return SP_ERR_CONFIG;
  v->n_nodes = g->n;
  v->name_bytes = (const uint8_t*)g->name_bytes.data();
  v->name_off = g->name_off.data();
  v->topo_rank = g->topo.data();
  v->op = g->op.data();
  v->act_rank = g->act_rank.data();
  v->act_shape = g->act_shape.data();
  v->act_bytes = g->act_bytes.data();
  v->w_rank = g->w_rank.data();
  v->w_shape = g->w_shape.data();
  v->w_bytes = g->w_bytes.data();
  v->w_trainable = g->w_train.data();
  v->in_off = g->in_off.data();
  v->in_idx = g->in_idx.data();
  if (n_raw) *n_raw = g->n_raw;
  if (n_aux) *n_aux = g->n_aux;
  return SP_OK;
}

void sp_ingest_free(sp_ingest* g) { delete g; }

}  // extern "C"
