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
#include <unordered_map>
#include <unordered_set>
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
  // ONNX conversion (sp_ingest_onnx): report and, in export mode, the document
  std::string json;
  std::vector<std::string> warnings, skipped;
  int64_t trainable = 0, skipped_elements = 0, initializer_elements = 0;
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

void build_graph(std::vector<Raw>& raw, std::vector<std::vector<std::string_view>>& in_names, sp_ingest* out,
                 PhaseTimer& tm);

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
  build_graph(raw, in_names, out, tm);
}

// ModelGraph(nodes) validation + toposort, trim_and_group and lowering of raw
// nodes (names / input names are views that must outlive the call).
void build_graph(std::vector<Raw>& raw, std::vector<std::vector<std::string_view>>& in_names, sp_ingest* out,
                 PhaseTimer& tm) {
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

// ---------------------------------------------------------------------------
// ONNX ingest: the reference's onnx_ingest package -- wire.py:27-97 (protobuf
// decoding), model.py:100-167 (structural subset), convert.py:55-274
// (conversion to the schema-1 document) -- followed by the same build_graph
// pipeline as JSON documents (= load_graph + trim_and_group of the converted
// document), or by a schema-1 JSON emission for export_graph.

struct OnnxError : std::runtime_error {
  int kind;  // SP_ERR_ONNX_PARSE (ModelParseError) / SP_ERR_ONNX_UNSUPPORTED (UnsupportedModel)
  OnnxError(int k, const std::string& m) : std::runtime_error(m), kind(k) {}
};

[[noreturn]] void model_error(const std::string& m) { throw OnnxError(SP_ERR_ONNX_PARSE, m); }
[[noreturn]] void unsupported(const std::string& m) { throw OnnxError(SP_ERR_ONNX_UNSUPPORTED, m); }

// Python repr() of a str: single quotes unless it contains ' and no "
std::string py_repr(std::string_view s) {
  const bool dq = s.find('\'') != std::string_view::npos && s.find('"') == std::string_view::npos;
  const char q = dq ? '"' : '\'';
  std::string o(1, q);
  for (char c : s) {
    if (c == '\\') o += "\\\\";
    else if (c == q) (o += '\\') += q;
    else if (c == '\n') o += "\\n";
    else if (c == '\r') o += "\\r";
    else if (c == '\t') o += "\\t";
    else o += c;
  }
  return o + q;
}

struct PbField {
  uint32_t field = 0;
  uint8_t wtype = 0;
  uint64_t v = 0;              // VARINT / FIXED64 / FIXED32
  const uint8_t* p = nullptr;  // LENGTH payload
  size_t n = 0;
};

bool pb_varint(const uint8_t* d, size_t n, size_t& pos, uint64_t& r) {
  r = 0;
  int shift = 0;
  while (true) {
    if (pos >= n) model_error("not a protobuf model file: truncated varint");
    const uint8_t b = d[pos++];
    r |= (uint64_t)(b & 0x7F) << shift;
    if (!(b & 0x80)) return true;
    shift += 7;
    if (shift > 63) model_error("not a protobuf model file: varint exceeds 64 bits");
  }
}

// iter_fields / fields_by_number (wire.py:42-83): all fields of a body, in order
std::vector<PbField> pb_fields(const uint8_t* d, size_t n) {
  std::vector<PbField> out;
  size_t pos = 0;
  while (pos < n) {
    uint64_t key;
    pb_varint(d, n, pos, key);
    PbField f;
    f.field = (uint32_t)(key >> 3);
    f.wtype = (uint8_t)(key & 7);
    if (f.field == 0) model_error("not a protobuf model file: field number 0");
    if (f.wtype == 0) {
      pb_varint(d, n, pos, f.v);
    } else if (f.wtype == 2) {
      uint64_t sz;
      pb_varint(d, n, pos, sz);
      if (sz > n - pos) model_error("not a protobuf model file: truncated length-delimited field");
      f.p = d + pos;
      f.n = (size_t)sz;
      pos += (size_t)sz;
    } else if (f.wtype == 1) {
      if (n - pos < 8) model_error("not a protobuf model file: truncated fixed64");
      std::memcpy(&f.v, d + pos, 8);
      pos += 8;
    } else if (f.wtype == 5) {
      if (n - pos < 4) model_error("not a protobuf model file: truncated fixed32");
      uint32_t x;
      std::memcpy(&x, d + pos, 4);
      f.v = x;
      pos += 4;
    } else {
      model_error("not a protobuf model file: unsupported wire type " + std::to_string(f.wtype));
    }
    out.push_back(f);
  }
  return out;
}

const PbField* pb_last(const std::vector<PbField>& fs, uint32_t field) {
  const PbField* r = nullptr;
  for (const PbField& f : fs)
    if (f.field == field) r = &f;
  return r;
}

const PbField& pb_body(const PbField& f, const char* what) {
  if (f.wtype != 2) model_error(std::string("malformed ") + what);
  return f;
}

// strict UTF-8 (Python's bytes.decode("utf-8"))
bool utf8_valid(const uint8_t* s, size_t n) {
  size_t i = 0;
  while (i < n) {
    const uint8_t c = s[i];
    if (c < 0x80) {
      i++;
      continue;
    }
    size_t k;
    uint32_t cp;
    if ((c & 0xE0) == 0xC0) {
      k = 1;
      cp = c & 0x1F;
    } else if ((c & 0xF0) == 0xE0) {
      k = 2;
      cp = c & 0x0F;
    } else if ((c & 0xF8) == 0xF0) {
      k = 3;
      cp = c & 0x07;
    } else {
      return false;
    }
    if (n - i <= k) return false;
    for (size_t j = 1; j <= k; j++) {
      if ((s[i + j] & 0xC0) != 0x80) return false;
      cp = (cp << 6) | (s[i + j] & 0x3F);
    }
    if ((k == 1 && cp < 0x80) || (k == 2 && cp < 0x800) || (k == 3 && (cp < 0x10000 || cp > 0x10FFFF)) ||
        (cp >= 0xD800 && cp < 0xE000))
      return false;
    i += k + 1;
  }
  return true;
}

std::string pb_str(const PbField& f) {
  if (f.wtype != 2) model_error("malformed string field");
  if (!utf8_valid(f.p, f.n)) model_error("invalid UTF-8 in string field");
  return std::string((const char*)f.p, f.n);
}

struct ODim {
  bool has_value = false;
  int64_t value = 0;
  std::string param;
};
struct OValueInfo {
  std::string name;
  int64_t elem_type = 0;
  std::vector<ODim> dims;
};
struct OTensor {
  std::string name;
  int64_t data_type = 0;
  std::vector<int64_t> dims;
  std::vector<int64_t> i64;  // int64 payload (shape operands), decoded for INT64 tensors
  int64_t num_elements() const {
    int64_t p = 1;
    for (int64_t d : dims) p *= d;
    return p;
  }
};
struct ONode {
  std::string op_type, name;
  std::vector<std::string> inputs, outputs;
  std::vector<std::pair<std::string, int64_t>> attrs_int;
  bool attr(const char* k, int64_t& v) const {  // dict semantics: the last one wins
    bool found = false;
    for (const auto& a : attrs_int)
      if (a.first == k) {
        v = a.second;
        found = true;
      }
    return found;
  }
};

void packed_varints(const PbField& x, std::vector<int64_t>& out) {
  size_t pos = 0;
  while (pos < x.n) {
    uint64_t r;
    pb_varint(x.p, x.n, pos, r);
    out.push_back((int64_t)r);
  }
}

// _parse_dims / _parse_value_info / _parse_tensor / _parse_node (model.py:100-140)
std::vector<ODim> parse_dims(const PbField& shape) {
  std::vector<ODim> dims;
  for (const PbField& df : pb_fields(shape.p, shape.n)) {
    if (df.field != 1) continue;
    const auto f = pb_fields(pb_body(df, "dimension").p, df.n);
    ODim d;
    if (const PbField* v = pb_last(f, 1)) {
      if (v->wtype == 2) model_error("malformed dimension value");
      d.has_value = true;
      d.value = (int64_t)v->v;
    } else if (const PbField* q = pb_last(f, 2)) {
      d.param = pb_str(*q);
    }
    dims.push_back(std::move(d));
  }
  return dims;
}

OValueInfo parse_value_info(const PbField& body) {
  const auto f = pb_fields(pb_body(body, "value info").p, body.n);
  OValueInfo vi;
  if (const PbField* nm = pb_last(f, 1)) vi.name = pb_str(*nm);
  if (const PbField* t = pb_last(f, 2)) {
    const auto tf = pb_fields(pb_body(*t, "type").p, t->n);
    if (const PbField* tt = pb_last(tf, 1)) {
      const auto ttf = pb_fields(pb_body(*tt, "tensor type").p, tt->n);
      if (const PbField* e = pb_last(ttf, 1)) vi.elem_type = (int64_t)e->v;
      if (const PbField* sh = pb_last(ttf, 2)) vi.dims = parse_dims(pb_body(*sh, "shape"));
    }
  }
  return vi;
}

OTensor parse_tensor(const PbField& body) {
  const auto f = pb_fields(pb_body(body, "tensor").p, body.n);
  OTensor t;
  for (const PbField& x : f)
    if (x.field == 1) {
      if (x.wtype == 2) packed_varints(x, t.dims);
      else t.dims.push_back((int64_t)x.v);
    }
  if (const PbField* dt = pb_last(f, 2)) t.data_type = (int64_t)dt->v;
  if (const PbField* nm = pb_last(f, 8)) t.name = pb_str(*nm);
  if (t.data_type == 7) {  // INT64: packed int64_data (7) or little-endian raw_data (9)
    bool any7 = false;
    for (const PbField& x : f)
      if (x.field == 7) {
        any7 = true;
        if (x.wtype == 2) packed_varints(x, t.i64);
        else model_error("malformed int64_data");
      }
    if (!any7)
      if (const PbField* raw = pb_last(f, 9)) {
        if (raw->wtype != 2) model_error("malformed raw_data");
        for (size_t i = 0; i < raw->n; i += 8) {
          const size_t k = std::min<size_t>(8, raw->n - i);
          uint64_t u = 0;
          for (size_t j = 0; j < k; j++) u |= (uint64_t)raw->p[i + j] << (8 * j);
          if (k < 8 && (raw->p[i + k - 1] & 0x80)) u |= ~0ULL << (8 * k);  // int.from_bytes(signed)
          t.i64.push_back((int64_t)u);
        }
      }
  }
  return t;
}

ONode parse_node(const PbField& body) {
  const auto f = pb_fields(pb_body(body, "node").p, body.n);
  ONode nd;
  for (const PbField& x : f) {
    if (x.field == 1) {
      nd.inputs.push_back(pb_str(x));
    } else if (x.field == 2) {
      nd.outputs.push_back(pb_str(x));
    } else if (x.field == 5) {
      const auto a = pb_fields(pb_body(x, "attribute").p, x.n);
      const PbField* an = pb_last(a, 1);
      const PbField* av = pb_last(a, 3);
      if (an && av) {
        if (av->wtype == 2) model_error("malformed attribute value");
        nd.attrs_int.emplace_back(pb_str(*an), (int64_t)av->v);
      }
    }
  }
  if (const PbField* o = pb_last(f, 4)) nd.op_type = pb_str(*o);
  if (const PbField* nm = pb_last(f, 3)) nd.name = pb_str(*nm);
  return nd;
}

// str.strip() on ASCII whitespace, str.strip("/")
bool py_ws(unsigned char c) { return c == ' ' || (c >= 0x09 && c <= 0x0d) || (c >= 0x1c && c <= 0x1f); }
std::string strip_ws(const std::string& s) {
  size_t a = 0, b = s.size();
  while (a < b && py_ws((unsigned char)s[a])) a++;
  while (b > a && py_ws((unsigned char)s[b - 1])) b--;
  return s.substr(a, b - a);
}
std::string strip_slash(const std::string& s) {
  size_t a = 0, b = s.size();
  while (a < b && s[a] == '/') a++;
  while (b > a && s[b - 1] == '/') b--;
  return s.substr(a, b - a);
}
std::string ascii_lower(std::string s) {
  for (char& c : s)
    if (c >= 'A' && c <= 'Z') c = (char)(c - 'A' + 'a');
  return s;
}

struct OutSpec {
  std::vector<int64_t> shape;
  std::string dtype;
};
struct OutNode {
  std::string name, op;
  std::vector<std::string> inputs;
  OutSpec out;
  bool has_w = false;
  OutSpec w;
  std::string fn;  // attrs {"fn": fn} when non-empty
};
struct OnnxResult {
  std::vector<OutNode> nodes;
  int64_t trainable = 0, skipped_elements = 0, initializer_elements = 0;
  std::vector<std::string> skipped, warnings;
};

const char* dtype_label(int64_t t) { return t == 1 ? "f32" : t == 11 ? "f64" : nullptr; }


// parse_model (model.py:143-167) + convert_graph (convert.py:84-269)
void convert_onnx(const uint8_t* data, size_t n, bool has_batch, int64_t batch, OnnxResult& R) {
  const auto model = pb_fields(data, n);
  const PbField* gf = pb_last(model, 7);
  if (!gf) model_error("model has no graph");
  const auto g = pb_fields(pb_body(*gf, "graph").p, gf->n);
  // initializers: dict name -> tensor (first position, last value)
  std::vector<OTensor> inits;
  std::unordered_map<std::string, size_t> init_at;
  for (const PbField& x : g)
    if (x.field == 5) {
      OTensor t = parse_tensor(x);
      if (t.name.empty()) model_error("initializer without a name");
      auto it = init_at.find(t.name);
      if (it == init_at.end()) {
        init_at.emplace(t.name, inits.size());
        inits.push_back(std::move(t));
      } else {
        inits[it->second] = std::move(t);
      }
    }
  if (const PbField* gn = pb_last(g, 2)) (void)pb_str(*gn);
  std::vector<ONode> nodes;
  std::vector<OValueInfo> g_in, g_out, g_vi;
  for (const PbField& x : g) {
    if (x.field == 1) nodes.push_back(parse_node(x));
    else if (x.field == 11) g_in.push_back(parse_value_info(x));
    else if (x.field == 12) g_out.push_back(parse_value_info(x));
    else if (x.field == 13) g_vi.push_back(parse_value_info(x));
  }
  // value_infos dict {vi.name: vi}: first position, last value
  std::vector<OValueInfo> vinfo;
  {
    std::unordered_map<std::string, size_t> at;
    for (OValueInfo& vi : g_vi) {
      auto it = at.find(vi.name);
      if (it == at.end()) {
        at.emplace(vi.name, vinfo.size());
        vinfo.push_back(std::move(vi));
      } else {
        vinfo[it->second] = std::move(vi);
      }
    }
  }
  for (const ONode& nd : nodes)
    if (nd.op_type == "Loop" || nd.op_type == "If" || nd.op_type == "Scan")
      unsupported("control-flow operator " + nd.op_type + " is not supported");
  for (const OTensor& t : inits) R.initializer_elements += t.num_elements();

  auto resolve = [&](const std::vector<ODim>& dims, const std::string& owner) {
    std::vector<int64_t> shape;
    for (size_t i = 0; i < dims.size(); i++) {
      if (dims[i].has_value && dims[i].value > 0) {
        shape.push_back(dims[i].value);
      } else if (i == 0 && has_batch) {
        shape.push_back(batch);
      } else {
        const std::string label = dims[i].param.empty() ? "?" : dims[i].param;
        unsupported("dynamic dimension " + py_repr(label) + " in " + py_repr(owner) +
                    "; static shapes are required (pass --batch N to fix a leading batch dimension)");
      }
    }
    return shape;
  };
  // value name -> (shape, dtype label)
  std::unordered_map<std::string, OutSpec> shapes;
  auto seed = [&](const OValueInfo& vi) {
    if (!vi.name.empty() && !vi.dims.empty()) {
      const char* lab = dtype_label(vi.elem_type);
      shapes[vi.name] = OutSpec{resolve(vi.dims, vi.name), lab ? lab : "f32"};
    }
  };
  for (const auto& vi : g_in) seed(vi);
  for (const auto& vi : g_out) seed(vi);
  for (const auto& vi : vinfo) seed(vi);

  std::unordered_set<std::string> taken;
  std::unordered_map<std::string, std::string> producer;  // ONNX value -> planner node name
  std::unordered_set<std::string> consumed;
  std::unordered_set<std::string> skipped_set;

  auto skip = [&](const OTensor& t, const char* why) {
    if (skipped_set.insert(t.name).second) {
      R.skipped.push_back(t.name);
      R.skipped_elements += t.num_elements();
      R.warnings.push_back("skipped non-trainable " + py_repr(t.name) + ": " + why);
    }
  };
  auto weight_spec = [&](const OTensor& t, const std::vector<int64_t>* dims) {
    const char* lab = dtype_label(t.data_type);
    if (!lab)
      unsupported("weight " + py_repr(t.name) + " has unsupported element type " + std::to_string(t.data_type));
    if (consumed.insert(t.name).second) R.trainable += t.num_elements();
    return OutSpec{dims && !dims->empty() ? *dims : t.dims, lab};
  };
  auto emit = [&](const std::string& name, const char* op, std::vector<std::string> ins, const OutSpec& out,
                  const OutSpec* w, const char* fn) -> std::string {
    OutNode o;
    o.name = name;
    o.op = op;
    o.inputs = std::move(ins);
    o.out = out;
    if (w) {
      o.has_w = true;
      o.w = *w;
    }
    if (fn) o.fn = fn;
    R.nodes.push_back(std::move(o));
    return name;
  };
  auto scope_name = [&](const std::string& nm, const std::string& op_type, size_t index) {
    std::string base = nm.empty() ? std::string() : strip_ws(strip_slash(nm));
    if (base.empty()) base = "block_" + std::to_string(index) + "/" + ascii_lower(op_type);
    for (char& c : base)
      if (c == '\\') c = '/';
    std::string name = base;
    int suffix = 1;
    while (taken.count(name)) {
      suffix++;
      name = base + "_" + std::to_string(suffix);
    }
    taken.insert(name);
    return name;
  };

  for (const OValueInfo& vi : g_in) {
    if (init_at.count(vi.name)) continue;
    OutSpec sp;
    auto it = shapes.find(vi.name);
    if (it != shapes.end()) {
      sp = it->second;
    } else {
      const char* lab = dtype_label(vi.elem_type);
      sp = OutSpec{resolve(vi.dims, vi.name), lab ? lab : "f32"};
    }
    std::string name = strip_ws(strip_slash(vi.name));
    if (name.empty()) name = "value";
    taken.insert(name);
    producer[vi.name] = emit(name, "input", {}, sp, nullptr, nullptr);
    shapes[vi.name] = sp;
  }

  static const std::pair<const char*, const char*> kMap[] = {
      {"Gemm", "matmul"},           {"MatMul", "matmul"},     {"Add", "elementwise"},    {"Mul", "elementwise"},
      {"Relu", "elementwise"},      {"LayerNormalization", "layernorm"}, {"Softmax", "softmax"},
      {"Gather", "embedding"},      {"Reshape", "reshape"},   {"Transpose", "reshape"},  {"Constant", "auxiliary"},
      {"Identity", "auxiliary"}};
  for (size_t index = 0; index < nodes.size(); index++) {
    const ONode& nd = nodes[index];
    std::string kind;
    for (const auto& m : kMap)
      if (nd.op_type == m.first) kind = m.second;
    if (kind.empty()) {
      kind = "elementwise";
      R.warnings.push_back("no mapping for operator " + py_repr(nd.op_type) + "; treating as elementwise");
    }
    std::string name = scope_name(nd.name, nd.op_type, index);
    std::vector<std::string> operands;
    std::vector<const OTensor*> wts;
    for (const std::string& v : nd.inputs) {
      auto it = init_at.find(v);
      if (it != init_at.end()) wts.push_back(&inits[it->second]);
      else if (!v.empty()) operands.push_back(v);
    }
    for (const std::string& v : operands)
      if (!producer.count(v)) unsupported("node " + py_repr(name) + " consumes undeclared value " + py_repr(v));
    std::vector<std::string> in_names;
    for (const std::string& v : operands) in_names.push_back(producer[v]);
    auto operand_shape = [&]() -> const OutSpec& {
      if (operands.empty()) unsupported("node " + py_repr(name) + " has no operand");
      auto it = shapes.find(operands[0]);
      if (it == shapes.end()) unsupported("no static shape known for value " + py_repr(operands[0]));
      return it->second;
    };
    const std::string out0 = nd.outputs.empty() ? std::string() : nd.outputs[0];
    if (nd.outputs.empty()) unsupported("node " + py_repr(name) + " has no output");
    OutSpec out;
    OutSpec w;
    bool has_w = false;
    const char* fn = nullptr;
    const OTensor* bias = nullptr;
    if (kind == "matmul") {
      if (wts.empty()) unsupported(nd.op_type + " node " + py_repr(name) + " has no constant weight operand");
      std::vector<int64_t> dims = wts[0]->dims;
      int64_t tb = 0;
      if (nd.op_type == "Gemm" && nd.attr("transB", tb) && tb) std::reverse(dims.begin(), dims.end());
      w = weight_spec(*wts[0], &dims);
      has_w = true;
      if (wts.size() > 1) bias = wts[1];
      const OutSpec& in = operand_shape();
      if (dims.empty()) unsupported("weight " + py_repr(wts[0]->name) + " has no dimensions");
      out.shape.assign(in.shape.begin(), in.shape.empty() ? in.shape.end() : in.shape.end() - 1);
      out.shape.push_back(dims.back());
      out.dtype = in.dtype;
    } else if (kind == "embedding") {
      int64_t axis = 0;
      nd.attr("axis", axis);
      if (wts.empty() || axis != 0) {
        kind = "elementwise";
        R.warnings.push_back("Gather node " + py_repr(name) + " is not an embedding lookup; treating as elementwise");
        out = operand_shape();
      } else {
        w = weight_spec(*wts[0], nullptr);
        has_w = true;
        out.shape = operand_shape().shape;
        out.shape.insert(out.shape.end(), wts[0]->dims.begin() + (wts[0]->dims.empty() ? 0 : 1), wts[0]->dims.end());
        out.dtype = w.dtype;
      }
    } else if (kind == "layernorm") {
      out = operand_shape();
      if (!wts.empty()) {
        w = weight_spec(*wts[0], nullptr);
        has_w = true;
      }
      if (wts.size() > 1) bias = wts[1];
    } else if (kind == "reshape") {
      for (const OTensor* t : wts) skip(*t, "shape operand");
      out.dtype = operand_shape().dtype;
      auto it = shapes.find(out0);
      bool pos = !wts.empty() && !wts[0]->i64.empty();
      if (pos)
        for (int64_t v : wts[0]->i64) pos = pos && v > 0;
      if (it != shapes.end()) {
        out.shape = it->second.shape;
      } else if (pos) {
        out.shape = wts[0]->i64;
      } else if (nd.op_type == "Transpose") {
        out.shape = operand_shape().shape;
        std::reverse(out.shape.begin(), out.shape.end());
      } else {
        unsupported("cannot determine output shape of " + py_repr(name));
      }
    } else if (kind == "auxiliary") {
      for (const OTensor* t : wts) skip(*t, "constant payload");
      if (!operands.empty()) {
        out = operand_shape();
      } else {
        auto it = shapes.find(out0);
        out = it != shapes.end() ? it->second : OutSpec{{1}, "f32"};
      }
    } else {  // elementwise, softmax, fallbacks
      out = operand_shape();
      if (kind == "elementwise") {
        fn = nd.op_type == "Mul" ? "mul" : "add";  // ELEMENTWISE_FN (Add/Relu -> add)
        if (!wts.empty()) {
          w = weight_spec(*wts[0], nullptr);
          has_w = true;
          for (size_t j = 1; j < wts.size(); j++) skip(*wts[j], "surplus constant operand");
        }
      }
    }
    if (auto it = shapes.find(out0); it != shapes.end()) out.shape = it->second.shape;
    emit(name, kind.c_str(), in_names, out, has_w ? &w : nullptr, fn);
    if (bias) {
      const std::string bias_name = scope_name(name + "_bias", "Add", index);
      const OutSpec bw = weight_spec(*bias, nullptr);
      emit(bias_name, "elementwise", {name}, out, &bw, "add");
      name = bias_name;
    }
    for (size_t j = 0; j < nd.outputs.size(); j++) {
      producer[nd.outputs[j]] = name;
      shapes[nd.outputs[j]] = out;
    }
  }
  for (size_t i = 0; i < g_out.size(); i++) {
    const OValueInfo& vi = g_out[i];
    auto pit = producer.find(vi.name);
    if (pit == producer.end()) unsupported("graph output " + py_repr(vi.name) + " is never produced");
    const OutSpec sp = shapes[vi.name];
    std::string name = g_out.size() == 1 ? "output" : "output_" + std::to_string(i);
    while (taken.count(name)) name += "_";
    taken.insert(name);
    emit(name, "output", {pit->second}, sp, nullptr, nullptr);
  }
  for (const OTensor& t : inits)
    if (!consumed.count(t.name) && !skipped_set.count(t.name)) skip(t, "unused initializer");
}

// json.dumps of the converted document (default separators, ensure_ascii)
void json_str(std::string& o, std::string_view s) {
  static const char* hex = "0123456789abcdef";
  o += '"';
  size_t i = 0;
  while (i < s.size()) {
    const unsigned char c = (unsigned char)s[i];
    if (c == '"') o += "\\\"";
    else if (c == '\\') o += "\\\\";
    else if (c == '\n') o += "\\n";
    else if (c == '\r') o += "\\r";
    else if (c == '\t') o += "\\t";
    else if (c == '\b') o += "\\b";
    else if (c == '\f') o += "\\f";
    else if (c < 0x20) {
      o += "\\u00";
      o += hex[c >> 4];
      o += hex[c & 15];
    } else if (c < 0x80) {
      o += (char)c;
    } else {  // decode UTF-8, emit \uXXXX (surrogate pairs above the BMP)
      uint32_t cp;
      size_t k;
      if ((c & 0xE0) == 0xC0) { cp = c & 0x1F; k = 1; }
      else if ((c & 0xF0) == 0xE0) { cp = c & 0x0F; k = 2; }
      else { cp = c & 0x07; k = 3; }
      for (size_t j = 1; j <= k && i + j < s.size(); j++) cp = (cp << 6) | ((unsigned char)s[i + j] & 0x3F);
      i += k;
      auto u16 = [&](uint32_t u) {
        o += "\\u";
        for (int sh = 12; sh >= 0; sh -= 4) o += hex[(u >> sh) & 15];
      };
      if (cp >= 0x10000) {
        cp -= 0x10000;
        u16(0xD800 + (cp >> 10));
        u16(0xDC00 + (cp & 0x3FF));
      } else {
        u16(cp);
      }
    }
    i++;
  }
  o += '"';
}

void json_shape(std::string& o, const OutSpec& s, bool trainable) {
  o += "{\"shape\": [";
  for (size_t i = 0; i < s.shape.size(); i++) {
    if (i) o += ", ";
    o += std::to_string(s.shape[i]);
  }
  o += "], \"dtype\": ";
  json_str(o, s.dtype);
  o += trainable ? ", \"trainable\": true}" : ", \"trainable\": false}";
}

std::string onnx_json(const OnnxResult& R) {
  std::string o = "{\"version\": 1, \"nodes\": [";
  for (size_t k = 0; k < R.nodes.size(); k++) {
    const OutNode& nd = R.nodes[k];
    if (k) o += ", ";
    o += "{\"name\": ";
    json_str(o, nd.name);
    o += ", \"op\": ";
    json_str(o, nd.op);
    o += ", \"inputs\": [";
    for (size_t j = 0; j < nd.inputs.size(); j++) {
      if (j) o += ", ";
      json_str(o, nd.inputs[j]);
    }
    o += "], \"weight\": ";
    if (nd.has_w) json_shape(o, nd.w, true);
    else o += "null";
    o += ", \"output\": ";
    json_shape(o, nd.out, false);
    if (!nd.fn.empty()) {
      o += ", \"attrs\": {\"fn\": ";
      json_str(o, nd.fn);
      o += "}";
    }
    o += "}";
  }
  return o + "]}";
}

// load_graph semantics of the converted document, straight into build_graph
void onnx_to_graph(const OnnxResult& R, sp_ingest* out) {
  PhaseTimer tm;
  const size_t n = R.nodes.size();
  std::vector<Raw> raw(n);
  std::vector<std::vector<std::string_view>> in_names(n);
  auto spec = [](const OutSpec& s, bool trainable) {
    Spec t;
    for (int64_t d : s.shape) t.shape.push_back(d);
    t.width = s.dtype == "f64" ? 8 : 4;
    t.trainable = trainable;
    if (t.shape.empty()) parse_error("tensor shape must be non-empty");
    if (t.shape.nonpos) parse_error("tensor dimensions must be positive integers");
    return t;
  };
  for (size_t k = 0; k < n; k++) {
    const OutNode& nd = R.nodes[k];
    Raw& r = raw[k];
    r.name = nd.name;
    r.op = ELEMENTWISE;
    for (int q = 0; q < 10; q++)
      if (nd.op == kOpLabels[q]) r.op = (Op)q;
    for (const std::string& s : nd.inputs) in_names[k].push_back(s);
    r.out = spec(nd.out, false);
    if (nd.has_w) {
      r.w = spec(nd.w, true);
      r.has_w = true;
    }
  }
  build_graph(raw, in_names, out, tm);
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

int sp_ingest_onnx(const uint8_t* data, int64_t len, int32_t has_batch, int64_t batch, int32_t export_only,
                   sp_ingest** out) {
  if (!data || len < 0 || !out) return SP_ERR_CONFIG;
  *out = nullptr;
  sp_ingest* g = new sp_ingest();
  try {
    OnnxResult R;
    convert_onnx(data, (size_t)len, has_batch != 0, batch, R);
    g->trainable = R.trainable;
    g->skipped_elements = R.skipped_elements;
    g->initializer_elements = R.initializer_elements;
    g->warnings = R.warnings;
    g->skipped = R.skipped;
    if (export_only) g->json = onnx_json(R);
    else onnx_to_graph(R, g);
  } catch (const OnnxError& e) {
    t_err = e.what();
    t_err_a.clear();
    t_err_b.clear();
    delete g;
    return e.kind;
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
    return SP_ERR_ONNX_PARSE;
  }
  *out = g;
  return SP_OK;
}

int sp_ingest_report(const sp_ingest* g, int64_t* counts) {
  if (!g || !counts) return SP_ERR_CONFIG;
  counts[0] = g->trainable;
  counts[1] = g->skipped_elements;
  counts[2] = g->initializer_elements;
  counts[3] = (int64_t)g->warnings.size();
  counts[4] = (int64_t)g->skipped.size();
  counts[5] = (int64_t)g->json.size();
  return SP_OK;
}

const char* sp_ingest_text(const sp_ingest* g, int32_t kind, int64_t i) {
  if (!g) return nullptr;
  if (kind == 0) return g->json.c_str();
  if (kind == 1 && i >= 0 && i < (int64_t)g->warnings.size()) return g->warnings[i].c_str();
  if (kind == 2 && i >= 0 && i < (int64_t)g->skipped.size()) return g->skipped[i].c_str();
  return nullptr;
}

}  // extern "C"
