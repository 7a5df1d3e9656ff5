/*
 * _lower: native lowering of a grouped ModelGraph to the flat sp_graph arrays
 * (the Python restatement is lowering.lower()).
 *
 * Walks the reference's object graph (ir.py:164-292: ModelGraph.topo_order,
 * ModelGraph.nodes[name] -> GraphNode{op, inputs, activation, weight},
 * TensorSpec{shape, dtype, trainable}) with the CPython API in two passes:
 * names -> row map (open addressing, no Python dict), then one pass over the
 * nodes filling bytearrays that lowering.py wraps as numpy arrays without
 * copying.  Enum members (OpKind,
 * DType) are mapped through small pointer-keyed caches filled by calling back
 * into the Python mapping functions on first sight, so string-valued and
 * enum-valued graphs (reference types or this package's) lower identically.
 */
#define PY_SSIZE_T_CLEAN
#include <Python.h>

/* The parallel walker reads CPython object layouts in place (compact-ASCII str
 * bytes and hash, compact ints via PyUnstable_Long_*): supported for the 3.12
 * and 3.13 layouts only.  The module records the version it was built for and
 * lowering.py uses it only under that interpreter (tests/test_lowering.py). */
#if PY_VERSION_HEX < 0x030C0000 || PY_VERSION_HEX >= 0x030E0000
#error "lower_ext.c reads the CPython 3.12/3.13 object layouts"
#endif
#include <stddef.h>
#include <stdint.h>
#include <string.h>
#include <time.h>

static double now_ms(void) {
  struct timespec ts;
  clock_gettime(CLOCK_MONOTONIC, &ts);
  return ts.tv_sec * 1e3 + ts.tv_nsec * 1e-6;
}


#define MAX_RANK 8
#define CACHE_N 64

typedef struct {
  PyObject* key[CACHE_N];
  long val[CACHE_N];
  int n;
} PtrCache;

static int cache_get(PtrCache* c, PyObject* key, PyObject* fn, long* out) {
  for (int i = 0; i < c->n; i++)
    if (c->key[i] == key) {
      *out = c->val[i];
      return 0;
    }
  PyObject* r = PyObject_CallOneArg(fn, key);
  if (!r) return -1;
  long v = PyLong_AsLong(r);
  Py_DECREF(r);
  if (v == -1 && PyErr_Occurred()) return -1;
  if (c->n < CACHE_N) {
    Py_INCREF(key);  /* keep the member alive while cached */
    c->key[c->n] = key;
    c->val[c->n] = v;
    c->n++;
  }
  *out = v;
  return 0;
}

/* string keys compare by value (JSON-loaded graphs carry one str object per node) */
static int cache_get_any(PtrCache* c, PyObject* key, PyObject* fn, long* out) {
  for (int i = 0; i < c->n; i++)
    if (c->key[i] == key) {
      *out = c->val[i];
      return 0;
    }
  if (PyUnicode_CheckExact(key))
    for (int i = 0; i < c->n; i++)
      if (PyUnicode_CheckExact(c->key[i]) && PyUnicode_Compare(c->key[i], key) == 0) {
        *out = c->val[i];
        return 0;
      }
  return cache_get(c, key, fn, out);
}

/* name -> topological index: open addressing over the names list (borrowed keys) */
typedef struct {
  PyObject** key;
  Py_hash_t* hash;
  int32_t* val;
  size_t mask;
} NameMap;

static int namemap_init(NameMap* m, Py_ssize_t n) {
  size_t cap = 16;
  while (cap < (size_t)n * 2) cap <<= 1;
  m->key = (PyObject**)PyMem_Calloc(cap, sizeof(PyObject*));
  m->hash = (Py_hash_t*)PyMem_Malloc(cap * sizeof(Py_hash_t));
  m->val = (int32_t*)PyMem_Malloc(cap * sizeof(int32_t));
  m->mask = cap - 1;
  if (!m->key || !m->hash || !m->val) {
    PyErr_NoMemory();
    return -1;
  }
  return 0;
}

static void namemap_free(NameMap* m) {
  PyMem_Free(m->key);
  PyMem_Free(m->hash);
  PyMem_Free(m->val);
}

static int namemap_put(NameMap* m, PyObject* k, int32_t v) {
  const Py_hash_t h = PyObject_Hash(k);
  if (h == -1) return -1;
  for (size_t i = (size_t)h & m->mask;; i = (i + 1) & m->mask)
    if (!m->key[i]) {
      m->key[i] = k;
      m->hash[i] = h;
      m->val[i] = v;
      return 0;
    }
}

/* -1 with no exception set: absent */
static int32_t namemap_get(const NameMap* m, PyObject* k) {
  const Py_hash_t h = PyObject_Hash(k);
  if (h == -1) return -1;
  for (size_t i = (size_t)h & m->mask;; i = (i + 1) & m->mask) {
    PyObject* q = m->key[i];
    if (!q) return -1;
    if (q == k) return m->val[i];
    if (m->hash[i] == h && PyUnicode_Check(k) && PyUnicode_Compare(q, k) == 0) return m->val[i];
  }
}

static void cache_clear(PtrCache* c) {
  for (int i = 0; i < c->n; i++) Py_DECREF(c->key[i]);
  c->n = 0;
}

/* shape tuple -> rank, dims[MAX_RANK] (unused 0), element product (double for the overflow check) */
static int read_shape(PyObject* shape, int64_t* dims, int* rank, int64_t* elems, double* felems) {
  PyObject* seq = PySequence_Fast(shape, "shape must be a sequence");
  if (!seq) return -1;
  Py_ssize_t r = PySequence_Fast_GET_SIZE(seq);
  PyObject** it = PySequence_Fast_ITEMS(seq);
  int64_t p = 1;
  double fp = 1.0;
  for (Py_ssize_t j = 0; j < r; j++) {
    long long v = PyLong_AsLongLong(it[j]);
    if (v == -1 && PyErr_Occurred()) {
      Py_DECREF(seq);
      return -1;
    }
    if (j < MAX_RANK) dims[j] = v;
    p *= v;
    fp *= (double)v;
  }
  for (Py_ssize_t j = r; j < MAX_RANK; j++) dims[j] = 0;
  Py_DECREF(seq);
  *rank = (int)r;
  *elems = p;
  *felems = fp;
  return 0;
}

static PyObject* new_bytearray(Py_ssize_t n) { return PyByteArray_FromStringAndSize(NULL, n > 0 ? n : 0); }

/*
 * Attribute read with a fast path for __slots__ classes (this package's IR
 * types): the member descriptor's offset is resolved once per (type, name)
 * and the value read straight from the instance; any other class goes
 * through PyObject_GetAttr.  Returns a new reference.
 */
typedef struct {
  PyObject* name;
  PyTypeObject* type;
  Py_ssize_t offset;  /* -1: generic getattr */
} FieldRef;

static PyObject* field_get(FieldRef* f, PyObject* obj) {
  PyTypeObject* tp = Py_TYPE(obj);
  if (tp != f->type) {
    f->type = tp;
    f->offset = -1;
    PyObject* d = PyObject_GetAttr((PyObject*)tp, f->name);
    if (d) {
      if (Py_IS_TYPE(d, &PyMemberDescr_Type)) {
        PyMemberDef* m = ((PyMemberDescrObject*)d)->d_member;
        if (m->type == Py_T_OBJECT_EX && !(m->flags & Py_RELATIVE_OFFSET)) f->offset = m->offset;
      }
      Py_DECREF(d);
    } else {
      PyErr_Clear();
    }
  }
  if (f->offset >= 0) {
    PyObject* v = *(PyObject**)((char*)obj + f->offset);
    if (v) {
      Py_INCREF(v);
      return v;
    }
  }
  return PyObject_GetAttr(obj, f->name);
}

/* reference on an object, kept in `keep` (new references released at the end) */
#define KEEP(slot, expr)                    \
  do {                                      \
    PyObject* _v = (expr);                  \
    if (!_v) goto done;                     \
    (slot) = _v;                            \
  } while (0)

/*
 * lower_arrays(topo_order, nodes, op_code, dtype_width)
 * -> (names, ascii, max_act_rank, max_w_rank, overflow_what,
 *     name_bytes, name_off, op, act_rank, act_shape, act_bytes,
 *     w_rank, w_shape, w_bytes, w_trainable, in_off, in_idx)
 *
 * The walk is a sequence of passes over pointer arrays (nodes, then their
 * fields, then the fields' fields) rather than one dependent chain per node:
 * the loads of a pass are independent across nodes, so the core overlaps the
 * cache misses of the scattered Python objects.
 */
static PyObject* lower_serial(PyObject* self, PyObject* args) {
  PyObject *topo, *nodes, *op_fn, *width_fn;
  if (!PyArg_ParseTuple(args, "OO!OO", &topo, &PyDict_Type, &nodes, &op_fn, &width_fn)) return NULL;
  PyObject* names = PySequence_List(topo);
  if (!names) return NULL;
  const Py_ssize_t n = PyList_GET_SIZE(names);
  NameMap index = {NULL, NULL, NULL, 0};
  PyObject *b_names = NULL, *b_noff = NULL, *b_op = NULL, *b_arank = NULL, *b_ashape = NULL, *b_abytes = NULL,
           *b_wrank = NULL, *b_wshape = NULL, *b_wbytes = NULL, *b_wtrain = NULL, *b_inoff = NULL, *b_inidx = NULL;
  PyObject* result = NULL;
  PtrCache opc = {{0}, {0}, 0}, wc = {{0}, {0}, 0};
  /* per-node object arrays: 0 node, 1 op, 2 activation, 3 weight, 4 inputs,
     5 act shape, 6 act dtype, 7 w shape, 8 w dtype, 9 w trainable */
  enum { K_NODE, K_OP, K_ACT, K_W, K_IN, K_ASH, K_ADT, K_WSH, K_WDT, K_WTR, K_N };
  PyObject** obj = NULL;
  int32_t* inidx = NULL;
  static PyObject *s_op, *s_inputs, *s_activation, *s_weight, *s_shape, *s_dtype, *s_trainable, *s_member,
      *s_output;
  if (!s_op) {
    s_op = PyUnicode_InternFromString("op");
    s_inputs = PyUnicode_InternFromString("inputs");
    s_activation = PyUnicode_InternFromString("activation");
    s_weight = PyUnicode_InternFromString("weight");
    s_shape = PyUnicode_InternFromString("shape");
    s_dtype = PyUnicode_InternFromString("dtype");
    s_trainable = PyUnicode_InternFromString("trainable");
    s_member = PyUnicode_InternFromString("member");
    s_output = PyUnicode_InternFromString("output");
  }
  FieldRef f_op = {s_op, NULL, -1}, f_inputs = {s_inputs, NULL, -1}, f_act = {s_activation, NULL, -1},
           f_weight = {s_weight, NULL, -1}, a_shape = {s_shape, NULL, -1}, a_dtype = {s_dtype, NULL, -1},
           w_shape_f = {s_shape, NULL, -1}, w_dtype_f = {s_dtype, NULL, -1}, w_train_f = {s_trainable, NULL, -1},
           f_member = {s_member, NULL, -1}, m_op = {s_op, NULL, -1}, m_out = {s_output, NULL, -1},
           m_weight = {s_weight, NULL, -1};
  const int trace = getenv("SP_LOWER_TRACE") != NULL;
  double tm[8];
  tm[0] = now_ms();
  if (namemap_init(&index, n) < 0) goto done;
  obj = (PyObject**)PyMem_Calloc((size_t)(n ? n : 1) * K_N, sizeof(PyObject*));
  if (!obj) {
    PyErr_NoMemory();
    goto done;
  }
#define O(i, k) obj[(size_t)(i) * K_N + (k)]
  /* pass 1: names -> row map, name bytes; node objects (borrowed from the dict) */
  Py_ssize_t nbytes = 0, E = 0;
  int ascii = 1;
  for (Py_ssize_t i = 0; i < n; i++) {
    PyObject* nm = PyList_GET_ITEM(names, i);
    if (!PyUnicode_Check(nm)) {
      PyErr_SetString(PyExc_TypeError, "node names must be str");
      goto done;
    }
    Py_ssize_t L;
    if (!PyUnicode_AsUTF8AndSize(nm, &L)) goto done;
    if (!PyUnicode_IS_ASCII(nm)) ascii = 0;
    nbytes += L;
    if (namemap_put(&index, nm, (int32_t)i) < 0) goto done;
  }
  tm[1] = now_ms();
  for (Py_ssize_t i = 0; i < n; i++) {
    PyObject* nm = PyList_GET_ITEM(names, i);
    PyObject* node = PyDict_GetItemWithError(nodes, nm);
    if (!node) {
      if (!PyErr_Occurred()) PyErr_SetObject(PyExc_KeyError, nm);
      goto done;
    }
    Py_INCREF(node);
    O(i, K_NODE) = node;
  }
  /* pass 2: op / activation / weight / inputs (the reference's GraphNode
     exposes op/activation/weight as properties over its RawNode `member`,
     ir.py:164-202: read the member's fields instead) */
  tm[2] = now_ms();
  const int via_member = n > 0 && PyObject_HasAttr(O(0, K_NODE), s_member);
  for (Py_ssize_t i = 0; i < n; i++) {
    PyObject* node = O(i, K_NODE);
    PyObject* src = node;
    if (via_member) KEEP(src, field_get(&f_member, node));
    PyObject *o = field_get(via_member ? &m_op : &f_op, src), *a = o ? field_get(via_member ? &m_out : &f_act, src) : NULL;
    PyObject* w = a ? field_get(via_member ? &m_weight : &f_weight, src) : NULL;
    PyObject* in = w ? field_get(&f_inputs, node) : NULL;
    if (via_member) Py_DECREF(src);
    if (!in) {
      Py_XDECREF(o);
      Py_XDECREF(a);
      Py_XDECREF(w);
      goto done;
    }
    O(i, K_OP) = o;
    O(i, K_ACT) = a;
    O(i, K_W) = w;
    O(i, K_IN) = in;
  }
  tm[3] = now_ms();
  /* pass 3: tensor spec fields */
  for (Py_ssize_t i = 0; i < n; i++) {
    KEEP(O(i, K_ASH), field_get(&a_shape, O(i, K_ACT)));
    KEEP(O(i, K_ADT), field_get(&a_dtype, O(i, K_ACT)));
    PyObject* w = O(i, K_W);
    if (w != Py_None) {
      KEEP(O(i, K_WSH), field_get(&w_shape_f, w));
      KEEP(O(i, K_WDT), field_get(&w_dtype_f, w));
      KEEP(O(i, K_WTR), field_get(&w_train_f, w));
    }
  }
  tm[4] = now_ms();
  b_names = new_bytearray(nbytes);
  b_noff = new_bytearray((n + 1) * 8);
  b_op = new_bytearray(n);
  b_arank = new_bytearray(n);
  b_ashape = new_bytearray(n * MAX_RANK * 8);
  b_abytes = new_bytearray(n * 8);
  b_wrank = new_bytearray(n);
  b_wshape = new_bytearray(n * MAX_RANK * 8);
  b_wbytes = new_bytearray(n * 8);
  b_wtrain = new_bytearray(n);
  b_inoff = new_bytearray((n + 1) * 8);
  if (!b_names || !b_noff || !b_op || !b_arank || !b_ashape || !b_abytes || !b_wrank || !b_wshape || !b_wbytes ||
      !b_wtrain || !b_inoff)
    goto done;
  char* pn = PyByteArray_AS_STRING(b_names);
  int64_t* noff = (int64_t*)PyByteArray_AS_STRING(b_noff);
  uint8_t* op = (uint8_t*)PyByteArray_AS_STRING(b_op);
  uint8_t* arank = (uint8_t*)PyByteArray_AS_STRING(b_arank);
  int64_t* ashape = (int64_t*)PyByteArray_AS_STRING(b_ashape);
  int64_t* abytes = (int64_t*)PyByteArray_AS_STRING(b_abytes);
  uint8_t* wrank = (uint8_t*)PyByteArray_AS_STRING(b_wrank);
  int64_t* wshape = (int64_t*)PyByteArray_AS_STRING(b_wshape);
  int64_t* wbytes = (int64_t*)PyByteArray_AS_STRING(b_wbytes);
  uint8_t* wtrain = (uint8_t*)PyByteArray_AS_STRING(b_wtrain);
  int64_t* inoff = (int64_t*)PyByteArray_AS_STRING(b_inoff);
  int max_ar = 0, max_wr = 0;
  const char* overflow = NULL;
  /* pass 4: values */
  Py_ssize_t off = 0;
  noff[0] = 0;
  for (Py_ssize_t i = 0; i < n; i++) {
    Py_ssize_t L;
    const char* u = PyUnicode_AsUTF8AndSize(PyList_GET_ITEM(names, i), &L);
    memcpy(pn + off, u, (size_t)L);
    off += L;
    noff[i + 1] = off;
    long v;
    if (cache_get_any(&opc, O(i, K_OP), op_fn, &v) < 0) goto done;
    op[i] = (uint8_t)v;
    int r;
    int64_t el;
    double fel;
    if (read_shape(O(i, K_ASH), ashape + i * MAX_RANK, &r, &el, &fel) < 0) goto done;
    if (cache_get_any(&wc, O(i, K_ADT), width_fn, &v) < 0) goto done;
    if (r > max_ar) max_ar = r;
    arank[i] = (uint8_t)(r > 255 ? 255 : r);
    abytes[i] = el * (int64_t)v;
    if (fel * 8.0 >= 9223372036854775808.0 && !overflow) overflow = "activation";
    if (O(i, K_W) == Py_None) {
      wrank[i] = 0;
      memset(wshape + i * MAX_RANK, 0, MAX_RANK * 8);
      wbytes[i] = 0;
      wtrain[i] = 0;
      continue;
    }
    if (read_shape(O(i, K_WSH), wshape + i * MAX_RANK, &r, &el, &fel) < 0) goto done;
    if (cache_get_any(&wc, O(i, K_WDT), width_fn, &v) < 0) goto done;
    const int tr = PyObject_IsTrue(O(i, K_WTR));
    if (tr < 0) goto done;
    if (r > max_wr) max_wr = r;
    wrank[i] = (uint8_t)(r > 255 ? 255 : r);
    wbytes[i] = el * (int64_t)v;
    wtrain[i] = (uint8_t)tr;
    if (fel * 8.0 >= 9223372036854775808.0 && !overflow) overflow = "weight";
  }
  tm[5] = now_ms();
  /* pass 5: producers, GraphNode.inputs order */
  Py_ssize_t cap = n * 2 + 16;
  inidx = (int32_t*)PyMem_Malloc((size_t)cap * sizeof(int32_t));
  if (!inidx) {
    PyErr_NoMemory();
    goto done;
  }
  inoff[0] = 0;
  for (Py_ssize_t i = 0; i < n; i++) {
    PyObject* seq = PySequence_Fast(O(i, K_IN), "inputs must be a sequence");
    if (!seq) goto done;
    const Py_ssize_t k = PySequence_Fast_GET_SIZE(seq);
    PyObject** it = PySequence_Fast_ITEMS(seq);
    if (E + k > cap) {
      while (E + k > cap) cap *= 2;
      int32_t* grown = (int32_t*)PyMem_Realloc(inidx, (size_t)cap * sizeof(int32_t));
      if (!grown) {
        Py_DECREF(seq);
        PyErr_NoMemory();
        goto done;
      }
      inidx = grown;
    }
    for (Py_ssize_t j = 0; j < k; j++) {
      const int32_t pi = namemap_get(&index, it[j]);
      if (pi < 0) {
        if (!PyErr_Occurred()) PyErr_SetObject(PyExc_KeyError, it[j]);
        Py_DECREF(seq);
        goto done;
      }
      inidx[E++] = pi;
    }
    Py_DECREF(seq);
    inoff[i + 1] = E;
  }
  tm[6] = now_ms();
  if (trace)
    fprintf(stderr, "[lower] names %.2f lookup %.2f fields %.2f specs %.2f values %.2f inputs %.2f ms\n", tm[1] - tm[0],
            tm[2] - tm[1], tm[3] - tm[2], tm[4] - tm[3], tm[5] - tm[4], tm[6] - tm[5]);
  b_inidx = PyByteArray_FromStringAndSize((const char*)inidx, E * 4);
  if (!b_inidx) goto done;
  result = Py_BuildValue("(OiiizOOOOOOOOOOOO)", names, ascii, max_ar, max_wr, overflow, b_names, b_noff, b_op,
                         b_arank, b_ashape, b_abytes, b_wrank, b_wshape, b_wbytes, b_wtrain, b_inoff, b_inidx);
done:
  if (obj) {
    for (size_t q = 0; q < (size_t)(n ? n : 1) * K_N; q++) Py_XDECREF(obj[q]);
    PyMem_Free(obj);
  }
#undef O
  PyMem_Free(inidx);
  cache_clear(&opc);
  cache_clear(&wc);
  Py_XDECREF(names);
  namemap_free(&index);
  Py_XDECREF(b_names);
  Py_XDECREF(b_noff);
  Py_XDECREF(b_op);
  Py_XDECREF(b_arank);
  Py_XDECREF(b_ashape);
  Py_XDECREF(b_abytes);
  Py_XDECREF(b_wrank);
  Py_XDECREF(b_wshape);
  Py_XDECREF(b_wbytes);
  Py_XDECREF(b_wtrain);
  Py_XDECREF(b_inoff);
  Py_XDECREF(b_inidx);
  return result;
}

/* ------------------------------------------------------------------------
 * Parallel walker.  The serial passes above are bound by cache misses on
 * the scattered Python objects (one or two per field), so the same walk is
 * spread over host threads.  The workers read the frozen object graph
 * without touching the interpreter: borrowed pointers only (the caller's
 * graph keeps every object alive and this thread keeps the GIL for the
 * whole call, so no Python code can run, mutate or free anything), exact
 * type checks, __slots__ offsets resolved up front, compact-ASCII str bytes
 * read in place and hashed with a private hash, compact ints read in place.
 * Anything outside that envelope (other node classes, non-ASCII names, big
 * ints, non-tuple shapes or inputs, unknown or duplicate names, byte-size
 * overflow) makes the call fall back to the serial walker, which produces
 * the identical arrays and raises the errors.
 * ---------------------------------------------------------------------- */
#include <pthread.h>
#include <sched.h>
#include <unistd.h>

#define PAR_MAX_THREADS 32
#define PAR_MIN_NODES 4096
#define PAR_DISTINCT 32

static Py_ssize_t slot_offset(PyTypeObject* tp, PyObject* name) {
  PyObject* d = PyObject_GetAttr((PyObject*)tp, name);
  Py_ssize_t off = -1;
  if (d) {
    if (Py_IS_TYPE(d, &PyMemberDescr_Type)) {
      PyMemberDef* m = ((PyMemberDescrObject*)d)->d_member;
      if (m->type == Py_T_OBJECT_EX && !(m->flags & Py_RELATIVE_OFFSET)) off = m->offset;
    }
    Py_DECREF(d);
  } else {
    PyErr_Clear();
  }
  return off;
}

static inline PyObject* slot_read(PyObject* o, Py_ssize_t off) { return *(PyObject**)((char*)o + off); }

static inline uint64_t name_hash(const char* p, Py_ssize_t n) {
  uint64_t h = 0x243F6A8885A308D3ull ^ (uint64_t)n;
  while (n >= 8) {
    uint64_t w;
    memcpy(&w, p, 8);
    h = (h ^ w) * 0x9E3779B97F4A7C15ull;
    h ^= h >> 29;
    p += 8;
    n -= 8;
  }
  if (n) {
    uint64_t w = 0;
    memcpy(&w, p, (size_t)n);
    h = (h ^ w) * 0x9E3779B97F4A7C15ull;
    h ^= h >> 29;
  }
  h *= 0xBF58476D1CE4E5B9ull;
  return h ^ (h >> 31);
}

/* exact compact-ASCII str -> its bytes in place; 0 outside the envelope */
static inline int ascii_view(PyObject* o, const char** p, Py_ssize_t* n) {
  if (!PyUnicode_CheckExact(o) || !PyUnicode_IS_COMPACT_ASCII(o)) return 0;
  *p = (const char*)(((PyASCIIObject*)o) + 1);
  *n = PyUnicode_GET_LENGTH(o);
  return 1;
}

/* exact tuple of compact ints -> read_shape's outputs; 0 outside the envelope */
static inline int shape_view(PyObject* t, int64_t* dims, int* rank, int64_t* elems, double* felems) {
  if (!PyTuple_CheckExact(t)) return 0;
  const Py_ssize_t r = PyTuple_GET_SIZE(t);
  int64_t p = 1;
  double fp = 1.0;
  for (Py_ssize_t j = 0; j < r; j++) {
    PyObject* v = PyTuple_GET_ITEM(t, j);
    if (!PyLong_CheckExact(v) || !PyUnstable_Long_IsCompact((PyLongObject*)v)) return 0;
    const int64_t x = (int64_t)PyUnstable_Long_CompactValue((PyLongObject*)v);
    if (j < MAX_RANK) dims[j] = x;
    p *= x;
    fp *= (double)x;
  }
  for (Py_ssize_t j = r; j < MAX_RANK; j++) dims[j] = 0;
  *rank = (int)r;
  *elems = p;
  *felems = fp;
  return 1;
}

typedef struct Par {
  Py_ssize_t n, nd;
  PyObject** names; /* topo names */
  PyObject** dkey;  /* nodes dict entries */
  PyObject** dval;
  PyTypeObject *t_node, *t_spec;
  Py_ssize_t o_op, o_in, o_act, o_w, o_shape, o_dtype, o_train;
  const char** np; /* name bytes, length, hash per row */
  Py_ssize_t* nl;
  uint64_t* nh;
  int32_t* tab; /* open-addressing row map: row + 1, 0 = empty */
  int32_t* ptab; /* the same rows keyed by the name object's address */
  size_t mask;
  PyObject** node;
  PyObject** inseq;
  int64_t *ael, *wel; /* element counts (bytes = count x dtype width, mapped after the join) */
  PyObject **opv, **adt, **wdt;
  char* pn;
  int64_t *noff, *ashape, *wshape, *inoff;
  uint8_t *arank, *wrank, *wtrain;
  int32_t* inidx;
  int nthreads, go, fail;
  /* the names list is built by the workers; name bytes allocated between phases */
  PyObject* names_list;
  PyObject* b_names;
  Py_ssize_t nbytes;
  /* enum members -> codes: distinct objects per thread (phase 3), mapped by
     thread 0 through the Python functions, applied in phase 4 */
  PyObject *op_fn, *width_fn;
  PyObject* dop[PAR_MAX_THREADS][PAR_DISTINCT];
  PyObject* ddt[PAR_MAX_THREADS][PAR_DISTINCT];
  int nop[PAR_MAX_THREADS], ndt[PAR_MAX_THREADS];
  PyObject* mop[PAR_MAX_THREADS * PAR_DISTINCT];
  PyObject* mdt[PAR_MAX_THREADS * PAR_DISTINCT];
  long cop[PAR_MAX_THREADS * PAR_DISTINCT], cdt[PAR_MAX_THREADS * PAR_DISTINCT];
  int nmop, nmdt;
  uint8_t* op;
  int64_t *abytes, *wbytes;
  Py_ssize_t bytes_part[PAR_MAX_THREADS], edges_part[PAR_MAX_THREADS];
  int max_ar[PAR_MAX_THREADS], max_wr[PAR_MAX_THREADS];
  double ph[8];  /* thread 0's clock at each phase boundary (SP_LOWER_TRACE) */
  int bar_count, bar_gen;  /* spin barrier: the phases last ~0.1-1 ms, a futex wake-up ~0.1 ms */
} Par;

typedef struct {
  Par* P;
  int t;
} ParArg;

static inline void par_fail(Par* P) { __atomic_store_n(&P->fail, 1, __ATOMIC_RELAXED); }
static inline int par_failed(Par* P) { return __atomic_load_n(&P->fail, __ATOMIC_RELAXED); }

static inline int32_t par_find(const Par* P, const char* p, Py_ssize_t n, uint64_t h) {
  for (size_t s = h & P->mask;; s = (s + 1) & P->mask) {
    const int32_t v = __atomic_load_n(&P->tab[s], __ATOMIC_ACQUIRE);
    if (!v) return -1;
    const int32_t j = v - 1;
    if (P->nh[j] == h && P->nl[j] == n && memcmp(P->np[j], p, (size_t)n) == 0) return j;
  }
}

static inline size_t ptr_slot(const void* o) {
  uint64_t h = (uint64_t)(uintptr_t)o * 0x9E3779B97F4A7C15ull;
  return (size_t)(h ^ (h >> 29));
}

/* row of a name object by address: the names of GraphNode.inputs and the
   dict keys are usually the very objects of topo_order, and this lookup does
   not touch them; -1 when absent (then compare by content) */
static inline int32_t par_find_ptr(const Par* P, PyObject* o) {
  for (size_t s = ptr_slot(o) & P->mask;; s = (s + 1) & P->mask) {
    const int32_t v = __atomic_load_n(&P->ptab[s], __ATOMIC_ACQUIRE);
    if (!v) return -1;
    if (P->names[v - 1] == o) return v - 1;
  }
}

static inline int32_t par_row_of(const Par* P, PyObject* o) {
  const int32_t r = par_find_ptr(P, o);
  if (r >= 0) return r;
  const char* p;
  Py_ssize_t L;
  if (!ascii_view(o, &p, &L)) return -2;
  return par_find(P, p, L, name_hash(p, L));
}

static void par_barrier(Par* P) {
  const int gen = __atomic_load_n(&P->bar_gen, __ATOMIC_ACQUIRE);
  if (__atomic_add_fetch(&P->bar_count, 1, __ATOMIC_ACQ_REL) == P->nthreads) {
    __atomic_store_n(&P->bar_count, 0, __ATOMIC_RELAXED);
    __atomic_store_n(&P->bar_gen, gen + 1, __ATOMIC_RELEASE);
    return;
  }
  for (unsigned spins = 0; __atomic_load_n(&P->bar_gen, __ATOMIC_ACQUIRE) == gen; spins++) {
    if (spins < 4096) {
#if defined(__x86_64__) || defined(__i386__)
      __builtin_ia32_pause();
#endif
    } else {
      sched_yield();  /* oversubscribed host: let the other threads run */
    }
  }
}

/* add o to a small distinct-pointer set; 0 when the set is full */
static inline int distinct_add(PyObject** set, int* n, PyObject* o) {
  for (int k = 0; k < *n; k++)
    if (set[k] == o) return 1;
  if (*n == PAR_DISTINCT) return 0;
  set[(*n)++] = o;
  return 1;
}

static inline long code_of(PyObject* const* keys, const long* vals, int n, PyObject* o) {
  for (int k = 0; k < n; k++)
    if (keys[k] == o) return vals[k];
  return -1;
}

/* thread 0 between phases 3 and 4 (it holds the GIL): map every distinct
   enum member through the Python functions; 0 on failure (error cleared) */
static int par_map_codes(Par* P) {
  P->nmop = P->nmdt = 0;
  for (int u = 0; u < P->nthreads; u++) {
    for (int k = 0; k < P->nop[u]; k++)
      if (code_of(P->mop, P->cop, P->nmop, P->dop[u][k]) < 0) P->mop[P->nmop++] = P->dop[u][k];
    for (int k = 0; k < P->ndt[u]; k++)
      if (code_of(P->mdt, P->cdt, P->nmdt, P->ddt[u][k]) < 0) P->mdt[P->nmdt++] = P->ddt[u][k];
  }
  for (int pass = 0; pass < 2; pass++) {
    PyObject* fn = pass ? P->width_fn : P->op_fn;
    PyObject** keys = pass ? P->mdt : P->mop;
    long* vals = pass ? P->cdt : P->cop;
    const int n = pass ? P->nmdt : P->nmop;
    for (int k = 0; k < n; k++) {
      PyObject* r = PyObject_CallOneArg(fn, keys[k]);
      long v = r ? PyLong_AsLong(r) : -1;
      Py_XDECREF(r);
      if (!r || (v == -1 && PyErr_Occurred()) || v < 0) {
        PyErr_Clear();
        return 0;
      }
      vals[k] = v;
    }
  }
  return 1;
}

static void par_phases(Par* P, int t) {
  if (t == 0) P->ph[0] = now_ms();
  const int T = P->nthreads;
  const Py_ssize_t n = P->n, lo = n * t / T, hi = n * (t + 1) / T;
  const Py_ssize_t dlo = P->nd * t / T, dhi = P->nd * (t + 1) / T;
  /* phase 1: name bytes and hash, lock-free insert into the row map */
  Py_ssize_t bytes = 0;
  for (Py_ssize_t i = lo; i < hi && !par_failed(P); i++) {
    const char* p;
    Py_ssize_t L;
    if (!ascii_view(P->names[i], &p, &L)) {
      par_fail(P);
      break;
    }
    const uint64_t h = name_hash(p, L);
    P->np[i] = p;
    P->nl[i] = L;
    P->nh[i] = h;
    bytes += L;
    for (size_t s = h & P->mask;; s = (s + 1) & P->mask) {
      int32_t expect = 0;
      if (__atomic_compare_exchange_n(&P->tab[s], &expect, (int32_t)(i + 1), 0, __ATOMIC_ACQ_REL,
                                      __ATOMIC_ACQUIRE))
        break;
      const int32_t j = expect - 1;
      if (P->nh[j] == h && P->nl[j] == L && memcmp(P->np[j], p, (size_t)L) == 0) {
        par_fail(P); /* duplicate name */
        break;
      }
    }
    for (size_t s = ptr_slot(P->names[i]) & P->mask;; s = (s + 1) & P->mask) {
      int32_t expect = 0;
      if (__atomic_compare_exchange_n(&P->ptab[s], &expect, (int32_t)(i + 1), 0, __ATOMIC_ACQ_REL,
                                      __ATOMIC_ACQUIRE))
        break;
    }
  }
  P->bytes_part[t] = bytes;
  if (t == 0) P->ph[1] = now_ms();
  par_barrier(P);
  if (t == 0 && !par_failed(P)) {  /* the name-byte buffer (this thread holds the GIL) */
    Py_ssize_t nb = 0;
    for (int u = 0; u < T; u++) nb += P->bytes_part[u];
    P->b_names = PyByteArray_FromStringAndSize(NULL, nb > 0 ? nb : 0);
    if (!P->b_names) {
      PyErr_Clear();
      par_fail(P);
    } else {
      P->pn = PyByteArray_AS_STRING(P->b_names);
    }
  }
  /* phase 2: dict entries -> rows */
  for (Py_ssize_t j = dlo; j < dhi && !par_failed(P); j++) {
    const int32_t r = par_row_of(P, P->dkey[j]);
    if (r == -2) {
      par_fail(P);
      break;
    }
    if (r >= 0) P->node[r] = P->dval[j];
  }
  Py_ssize_t base = 0;
  for (int u = 0; u < t; u++) base += P->bytes_part[u];
  if (t == 0) P->ph[2] = now_ms();
  par_barrier(P);
  /* phase 3: node fields, tensor specs, shapes, name bytes, input counts */
  Py_ssize_t edges = 0;
  int mar = 0, mwr = 0;
  for (Py_ssize_t i = lo; i < hi && !par_failed(P); i++) {
    PyObject* nd = P->node[i];
    if (!nd || Py_TYPE(nd) != P->t_node) goto bad;
    PyObject *op = slot_read(nd, P->o_op), *in = slot_read(nd, P->o_in), *a = slot_read(nd, P->o_act),
             *w = slot_read(nd, P->o_w);
    if (!op || !in || !a || !w || Py_TYPE(a) != P->t_spec || !PyTuple_CheckExact(in)) goto bad;
    memcpy(P->pn + base, P->np[i], (size_t)P->nl[i]);
    base += P->nl[i];
    P->noff[i + 1] = base;
    P->opv[i] = op;
    if (!distinct_add(P->dop[t], &P->nop[t], op)) goto bad;
    Py_INCREF(P->names[i]);  /* distinct objects (duplicates failed phase 1) */
    PyList_SET_ITEM(P->names_list, i, P->names[i]);
    PyObject *sh = slot_read(a, P->o_shape), *dt = slot_read(a, P->o_dtype);
    int r;
    int64_t el;
    double fel;
    if (!sh || !dt || !shape_view(sh, P->ashape + i * MAX_RANK, &r, &el, &fel)) goto bad;
    if (fel * 8.0 >= 9223372036854775808.0) goto bad;
    if (r > mar) mar = r;
    P->arank[i] = (uint8_t)(r > 255 ? 255 : r);
    P->ael[i] = el;
    P->adt[i] = dt;
    if (!distinct_add(P->ddt[t], &P->ndt[t], dt)) goto bad;
    if (w == Py_None) {
      P->wrank[i] = 0;
      memset(P->wshape + i * MAX_RANK, 0, MAX_RANK * 8);
      P->wel[i] = 0;
      P->wtrain[i] = 0;
      P->wdt[i] = NULL;
    } else {
      if (Py_TYPE(w) != P->t_spec) goto bad;
      PyObject *wsh = slot_read(w, P->o_shape), *wdt = slot_read(w, P->o_dtype), *tr = slot_read(w, P->o_train);
      if (!wsh || !wdt || (tr != Py_True && tr != Py_False)) goto bad;
      if (!shape_view(wsh, P->wshape + i * MAX_RANK, &r, &el, &fel)) goto bad;
      if (fel * 8.0 >= 9223372036854775808.0) goto bad;
      if (r > mwr) mwr = r;
      P->wrank[i] = (uint8_t)(r > 255 ? 255 : r);
      P->wel[i] = el;
      P->wdt[i] = wdt;
      if (!distinct_add(P->ddt[t], &P->ndt[t], wdt)) goto bad;
      P->wtrain[i] = tr == Py_True;
    }
    P->inseq[i] = in;
    edges += PyTuple_GET_SIZE(in);
    continue;
  bad:
    par_fail(P);
    break;
  }
  P->edges_part[t] = edges;
  P->max_ar[t] = mar;
  P->max_wr[t] = mwr;
  if (t == 0) P->ph[3] = now_ms();
  par_barrier(P);
  if (t == 0 && !par_failed(P)) {
    Py_ssize_t E = 0;
    for (int u = 0; u < T; u++) E += P->edges_part[u];
    P->inidx = (int32_t*)malloc((size_t)(E ? E : 1) * sizeof(int32_t));
    if (!P->inidx || !par_map_codes(P)) par_fail(P);
  }
  if (t == 0) P->ph[4] = now_ms();
  par_barrier(P);
  if (par_failed(P)) return;
  /* phase 4: producer rows in GraphNode.inputs order */
  Py_ssize_t e = 0;
  for (int u = 0; u < t; u++) e += P->edges_part[u];
  for (Py_ssize_t i = lo; i < hi; i++) {
    P->op[i] = (uint8_t)code_of(P->mop, P->cop, P->nmop, P->opv[i]);
    P->abytes[i] = P->ael[i] * (int64_t)code_of(P->mdt, P->cdt, P->nmdt, P->adt[i]);
    P->wbytes[i] = P->wdt[i] ? P->wel[i] * (int64_t)code_of(P->mdt, P->cdt, P->nmdt, P->wdt[i]) : 0;
    PyObject* in = P->inseq[i];
    const Py_ssize_t k = PyTuple_GET_SIZE(in);
    for (Py_ssize_t j = 0; j < k; j++) {
      const int32_t r = par_row_of(P, PyTuple_GET_ITEM(in, j));
      if (r < 0) {
        par_fail(P);
        return;
      }
      P->inidx[e++] = r;
    }
    P->inoff[i + 1] = e;
  }
}

/* Persistent workers (created on first use, kept for the process): a call
   hands them its Par through a generation counter instead of creating
   threads (~20 us each).  Idle workers sleep on a condition variable. */
static struct {
  pthread_mutex_t mu;
  pthread_cond_t cv;
  int size;          /* workers started (thread ids 1..size) */
  unsigned gen;      /* bumped per job */
  Par* job;
  int done;          /* workers finished with the current job */
} g_pool = {PTHREAD_MUTEX_INITIALIZER, PTHREAD_COND_INITIALIZER, 0, 0, NULL, 0};

static void* pool_worker(void* arg) {
  /* arg = worker id | the job generation at creation << 8: a worker started
     for a call must take part in that call even if it reaches the lock late */
  const int t = (int)((uintptr_t)arg & 0xff);
  unsigned seen = (unsigned)((uintptr_t)arg >> 8);
  pthread_mutex_lock(&g_pool.mu);
  for (;;) {
    while (g_pool.gen == seen) pthread_cond_wait(&g_pool.cv, &g_pool.mu);
    seen = g_pool.gen;
    Par* P = g_pool.job;
    pthread_mutex_unlock(&g_pool.mu);
    if (P && t < P->nthreads) par_phases(P, t);
    __atomic_add_fetch(&g_pool.done, 1, __ATOMIC_ACQ_REL);
    pthread_mutex_lock(&g_pool.mu);
  }
  return NULL;
}

static void pool_after_fork(void) {  /* the child has none of the parent's threads */
  pthread_mutex_init(&g_pool.mu, NULL);
  pthread_cond_init(&g_pool.cv, NULL);
  g_pool.size = 0;
  g_pool.job = NULL;
}

/* grow the pool to `want` workers (best effort); returns the worker count */
static int pool_ensure(int want) {
  static int atfork = 0;
  if (!atfork) {
    pthread_atfork(NULL, NULL, pool_after_fork);
    atfork = 1;
  }
  while (g_pool.size < want) {
    pthread_t th;
    pthread_attr_t at;
    pthread_attr_init(&at);
    pthread_attr_setdetachstate(&at, PTHREAD_CREATE_DETACHED);
    const uintptr_t arg = (uintptr_t)(g_pool.size + 1) | ((uintptr_t)g_pool.gen << 8);
    const int rc = pthread_create(&th, &at, pool_worker, (void*)arg);
    pthread_attr_destroy(&at);
    if (rc) break;
    g_pool.size++;
  }
  return g_pool.size;
}

/* run par_phases on this thread (t = 0) and workers 1..nthreads-1; every
   started worker takes part in the handshake (idle ones return at once) */
static void pool_run(Par* P) {
  const int workers = g_pool.size;
  __atomic_store_n(&g_pool.done, 0, __ATOMIC_RELAXED);
  pthread_mutex_lock(&g_pool.mu);
  g_pool.job = P;
  g_pool.gen++;
  pthread_cond_broadcast(&g_pool.cv);
  pthread_mutex_unlock(&g_pool.mu);
  par_phases(P, 0);
  for (unsigned spins = 0; __atomic_load_n(&g_pool.done, __ATOMIC_ACQUIRE) < workers; spins++)
    if (spins > 4096) sched_yield();
  g_pool.job = NULL;
}

/* NULL with no exception set: outside the envelope (use the serial walker) */
static PyObject* lower_parallel(PyObject* topo, PyObject* nodes, PyObject* op_fn, PyObject* width_fn) {
  if (!PyList_CheckExact(topo) && !PyTuple_CheckExact(topo)) return NULL;
  const Py_ssize_t n = PySequence_Fast_GET_SIZE(topo);
  long ncpu = sysconf(_SC_NPROCESSORS_ONLN);
  const char* env = getenv("SP_LOWER_THREADS");
  if (env) ncpu = atol(env);
  int T = (int)(ncpu < PAR_MAX_THREADS ? ncpu : PAR_MAX_THREADS);
  if (T > n / 2048) T = (int)(n / 2048);
  if (n < PAR_MIN_NODES || T < 2 || n >= INT32_MAX / 4 || PyDict_GET_SIZE(nodes) == 0) return NULL;
  PyObject* n0 = PyDict_GetItemWithError(nodes, PySequence_Fast_ITEMS(topo)[0]);
  if (!n0) {
    PyErr_Clear();
    return NULL;
  }
  static PyObject *s_op, *s_inputs, *s_activation, *s_weight, *s_shape, *s_dtype, *s_trainable;
  if (!s_op) {
    s_op = PyUnicode_InternFromString("op");
    s_inputs = PyUnicode_InternFromString("inputs");
    s_activation = PyUnicode_InternFromString("activation");
    s_weight = PyUnicode_InternFromString("weight");
    s_shape = PyUnicode_InternFromString("shape");
    s_dtype = PyUnicode_InternFromString("dtype");
    s_trainable = PyUnicode_InternFromString("trainable");
  }
  Par* P = (Par*)calloc(1, sizeof(Par));
  if (!P) return NULL;
  PyObject *result = NULL, *names = NULL;
  PyObject *b_names = NULL, *b_noff = NULL, *b_op = NULL, *b_arank = NULL, *b_ashape = NULL, *b_abytes = NULL,
           *b_wrank = NULL, *b_wshape = NULL, *b_wbytes = NULL, *b_wtrain = NULL, *b_inoff = NULL, *b_inidx = NULL;
  P->n = n;
  P->t_node = Py_TYPE(n0);
  P->o_op = slot_offset(P->t_node, s_op);
  P->o_in = slot_offset(P->t_node, s_inputs);
  P->o_act = slot_offset(P->t_node, s_activation);
  P->o_w = slot_offset(P->t_node, s_weight);
  PyObject* a0 = P->o_act >= 0 ? slot_read(n0, P->o_act) : NULL;
  if (!a0 || P->o_op < 0 || P->o_in < 0 || P->o_w < 0) goto out;
  P->t_spec = Py_TYPE(a0);
  P->o_shape = slot_offset(P->t_spec, s_shape);
  P->o_dtype = slot_offset(P->t_spec, s_dtype);
  P->o_train = slot_offset(P->t_spec, s_trainable);
  if (P->o_shape < 0 || P->o_dtype < 0 || P->o_train < 0) goto out;
  double tp[8];
  tp[0] = now_ms();
  /* the workers fill the returned names list (one reference per distinct name) */
  names = PyList_New(n);
  if (!names) {
    PyErr_Clear();
    goto out;
  }
  P->names_list = names;
  P->names = PySequence_Fast_ITEMS(topo);
  P->op_fn = op_fn;
  P->width_fn = width_fn;
  tp[1] = tp[2] = now_ms();
  P->nd = PyDict_GET_SIZE(nodes);
  P->dkey = (PyObject**)malloc((size_t)P->nd * sizeof(PyObject*));
  P->dval = (PyObject**)malloc((size_t)P->nd * sizeof(PyObject*));
  if (!P->dkey || !P->dval) goto out;
  {
    Py_ssize_t pos = 0, j = 0;
    PyObject *k, *v;
    while (j < P->nd && PyDict_Next(nodes, &pos, &k, &v)) {
      P->dkey[j] = k;
      P->dval[j] = v;
      j++;
    }
    P->nd = j;
  }
  tp[3] = now_ms();
  size_t cap = 16;
  while (cap < (size_t)n * 2) cap <<= 1;
  P->mask = cap - 1;
  P->tab = (int32_t*)calloc(cap, sizeof(int32_t));
  P->ptab = (int32_t*)calloc(cap, sizeof(int32_t));
  P->np = (const char**)malloc((size_t)n * sizeof(char*));
  P->nl = (Py_ssize_t*)malloc((size_t)n * sizeof(Py_ssize_t));
  P->nh = (uint64_t*)malloc((size_t)n * 8);
  P->node = (PyObject**)calloc((size_t)n, sizeof(PyObject*));
  P->inseq = (PyObject**)malloc((size_t)n * sizeof(PyObject*));
  P->ael = (int64_t*)malloc((size_t)n * 8);
  P->wel = (int64_t*)malloc((size_t)n * 8);
  P->opv = (PyObject**)malloc((size_t)n * sizeof(PyObject*));
  P->adt = (PyObject**)malloc((size_t)n * sizeof(PyObject*));
  P->wdt = (PyObject**)malloc((size_t)n * sizeof(PyObject*));
  if (!P->tab || !P->ptab || !P->np || !P->nl || !P->nh || !P->node || !P->inseq || !P->ael || !P->wel || !P->opv || !P->adt ||
      !P->wdt)
    goto out;
  b_noff = new_bytearray((n + 1) * 8);
  b_op = new_bytearray(n);
  b_arank = new_bytearray(n);
  b_ashape = new_bytearray(n * MAX_RANK * 8);
  b_abytes = new_bytearray(n * 8);
  b_wrank = new_bytearray(n);
  b_wshape = new_bytearray(n * MAX_RANK * 8);
  b_wbytes = new_bytearray(n * 8);
  b_wtrain = new_bytearray(n);
  b_inoff = new_bytearray((n + 1) * 8);
  if (!b_noff || !b_op || !b_arank || !b_ashape || !b_abytes || !b_wrank || !b_wshape || !b_wbytes || !b_wtrain ||
      !b_inoff) {
    PyErr_Clear();
    goto out;
  }
  P->op = (uint8_t*)PyByteArray_AS_STRING(b_op);
  P->abytes = (int64_t*)PyByteArray_AS_STRING(b_abytes);
  P->wbytes = (int64_t*)PyByteArray_AS_STRING(b_wbytes);
  P->noff = (int64_t*)PyByteArray_AS_STRING(b_noff);
  P->arank = (uint8_t*)PyByteArray_AS_STRING(b_arank);
  P->ashape = (int64_t*)PyByteArray_AS_STRING(b_ashape);
  P->wrank = (uint8_t*)PyByteArray_AS_STRING(b_wrank);
  P->wshape = (int64_t*)PyByteArray_AS_STRING(b_wshape);
  P->wtrain = (uint8_t*)PyByteArray_AS_STRING(b_wtrain);
  P->inoff = (int64_t*)PyByteArray_AS_STRING(b_inoff);
  P->noff[0] = 0;
  P->inoff[0] = 0;
  /* the GIL stays with this thread throughout */
  const int created = 1 + (pool_ensure(T - 1) < T - 1 ? g_pool.size : T - 1);
  P->nthreads = created;
  if (created < 2) goto out;
  tp[4] = now_ms();
  {
    /* no collection while the workers read the object graph (thread 0
       allocates between phases) */
    const int gc_was = PyGC_Disable();
    pool_run(P);
    if (gc_was) PyGC_Enable();
  }
  tp[5] = now_ms();
  b_names = P->b_names;  /* owned from here on */
  P->b_names = NULL;
  if (par_failed(P)) goto out;
  {
    int max_ar = 0, max_wr = 0;
    for (int u = 0; u < created; u++) {
      if (P->max_ar[u] > max_ar) max_ar = P->max_ar[u];
      if (P->max_wr[u] > max_wr) max_wr = P->max_wr[u];
    }
    const Py_ssize_t E = P->inoff[n];
    b_inidx = PyByteArray_FromStringAndSize((const char*)P->inidx, E * 4);
    if (!b_inidx) goto err;
    result = Py_BuildValue("(OiiizOOOOOOOOOOOO)", names, 1, max_ar, max_wr, NULL, b_names, b_noff, b_op, b_arank,
                           b_ashape, b_abytes, b_wrank, b_wshape, b_wbytes, b_wtrain, b_inoff, b_inidx);
    if (!result) goto err;
    if (getenv("SP_LOWER_TRACE"))
      fprintf(stderr,
              "[lower-par] setup %.2f dict %.2f alloc %.2f threads %.2f (p1 %.2f p2 %.2f p3 %.2f p3b %.2f p4 %.2f) "
              "post %.2f ms (%d threads)\n",
              tp[1] - tp[0], tp[3] - tp[2], tp[4] - tp[3], tp[5] - tp[4], P->ph[1] - P->ph[0], P->ph[2] - P->ph[1],
              P->ph[3] - P->ph[2], P->ph[4] - P->ph[3], tp[5] - P->ph[4], now_ms() - tp[5], created);
    goto out;
  err:
    /* a Python mapping call failed: let the serial walker raise it */
    PyErr_Clear();
  }
out:
  Py_XDECREF(names);
  Py_XDECREF(b_names);
  Py_XDECREF(b_noff);
  Py_XDECREF(b_op);
  Py_XDECREF(b_arank);
  Py_XDECREF(b_ashape);
  Py_XDECREF(b_abytes);
  Py_XDECREF(b_wrank);
  Py_XDECREF(b_wshape);
  Py_XDECREF(b_wbytes);
  Py_XDECREF(b_wtrain);
  Py_XDECREF(b_inoff);
  Py_XDECREF(b_inidx);
  free(P->dkey);
  free(P->dval);
  free(P->tab);
  free(P->ptab);
  free(P->np);
  free(P->nl);
  free(P->nh);
  free(P->node);
  free(P->inseq);
  free(P->ael);
  free(P->wel);
  free(P->opv);
  free(P->adt);
  free(P->wdt);
  free(P->inidx);
  free(P);
  return result;
}

/* lower_arrays(topo_order, nodes, op_code, dtype_width): the parallel walker
   when the graph is inside its envelope, else the serial one */
static PyObject* lower_arrays(PyObject* self, PyObject* args) {
  PyObject *topo, *nodes, *op_fn, *width_fn;
  if (!PyArg_ParseTuple(args, "OO!OO", &topo, &PyDict_Type, &nodes, &op_fn, &width_fn)) return NULL;
  const char* mode = getenv("SP_LOWER_SERIAL");
  if (!mode || !*mode || *mode == '0') {
    const double t0 = now_ms();
    PyObject* r = lower_parallel(topo, nodes, op_fn, width_fn);
    if (getenv("SP_LOWER_TRACE"))
      fprintf(stderr, "[lower] parallel %s %.2f ms\n", r ? "ok" : "declined", now_ms() - t0);
    if (r) return r;
  }
  return lower_serial(self, args);
}

/*
 * block_instances(names, members, prefix_node, prefix_len, inst_off, block_T, ascii)
 * -> [ (instances tuple) per block ], instance = (prefix str, member scopes tuple)
 * (Subgraph.instances, pruning.py:33-55) straight from the fold's flat arrays:
 * members int32, prefix_node/prefix_len/inst_off/block_T int64 buffers.
 */
static PyObject* block_instances(PyObject* self, PyObject* args) {
  PyObject *names, *ascii_o;
  Py_buffer mem, pn, pl, io, bt;
  if (!PyArg_ParseTuple(args, "O!y*y*y*y*y*O", &PyList_Type, &names, &mem, &pn, &pl, &io, &bt, &ascii_o)) return NULL;
  PyObject* out = NULL;
  const int ascii = PyObject_IsTrue(ascii_o);
  const int32_t* m = (const int32_t*)mem.buf;
  const int64_t* pnode = (const int64_t*)pn.buf;
  const int64_t* plen = (const int64_t*)pl.buf;
  const int64_t* ioff = (const int64_t*)io.buf;
  const int64_t* T = (const int64_t*)bt.buf;
  const Py_ssize_t nb = bt.len / 8, nn = PyList_GET_SIZE(names), nm = mem.len / 4;
  out = PyList_New(nb);
  if (!out) goto done;
  Py_ssize_t mo = 0;
  for (Py_ssize_t b = 0; b < nb; b++) {
    const Py_ssize_t R = ioff[b + 1] - ioff[b];
    PyObject* insts = PyTuple_New(R);
    if (!insts) goto fail;
    PyList_SET_ITEM(out, b, insts);
    for (Py_ssize_t i = 0; i < R; i++) {
      const int64_t j = ioff[b] + i;
      if (pnode[j] < 0 || pnode[j] >= nn || mo + T[b] > nm) {
        PyErr_SetString(PyExc_IndexError, "fold arrays out of range");
        goto fail;
      }
      PyObject* full = PyList_GET_ITEM(names, pnode[j]);
      PyObject* pre;
      if (ascii) {
        pre = PyUnicode_Substring(full, 0, plen[j]);
      } else {  /* prefix length is in UTF-8 bytes */
        Py_ssize_t L;
        const char* u = PyUnicode_AsUTF8AndSize(full, &L);
        pre = u ? PyUnicode_DecodeUTF8(u, plen[j] < L ? plen[j] : L, "strict") : NULL;
      }
      if (!pre) goto fail;
      PyObject* tup = PyTuple_New(T[b]);
      if (!tup) {
        Py_DECREF(pre);
        goto fail;
      }
      for (int64_t t = 0; t < T[b]; t++) {
        const int32_t v = m[mo + t];
        if (v < 0 || v >= nn) {
          Py_DECREF(pre);
          Py_DECREF(tup);
          PyErr_SetString(PyExc_IndexError, "member index out of range");
          goto fail;
        }
        PyObject* s = PyList_GET_ITEM(names, v);
        Py_INCREF(s);
        PyTuple_SET_ITEM(tup, t, s);
      }
      mo += T[b];
      /* tuples of strings cannot be part of a reference cycle: untracked now,
         as the collector would untrack them at its first pass over them
         (_PyTuple_MaybeUntrack) -- the pass itself (~10^5 referents for c5)
         is then never paid */
      PyObject_GC_UnTrack(tup);
      PyObject* pair = PyTuple_Pack(2, pre, tup);
      Py_DECREF(pre);
      Py_DECREF(tup);
      if (!pair) goto fail;
      PyObject_GC_UnTrack(pair);
      PyTuple_SET_ITEM(insts, i, pair);
    }
    PyObject_GC_UnTrack(insts);
  }
  goto done;
fail:
  Py_CLEAR(out);
done:
  PyBuffer_Release(&mem);
  PyBuffer_Release(&pn);
  PyBuffer_Release(&pl);
  PyBuffer_Release(&io);
  PyBuffer_Release(&bt);
  return out;
}




/*
 * Ctor(cls, field_names): a callable that builds instances of a dataclass
 * from positional field values without running its generated __init__
 * (object.__new__ + generic attribute stores; frozen classes included).  For
 * the result objects of a search (~10^4 per c5 step) the generated __init__,
 * which goes through object.__setattr__ once per field for frozen classes,
 * is most of the assembly time.  Only for classes without __post_init__ and
 * with every field passed.
 */
typedef struct {
  PyObject_HEAD
  PyTypeObject* cls;
  PyObject* names;  /* tuple of interned str: the positional fields */
  PyObject* fixed_names;  /* remaining fields, set to shared default values */
  PyObject* fixed_values;
  vectorcallfunc vectorcall;
} CtorObject;

static PyObject* ctor_vectorcall(PyObject* self, PyObject* const* args, size_t nargsf, PyObject* kwnames) {
  CtorObject* c = (CtorObject*)self;
  const Py_ssize_t n = PyVectorcall_NARGS(nargsf);
  const Py_ssize_t nf = PyTuple_GET_SIZE(c->names);
  if (kwnames || n != nf) {
    PyErr_Format(PyExc_TypeError, "%s ctor takes exactly %zd positional arguments", c->cls->tp_name, nf);
    return NULL;
  }
  static PyObject* empty = NULL;
  if (!empty && !(empty = PyTuple_New(0))) return NULL;
  PyObject* o = c->cls->tp_new(c->cls, empty, NULL);
  if (!o) return NULL;
  for (Py_ssize_t i = 0; i < nf; i++)
    if (PyObject_GenericSetAttr(o, PyTuple_GET_ITEM(c->names, i), args[i]) < 0) {
      Py_DECREF(o);
      return NULL;
    }
  for (Py_ssize_t i = 0; i < PyTuple_GET_SIZE(c->fixed_names); i++)
    if (PyObject_GenericSetAttr(o, PyTuple_GET_ITEM(c->fixed_names, i), PyTuple_GET_ITEM(c->fixed_values, i)) < 0) {
      Py_DECREF(o);
      return NULL;
    }
  return o;
}

static void ctor_dealloc(PyObject* self) {
  CtorObject* c = (CtorObject*)self;
  Py_XDECREF(c->cls);
  Py_XDECREF(c->names);
  Py_XDECREF(c->fixed_names);
  Py_XDECREF(c->fixed_values);
  Py_TYPE(self)->tp_free(self);
}

static PyTypeObject CtorType = {
    PyVarObject_HEAD_INIT(NULL, 0).tp_name = "_lower.Ctor",
    .tp_basicsize = sizeof(CtorObject),
    .tp_dealloc = ctor_dealloc,
    .tp_call = PyVectorcall_Call,
    .tp_vectorcall_offset = offsetof(CtorObject, vectorcall),
    .tp_flags = Py_TPFLAGS_DEFAULT | Py_TPFLAGS_HAVE_VECTORCALL,
};

static PyObject* make_ctor(PyObject* self, PyObject* args) {
  PyObject *cls, *names, *fixed_names = NULL, *fixed_values = NULL;
  if (!PyArg_ParseTuple(args, "O!O!|O!O!", &PyType_Type, &cls, &PyTuple_Type, &names, &PyTuple_Type, &fixed_names,
                        &PyTuple_Type, &fixed_values))
    return NULL;
  if ((fixed_names ? PyTuple_GET_SIZE(fixed_names) : 0) != (fixed_values ? PyTuple_GET_SIZE(fixed_values) : 0)) {
    PyErr_SetString(PyExc_ValueError, "fixed names and values differ in length");
    return NULL;
  }
  if (PyType_Ready(&CtorType) < 0) return NULL;
  CtorObject* c = PyObject_New(CtorObject, &CtorType);
  if (!c) return NULL;
  c->cls = NULL;
  c->names = c->fixed_names = c->fixed_values = NULL;
  Py_INCREF(cls);
  c->cls = (PyTypeObject*)cls;
  c->fixed_names = fixed_names ? fixed_names : PyTuple_New(0);
  c->fixed_values = fixed_values ? fixed_values : PyTuple_New(0);
  if (fixed_names) Py_INCREF(fixed_names);
  if (fixed_values) Py_INCREF(fixed_values);
  c->names = PyTuple_New(PyTuple_GET_SIZE(names));
  if (!c->names) {
    Py_DECREF(c);
    return NULL;
  }
  for (Py_ssize_t i = 0; i < PyTuple_GET_SIZE(names); i++) {
    PyObject* nm = PyTuple_GET_ITEM(names, i);
    if (!PyUnicode_Check(nm)) {
      PyErr_SetString(PyExc_TypeError, "field names must be str");
      Py_DECREF(c);
      return NULL;
    }
    Py_INCREF(nm);
    PyUnicode_InternInPlace(&nm);
    PyTuple_SET_ITEM(c->names, i, nm);
  }
  c->vectorcall = ctor_vectorcall;
  return (PyObject*)c;
}


/*
 * singleton_results(ctors, subs, sel, recs, xblocks, node, toff, op, radix,
 *                   obytes, flops, pnames, pallred, specs, identity, gather,
 *                   kind_labels, overlap)
 * -> [SubgraphResult or None] for the blocks `sel` of a search whose template
 * is ONE node (c5: ~1000 residual ops).  The same objects routed_plans_all +
 * collect build in Python (search.py), straight from the raw sp_score_out /
 * sp_explain_block records: CandidatePlan, NodeRouting, exits, CostReport,
 * RoutedPlan, SubgraphResult.  None where the block has no winner, its
 * winner did not route, or the explained total differs from the scored one:
 * the caller's Python path handles (and raises for) those.
 *   ctors: (CandidatePlan, NodeRouting, RoutedPlan, CostReport, SubgraphResult)
 *   recs: raw sp_score_out [nb] (40 B), xblocks: raw sp_explain_block [nb] (104 B)
 *   node: int8 [ne, 4]; toff: int64 [nb + 1]; op, radix: uint8 [nb];
 *   obytes, flops: int64 [nb]; pnames / pallred: per op code tuples
 *   specs: (replica, split(0), ..., split(7)); gather: allgather per axis
 */
typedef struct {
  uint64_t candidates, valid, best_index;
  double best_total;
  int32_t best_num_split, has_best;
} RecView;

typedef struct {
  int32_t valid, fail_pos;
  double forward_comm, backward_comm, total;
  int64_t bytes[4], calls[4], collective_calls;
} XView;

static PyObject* call_n(PyObject* f, PyObject** a, size_t n) { return PyObject_Vectorcall(f, a, n, NULL); }

static PyObject* singleton_results(PyObject* self, PyObject* args) {
  PyObject *ctors, *subs, *pnames, *pallred, *specs, *identity, *allreduce, *gather, *kinds;
  Py_buffer sel, recs, xb, node, toff, op, radix, ob, fl;
  double overlap;
  if (!PyArg_ParseTuple(args, "O!O!y*y*y*y*y*y*y*y*y*O!O!O!OOO!O!d", &PyTuple_Type, &ctors, &PyList_Type, &subs, &sel,
                        &recs, &xb, &node, &toff, &op, &radix, &ob, &fl, &PyTuple_Type, &pnames, &PyTuple_Type,
                        &pallred, &PyTuple_Type, &specs, &identity, &allreduce, &PyTuple_Type, &gather,
                        &PyTuple_Type, &kinds, &overlap))
    return NULL;
  PyObject* out = NULL;
  static PyObject* s_template = NULL;
  if (!s_template) s_template = PyUnicode_InternFromString("template");
  const int64_t* selp = (const int64_t*)sel.buf;
  const Py_ssize_t ns = sel.len / 8, nb = PyList_GET_SIZE(subs);
  const RecView* R = (const RecView*)recs.buf;
  const XView* X = (const XView*)xb.buf;
  const int8_t* nd = (const int8_t*)node.buf;
  const int64_t* to = (const int64_t*)toff.buf;
  const uint8_t* opc = (const uint8_t*)op.buf;
  const uint8_t* rdx = (const uint8_t*)radix.buf;
  const int64_t* obp = (const int64_t*)ob.buf;
  const int64_t* flp = (const int64_t*)fl.buf;
  if (PyTuple_GET_SIZE(ctors) != 5 || PyTuple_GET_SIZE(specs) < 9 || PyTuple_GET_SIZE(gather) < 8 ||
      PyTuple_GET_SIZE(kinds) != 4 || recs.len < nb * (Py_ssize_t)sizeof(RecView) ||
      xb.len < nb * (Py_ssize_t)sizeof(XView) || toff.len < (nb + 1) * 8 || op.len < nb || radix.len < nb ||
      ob.len < nb * 8 || fl.len < nb * 8) {
    PyErr_SetString(PyExc_ValueError, "singleton_results: inconsistent arguments");
    goto done;
  }
  PyObject *mkPlan = PyTuple_GET_ITEM(ctors, 0), *mkNR = PyTuple_GET_ITEM(ctors, 1),
           *mkRP = PyTuple_GET_ITEM(ctors, 2), *mkCR = PyTuple_GET_ITEM(ctors, 3),
           *mkRes = PyTuple_GET_ITEM(ctors, 4);
  PyObject* py_overlap = PyFloat_FromDouble(overlap);
  PyObject* empty = PyTuple_New(0);
  if (!py_overlap || !empty) {
    Py_XDECREF(py_overlap);
    Py_XDECREF(empty);
    goto done;
  }
  out = PyList_New(ns);
  if (!out) goto fail0;
  for (Py_ssize_t q = 0; q < ns; q++) {
    const int64_t b = selp[q];
    if (b < 0 || b >= nb || to[b + 1] - to[b] != 1) {
      PyErr_SetString(PyExc_ValueError, "singleton_results: not a one-node block");
      goto fail;
    }
    const RecView r = R[b];
    const XView x = X[b];
    /* CostReport.total = forward + backward * (1 - overlap), rounded in that order */
    const double total = x.forward_comm + x.backward_comm * (1.0 - overlap);
    if (!r.has_best || !x.valid || (r.best_total == r.best_total && total != r.best_total)) {
      Py_INCREF(Py_None);
      PyList_SET_ITEM(out, q, Py_None);
      continue;
    }
    const int64_t e0 = to[b];
    const int pidx = nd[4 * e0], sax = nd[4 * e0 + 1], xax = nd[4 * e0 + 2];
    const int oc = opc[b];
    if (oc >= PyTuple_GET_SIZE(pnames) || oc >= PyTuple_GET_SIZE(pallred) || pidx < 0 ||
        pidx >= PyTuple_GET_SIZE(PyTuple_GET_ITEM(pnames, oc)) || sax >= 8 || xax >= 8) {
      PyErr_SetString(PyExc_ValueError, "singleton_results: detail out of range");
      goto fail;
    }
    PyObject* sub = PyList_GET_ITEM(subs, b);
    PyObject* tmpl = PyObject_GetAttr(sub, s_template);
    if (!tmpl) goto fail;
    PyObject* scope = PySequence_GetItem(tmpl, 0);
    Py_DECREF(tmpl);
    if (!scope) goto fail;
    /* assignments: the one weight slot takes digit index % radix */
    PyObject* asg;
    if (rdx[b]) {
      PyObject* pair = PyTuple_Pack(2, scope, PyTuple_GET_ITEM(specs, (Py_ssize_t)(r.best_index % rdx[b])));
      asg = pair ? PyTuple_Pack(1, pair) : NULL;
      Py_XDECREF(pair);
    } else {
      asg = empty;
      Py_INCREF(asg);
    }
    PyObject* idx = PyLong_FromUnsignedLongLong(r.best_index);
    PyObject* plan = NULL;
    if (asg && idx) {
      PyObject* a[3] = {sub, asg, idx};
      plan = call_n(mkPlan, a, 3);
    }
    Py_XDECREF(asg);
    Py_XDECREF(idx);
    PyObject* obytes = PyLong_FromLongLong(obp[b]);
    PyObject* nr = NULL;
    if (plan && obytes) {
      PyObject* a[6] = {scope, PyTuple_GET_ITEM(PyTuple_GET_ITEM(pnames, oc), pidx), empty,
                        PyObject_IsTrue(PyTuple_GET_ITEM(PyTuple_GET_ITEM(pallred, oc), pidx)) ? allreduce : identity,
                        obytes, PyTuple_GET_ITEM(specs, sax < 0 ? 0 : 1 + sax)};
      nr = call_n(mkNR, a, 6);
    }
    PyObject* exits = NULL;
    if (nr) {
      if (xax >= 0) {
        PyObject* ex = PyTuple_Pack(3, scope, PyTuple_GET_ITEM(gather, xax), obytes);
        exits = ex ? PyTuple_Pack(1, ex) : NULL;
        Py_XDECREF(ex);
      } else {
        exits = empty;
        Py_INCREF(exits);
      }
    }
    Py_DECREF(scope);
    Py_XDECREF(obytes);
    PyObject* bbc = exits ? PyDict_New() : NULL;
    int ok = bbc != NULL;
    for (int j = 0; j < 4 && ok; j++)
      if (x.calls[j]) {
        PyObject* v = PyLong_FromLongLong(x.bytes[j]);
        ok = v && PyDict_SetItem(bbc, PyTuple_GET_ITEM(kinds, j), v) == 0;
        Py_XDECREF(v);
      }
    PyObject *fwd = PyFloat_FromDouble(x.forward_comm), *bwd = PyFloat_FromDouble(x.backward_comm),
             *cc = PyLong_FromLongLong(x.collective_calls), *fp = PyLong_FromLongLong(flp[b]);
    PyObject* cost = NULL;
    if (ok && fwd && bwd && cc && fp) {
      PyObject* a[6] = {fwd, bwd, py_overlap, bbc, cc, fp};
      cost = call_n(mkCR, a, 6);
    }
    Py_XDECREF(fwd);
    Py_XDECREF(bwd);
    Py_XDECREF(cc);
    Py_XDECREF(fp);
    Py_XDECREF(bbc);
    PyObject* routings = nr ? PyTuple_Pack(1, nr) : NULL;
    PyObject* rp = NULL;
    if (cost && routings) {
      PyObject* a[4] = {plan, routings, exits, cost};
      rp = call_n(mkRP, a, 4);
    }
    Py_XDECREF(plan);
    Py_XDECREF(nr);
    Py_XDECREF(routings);
    Py_XDECREF(exits);
    Py_XDECREF(cost);
    PyObject *cand = PyLong_FromUnsignedLongLong(r.candidates), *val = PyLong_FromUnsignedLongLong(r.valid),
             *table = PyList_New(0);
    PyObject* res = NULL;
    if (rp && cand && val && table) {
      PyObject* a[5] = {sub, rp, cand, val, table};
      res = call_n(mkRes, a, 5);
    }
    Py_XDECREF(rp);
    Py_XDECREF(cand);
    Py_XDECREF(val);
    Py_XDECREF(table);
    if (!res) goto fail;
    PyList_SET_ITEM(out, q, res);
  }
  goto fail0;
fail:
  Py_CLEAR(out);
fail0:
  Py_DECREF(py_overlap);
  Py_DECREF(empty);
done:
  PyBuffer_Release(&sel);
  PyBuffer_Release(&recs);
  PyBuffer_Release(&xb);
  PyBuffer_Release(&node);
  PyBuffer_Release(&toff);
  PyBuffer_Release(&op);
  PyBuffer_Release(&radix);
  PyBuffer_Release(&ob);
  PyBuffer_Release(&fl);
  return out;
}


/*
 * assignments_dict(names, key_ids, key_slot, slot_labels) -> dict
 * {names[key_ids[i]]: slot_labels[key_slot[i]]} in i order: derive_plan's
 * instance-scope -> label map (search.py:374-376) without materialising the
 * key and value lists; the scattered name objects are prefetched.
 *   key_ids int32 [K] (node rows), key_slot int32 [K] (index into slot_labels)
 */
static PyObject* assignments_dict(PyObject* self, PyObject* args) {
  PyObject *names, *labels;
  Py_buffer ids, slot;
  if (!PyArg_ParseTuple(args, "O!y*y*O!", &PyList_Type, &names, &ids, &slot, &PyList_Type, &labels)) return NULL;
  PyObject* d = NULL;
  const int32_t* I = (const int32_t*)ids.buf;
  const int32_t* Sl = (const int32_t*)slot.buf;
  const Py_ssize_t K = ids.len / 4, nn = PyList_GET_SIZE(names), nl = PyList_GET_SIZE(labels);
  if (slot.len / 4 != K) {
    PyErr_SetString(PyExc_ValueError, "key_ids and key_slot differ in length");
    goto done;
  }
  d = _PyDict_NewPresized(K);
  if (!d) goto done;
  enum { AHEAD = 24 };
  for (Py_ssize_t i = 0; i < K; i++) {
    if (i + AHEAD < K && I[i + AHEAD] >= 0 && I[i + AHEAD] < nn)
      __builtin_prefetch(PyList_GET_ITEM(names, I[i + AHEAD]), 1, 0);
    if (I[i] < 0 || I[i] >= nn || Sl[i] < 0 || Sl[i] >= nl) {
      PyErr_SetString(PyExc_IndexError, "assignments_dict: index out of range");
      Py_CLEAR(d);
      goto done;
    }
    PyObject* k = PyList_GET_ITEM(names, I[i]);
    Py_hash_t h;
    if (!PyUnicode_CheckExact(k) || (h = ((PyASCIIObject*)k)->hash) == -1) {
      h = PyObject_Hash(k);
      if (h == -1) {
        Py_CLEAR(d);
        goto done;
      }
    }
    if (_PyDict_SetItem_KnownHash(d, k, PyList_GET_ITEM(labels, Sl[i]), h) < 0) {
      Py_CLEAR(d);
      goto done;
    }
  }
done:
  PyBuffer_Release(&ids);
  PyBuffer_Release(&slot);
  return d;
}

/*
 * The same map in two halves, so the expensive one overlaps the device search:
 * assignments_keys(names, key_ids) -> (dict {names[key_ids[i]]: None} in i
 * order, bytes of the keys' hashes) touches every scattered key object once;
 * assignments_fill(d, names, key_ids, hashes, key_slot, slot_labels) then sets
 * the winners' labels with the saved hashes (the dict probe compares the key
 * pointers it already holds; the key objects are not read again).
 */
static PyObject* assignments_keys(PyObject* self, PyObject* args) {
  PyObject* names;
  Py_buffer ids;
  if (!PyArg_ParseTuple(args, "O!y*", &PyList_Type, &names, &ids)) return NULL;
  PyObject *d = NULL, *hb = NULL, *out = NULL;
  const int32_t* I = (const int32_t*)ids.buf;
  const Py_ssize_t K = ids.len / 4, nn = PyList_GET_SIZE(names);
  d = _PyDict_NewPresized(K);
  hb = PyBytes_FromStringAndSize(NULL, K * (Py_ssize_t)sizeof(Py_hash_t));
  if (!d || !hb) goto done;
  Py_hash_t* H = (Py_hash_t*)PyBytes_AS_STRING(hb);
  enum { AHEAD = 24 };
  for (Py_ssize_t i = 0; i < K; i++) {
    if (i + AHEAD < K && I[i + AHEAD] >= 0 && I[i + AHEAD] < nn)
      __builtin_prefetch(PyList_GET_ITEM(names, I[i + AHEAD]), 1, 0);
    if (I[i] < 0 || I[i] >= nn) {
      PyErr_SetString(PyExc_IndexError, "assignments_keys: index out of range");
      goto done;
    }
    PyObject* k = PyList_GET_ITEM(names, I[i]);
    Py_hash_t h;
    if (!PyUnicode_CheckExact(k) || (h = ((PyASCIIObject*)k)->hash) == -1) {
      h = PyObject_Hash(k);
      if (h == -1) goto done;
    }
    H[i] = h;
    if (_PyDict_SetItem_KnownHash(d, k, Py_None, h) < 0) goto done;
  }
  out = PyTuple_Pack(2, d, hb);
done:
  Py_XDECREF(d);
  Py_XDECREF(hb);
  PyBuffer_Release(&ids);
  return out;
}

/* The entry array of a combined-table dict (CPython 3.12 layout,
 * Include/internal/pycore_dict.h): assignments_keys inserted the K keys in
 * order with no deletion, so entry i holds key i.  assignments_fill writes the
 * values there directly when every entry's key is the expected key object
 * (pointer check per entry); anything else takes the probing path.  The dict
 * is still private to derive_plan (no watchers, not a namespace). */
#if PY_VERSION_HEX >= 0x030C0000 && PY_VERSION_HEX < 0x030D0000
#define DIRECT_FILL 1
typedef struct {
  Py_ssize_t dk_refcnt;
  uint8_t dk_log2_size;
  uint8_t dk_log2_index_bytes;
  uint8_t dk_kind;
  uint32_t dk_version;
  Py_ssize_t dk_usable;
  Py_ssize_t dk_nentries;
  char dk_indices[];
} DictKeys312;
typedef struct {
  PyObject* me_key;
  PyObject* me_value;
} DictUEntry312;
typedef struct {
  Py_hash_t me_hash;
  PyObject* me_key;
  PyObject* me_value;
} DictGEntry312;
#endif

static PyObject* assignments_fill(PyObject* self, PyObject* args) {
  PyObject *d, *names, *labels;
  Py_buffer ids, hashes, slot;
  if (!PyArg_ParseTuple(args, "O!O!y*y*y*O!", &PyDict_Type, &d, &PyList_Type, &names, &ids, &hashes, &slot,
                        &PyList_Type, &labels))
    return NULL;
  PyObject* ret = NULL;
  const int32_t* I = (const int32_t*)ids.buf;
  const int32_t* Sl = (const int32_t*)slot.buf;
  const Py_hash_t* H = (const Py_hash_t*)hashes.buf;
  const Py_ssize_t K = ids.len / 4, nn = PyList_GET_SIZE(names), nl = PyList_GET_SIZE(labels);
  if (slot.len / 4 != K || hashes.len / (Py_ssize_t)sizeof(Py_hash_t) != K) {
    PyErr_SetString(PyExc_ValueError, "assignments_fill: lengths differ");
    goto done;
  }
  Py_ssize_t i = 0;
#ifdef DIRECT_FILL
  {
    PyDictObject* mp = (PyDictObject*)d;
    DictKeys312* dk = (DictKeys312*)mp->ma_keys;
    if (PyDict_CheckExact(d) && mp->ma_values == NULL && mp->ma_used == K && dk->dk_nentries == K &&
        dk->dk_kind <= 1) {
      char* ent = dk->dk_indices + ((size_t)1 << dk->dk_log2_index_bytes);
      for (; i < K; i++) {
        if (I[i] < 0 || I[i] >= nn || Sl[i] < 0 || Sl[i] >= nl) break;
        PyObject* key = PyList_GET_ITEM(names, I[i]);
        PyObject** slot;
        if (dk->dk_kind == 1) {
          DictUEntry312* e = (DictUEntry312*)ent + i;
          if (e->me_key != key) break;
          slot = &e->me_value;
        } else {
          DictGEntry312* e = (DictGEntry312*)ent + i;
          if (e->me_key != key) break;
          slot = &e->me_value;
        }
        PyObject* v = PyList_GET_ITEM(labels, Sl[i]);
        Py_INCREF(v);
        PyObject* old = *slot;
        *slot = v;
        Py_XDECREF(old);
      }
    }
  }
#endif
  for (; i < K; i++) {
    if (I[i] < 0 || I[i] >= nn || Sl[i] < 0 || Sl[i] >= nl) {
      PyErr_SetString(PyExc_IndexError, "assignments_fill: index out of range");
      goto done;
    }
    if (_PyDict_SetItem_KnownHash(d, PyList_GET_ITEM(names, I[i]), PyList_GET_ITEM(labels, Sl[i]), H[i]) < 0)
      goto done;
  }
  ret = Py_NewRef(d);
done:
  PyBuffer_Release(&ids);
  PyBuffer_Release(&hashes);
  PyBuffer_Release(&slot);
  return ret;
}

/*
 * save_graph_json(topo_order, nodes, version, op_label, dtype_label, dumps) -> bytes
 *
 * The reference's save_graph (ir.py:358-367): every node of a ModelGraph in
 * topo_order (a GraphNode contributes its member RawNode, ir.py:363-364) as
 * _node_to_json (ir.py:342-355), the document {"nodes": [...], "version": v}
 * written exactly as json.dumps(doc, sort_keys=True, separators=(",", ":"))
 * + "\n", UTF-8.  Keys in sorted order: attrs, collective, device, inputs,
 * name, op, output, weight; tensor specs dtype, shape, trainable.  Strings are
 * escaped like json's ensure_ascii; attribute VALUES (arbitrary JSON) go
 * through `dumps` (json.dumps with the same options), enum labels through
 * op_label / dtype_label with pointer caches.
 */
typedef struct {
  char* p;
  Py_ssize_t n, cap;
} SBuf;

/* interned attribute names (module init) */
static PyObject *S_name, *S_op, *S_inputs, *S_output, *S_weight, *S_attrs, *S_member, *S_shape, *S_dtype,
    *S_trainable;

static int sb_grow(SBuf* b, Py_ssize_t need) {
  if (b->n + need <= b->cap) return 0;
  Py_ssize_t c = b->cap ? b->cap : 4096;
  while (c < b->n + need) c *= 2;
  char* q = (char*)PyMem_Realloc(b->p, (size_t)c);
  if (!q) {
    PyErr_NoMemory();
    return -1;
  }
  b->p = q;
  b->cap = c;
  return 0;
}
static int sb_put(SBuf* b, const char* s, Py_ssize_t len) {
  if (sb_grow(b, len) < 0) return -1;
  memcpy(b->p + b->n, s, (size_t)len);
  b->n += len;
  return 0;
}
#define SB_LIT(b, s) sb_put((b), (s), (Py_ssize_t)(sizeof(s) - 1))

/* a str as a JSON string literal, ensure_ascii escaping (json.encoder) */
static int sb_jstr(SBuf* b, PyObject* s) {
  if (!PyUnicode_Check(s)) {
    PyErr_SetString(PyExc_TypeError, "save_graph: expected str");
    return -1;
  }
  const Py_ssize_t L = PyUnicode_GET_LENGTH(s);
  const int kind = PyUnicode_KIND(s);
  const void* data = PyUnicode_DATA(s);
  if (sb_grow(b, L + 2) < 0) return -1;
  b->p[b->n++] = '"';
  static const char hex[] = "0123456789abcdef";
  for (Py_ssize_t i = 0; i < L; i++) {
    const Py_UCS4 c = PyUnicode_READ(kind, data, i);
    if (c >= 0x20 && c < 0x7f && c != '"' && c != '\\') {
      if (sb_grow(b, 1) < 0) return -1;
      b->p[b->n++] = (char)c;
      continue;
    }
    char e[12];
    int k = 0;
    switch (c) {
      case '"': e[k++] = '\\'; e[k++] = '"'; break;
      case '\\': e[k++] = '\\'; e[k++] = '\\'; break;
      case '\n': e[k++] = '\\'; e[k++] = 'n'; break;
      case '\r': e[k++] = '\\'; e[k++] = 'r'; break;
      case '\t': e[k++] = '\\'; e[k++] = 't'; break;
      case '\b': e[k++] = '\\'; e[k++] = 'b'; break;
      case '\f': e[k++] = '\\'; e[k++] = 'f'; break;
      default: {
        Py_UCS4 u = c;
        if (u >= 0x10000) {  /* surrogate pair */
          u -= 0x10000;
          const Py_UCS4 hi = 0xd800 | ((u >> 10) & 0x3ff), lo = 0xdc00 | (u & 0x3ff);
          const Py_UCS4 pr[2] = {hi, lo};
          for (int t = 0; t < 2; t++) {
            e[k++] = '\\'; e[k++] = 'u';
            for (int sh = 12; sh >= 0; sh -= 4) e[k++] = hex[(pr[t] >> sh) & 0xf];
          }
        } else {
          e[k++] = '\\'; e[k++] = 'u';
          for (int sh = 12; sh >= 0; sh -= 4) e[k++] = hex[(u >> sh) & 0xf];
        }
      }
    }
    if (sb_put(b, e, k) < 0) return -1;
  }
  if (sb_grow(b, 1) < 0) return -1;
  b->p[b->n++] = '"';
  return 0;
}

/* str(o) appended verbatim (ints, the `dumps` results) */
static int sb_str_of(SBuf* b, PyObject* o) {
  PyObject* s = PyObject_Str(o);
  if (!s) return -1;
  Py_ssize_t len;
  const char* u = PyUnicode_AsUTF8AndSize(s, &len);
  const int rc = u ? sb_put(b, u, len) : -1;
  Py_DECREF(s);
  return rc;
}

/* a JSON value as json.dumps(v, sort_keys=True, separators=(",", ":")) writes it;
 * types outside the plain JSON ones (and dicts with non-str keys) through `dumps` */
static int sb_json(SBuf* b, PyObject* v, PyObject* dumps, int depth) {
  if (v == Py_None) return SB_LIT(b, "null");
  if (v == Py_True) return SB_LIT(b, "true");
  if (v == Py_False) return SB_LIT(b, "false");
  if (PyLong_CheckExact(v)) return sb_str_of(b, v);
  if (PyUnicode_CheckExact(v)) return sb_jstr(b, v);
  if (PyFloat_CheckExact(v)) {
    const double x = PyFloat_AS_DOUBLE(v);
    if (x != x) return SB_LIT(b, "NaN");
    if (x == Py_HUGE_VAL) return SB_LIT(b, "Infinity");
    if (x == -Py_HUGE_VAL) return SB_LIT(b, "-Infinity");
    PyObject* r = PyObject_Repr(v);  /* float.__repr__, as json's encoder */
    if (!r) return -1;
    const int rc = sb_str_of(b, r);
    Py_DECREF(r);
    return rc;
  }
  if (depth < 64 && (PyList_CheckExact(v) || PyTuple_CheckExact(v))) {
    PyObject* seq = PySequence_Fast(v, "");
    if (!seq) return -1;
    int rc = SB_LIT(b, "[");
    for (Py_ssize_t i = 0; rc == 0 && i < PySequence_Fast_GET_SIZE(seq); i++) {
      if (i) rc = SB_LIT(b, ",");
      if (rc == 0) rc = sb_json(b, PySequence_Fast_GET_ITEM(seq, i), dumps, depth + 1);
    }
    Py_DECREF(seq);
    return rc ? rc : SB_LIT(b, "]");
  }
  if (depth < 64 && PyDict_CheckExact(v)) {
    PyObject* keys = PyDict_Keys(v);
    if (!keys) return -1;
    int plain = 1;
    for (Py_ssize_t i = 0; i < PyList_GET_SIZE(keys); i++) plain = plain && PyUnicode_CheckExact(PyList_GET_ITEM(keys, i));
    if (plain && PyList_Sort(keys) == 0) {
      int rc = SB_LIT(b, "{");
      for (Py_ssize_t i = 0; rc == 0 && i < PyList_GET_SIZE(keys); i++) {
        PyObject* k = PyList_GET_ITEM(keys, i);
        if (i) rc = SB_LIT(b, ",");
        if (rc == 0) rc = sb_jstr(b, k);
        if (rc == 0) rc = SB_LIT(b, ":");
        if (rc == 0) rc = sb_json(b, PyDict_GetItem(v, k), dumps, depth + 1);
      }
      Py_DECREF(keys);
      return rc ? rc : SB_LIT(b, "}");
    }
    Py_DECREF(keys);
    if (PyErr_Occurred()) return -1;
  }
  PyObject* js = PyObject_CallOneArg(dumps, v);
  if (!js) return -1;
  const int rc = sb_str_of(b, js);
  Py_DECREF(js);
  return rc;
}

static int sb_label(SBuf* b, PtrCache* cache, PyObject* enum_val, PyObject* fn) {
  /* label strings through the cache's Python call (value cached as a str object pointer) */
  for (int i = 0; i < cache->n; i++)
    if (cache->key[i] == enum_val) return sb_jstr(b, (PyObject*)cache->val[i]);
  PyObject* r = PyObject_CallOneArg(fn, enum_val);
  if (!r) return -1;
  const int rc = sb_jstr(b, r);
  if (cache->n < CACHE_N) {
    Py_INCREF(enum_val);
    cache->key[cache->n] = enum_val;
    cache->val[cache->n] = (long)r;  /* owns the reference */
    cache->n++;
  } else {
    Py_DECREF(r);
  }
  return rc;
}

static void label_cache_clear(PtrCache* c) {
  for (int i = 0; i < c->n; i++) {
    Py_DECREF(c->key[i]);
    Py_DECREF((PyObject*)c->val[i]);
  }
  c->n = 0;
}

static int sb_spec(SBuf* b, PyObject* spec, PtrCache* dcache, PyObject* dtype_label) {
  PyObject *shape = PyObject_GetAttr(spec, S_shape), *dt = PyObject_GetAttr(spec, S_dtype),
           *tr = PyObject_GetAttr(spec, S_trainable);
  int rc = -1;
  if (!shape || !dt || !tr) goto done;
  if (SB_LIT(b, "{\"dtype\":") < 0 || sb_label(b, dcache, dt, dtype_label) < 0 || SB_LIT(b, ",\"shape\":[") < 0)
    goto done;
  {
    PyObject* seq = PySequence_Fast(shape, "shape must be a sequence");
    if (!seq) goto done;
    const Py_ssize_t r = PySequence_Fast_GET_SIZE(seq);
    for (Py_ssize_t i = 0; i < r; i++) {
      if ((i && SB_LIT(b, ",") < 0) || sb_str_of(b, PySequence_Fast_GET_ITEM(seq, i)) < 0) {
        Py_DECREF(seq);
        goto done;
      }
    }
    Py_DECREF(seq);
  }
  {
    const int t = PyObject_IsTrue(tr);
    if (t < 0) goto done;
    if ((t ? SB_LIT(b, "],\"trainable\":true}") : SB_LIT(b, "],\"trainable\":false}")) < 0) goto done;
  }
  rc = 0;
done:
  Py_XDECREF(shape);
  Py_XDECREF(dt);
  Py_XDECREF(tr);
  return rc;
}

static PyObject* save_graph_json(PyObject* self, PyObject* args) {
  PyObject *topo, *nodes, *op_label, *dtype_label, *dumps;
  long version;
  if (!PyArg_ParseTuple(args, "OO!lOOO", &topo, &PyDict_Type, &nodes, &version, &op_label, &dtype_label, &dumps))
    return NULL;
  PyObject* seq = PySequence_Fast(topo, "topo_order must be a sequence");
  if (!seq) return NULL;
  SBuf b = {NULL, 0, 0};
  PtrCache ocache = {{0}, {0}, 0}, dcache = {{0}, {0}, 0};
  PyObject* out = NULL;
  const Py_ssize_t N = PySequence_Fast_GET_SIZE(seq);
  if (SB_LIT(&b, "{\"nodes\":[") < 0) goto done;
  for (Py_ssize_t i = 0; i < N; i++) {
    PyObject* name = PySequence_Fast_GET_ITEM(seq, i);
    PyObject* node = PyDict_GetItemWithError(nodes, name);
    if (!node) {
      if (!PyErr_Occurred()) PyErr_SetObject(PyExc_KeyError, name);
      goto done;
    }
    Py_INCREF(node);
    if (PyObject_HasAttr(node, S_member)) {  /* GraphNode -> its member RawNode */
      PyObject* m = PyObject_GetAttr(node, S_member);
      Py_DECREF(node);
      if (!m) goto done;
      node = m;
    }
    PyObject *nm = PyObject_GetAttr(node, S_name), *op = PyObject_GetAttr(node, S_op),
             *ins = PyObject_GetAttr(node, S_inputs), *outp = PyObject_GetAttr(node, S_output),
             *w = PyObject_GetAttr(node, S_weight), *attrs = PyObject_GetAttr(node, S_attrs);
    int ok = nm && op && ins && outp && w && attrs;
    PyObject *dev = NULL, *coll = NULL, *attr_seq = NULL;
    if (ok && (i ? SB_LIT(&b, ",{") : SB_LIT(&b, "{")) < 0) ok = 0;
    if (ok) {
      attr_seq = PySequence_Fast(attrs, "attrs must be a sequence");
      if (!attr_seq) ok = 0;
    }
    if (ok) {
      /* "attrs": the non device/collective pairs in their (sorted) order, values via dumps */
      const Py_ssize_t na = PySequence_Fast_GET_SIZE(attr_seq);
      int first = 1;
      for (Py_ssize_t a = 0; a < na && ok; a++) {
        PyObject* kv = PySequence_Fast_GET_ITEM(attr_seq, a);
        PyObject *k = PySequence_GetItem(kv, 0), *v = PySequence_GetItem(kv, 1);
        if (!k || !v) {
          ok = 0;
        } else if (PyUnicode_Check(k) && (PyUnicode_CompareWithASCIIString(k, "device") == 0 ||
                                          PyUnicode_CompareWithASCIIString(k, "collective") == 0)) {
          /* the last pair of a key wins, as the dict literal of _node_to_json does */
          PyObject** slot = PyUnicode_CompareWithASCIIString(k, "device") == 0 ? &dev : &coll;
          Py_XDECREF(*slot);
          *slot = Py_NewRef(v);
        } else {
          (void)first;
        }
        Py_XDECREF(k);
        Py_XDECREF(v);
      }
      /* the reference builds {k: v} (later duplicates win, first position kept) and
       * sort_keys orders it: delegate the attrs object to dumps when there is one */
      if (ok) {
        PyObject* d = PyDict_New();
        if (!d) ok = 0;
        for (Py_ssize_t a = 0; a < na && ok; a++) {
          PyObject* kv = PySequence_Fast_GET_ITEM(attr_seq, a);
          PyObject *k = PySequence_GetItem(kv, 0), *v = PySequence_GetItem(kv, 1);
          if (!k || !v) ok = 0;
          else if (!(PyUnicode_Check(k) && (PyUnicode_CompareWithASCIIString(k, "device") == 0 ||
                                             PyUnicode_CompareWithASCIIString(k, "collective") == 0)))
            ok = PyDict_SetItem(d, k, v) == 0;
          Py_XDECREF(k);
          Py_XDECREF(v);
        }
        if (ok && PyDict_GET_SIZE(d))
          ok = SB_LIT(&b, "\"attrs\":") == 0 && sb_json(&b, d, dumps, 0) == 0 && SB_LIT(&b, ",") == 0;
        Py_XDECREF(d);
      }
    }
    if (ok && coll) ok = SB_LIT(&b, "\"collective\":") == 0 && sb_json(&b, coll, dumps, 0) == 0 && SB_LIT(&b, ",") == 0;
    if (ok && dev) ok = SB_LIT(&b, "\"device\":") == 0 && sb_json(&b, dev, dumps, 0) == 0 && SB_LIT(&b, ",") == 0;
    if (ok) {
      ok = SB_LIT(&b, "\"inputs\":[") == 0;
      PyObject* iseq = ok ? PySequence_Fast(ins, "inputs must be a sequence") : NULL;
      if (!iseq) ok = 0;
      for (Py_ssize_t k = 0; ok && k < PySequence_Fast_GET_SIZE(iseq); k++)
        ok = (!k || SB_LIT(&b, ",") == 0) && sb_jstr(&b, PySequence_Fast_GET_ITEM(iseq, k)) == 0;
      Py_XDECREF(iseq);
    }
    ok = ok && SB_LIT(&b, "],\"name\":") == 0 && sb_jstr(&b, nm) == 0 && SB_LIT(&b, ",\"op\":") == 0 &&
         sb_label(&b, &ocache, op, op_label) == 0 && SB_LIT(&b, ",\"output\":") == 0 &&
         sb_spec(&b, outp, &dcache, dtype_label) == 0 && SB_LIT(&b, ",\"weight\":") == 0;
    if (ok) {
      const int has_w = w != Py_None ? PyObject_IsTrue(w) : 0;  /* `if node.weight` */
      if (has_w < 0) ok = 0;
      else if (has_w) ok = sb_spec(&b, w, &dcache, dtype_label) == 0;
      else ok = SB_LIT(&b, "null") == 0;
    }
    ok = ok && SB_LIT(&b, "}") == 0;
    Py_XDECREF(nm);
    Py_XDECREF(op);
    Py_XDECREF(ins);
    Py_XDECREF(outp);
    Py_XDECREF(w);
    Py_XDECREF(attrs);
    Py_XDECREF(attr_seq);
    Py_XDECREF(dev);
    Py_XDECREF(coll);
    Py_DECREF(node);
    if (!ok) goto done;
  }
  {
    char tail[64];
    const int k = snprintf(tail, sizeof tail, "],\"version\":%ld}\n", version);
    if (sb_put(&b, tail, k) < 0) goto done;
  }
  out = PyBytes_FromStringAndSize(b.p, b.n);
done:
  label_cache_clear(&ocache);
  label_cache_clear(&dcache);
  PyMem_Free(b.p);
  Py_DECREF(seq);
  return out;
}

/*
 * slot_positions(names, toff, tnodes, w_rank) -> (slot_off, slot_pos, radix) as bytes
 *   slot_off int64 [nb + 1], slot_pos int32 [S], radix uint8 [S]
 * Per block: the template positions of its nodes with a weight in weight_nodes
 * order (the scopes sorted by name, search.py:85-88) and their option counts
 * (_options, search.py:91-93: 3 for a weight of rank >= 2, else 2).
 */
static PyObject* slot_positions(PyObject* self, PyObject* args) {
  PyObject* names;
  Py_buffer toff, tn, wr;
  if (!PyArg_ParseTuple(args, "O!y*y*y*", &PyList_Type, &names, &toff, &tn, &wr)) return NULL;
  PyObject *bo = NULL, *bp = NULL, *br = NULL, *out = NULL;
  const int64_t* to = (const int64_t*)toff.buf;
  const int32_t* T = (const int32_t*)tn.buf;
  const uint8_t* W = (const uint8_t*)wr.buf;
  const Py_ssize_t nb = toff.len / 8 - 1, ne = tn.len / 4, nn = PyList_GET_SIZE(names);
  if (nb < 0 || wr.len < nn || (nb >= 0 && (to[0] != 0 || to[nb] > ne))) {
    PyErr_SetString(PyExc_ValueError, "slot_positions: inconsistent arguments");
    goto done;
  }
  Py_ssize_t S = 0;
  for (Py_ssize_t e = 0; e < to[nb]; e++) {
    if (T[e] < 0 || T[e] >= nn) {
      PyErr_SetString(PyExc_IndexError, "slot_positions: node out of range");
      goto done;
    }
    S += W[T[e]] != 0;
  }
  bo = PyBytes_FromStringAndSize(NULL, (nb + 1) * 8);
  bp = PyBytes_FromStringAndSize(NULL, S * 4);
  br = PyBytes_FromStringAndSize(NULL, S);
  if (!bo || !bp || !br) goto done;
  int64_t* so = (int64_t*)PyBytes_AS_STRING(bo);
  int32_t* sp = (int32_t*)PyBytes_AS_STRING(bp);
  uint8_t* rx = (uint8_t*)PyBytes_AS_STRING(br);
  Py_ssize_t k = 0;
  so[0] = 0;
  for (Py_ssize_t b = 0; b < nb; b++) {
    const Py_ssize_t k0 = k;
    for (int64_t e = to[b]; e < to[b + 1]; e++) {
      const int32_t v = T[e];
      if (!W[v]) continue;
      /* insertion by name (str order); names within a template are distinct */
      PyObject* nv = PyList_GET_ITEM(names, v);
      Py_ssize_t j = k;
      while (j > k0) {
        const int c = PyUnicode_Compare(PyList_GET_ITEM(names, T[to[b] + sp[j - 1]]), nv);
        if (c == -1 && PyErr_Occurred()) goto done;
        if (c <= 0) break;
        sp[j] = sp[j - 1];
        rx[j] = rx[j - 1];
        j--;
      }
      sp[j] = (int32_t)(e - to[b]);
      rx[j] = W[v] >= 2 ? 3 : 2;
      k++;
    }
    so[b + 1] = k;
  }
  out = PyTuple_Pack(3, bo, bp, br);
done:
  Py_XDECREF(bo);
  Py_XDECREF(bp);
  Py_XDECREF(br);
  PyBuffer_Release(&toff);
  PyBuffer_Release(&tn);
  PyBuffer_Release(&wr);
  return out;
}

/* flops of one template (costmodel.py:185-190): 2 x the activation's elements x
 * the weight's first dim, summed over matmuls (op 0) with a weight; Python
 * integers when the sum leaves int64 */
static PyObject* template_flops(const int32_t* tn, int64_t T, const uint8_t* op, const uint8_t* ar, const int64_t* as,
                                Py_ssize_t aw, const uint8_t* wr, const int64_t* ws, Py_ssize_t ww) {
  int64_t acc = 0;
  int over = 0;
  for (int64_t t = 0; t < T && !over; t++) {
    const int32_t v = tn[t];
    if (op[v] != 0 || !wr[v]) continue;
    int64_t x = 2;
    for (int d = 0; d < ar[v] && !over; d++) over = __builtin_mul_overflow(x, as[(int64_t)v * aw + d], &x);
    if (!over) over = __builtin_mul_overflow(x, ws[(int64_t)v * ww], &x);
    if (!over) over = __builtin_add_overflow(acc, x, &acc);
  }
  if (!over) return PyLong_FromLongLong(acc);
  PyObject* sum = PyLong_FromLong(0);
  for (int64_t t = 0; t < T && sum; t++) {
    const int32_t v = tn[t];
    if (op[v] != 0 || !wr[v]) continue;
    PyObject* x = PyLong_FromLong(2);
    for (int d = 0; d <= ar[v] && x; d++) {
      PyObject* f = PyLong_FromLongLong(d < ar[v] ? as[(int64_t)v * aw + d] : ws[(int64_t)v * ww]);
      PyObject* y = f ? PyNumber_Multiply(x, f) : NULL;
      Py_XDECREF(f);
      Py_DECREF(x);
      x = y;
    }
    PyObject* s2 = x ? PyNumber_Add(sum, x) : NULL;
    Py_XDECREF(x);
    Py_DECREF(sum);
    sum = s2;
  }
  return sum;
}

/*
 * block_results(ctors, subs, names, graph, blocks, recs, xblocks, node, edge, eoff,
 *               pnames, pallred, specs, labels, identity, allreduce, colls, kinds, overlap)
 *   -> (results, terms, slot_labels)
 * The SubgraphResult of every block's winner (search.py:317-345) built from the
 * raw score and winner-detail records -- routed_plans_all in C for blocks of any
 * size: CandidatePlan (assignments in weight_nodes order, digits of the
 * winner's reference index), NodeRouting per template node (pattern, internal
 * producers' conversions in GraphNode.inputs order, output collective, state),
 * exit conversions, CostReport (+ flops).  None for a block without a winner,
 * whose winner did not route, or whose explained total differs from the scored
 * one: the Python path handles (and raises for) those.  terms[b] = the block's
 * cost x multiplicity (search.py:373), slot_labels[b] = its weight labels in
 * weight_nodes order (search.py:374-376), None where results[b] is None.
 *   graph: (op u8[n], act_rank u8[n], act_shape i64[n, aw], aw, w_rank u8[n],
 *           w_shape i64[n, ww], ww, act_bytes i64[n], in_off i64[n+1], in_idx i32[m])
 *   blocks: (toff i64[nb+1], tnodes i32[ne], slot_off i64[nb+1], slot_pos i32[S],
 *            radix u8[S], inst_off i64[nb+1])
 *   recs: sp_score_out [nb]; xblocks: sp_explain_block [nb]; node: int8 [ne, 4];
 *   edge: int8 [nedge, 2]; eoff: int64 [nb + 1]
 *   specs / labels: (replica, split(0), ..., split(7)) and their labels;
 *   colls: 4 tuples (allreduce, allgather, reducescatter, alltoall) of 8 Collectives (by axis)
 */
static PyObject* block_results(PyObject* self, PyObject* args) {
  PyObject *ctors, *subs, *names, *pnames, *pallred, *specs, *labels, *identity, *allreduce, *colls, *kinds;
  Py_buffer op, ar, as, wr, ws, ab, ino, ini, to_, tn_, so_, sp_, rx_, io_, recs, xb, node, edge, eo;
  Py_ssize_t aw, ww;
  double overlap;
  if (!PyArg_ParseTuple(args, "O!O!O!(y*y*y*ny*y*ny*y*y*)(y*y*y*y*y*y*)y*y*y*y*y*O!O!O!O!OOO!O!d", &PyTuple_Type,
                        &ctors, &PyList_Type, &subs, &PyList_Type, &names, &op, &ar, &as, &aw, &wr, &ws, &ww, &ab,
                        &ino, &ini, &to_, &tn_, &so_, &sp_, &rx_, &io_, &recs, &xb, &node, &edge, &eo, &PyTuple_Type,
                        &pnames, &PyTuple_Type, &pallred, &PyTuple_Type, &specs, &PyTuple_Type, &labels, &identity,
                        &allreduce, &PyTuple_Type, &colls, &PyTuple_Type, &kinds, &overlap))
    return NULL;
  PyObject *res_l = NULL, *terms = NULL, *labs = NULL, *out = NULL, *py_overlap = NULL, *empty = NULL;
  int32_t* pos_of = NULL;
  static PyObject* s_template = NULL;
  if (!s_template) s_template = PyUnicode_InternFromString("template");
  const uint8_t* OP = (const uint8_t*)op.buf;
  const uint8_t* AR = (const uint8_t*)ar.buf;
  const int64_t* AS = (const int64_t*)as.buf;
  const uint8_t* WR = (const uint8_t*)wr.buf;
  const int64_t* WS = (const int64_t*)ws.buf;
  const int64_t* AB = (const int64_t*)ab.buf;
  const int64_t* INO = (const int64_t*)ino.buf;
  const int32_t* INI = (const int32_t*)ini.buf;
  const int64_t* TO = (const int64_t*)to_.buf;
  const int32_t* TN = (const int32_t*)tn_.buf;
  const int64_t* SO = (const int64_t*)so_.buf;
  const int32_t* SP = (const int32_t*)sp_.buf;
  const uint8_t* RX = (const uint8_t*)rx_.buf;
  const int64_t* IO = (const int64_t*)io_.buf;
  const RecView* R = (const RecView*)recs.buf;
  const XView* X = (const XView*)xb.buf;
  const int8_t* ND = (const int8_t*)node.buf;
  const int8_t* ED = (const int8_t*)edge.buf;
  const int64_t* EO = (const int64_t*)eo.buf;
  const Py_ssize_t n = op.len, nb = PyList_GET_SIZE(subs), nn = PyList_GET_SIZE(names);
  const Py_ssize_t nedge = edge.len / 2, ne = tn_.len / 4, nin = ini.len / 4;
  int ok = n == nn && ar.len >= n && wr.len >= n && aw >= 1 && ww >= 1 && as.len >= n * aw * 8 &&
           ws.len >= n * ww * 8 && ab.len >= n * 8 && ino.len >= (n + 1) * 8 && to_.len >= (nb + 1) * 8 &&
           so_.len >= (nb + 1) * 8 && io_.len >= (nb + 1) * 8 && eo.len >= (nb + 1) * 8 &&
           recs.len >= nb * (Py_ssize_t)sizeof(RecView) && xb.len >= nb * (Py_ssize_t)sizeof(XView) &&
           PyTuple_GET_SIZE(ctors) == 5 && PyTuple_GET_SIZE(specs) >= 9 && PyTuple_GET_SIZE(labels) >= 9 &&
           PyTuple_GET_SIZE(colls) == 4 && PyTuple_GET_SIZE(kinds) == 4;
  for (int j = 0; ok && j < 4; j++)
    ok = PyTuple_Check(PyTuple_GET_ITEM(colls, j)) && PyTuple_GET_SIZE(PyTuple_GET_ITEM(colls, j)) >= 8;
  if (ok) ok = TO[nb] <= ne && node.len >= TO[nb] * 4 && SO[nb] * 4 <= sp_.len && SO[nb] <= rx_.len &&
               EO[nb] <= nedge && INO[n] <= nin;
  if (!ok) {
    PyErr_SetString(PyExc_ValueError, "block_results: inconsistent arguments");
    goto done;
  }
  PyObject *mkPlan = PyTuple_GET_ITEM(ctors, 0), *mkNR = PyTuple_GET_ITEM(ctors, 1),
           *mkRP = PyTuple_GET_ITEM(ctors, 2), *mkCR = PyTuple_GET_ITEM(ctors, 3),
           *mkRes = PyTuple_GET_ITEM(ctors, 4);
  py_overlap = PyFloat_FromDouble(overlap);
  empty = PyTuple_New(0);
  res_l = PyList_New(nb);
  terms = PyList_New(nb);
  labs = PyList_New(nb);
  pos_of = (int32_t*)PyMem_Malloc((n > 0 ? n : 1) * sizeof(int32_t));
  if (!py_overlap || !empty || !res_l || !terms || !labs || !pos_of) {
    if (!pos_of) PyErr_NoMemory();
    goto fail;
  }
  for (Py_ssize_t v = 0; v < n; v++) pos_of[v] = -1;
  for (Py_ssize_t b = 0; b < nb; b++) {
    const RecView r = R[b];
    const XView x = X[b];
    /* CostReport.total = forward + backward * (1 - overlap), rounded in that order */
    const double total = x.forward_comm + x.backward_comm * (1.0 - overlap);
    if (!r.has_best || !x.valid || (r.best_total == r.best_total && total != r.best_total)) {
      PyList_SET_ITEM(res_l, b, Py_NewRef(Py_None));
      PyList_SET_ITEM(terms, b, Py_NewRef(Py_None));
      PyList_SET_ITEM(labs, b, Py_NewRef(Py_None));
      continue;
    }
    const int64_t e0 = TO[b], T = TO[b + 1] - TO[b];
    PyObject* sub = PyList_GET_ITEM(subs, b);
    PyObject* tmpl = PyObject_GetAttr(sub, s_template);
    if (!tmpl) goto fail;
    if (!PyTuple_Check(tmpl) || PyTuple_GET_SIZE(tmpl) != T) {
      Py_DECREF(tmpl);
      PyErr_SetString(PyExc_ValueError, "block_results: template size differs from the tables");
      goto fail;
    }
    /* assignments in weight_nodes order: digits of the winner's reference index,
       the last slot fastest (candidate_by_index, search.py:103-116) */
    const int64_t s0 = SO[b], S = SO[b + 1] - SO[b];
    PyObject* asg = PyTuple_New(S);
    PyObject* lab = PyList_New(S);
    if (!asg || !lab) {
      Py_XDECREF(asg);
      Py_XDECREF(lab);
      Py_DECREF(tmpl);
      goto fail;
    }
    {
      uint64_t rem = r.best_index;
      for (int64_t k = S - 1; k >= 0; k--) {
        const int rdx = RX[s0 + k] ? RX[s0 + k] : 2;
        const int d = (int)(rem % (uint64_t)rdx);
        rem /= (uint64_t)rdx;
        const int32_t q = SP[s0 + k];
        PyObject* pair = (q >= 0 && q < T) ? PyTuple_Pack(2, PyTuple_GET_ITEM(tmpl, q), PyTuple_GET_ITEM(specs, d))
                                           : NULL;
        if (!pair) {
          if (!PyErr_Occurred()) PyErr_SetString(PyExc_IndexError, "block_results: slot out of range");
          Py_DECREF(asg);
          Py_DECREF(lab);
          Py_DECREF(tmpl);
          goto fail;
        }
        PyTuple_SET_ITEM(asg, k, pair);
        PyList_SET_ITEM(lab, k, Py_NewRef(PyTuple_GET_ITEM(labels, d)));
      }
    }
    PyObject* idx = PyLong_FromUnsignedLongLong(r.best_index);
    PyObject* plan = NULL;
    if (idx) {
      PyObject* a[3] = {sub, asg, idx};
      plan = call_n(mkPlan, a, 3);
    }
    Py_XDECREF(idx);
    Py_DECREF(asg);
    PyObject* routings = plan ? PyTuple_New(T) : NULL;
    PyObject* exits = routings ? PyList_New(0) : NULL;
    int bad = !exits;
    for (int64_t t = 0; t < T; t++) {
      if (TN[e0 + t] < 0 || TN[e0 + t] >= n) {
        PyErr_SetString(PyExc_IndexError, "block_results: node out of range");
        bad = 1;
        break;
      }
      pos_of[TN[e0 + t]] = (int32_t)t;
    }
    int64_t k = EO[b];
    for (int64_t i = 0; i < T && !bad; i++) {
      const int32_t v = TN[e0 + i];
      PyObject* scope = PyTuple_GET_ITEM(tmpl, i);
      const int oc = OP[v];
      const int pidx = ND[4 * (e0 + i)], sax = ND[4 * (e0 + i) + 1], xax = ND[4 * (e0 + i) + 2];
      if (oc >= PyTuple_GET_SIZE(pnames) || oc >= PyTuple_GET_SIZE(pallred) || pidx < 0 ||
          pidx >= PyTuple_GET_SIZE(PyTuple_GET_ITEM(pnames, oc)) || sax >= 8 || xax >= 8) {
        PyErr_SetString(PyExc_ValueError, "block_results: detail out of range");
        bad = 1;
        break;
      }
      PyObject* convs = PyList_New(0);
      if (!convs) {
        bad = 1;
        break;
      }
      for (int64_t e = INO[v]; e < INO[v + 1] && !bad; e++) {
        const int32_t p = INI[e];
        if (p < 0 || p >= n || pos_of[p] < 0) continue;  /* not a member of this template */
        if (k >= EO[b + 1]) {
          PyErr_SetString(PyExc_ValueError, "block_results: more internal edges than the detail holds");
          bad = 1;
          break;
        }
        const int kind = ED[2 * k], axis = ED[2 * k + 1];
        k++;
        if (!kind) continue;
        if (kind < 1 || kind > 4 || (kind > 1 && (axis < 0 || axis >= 8))) {
          PyErr_SetString(PyExc_ValueError, "block_results: edge detail out of range");
          bad = 1;
          break;
        }
        PyObject* pb = PyLong_FromLongLong(AB[p]);
        PyObject* c = pb ? PyTuple_Pack(3, PyList_GET_ITEM(names, p),
                                        PyTuple_GET_ITEM(PyTuple_GET_ITEM(colls, kind - 1), kind == 1 ? 0 : axis), pb)
                         : NULL;
        Py_XDECREF(pb);
        if (!c || PyList_Append(convs, c) < 0) bad = 1;
        Py_XDECREF(c);
      }
      PyObject* ct = bad ? NULL : PyList_AsTuple(convs);
      Py_DECREF(convs);
      PyObject* obytes = ct ? PyLong_FromLongLong(AB[v]) : NULL;
      PyObject* nr = NULL;
      if (obytes) {
        const int ar_ = PyObject_IsTrue(PyTuple_GET_ITEM(PyTuple_GET_ITEM(pallred, oc), pidx));
        PyObject* a[6] = {scope, PyTuple_GET_ITEM(PyTuple_GET_ITEM(pnames, oc), pidx), ct,
                          ar_ ? allreduce : identity, obytes, PyTuple_GET_ITEM(specs, sax < 0 ? 0 : 1 + sax)};
        nr = call_n(mkNR, a, 6);
      }
      Py_XDECREF(ct);
      if (!nr) {
        Py_XDECREF(obytes);
        bad = 1;
        break;
      }
      PyTuple_SET_ITEM(routings, i, nr);
      if (xax >= 0) {
        PyObject* ex = PyTuple_Pack(3, scope, PyTuple_GET_ITEM(PyTuple_GET_ITEM(colls, 1), xax), obytes);
        if (!ex || PyList_Append(exits, ex) < 0) bad = 1;
        Py_XDECREF(ex);
      }
      Py_DECREF(obytes);
    }
    for (int64_t t = 0; t < T; t++)
      if (TN[e0 + t] >= 0 && TN[e0 + t] < n) pos_of[TN[e0 + t]] = -1;
    if (!bad && k != EO[b + 1]) {
      PyErr_SetString(PyExc_ValueError, "block_results: internal edges differ from the detail");
      bad = 1;
    }
    Py_DECREF(tmpl);
    PyObject* exits_t = bad ? NULL : PyList_AsTuple(exits);
    Py_XDECREF(exits);
    PyObject* bbc = exits_t ? PyDict_New() : NULL;
    int okd = bbc != NULL;
    for (int j = 0; j < 4 && okd; j++)
      if (x.calls[j]) {
        PyObject* v = PyLong_FromLongLong(x.bytes[j]);
        okd = v && PyDict_SetItem(bbc, PyTuple_GET_ITEM(kinds, j), v) == 0;
        Py_XDECREF(v);
      }
    PyObject *fwd = PyFloat_FromDouble(x.forward_comm), *bwd = PyFloat_FromDouble(x.backward_comm),
             *cc = PyLong_FromLongLong(x.collective_calls),
             *fp = okd ? template_flops(TN + e0, T, OP, AR, AS, aw, WR, WS, ww) : NULL;
    PyObject* cost = NULL;
    if (okd && fwd && bwd && cc && fp) {
      PyObject* a[6] = {fwd, bwd, py_overlap, bbc, cc, fp};
      cost = call_n(mkCR, a, 6);
    }
    Py_XDECREF(fwd);
    Py_XDECREF(bwd);
    Py_XDECREF(cc);
    Py_XDECREF(fp);
    Py_XDECREF(bbc);
    PyObject* rp = NULL;
    if (cost) {
      PyObject* a[4] = {plan, routings, exits_t, cost};
      rp = call_n(mkRP, a, 4);
    }
    Py_XDECREF(plan);
    Py_XDECREF(routings);
    Py_XDECREF(exits_t);
    Py_XDECREF(cost);
    PyObject *cand = PyLong_FromUnsignedLongLong(r.candidates), *val = PyLong_FromUnsignedLongLong(r.valid),
             *table = PyList_New(0);
    PyObject* res = NULL;
    if (rp && cand && val && table) {
      PyObject* a[5] = {sub, rp, cand, val, table};
      res = call_n(mkRes, a, 5);
    }
    Py_XDECREF(rp);
    Py_XDECREF(cand);
    Py_XDECREF(val);
    Py_XDECREF(table);
    PyObject* term = res ? PyFloat_FromDouble(total * (double)(IO[b + 1] - IO[b])) : NULL;
    if (!term) {
      Py_XDECREF(res);
      Py_DECREF(lab);
      goto fail;
    }
    PyList_SET_ITEM(res_l, b, res);
    PyList_SET_ITEM(terms, b, term);
    PyList_SET_ITEM(labs, b, lab);
  }
  out = PyTuple_Pack(3, res_l, terms, labs);
fail:
  Py_XDECREF(res_l);
  Py_XDECREF(terms);
  Py_XDECREF(labs);
  Py_XDECREF(py_overlap);
  Py_XDECREF(empty);
  PyMem_Free(pos_of);
done:
  PyBuffer_Release(&op);
  PyBuffer_Release(&ar);
  PyBuffer_Release(&as);
  PyBuffer_Release(&wr);
  PyBuffer_Release(&ws);
  PyBuffer_Release(&ab);
  PyBuffer_Release(&ino);
  PyBuffer_Release(&ini);
  PyBuffer_Release(&to_);
  PyBuffer_Release(&tn_);
  PyBuffer_Release(&so_);
  PyBuffer_Release(&sp_);
  PyBuffer_Release(&rx_);
  PyBuffer_Release(&io_);
  PyBuffer_Release(&recs);
  PyBuffer_Release(&xb);
  PyBuffer_Release(&node);
  PyBuffer_Release(&edge);
  PyBuffer_Release(&eo);
  return out;
}

/*
 * label_rows(members, block_T, inst_off, member_off, slot_off, slot_pos) -> (rows, slots) as bytes
 * The (member row, slot) of every entry of derive_plan's assignment map, in
 * its order (search.py:374-376): block by block, instance by instance, the
 * block's weight slots in weight_nodes order; slots numbered over all
 * blocks.  int32 outputs.
 */
static PyObject* label_rows(PyObject* self, PyObject* args) {
  Py_buffer mem, bt, io, mo, so, sp;
  if (!PyArg_ParseTuple(args, "y*y*y*y*y*y*", &mem, &bt, &io, &mo, &so, &sp)) return NULL;
  PyObject *rows = NULL, *slots = NULL, *out = NULL;
  const int32_t* M = (const int32_t*)mem.buf;
  const int64_t* T = (const int64_t*)bt.buf;
  const int64_t* IO = (const int64_t*)io.buf;
  const int64_t* MO = (const int64_t*)mo.buf;
  const int64_t* SO = (const int64_t*)so.buf;
  const int32_t* SP = (const int32_t*)sp.buf;
  const Py_ssize_t nb = bt.len / 8, nm = mem.len / 4, ns = sp.len / 4;
  if (io.len < (nb + 1) * 8 || mo.len < (nb + 1) * 8 || so.len < (nb + 1) * 8 || SO[nb] > ns) {
    PyErr_SetString(PyExc_ValueError, "label_rows: inconsistent arguments");
    goto done;
  }
  Py_ssize_t K = 0;
  for (Py_ssize_t b = 0; b < nb; b++) K += (IO[b + 1] - IO[b]) * (SO[b + 1] - SO[b]);
  rows = PyBytes_FromStringAndSize(NULL, K * 4);
  slots = PyBytes_FromStringAndSize(NULL, K * 4);
  if (!rows || !slots) goto done;
  int32_t* R = (int32_t*)PyBytes_AS_STRING(rows);
  int32_t* S = (int32_t*)PyBytes_AS_STRING(slots);
  Py_ssize_t k = 0;
  for (Py_ssize_t b = 0; b < nb; b++) {
    const int64_t s0 = SO[b], s1 = SO[b + 1];
    if (s1 == s0) continue;
    for (int64_t i = 0; i < IO[b + 1] - IO[b]; i++) {
      const int64_t base = MO[b] + i * T[b];
      for (int64_t q = s0; q < s1; q++) {
        const int64_t at = base + SP[q];
        if (SP[q] < 0 || SP[q] >= T[b] || at < 0 || at >= nm) {
          PyErr_SetString(PyExc_IndexError, "label_rows: slot out of range");
          goto done;
        }
        R[k] = M[at];
        S[k] = (int32_t)q;
        k++;
      }
    }
  }
  out = PyTuple_Pack(2, rows, slots);
done:
  Py_XDECREF(rows);
  Py_XDECREF(slots);
  PyBuffer_Release(&mem);
  PyBuffer_Release(&bt);
  PyBuffer_Release(&io);
  PyBuffer_Release(&mo);
  PyBuffer_Release(&so);
  PyBuffer_Release(&sp);
  return out;
}

static PyMethodDef methods[] = {
    {"label_rows", label_rows, METH_VARARGS, "(member row, slot) of every assignment-map entry."},
    {"slot_positions", slot_positions, METH_VARARGS, "Weight slots (weight_nodes order) of every template."},
    {"block_results", block_results, METH_VARARGS, "SubgraphResults of every block from raw records."},
    {"lower_arrays", lower_arrays, METH_VARARGS, "Lower a grouped ModelGraph to flat sp_graph arrays."},
    {"singleton_results", singleton_results, METH_VARARGS, "SubgraphResults of one-node blocks from raw records."},
    {"assignments_dict", assignments_dict, METH_VARARGS, "Instance-scope -> label dict from member ids."},
    {"assignments_keys", assignments_keys, METH_VARARGS, "The keys half of assignments_dict (values None)."},
    {"save_graph_json", save_graph_json, METH_VARARGS, "The reference's save_graph document bytes."},
    {"assignments_fill", assignments_fill, METH_VARARGS, "The values half of assignments_dict."},
    {"make_ctor", make_ctor, METH_VARARGS, "Fast positional constructor for a dataclass."},
    {"block_instances", block_instances, METH_VARARGS, "Subgraph.instances of every block from fold arrays."},
    {NULL, NULL, 0, NULL}};

static struct PyModuleDef module = {PyModuleDef_HEAD_INIT, "_lower", NULL, -1, methods};

PyMODINIT_FUNC PyInit__lower(void) {
  S_name = PyUnicode_InternFromString("name");
  S_op = PyUnicode_InternFromString("op");
  S_inputs = PyUnicode_InternFromString("inputs");
  S_output = PyUnicode_InternFromString("output");
  S_weight = PyUnicode_InternFromString("weight");
  S_attrs = PyUnicode_InternFromString("attrs");
  S_member = PyUnicode_InternFromString("member");
  S_shape = PyUnicode_InternFromString("shape");
  S_dtype = PyUnicode_InternFromString("dtype");
  S_trainable = PyUnicode_InternFromString("trainable");
  if (!S_name || !S_op || !S_inputs || !S_output || !S_weight || !S_attrs || !S_member || !S_shape || !S_dtype ||
      !S_trainable)
    return NULL;
  PyObject* m = PyModule_Create(&module);
  if (m && PyModule_AddIntConstant(m, "built_for_hexversion", PY_VERSION_HEX) < 0) {
    Py_DECREF(m);
    return NULL;
  }
  return m;
}
