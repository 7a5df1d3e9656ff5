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
#include <stdint.h>
#include <string.h>

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
 * lower_arrays(topo_order, nodes, op_code, dtype_width)
 * -> (names, ascii, max_act_rank, max_w_rank, overflow_what,
 *     name_bytes, name_off, op, act_rank, act_shape, act_bytes,
 *     w_rank, w_shape, w_bytes, w_trainable, in_off, in_idx)
 */
static PyObject* lower_arrays(PyObject* self, PyObject* args) {
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
  if (namemap_init(&index, n) < 0) goto done;
  /* pass 1: name -> index map, name byte count */
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
  /* in_idx grows as inputs are seen (E unknown until the node pass) */
  Py_ssize_t cap = n * 2 + 16;
  int32_t* inidx = (int32_t*)PyMem_Malloc((size_t)cap * sizeof(int32_t));
  if (!inidx) {
    PyErr_NoMemory();
    goto done;
  }
  int max_ar = 0, max_wr = 0;
  const char* overflow = NULL;
  Py_ssize_t off = 0;
  noff[0] = 0;
  inoff[0] = 0;
  for (Py_ssize_t i = 0; i < n; i++) {
    PyObject* nm = PyList_GET_ITEM(names, i);
    Py_ssize_t L;
    const char* u = PyUnicode_AsUTF8AndSize(nm, &L);
    memcpy(pn + off, u, (size_t)L);
    off += L;
    noff[i + 1] = off;
    PyObject* node = PyDict_GetItemWithError(nodes, nm);
    if (!node) {
      if (!PyErr_Occurred()) PyErr_SetObject(PyExc_KeyError, nm);
      goto fail_idx;
    }
    long v;
    PyObject* o = PyObject_GetAttr(node, s_op);
    if (!o) goto fail_idx;
    int rc = cache_get_any(&opc, o, op_fn, &v);
    Py_DECREF(o);
    if (rc < 0) goto fail_idx;
    op[i] = (uint8_t)v;
    /* activation */
    PyObject* act = PyObject_GetAttr(node, s_activation);
    if (!act) goto fail_idx;
    PyObject* shp = PyObject_GetAttr(act, s_shape);
    PyObject* dt = shp ? PyObject_GetAttr(act, s_dtype) : NULL;
    Py_DECREF(act);
    if (!dt) {
      Py_XDECREF(shp);
      goto fail_idx;
    }
    int r;
    int64_t el;
    double fel;
    rc = read_shape(shp, ashape + i * MAX_RANK, &r, &el, &fel);
    Py_DECREF(shp);
    if (rc == 0) rc = cache_get_any(&wc, dt, width_fn, &v);
    Py_DECREF(dt);
    if (rc < 0) goto fail_idx;
    if (r > max_ar) max_ar = r;
    arank[i] = (uint8_t)(r > 255 ? 255 : r);
    abytes[i] = el * (int64_t)v;
    if (fel * 8.0 >= 9223372036854775808.0 && !overflow) overflow = "activation";
    /* weight */
    PyObject* w = PyObject_GetAttr(node, s_weight);
    if (!w) goto fail_idx;
    if (w == Py_None) {
      wrank[i] = 0;
      memset(wshape + i * MAX_RANK, 0, MAX_RANK * 8);
      wbytes[i] = 0;
      wtrain[i] = 0;
    } else {
      PyObject* ws = PyObject_GetAttr(w, s_shape);
      PyObject* wd = ws ? PyObject_GetAttr(w, s_dtype) : NULL;
      PyObject* wt = wd ? PyObject_GetAttr(w, s_trainable) : NULL;
      if (!wt) {
        Py_XDECREF(ws);
        Py_XDECREF(wd);
        Py_DECREF(w);
        goto fail_idx;
      }
      rc = read_shape(ws, wshape + i * MAX_RANK, &r, &el, &fel);
      if (rc == 0) rc = cache_get_any(&wc, wd, width_fn, &v);
      int tr = rc == 0 ? PyObject_IsTrue(wt) : 0;
      Py_DECREF(ws);
      Py_DECREF(wd);
      Py_DECREF(wt);
      if (rc < 0 || tr < 0) {
        Py_DECREF(w);
        goto fail_idx;
      }
      if (r > max_wr) max_wr = r;
      wrank[i] = (uint8_t)(r > 255 ? 255 : r);
      wbytes[i] = el * (int64_t)v;
      wtrain[i] = (uint8_t)tr;
      if (fel * 8.0 >= 9223372036854775808.0 && !overflow) overflow = "weight";
    }
    Py_DECREF(w);
    /* producers, GraphNode.inputs order */
    PyObject* ins = PyObject_GetAttr(node, s_inputs);
    if (!ins) goto fail_idx;
    PyObject* seq = PySequence_Fast(ins, "inputs must be a sequence");
    Py_DECREF(ins);
    if (!seq) goto fail_idx;
    const Py_ssize_t k = PySequence_Fast_GET_SIZE(seq);
    PyObject** it = PySequence_Fast_ITEMS(seq);
    if (E + k > cap) {
      while (E + k > cap) cap *= 2;
      int32_t* grown = (int32_t*)PyMem_Realloc(inidx, (size_t)cap * sizeof(int32_t));
      if (!grown) {
        Py_DECREF(seq);
        PyErr_NoMemory();
        goto fail_idx;
      }
      inidx = grown;
    }
    for (Py_ssize_t j = 0; j < k; j++) {
      const int32_t pi = namemap_get(&index, it[j]);
      if (pi < 0) {
        if (!PyErr_Occurred()) PyErr_SetObject(PyExc_KeyError, it[j]);
        Py_DECREF(seq);
        goto fail_idx;
      }
      inidx[E++] = pi;
    }
    Py_DECREF(seq);
    inoff[i + 1] = E;
  }
  b_inidx = PyByteArray_FromStringAndSize((const char*)inidx, E * 4);
  PyMem_Free(inidx);
  inidx = NULL;
  if (!b_inidx) goto done;
  result = Py_BuildValue("(OiiizOOOOOOOOOOOO)", names, ascii, max_ar, max_wr, overflow, b_names, b_noff,
                         b_op, b_arank, b_ashape, b_abytes, b_wrank, b_wshape, b_wbytes, b_wtrain, b_inoff, b_inidx);
  goto done;
fail_idx:
  PyMem_Free(inidx);
done:
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
      PyObject* pair = PyTuple_Pack(2, pre, tup);
      Py_DECREF(pre);
      Py_DECREF(tup);
      if (!pair) goto fail;
      PyTuple_SET_ITEM(insts, i, pair);
    }
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

static PyMethodDef methods[] = {
    {"lower_arrays", lower_arrays, METH_VARARGS, "Lower a grouped ModelGraph to flat sp_graph arrays."},
    {"block_instances", block_instances, METH_VARARGS, "Subgraph.instances of every block from fold arrays."},
    {NULL, NULL, 0, NULL}};

static struct PyModuleDef module = {PyModuleDef_HEAD_INIT, "_lower", NULL, -1, methods};

PyMODINIT_FUNC PyInit__lower(void) { return PyModule_Create(&module); }
