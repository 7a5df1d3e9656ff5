/*
 * oracle.c -- CPU restatement of the TAP search hot path.  TEST
 * INFRASTRUCTURE ONLY: the parity checker for the CUDA backend and the
 * `cpu_baseline` / `--impl reference` arm of bench.py.  Nothing in the
 * product package links or calls this file.
 *
 * It follows the reference literally (string-based folding, per-candidate
 * routing with explicit shard specs, no precomputed tables), so it is an
 * independent check of the table-driven GPU kernels:
 *   prune_graph          pkg/src/shardplan/pruning.py:123-201
 *   _template_key        pruning.py:97-111
 *   candidate_by_index   search.py:103-116
 *   pattern_routing      search.py:134-224  (+ _convert 227-233, _divisible 128-131)
 *   conversion_collective patterns.py:202-221, apply_collective 173-185,
 *                        ShardSpec.normalized 44-50, registry 118-159
 *   collective costs     costmodel.py:122-145
 *   plan_cost            costmodel.py:193-267, pack_gradients rewrite.py:78-111
 *   _plan_key/_eval_range search.py:284-310
 *
 * Parity pin: tests/test_oracle.py checks every function against the golden
 * vectors in tests/golden/cases.json produced by the reference itself
 * (tests/golden/make_golden.py).
 *
 * Build: make -C oracle   (-> oracle/lib/liboracle.so).  fp64 arithmetic is
 * compiled with -ffp-contract=off so every operation rounds like CPython.
 */
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include "../include/shardsearch.h"

/* templates the restatement handles (stack arrays per candidate; the
 * reference has no limit, the route search of the backend none below 2^64
 * candidates) */
#define ORACLE_MAX_T 2048

/* ------------------------------------------------------------------------- */
/* graph helpers                                                             */

typedef struct {
  const sp_graph* g;
  sp_graph gcopy;      /* owned copy of the caller's struct (arrays stay caller-owned) */
  int64_t* pos;        /* node -> template position scratch, kept at -1 between calls */
  int64_t n;
  int32_t* depth;      /* number of '/'-separated parts */
  int64_t* slash;      /* [n*maxd] byte position of the d-th '/' (d=1..), or name len */
  int32_t maxd;
  int64_t* by_name;    /* node indices sorted by name */
  int64_t* cons_off;   /* consumers CSR */
  int64_t* cons_idx;
} og;

static inline const uint8_t* nm(const og* G, int64_t i) { return G->g->name_bytes + G->g->name_off[i]; }
static inline int64_t nl(const og* G, int64_t i) { return G->g->name_off[i + 1] - G->g->name_off[i]; }

/* Python str ordering == UTF-8 byte ordering, shorter string first on a tie. */
static int strcmp_py(const uint8_t* a, int64_t la, const uint8_t* b, int64_t lb) {
  int64_t m = la < lb ? la : lb;
  int c = m ? memcmp(a, b, (size_t)m) : 0;
  if (c) return c;
  return (la > lb) - (la < lb);
}

/* _prefix(scope, depth): "/".join(scope.split("/")[:depth])  (pruning.py:58-59) */
static inline int64_t prefix_len(const og* G, int64_t i, int d) {
  if (d >= G->depth[i]) return nl(G, i);
  return G->slash[i * G->maxd + (d - 1)];
}

static const og* g_sort_ctx;
static int cmp_by_name(const void* x, const void* y) {
  int64_t a = *(const int64_t*)x, b = *(const int64_t*)y;
  return strcmp_py(nm(g_sort_ctx, a), nl(g_sort_ctx, a), nm(g_sort_ctx, b), nl(g_sort_ctx, b));
}

static int og_init(og* G, const sp_graph* g) {
  memset(G, 0, sizeof(*G));
  G->gcopy = *g;
  g = &G->gcopy;
  G->g = g;
  G->n = g->n_nodes;
  int64_t n = G->n;
  G->depth = (int32_t*)malloc(sizeof(int32_t) * (size_t)(n ? n : 1));
  int32_t maxd = 1;
  for (int64_t i = 0; i < n; i++) {
    int32_t d = 1;
    const uint8_t* s = nm(G, i);
    for (int64_t k = 0; k < nl(G, i); k++) d += (s[k] == '/');
    G->depth[i] = d;
    if (d > maxd) maxd = d;
  }
  G->maxd = maxd;
  G->slash = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n ? n : 1) * (size_t)maxd);
  for (int64_t i = 0; i < n; i++) {
    const uint8_t* s = nm(G, i);
    int64_t L = nl(G, i);
    int d = 0;
    for (int64_t k = 0; k < L; k++)
      if (s[k] == '/') G->slash[i * maxd + d++] = k;
    for (; d < maxd; d++) G->slash[i * maxd + d] = L;
  }
  G->by_name = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n ? n : 1));
  for (int64_t i = 0; i < n; i++) G->by_name[i] = i;
  g_sort_ctx = G;
  qsort(G->by_name, (size_t)n, sizeof(int64_t), cmp_by_name);
  /* consumers (ir.py:243-248); order is irrelevant for the boundary test */
  G->cons_off = (int64_t*)calloc((size_t)n + 1, sizeof(int64_t));
  int64_t E = g->in_off[n];
  G->cons_idx = (int64_t*)malloc(sizeof(int64_t) * (size_t)(E ? E : 1));
  for (int64_t e = 0; e < E; e++) G->cons_off[g->in_idx[e] + 1]++;
  for (int64_t i = 0; i < n; i++) G->cons_off[i + 1] += G->cons_off[i];
  int64_t* fill = (int64_t*)calloc((size_t)n + 1, sizeof(int64_t));
  for (int64_t i = 0; i < n; i++)
    for (int64_t e = g->in_off[i]; e < g->in_off[i + 1]; e++) {
      int64_t p = g->in_idx[e];
      G->cons_idx[G->cons_off[p] + fill[p]++] = i;
    }
  free(fill);
  G->pos = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n ? n : 1));
  for (int64_t i = 0; i < n; i++) G->pos[i] = -1;
  return 0;
}

static void og_free(og* G) {
  free(G->pos);
  free(G->depth);
  free(G->slash);
  free(G->by_name);
  free(G->cons_off);
  free(G->cons_idx);
}

/* name -> node index (exact), -1 when absent */
static int64_t og_lookup(const og* G, const uint8_t* s, int64_t L) {
  int64_t lo = 0, hi = G->n;
  while (lo < hi) {
    int64_t mid = (lo + hi) / 2;
    int64_t j = G->by_name[mid];
    int c = strcmp_py(nm(G, j), nl(G, j), s, L);
    if (c < 0) lo = mid + 1;
    else hi = mid;
  }
  if (lo < G->n) {
    int64_t j = G->by_name[lo];
    if (strcmp_py(nm(G, j), nl(G, j), s, L) == 0) return j;
  }
  return -1;
}

/* ------------------------------------------------------------------------- */
/* byte buffer                                                               */

typedef struct {
  uint8_t* p;
  size_t n, cap;
} buf;
static void bput(buf* b, const void* x, size_t k) {
  if (b->n + k > b->cap) {
    b->cap = (b->n + k) * 2 + 64;
    b->p = (uint8_t*)realloc(b->p, b->cap);
  }
  if (k) memcpy(b->p + b->n, x, k);
  b->n += k;
}

/* ------------------------------------------------------------------------- */
/* prune_graph (pruning.py:123-201)                                          */

typedef struct {
  int64_t pnode, plen; /* prefix = first plen bytes of node pnode's name */
  int64_t* mem;
  int64_t nmem;
} group;

typedef struct {
  int64_t pnode, plen;   /* template prefix */
  int64_t T, R;
  int64_t* inst_pnode;   /* [R] */
  int64_t* inst_plen;    /* [R] */
  int32_t* members;      /* [R*T] */
} subgraph;

typedef struct {
  og* G;
  int min_dup;
  subgraph* out;
  int64_t nout, capout;
  int32_t* mark;  /* member-set stamp per node */
  int32_t stamp;
} pruner;

static void push_sub(pruner* P, subgraph s) {
  if (P->nout == P->capout) {
    P->capout = P->capout * 2 + 16;
    P->out = (subgraph*)realloc(P->out, sizeof(subgraph) * (size_t)P->capout);
  }
  P->out[P->nout++] = s;
}

static const og* g_cmp_G;
static int cmp_group_prefix(const void* x, const void* y) {
  const group* a = (const group*)x;
  const group* b = (const group*)y;
  return strcmp_py(nm(g_cmp_G, a->pnode), a->plen, nm(g_cmp_G, b->pnode), b->plen);
}
static int cmp_topo(const void* x, const void* y) {
  int64_t a = *(const int64_t*)x, b = *(const int64_t*)y;
  int64_t ra = g_cmp_G->g->topo_rank[a], rb = g_cmp_G->g->topo_rank[b];
  if (ra != rb) return (ra > rb) - (ra < rb);
  return cmp_by_name(x, y);
}

/* accept(bucket) (pruning.py:136-148) */
static void accept(pruner* P, group* grp, int64_t k) {
  og* G = P->G;
  g_cmp_G = G;
  g_sort_ctx = G;
  qsort(grp, (size_t)k, sizeof(group), cmp_group_prefix);
  group* t = &grp[0];
  int64_t T = t->nmem;
  int64_t* tmpl = (int64_t*)malloc(sizeof(int64_t) * (size_t)T);
  memcpy(tmpl, t->mem, sizeof(int64_t) * (size_t)T);
  qsort(tmpl, (size_t)T, sizeof(int64_t), cmp_topo);
  subgraph s;
  s.pnode = t->pnode;
  s.plen = t->plen;
  s.T = T;
  s.R = k;
  s.inst_pnode = (int64_t*)malloc(sizeof(int64_t) * (size_t)k);
  s.inst_plen = (int64_t*)malloc(sizeof(int64_t) * (size_t)k);
  s.members = (int32_t*)malloc(sizeof(int32_t) * (size_t)(k * T));
  buf nbuf = {0};
  for (int64_t r = 0; r < k; r++) {
    s.inst_pnode[r] = grp[r].pnode;
    s.inst_plen[r] = grp[r].plen;
    for (int64_t j = 0; j < T; j++) {
      /* inst_prefix + t[len(prefix):] */
      nbuf.n = 0;
      bput(&nbuf, nm(G, grp[r].pnode), (size_t)grp[r].plen);
      bput(&nbuf, nm(G, tmpl[j]) + t->plen, (size_t)(nl(G, tmpl[j]) - t->plen));
      int64_t idx = og_lookup(G, nbuf.p, (int64_t)nbuf.n);
      s.members[r * T + j] = (int32_t)idx;
    }
  }
  free(nbuf.p);
  free(tmpl);
  push_sub(P, s);
}

static void accept_single(pruner* P, int64_t node) {
  group g1;
  int64_t m = node;
  g1.pnode = node;
  g1.plen = nl(P->G, node);
  g1.mem = &m;
  g1.nmem = 1;
  accept(P, &g1, 1);
}

/* _template_key serialisation (pruning.py:97-111): equal bytes <=> equal tuples */
typedef struct {
  const uint8_t* p;
  int64_t n;
} sv;
static int cmp_sv(const void* x, const void* y) {
  const sv* a = (const sv*)x;
  const sv* b = (const sv*)y;
  return strcmp_py(a->p, a->n, b->p, b->n);
}

static void template_key(pruner* P, const group* gr, buf* out) {
  og* G = P->G;
  const sp_graph* g = G->g;
  int64_t start = gr->plen ? gr->plen + 1 : 0;
  P->stamp++;
  for (int64_t i = 0; i < gr->nmem; i++) P->mark[gr->mem[i]] = P->stamp;
  int64_t* ms = (int64_t*)malloc(sizeof(int64_t) * (size_t)gr->nmem);
  memcpy(ms, gr->mem, sizeof(int64_t) * (size_t)gr->nmem);
  g_sort_ctx = G;
  qsort(ms, (size_t)gr->nmem, sizeof(int64_t), cmp_by_name);
  sv* rels = NULL;
  int64_t cap = 0;
  out->n = 0;
  for (int64_t i = 0; i < gr->nmem; i++) {
    int64_t m = ms[i];
    int64_t L = nl(G, m);
    uint32_t rl = (uint32_t)(start < L ? L - start : 0);
    bput(out, &rl, 4);
    bput(out, nm(G, m) + (start < L ? start : L), rl);
    uint8_t op = g->op[m];
    bput(out, &op, 1);
    uint8_t wr = g->w_rank[m];
    bput(out, &wr, 1);
    if (wr) {
      bput(out, &g->w_shape[m * SP_MAX_RANK], sizeof(int64_t) * wr);
      uint8_t tr = g->w_trainable[m] ? 1 : 0;
      bput(out, &tr, 1);
    }
    int64_t k = 0;
    int64_t deg = g->in_off[m + 1] - g->in_off[m];
    if (deg > cap) {
      cap = deg;
      rels = (sv*)realloc(rels, sizeof(sv) * (size_t)cap);
    }
    for (int64_t e = g->in_off[m]; e < g->in_off[m + 1]; e++) {
      int64_t r = g->in_idx[e];
      if (P->mark[r] != P->stamp) continue;
      int64_t Lr = nl(G, r);
      rels[k].p = nm(G, r) + (start < Lr ? start : Lr);
      rels[k].n = start < Lr ? Lr - start : 0;
      k++;
    }
    qsort(rels, (size_t)k, sizeof(sv), cmp_sv);
    uint32_t kk = (uint32_t)k;
    bput(out, &kk, 4);
    for (int64_t j = 0; j < k; j++) {
      uint32_t l = (uint32_t)rels[j].n;
      bput(out, &l, 4);
      bput(out, rels[j].p, l);
    }
  }
  free(rels);
  free(ms);
}

typedef struct {
  int64_t gi;
  uint8_t* key;
  size_t klen;
} keyed;
static int cmp_keyed(const void* x, const void* y) {
  const keyed* a = (const keyed*)x;
  const keyed* b = (const keyed*)y;
  size_t m = a->klen < b->klen ? a->klen : b->klen;
  int c = m ? memcmp(a->key, b->key, m) : 0;
  if (c) return c;
  if (a->klen != b->klen) return (a->klen > b->klen) - (a->klen < b->klen);
  return (a->gi > b->gi) - (a->gi < b->gi);
}

static void refine(pruner* P, group* groups, int64_t ng, int depth);

/* descend(groups, depth) (pruning.py:150-174).  A signature bucket of >= min_dup
 * groups accepts each exact template class of >= min_dup; smaller buckets only
 * hold smaller classes, so accepting every template class of >= min_dup among
 * the siblings and refining the rest is the same partition. */
static void descend(pruner* P, group* groups, int64_t ng, int depth) {
  keyed* ks = (keyed*)malloc(sizeof(keyed) * (size_t)ng);
  buf b = {0};
  for (int64_t i = 0; i < ng; i++) {
    template_key(P, &groups[i], &b);
    ks[i].gi = i;
    ks[i].klen = b.n;
    ks[i].key = (uint8_t*)malloc(b.n ? b.n : 1);
    memcpy(ks[i].key, b.p, b.n);
  }
  free(b.p);
  qsort(ks, (size_t)ng, sizeof(keyed), cmp_keyed);
  group* left = (group*)malloc(sizeof(group) * (size_t)ng);
  int64_t nleft = 0;
  group* cls = (group*)malloc(sizeof(group) * (size_t)ng);
  for (int64_t i = 0; i < ng;) {
    int64_t j = i + 1;
    while (j < ng && ks[j].klen == ks[i].klen && memcmp(ks[j].key, ks[i].key, ks[i].klen) == 0) j++;
    if (j - i >= P->min_dup) {
      for (int64_t t = i; t < j; t++) cls[t - i] = groups[ks[t].gi];
      accept(P, cls, j - i);
    } else {
      for (int64_t t = i; t < j; t++) left[nleft++] = groups[ks[t].gi];
    }
    i = j;
  }
  for (int64_t i = 0; i < ng; i++) free(ks[i].key);
  free(ks);
  free(cls);
  if (nleft) refine(P, left, nleft, depth);
  free(left);
}

static int g_cmp_depth;
static int cmp_child(const void* x, const void* y) {
  int64_t a = *(const int64_t*)x, b = *(const int64_t*)y;
  int c = strcmp_py(nm(g_cmp_G, a), prefix_len(g_cmp_G, a, g_cmp_depth), nm(g_cmp_G, b),
                    prefix_len(g_cmp_G, b, g_cmp_depth));
  if (c) return c;
  return cmp_by_name(x, y);
}

/* refine(groups, depth) (pruning.py:176-193) */
static void refine(pruner* P, group* groups, int64_t ng, int depth) {
  og* G = P->G;
  for (int64_t gi = 0; gi < ng; gi++) {
    group* gr = &groups[gi];
    int64_t* kids = (int64_t*)malloc(sizeof(int64_t) * (size_t)gr->nmem);
    int64_t nk = 0;
    for (int64_t i = 0; i < gr->nmem; i++) {
      int64_t m = gr->mem[i];
      if (G->depth[m] <= depth) accept_single(P, m);
      else kids[nk++] = m;
    }
    if (nk) {
      g_cmp_G = G;
      g_sort_ctx = G;
      g_cmp_depth = depth + 1;
      qsort(kids, (size_t)nk, sizeof(int64_t), cmp_child);
      group* ch = (group*)malloc(sizeof(group) * (size_t)nk);
      int64_t nch = 0;
      for (int64_t i = 0; i < nk;) {
        int64_t L = prefix_len(G, kids[i], depth + 1);
        int64_t j = i + 1;
        while (j < nk && prefix_len(G, kids[j], depth + 1) == L &&
               memcmp(nm(G, kids[j]), nm(G, kids[i]), (size_t)L) == 0)
          j++;
        ch[nch].pnode = kids[i];
        ch[nch].plen = L;
        ch[nch].mem = kids + i;
        ch[nch].nmem = j - i;
        nch++;
        i = j;
      }
      descend(P, ch, nch, depth + 1);
      free(ch);
    }
    free(kids);
  }
}

static int cmp_sub_prefix(const void* x, const void* y) {
  const subgraph* a = (const subgraph*)x;
  const subgraph* b = (const subgraph*)y;
  return strcmp_py(nm(g_cmp_G, a->pnode), a->plen, nm(g_cmp_G, b->pnode), b->plen);
}

typedef struct oracle_blocks {
  sp_blocks view;
  int64_t* block_T;
  int64_t* block_inst_off;
  int64_t* block_member_off;
  int64_t* inst_prefix_node;
  int64_t* inst_prefix_len;
  int32_t* members;
} oracle_blocks;

int oracle_prune(const sp_graph* g, int32_t min_dup, oracle_blocks** out) {
  if (min_dup < 1) return SP_ERR_CONFIG; /* BadConfig("min_duplicates must be >= 1") */
  og G;
  og_init(&G, g);
  pruner P;
  memset(&P, 0, sizeof(P));
  P.G = &G;
  P.min_dup = min_dup;
  P.mark = (int32_t*)calloc((size_t)G.n + 1, sizeof(int32_t));
  /* top-level groups by _prefix(name, 1) over sorted names (pruning.py:195-198) */
  int64_t* all = (int64_t*)malloc(sizeof(int64_t) * (size_t)(G.n ? G.n : 1));
  memcpy(all, G.by_name, sizeof(int64_t) * (size_t)G.n);
  g_cmp_G = &G;
  g_sort_ctx = &G;
  g_cmp_depth = 1;
  qsort(all, (size_t)G.n, sizeof(int64_t), cmp_child);
  group* top = (group*)malloc(sizeof(group) * (size_t)(G.n ? G.n : 1));
  int64_t nt = 0;
  for (int64_t i = 0; i < G.n;) {
    int64_t L = prefix_len(&G, all[i], 1);
    int64_t j = i + 1;
    while (j < G.n && prefix_len(&G, all[j], 1) == L && memcmp(nm(&G, all[j]), nm(&G, all[i]), (size_t)L) == 0) j++;
    top[nt].pnode = all[i];
    top[nt].plen = L;
    top[nt].mem = all + i;
    top[nt].nmem = j - i;
    nt++;
    i = j;
  }
  descend(&P, top, nt, 1);
  g_cmp_G = &G;
  qsort(P.out, (size_t)P.nout, sizeof(subgraph), cmp_sub_prefix); /* pruning.py:200 */

  oracle_blocks* ob = (oracle_blocks*)calloc(1, sizeof(oracle_blocks));
  int64_t nb = P.nout, ni = 0, nmem = 0;
  for (int64_t b = 0; b < nb; b++) {
    ni += P.out[b].R;
    nmem += P.out[b].R * P.out[b].T;
  }
  ob->block_T = (int64_t*)malloc(sizeof(int64_t) * (size_t)(nb + 1));
  ob->block_inst_off = (int64_t*)malloc(sizeof(int64_t) * (size_t)(nb + 1));
  ob->block_member_off = (int64_t*)malloc(sizeof(int64_t) * (size_t)(nb + 1));
  ob->inst_prefix_node = (int64_t*)malloc(sizeof(int64_t) * (size_t)(ni + 1));
  ob->inst_prefix_len = (int64_t*)malloc(sizeof(int64_t) * (size_t)(ni + 1));
  ob->members = (int32_t*)malloc(sizeof(int32_t) * (size_t)(nmem + 1));
  int64_t io = 0, mo = 0;
  for (int64_t b = 0; b < nb; b++) {
    subgraph* s = &P.out[b];
    ob->block_T[b] = s->T;
    ob->block_inst_off[b] = io;
    ob->block_member_off[b] = mo;
    for (int64_t r = 0; r < s->R; r++) {
      ob->inst_prefix_node[io] = s->inst_pnode[r];
      ob->inst_prefix_len[io] = s->inst_plen[r];
      io++;
    }
    memcpy(ob->members + mo, s->members, sizeof(int32_t) * (size_t)(s->R * s->T));
    mo += s->R * s->T;
    free(s->inst_pnode);
    free(s->inst_plen);
    free(s->members);
  }
  ob->block_inst_off[nb] = io;
  ob->block_member_off[nb] = mo;
  ob->view.n_blocks = nb;
  ob->view.n_instances = ni;
  ob->view.n_members = nmem;
  ob->view.block_T = ob->block_T;
  ob->view.block_inst_off = ob->block_inst_off;
  ob->view.block_member_off = ob->block_member_off;
  ob->view.inst_prefix_node = ob->inst_prefix_node;
  ob->view.inst_prefix_len = ob->inst_prefix_len;
  ob->view.members = ob->members;
  free(P.out);
  free(P.mark);
  free(all);
  free(top);
  og_free(&G);
  *out = ob;
  return SP_OK;
}

const sp_blocks* oracle_blocks_view(const oracle_blocks* ob) { return &ob->view; }

void oracle_blocks_free(oracle_blocks* ob) {
  if (!ob) return;
  free(ob->block_T);
  free(ob->block_inst_off);
  free(ob->block_member_off);
  free(ob->inst_prefix_node);
  free(ob->inst_prefix_len);
  free(ob->members);
  free(ob);
}

/* ------------------------------------------------------------------------- */
/* shard specs, registry, collectives (patterns.py)                          */

enum { K_REPLICA = 0, K_SPLIT = 1, K_PARTIAL = 2, K_NONE = 3 };
enum { C_ID = 0, C_AR = 1, C_AG = 2, C_RS = 3, C_A2A = 4 };

typedef struct {
  int kind;
  int axis;
} spec;
typedef struct {
  int kind;
  int axis;
} coll;
typedef struct {
  spec in, w, out;
  int coll;
} pattern;

#define R_ {K_REPLICA, 0}
#define S_(a) {K_SPLIT, a}
#define P_ {K_PARTIAL, 0}
#define N_ {K_NONE, 0}

/* _REGISTRY (patterns.py:118-159), LAST = -1 */
static const pattern PAT_MATMUL[] = {{R_, R_, R_, C_ID},
                                     {R_, S_(1), S_(-1), C_ID},
                                     {S_(-1), S_(0), P_, C_AR},
                                     {S_(0), R_, S_(0), C_ID}};
static const pattern PAT_ELEM[] = {{R_, R_, R_, C_ID}, {S_(0), R_, S_(0), C_ID}, {S_(-1), S_(0), S_(-1), C_ID}};
static const pattern PAT_NORM[] = {{R_, N_, R_, C_ID}, {S_(0), N_, S_(0), C_ID}};
static const pattern PAT_EMB[] = {{R_, R_, R_, C_ID}, {R_, S_(1), S_(-1), C_ID}, {S_(0), R_, S_(0), C_ID}};
static const pattern PAT_ONE[] = {{R_, N_, R_, C_ID}};

static int patterns_for(int op, const pattern** out) {
  switch (op) {
    case SP_OP_MATMUL: *out = PAT_MATMUL; return 4;
    case SP_OP_ELEMENTWISE: *out = PAT_ELEM; return 3;
    case SP_OP_LAYERNORM:
    case SP_OP_SOFTMAX: *out = PAT_NORM; return 2;
    case SP_OP_EMBEDDING: *out = PAT_EMB; return 3;
    case SP_OP_RESHAPE:
    case SP_OP_INPUT:
    case SP_OP_OUTPUT: *out = PAT_ONE; return 1;
    default: *out = NULL; return -1; /* SpecMismatch: not a shardable compute kind */
  }
}

/* ShardSpec.normalized (patterns.py:44-50); returns 0 on SpecMismatch */
static int normalized(spec s, int rank, spec* out) {
  if (s.kind == K_SPLIT) {
    int a = s.axis >= 0 ? s.axis : rank + s.axis;
    if (!(0 <= a && a < rank)) return 0;
    out->kind = K_SPLIT;
    out->axis = a;
    return 1;
  }
  *out = s;
  out->axis = 0;
  return 1;
}

static int spec_eq(spec a, spec b) { return a.kind == b.kind && (a.kind != K_SPLIT || a.axis == b.axis); }

/* conversion_collective (patterns.py:202-221) + _convert divisibility (search.py:227-233);
 * returns 0 on NoRouteError */
static int convert(spec frm, spec to, int rank, const int64_t* shape, int64_t d, coll* c) {
  spec a, b;
  if (!normalized(frm, rank, &a) || !normalized(to, rank, &b)) return 0;
  if (spec_eq(a, b)) {
    c->kind = C_ID;
    c->axis = -1;
  } else if (b.kind == K_REPLICA && a.kind == K_SPLIT) {
    c->kind = C_AG;
    c->axis = a.axis;
  } else if (b.kind == K_REPLICA && a.kind == K_PARTIAL) {
    c->kind = C_AR;
    c->axis = -1;
  } else if (a.kind == K_SPLIT && b.kind == K_SPLIT && a.axis != b.axis) {
    c->kind = C_A2A;
    c->axis = b.axis;
  } else if (a.kind == K_PARTIAL && b.kind == K_SPLIT) {
    c->kind = C_RS;
    c->axis = b.axis;
  } else {
    return 0;
  }
  if (to.kind == K_SPLIT) {
    spec tn = {K_REPLICA, 0};
    normalized(to, rank, &tn);
    if (shape[tn.axis] % d) return 0;
  }
  return 1;
}

/* apply_collective (patterns.py:173-185) */
static spec apply_coll(spec s, coll c) {
  spec r = s;
  if (c.kind == C_AR || c.kind == C_AG) {
    r.kind = K_REPLICA;
    r.axis = 0;
  } else if (c.kind == C_RS || c.kind == C_A2A) {
    r.kind = K_SPLIT;
    r.axis = c.axis;
  }
  return r;
}

/* collective_cost_bytes (costmodel.py:122-134) */
static double cost_bytes(int kind, int64_t nbytes, const sp_mesh* M) {
  if (kind == C_ID) return 0.0;
  int64_t d = M->m * M->n;
  if (d == 1) return 0.0;
  double bw = M->m > 1 ? M->inter_bw : M->intra_bw;
  double vol;
  if (kind == C_AR) vol = 2.0 * (double)(d - 1) / (double)d * (double)nbytes;
  else vol = (double)(d - 1) / (double)d * (double)nbytes;
  double eff = kind == C_AR ? M->eff_allreduce
             : kind == C_AG ? M->eff_allgather
             : kind == C_RS ? M->eff_reducescatter
                            : M->eff_alltoall;
  return vol / bw * eff;
}

/* collective_call_cost (costmodel.py:141-145) */
static double call_cost(int kind, int64_t nbytes, const sp_mesh* M) {
  if (kind == C_ID || M->m * M->n == 1) return 0.0;
  return M->setup_latency_s + cost_bytes(kind, nbytes, M);
}

/* ------------------------------------------------------------------------- */
/* per-candidate routing and cost                                            */

typedef struct {
  const sp_graph* g;
  const sp_mesh* M;
  int64_t d;
  int64_t T;
  const int64_t* tn;   /* template node indices in template order */
  int64_t* pos;        /* node -> template position or -1  ([n]) */
  int32_t* slot;       /* template position -> weight slot or -1 */
  int32_t V;
  int32_t* slot_pos;   /* weight slot -> template position */
  int32_t* radix;      /* per slot */
  uint8_t* boundary;   /* per template position */
  int64_t mu, chunk;
} block_ctx;

typedef struct {
  int valid;
  int fail_pos;
  int pat[ORACLE_MAX_T];
  spec state[ORACLE_MAX_T];
  int exit_axis[ORACLE_MAX_T];
  double forward, backward, total;
  int num_split;
  int64_t bytes[5], calls[5];
} cand_result;

static spec weight_option(int radix, int digit) {
  /* WEIGHT_OPTIONS_2D/1D (search.py:35-36) */
  spec s;
  (void)radix;
  if (digit == 0) {
    s.kind = K_REPLICA;
    s.axis = 0;
  } else {
    s.kind = K_SPLIT;
    s.axis = digit - 1;
  }
  return s;
}

static void eval_candidate(const block_ctx* B, uint64_t index, cand_result* R, int detail) {
  const sp_graph* g = B->g;
  int digits[ORACLE_MAX_T];
  /* candidate_by_index (search.py:103-116): last weight varies fastest */
  uint64_t rem = index;
  for (int s = B->V - 1; s >= 0; s--) {
    digits[s] = (int)(rem % (uint64_t)B->radix[s]);
    rem /= (uint64_t)B->radix[s];
  }
  int num_split = 0;
  for (int s = 0; s < B->V; s++) num_split += digits[s] != 0;
  R->num_split = num_split;
  R->valid = 0;
  R->fail_pos = -1;
  int64_t T = B->T;
  spec* st = R->state;
  int pc[ORACLE_MAX_T];          /* chosen pattern collective */
  /* pattern_routing (search.py:134-224) */
  for (int64_t i = 0; i < T; i++) {
    int64_t n = B->tn[i];
    const pattern* pats;
    int np = patterns_for(g->op[n], &pats);
    int arank = g->act_rank[n];
    const int64_t* ashape = &g->act_shape[n * SP_MAX_RANK];
    double best_c = 0.0;
    int best = -1;
    spec best_out = {0, 0};
    for (int p = 0; p < np; p++) {
      const pattern* pt = &pats[p];
      if (g->w_rank[n]) {
        int wr = g->w_rank[n];
        spec want = {K_NONE, 0}, assigned = {K_REPLICA, 0};
        int have_want = 0;
        if (pt->w.kind != K_NONE) {
          if (!normalized(pt->w, wr, &want)) continue;
          have_want = 1;
        }
        spec opt = weight_option(B->radix[B->slot[i]], digits[B->slot[i]]);
        normalized(opt, wr, &assigned);
        if (!have_want || !spec_eq(want, assigned)) continue;
        /* _divisible(assigned, weight.shape, devices) */
        if (assigned.kind == K_SPLIT && g->w_shape[n * SP_MAX_RANK + assigned.axis] % B->d) continue;
      }
      double c = 0.0;
      int feasible = 1;
      for (int64_t e = g->in_off[n]; e < g->in_off[n + 1]; e++) {
        int64_t pr = g->in_idx[e];
        int64_t pp = B->pos[pr];
        spec ps;
        if (pp >= 0 && pp < i) ps = st[pp];
        else {
          ps.kind = K_REPLICA; /* entry edges are replica */
          ps.axis = 0;
        }
        spec req;
        coll cv;
        if (!normalized(pt->in, g->act_rank[pr], &req) ||
            !convert(ps, req, g->act_rank[pr], &g->act_shape[pr * SP_MAX_RANK], B->d, &cv)) {
          feasible = 0;
          break;
        }
        if (cv.kind != C_ID) c += call_cost(cv.kind, g->act_bytes[pr], B->M);
      }
      if (!feasible) continue;
      spec out;
      if (!normalized(pt->out, arank, &out)) continue;
      if (out.kind == K_SPLIT && ashape[out.axis] % B->d) continue;
      c += call_cost(pt->coll, g->act_bytes[n], B->M);
      if (best < 0 || c < best_c) { /* min by (cost, pattern index) */
        best = p;
        best_c = c;
        best_out = out;
      }
    }
    if (best < 0) {
      R->fail_pos = (int)i;
      return;
    }
    coll pcoll = {pats[best].coll, -1};
    st[i] = apply_coll(best_out, pcoll);
    R->pat[i] = best;
    pc[i] = pats[best].coll;
  }
  R->valid = 1;
  /* exits (search.py:213-223): boundary nodes not in replica gather back */
  for (int64_t i = 0; i < T; i++) {
    R->exit_axis[i] = -1;
    if (B->boundary[i] && st[i].kind != K_REPLICA) R->exit_axis[i] = st[i].kind == K_SPLIT ? st[i].axis : -2;
  }
  /* plan_cost (costmodel.py:193-267) */
  double reach[ORACLE_MAX_T];
  for (int k = 0; k < 5; k++) R->bytes[k] = R->calls[k] = 0;
  for (int64_t i = 0; i < T; i++) {
    int64_t n = B->tn[i];
    const pattern* pats;
    patterns_for(g->op[n], &pats);
    const pattern* pt = &pats[R->pat[i]];
    double base = 0.0;
    for (int64_t e = g->in_off[n]; e < g->in_off[n + 1]; e++) {
      int64_t pr = g->in_idx[e];
      int64_t pp = B->pos[pr];
      if (pp < 0) continue; /* external producer */
      spec req;
      coll cv;
      normalized(pt->in, g->act_rank[pr], &req);
      convert(st[pp], req, g->act_rank[pr], &g->act_shape[pr * SP_MAX_RANK], B->d, &cv);
      double cc = 0.0;
      if (cv.kind != C_ID) {
        cc = call_cost(cv.kind, g->act_bytes[pr], B->M);
        R->bytes[cv.kind] += g->act_bytes[pr];
        R->calls[cv.kind]++;
      }
      double v = reach[pp] + cc;
      if (v > base) base = v;
    }
    double own = call_cost(pc[i], g->act_bytes[n], B->M);
    if (pc[i] != C_ID) {
      R->bytes[pc[i]] += g->act_bytes[n];
      R->calls[pc[i]]++;
    }
    reach[i] = base + own;
  }
  double fwd = 0.0;
  for (int64_t i = 0; i < T; i++) {
    double tail = reach[i];
    if (R->exit_axis[i] != -1) {
      int64_t n = B->tn[i];
      tail += call_cost(C_AG, g->act_bytes[n], B->M);
      R->bytes[C_AG] += g->act_bytes[n];
      R->calls[C_AG]++;
    }
    if (tail > fwd) fwd = tail;
  }
  /* backward: pack_gradients (rewrite.py:78-111) over replicated trainable weights */
  int64_t buckets[ORACLE_MAX_T], unfused[ORACLE_MAX_T];
  int nb = 0, nu = 0;
  int64_t cur = 0;
  int cur_n = 0;
  for (int64_t i = 0; i < T; i++) {
    int64_t n = B->tn[i];
    if (!g->w_rank[n] || !g->w_trainable[n]) continue;
    if (digits[B->slot[i]] != 0) continue; /* split weights own their gradient shard */
    int64_t size = g->w_bytes[n];
    if (size >= B->mu) {
      unfused[nu++] = size;
      continue;
    }
    if (cur + size > B->chunk && cur_n) {
      buckets[nb++] = cur;
      cur = 0;
      cur_n = 0;
    }
    cur += size;
    cur_n++;
  }
  if (cur_n) buckets[nb++] = cur;
  double bwd = 0.0;
  if (B->d > 1) {
    for (int k = 0; k < nb; k++) {
      bwd += B->M->setup_latency_s + cost_bytes(C_AR, buckets[k], B->M);
      R->bytes[C_AR] += buckets[k];
      R->calls[C_AR]++;
    }
    for (int k = 0; k < nu; k++) {
      bwd += B->M->setup_latency_s + cost_bytes(C_AR, unfused[k], B->M);
      R->bytes[C_AR] += unfused[k];
      R->calls[C_AR]++;
    }
  }
  R->forward = fwd;
  R->backward = bwd;
  /* CostReport.total (costmodel.py:157-163) */
  double eff_b = bwd * (1.0 - B->M->overlap_fraction);
  R->total = fwd + eff_b;
  (void)detail;
}

static const og* g_slot_G;
static int cmp_slot_name(const void* x, const void* y) { return cmp_by_name(x, y); }

/* builds block context; returns SP_OK / error */
static int block_init(block_ctx* B, og* G, const int32_t* tmpl, int64_t T, const sp_mesh* M,
                      int64_t mu, int64_t chunk) {
  const sp_graph* g = G->g;
  memset(B, 0, sizeof(*B));
  if (T < 0) return SP_ERR_CONFIG;
  if (T > ORACLE_MAX_T) return SP_ERR_UNSUPPORTED;
  B->g = g;
  B->M = M;
  B->d = M->m * M->n;
  B->T = T;
  B->mu = mu;
  B->chunk = chunk;
  int64_t* tn = (int64_t*)malloc(sizeof(int64_t) * (size_t)(T ? T : 1));
  for (int64_t i = 0; i < T; i++) tn[i] = tmpl[i];
  B->tn = tn;
  B->pos = G->pos;  /* all -1 outside this template; restored by block_free */
  for (int64_t i = 0; i < T; i++) B->pos[tn[i]] = i;
  for (int64_t i = 0; i < T; i++) {
    const pattern* pats;
    if (patterns_for(g->op[tn[i]], &pats) < 0) return SP_ERR_SPEC;
  }
  /* weight_nodes: weighted template scopes sorted by name (search.py:85-88) */
  int64_t* ws = (int64_t*)malloc(sizeof(int64_t) * (size_t)(T ? T : 1));
  int V = 0;
  for (int64_t i = 0; i < T; i++)
    if (g->w_rank[tn[i]]) ws[V++] = tn[i];
  g_sort_ctx = G;
  g_slot_G = G;
  qsort(ws, (size_t)V, sizeof(int64_t), cmp_slot_name);
  B->V = V;
  B->slot = (int32_t*)malloc(sizeof(int32_t) * (size_t)(T ? T : 1));
  B->slot_pos = (int32_t*)malloc(sizeof(int32_t) * (size_t)(V ? V : 1));
  B->radix = (int32_t*)malloc(sizeof(int32_t) * (size_t)(V ? V : 1));
  for (int64_t i = 0; i < T; i++) B->slot[i] = -1;
  for (int s = 0; s < V; s++) {
    int64_t p = B->pos[ws[s]];
    B->slot[p] = s;
    B->slot_pos[s] = (int32_t)p;
    B->radix[s] = g->w_rank[ws[s]] >= 2 ? 3 : 2; /* _options (search.py:91-93) */
  }
  free(ws);
  B->boundary = (uint8_t*)malloc((size_t)(T ? T : 1));
  for (int64_t i = 0; i < T; i++) {
    int64_t n = tn[i];
    int b = G->cons_off[n + 1] == G->cons_off[n];
    for (int64_t e = G->cons_off[n]; e < G->cons_off[n + 1]; e++)
      if (B->pos[G->cons_idx[e]] < 0) b = 1;
    B->boundary[i] = (uint8_t)b;
  }
  return SP_OK;
}

static void block_free(block_ctx* B) {
  for (int64_t i = 0; i < B->T; i++) B->pos[B->tn[i]] = -1;
  free((void*)B->tn);
  free(B->slot);
  free(B->slot_pos);
  free(B->radix);
  free(B->boundary);
}

/* count_candidates (search.py:96-100); 0 on u64 overflow */
static int block_count(const block_ctx* B, uint64_t* C) {
  uint64_t c = 1;
  for (int s = 0; s < B->V; s++) {
    if (c > UINT64_MAX / (uint64_t)B->radix[s]) return 0;
    c *= (uint64_t)B->radix[s];
  }
  *C = c;
  return 1;
}

/* _plan_key comparison (search.py:284-286) */
static int key_less(double t, int ns, uint64_t idx, const sp_score_out* b) {
  if (!b->has_best) return 1;
  if (t != b->best_total) return t < b->best_total;
  if (ns != b->best_num_split) return ns < b->best_num_split;
  return idx < b->best_index;
}

typedef struct {
  const block_ctx* B;
  uint64_t lo, hi;
  double* totals;
  sp_score_out res;
} worker;

static void* work(void* arg) {
  worker* w = (worker*)arg;
  cand_result R;
  memset(&w->res, 0, sizeof(w->res));
  for (uint64_t idx = w->lo; idx < w->hi; idx++) {
    eval_candidate(w->B, idx, &R, 0);
    if (!R.valid) {
      if (w->totals) w->totals[idx - w->lo] = __builtin_nan("");
      continue;
    }
    if (w->totals) w->totals[idx - w->lo] = R.total;
    w->res.valid++;
    if (key_less(R.total, R.num_split, idx, &w->res)) {
      w->res.has_best = 1;
      w->res.best_total = R.total;
      w->res.best_num_split = R.num_split;
      w->res.best_index = idx;
    }
  }
  return NULL;
}

/*
 * _eval_range over [lo, hi) of one block (search.py:289-310), split over
 * `threads` pthreads like search_subgraph's worker pool (search.py:331-343).
 * totals (optional, [hi-lo]) receives CostReport.total or NaN for invalid.
 */
static int score_core(og* Gp, const int32_t* tmpl, int64_t T, const sp_mesh* M, int64_t mu, int64_t chunk,
                      uint64_t lo, uint64_t hi, int32_t threads, double* totals, sp_score_out* out);

/* Graph handle: build the per-graph structures (name order, consumers) once. */
void* oracle_graph_open(const sp_graph* g) {
  og* G = (og*)malloc(sizeof(og));
  og_init(G, g);
  return G;
}

void oracle_graph_close(void* h) {
  if (!h) return;
  og_free((og*)h);
  free(h);
}

int oracle_score_h(void* h, const int32_t* tmpl, int64_t T, const sp_mesh* M, int64_t mu, int64_t chunk,
                   uint64_t lo, uint64_t hi, int32_t threads, double* totals, sp_score_out* out) {
  return score_core((og*)h, tmpl, T, M, mu, chunk, lo, hi, threads, totals, out);
}

int oracle_score(const sp_graph* g, const int32_t* tmpl, int64_t T, const sp_mesh* M, int64_t mu,
                 int64_t chunk, uint64_t lo, uint64_t hi, int32_t threads, double* totals,
                 sp_score_out* out) {
  og G;
  og_init(&G, g);
  int rc = score_core(&G, tmpl, T, M, mu, chunk, lo, hi, threads, totals, out);
  og_free(&G);
  return rc;
}

static int score_core(og* Gp, const int32_t* tmpl, int64_t T, const sp_mesh* M, int64_t mu, int64_t chunk,
                      uint64_t lo, uint64_t hi, int32_t threads, double* totals, sp_score_out* out) {
  block_ctx B;
  int rc = block_init(&B, Gp, tmpl, T, M, mu, chunk);
  if (rc != SP_OK) return rc;
  memset(out, 0, sizeof(*out));
  uint64_t C;
  if (!block_count(&B, &C)) {
    block_free(&B);
    return SP_ERR_UNSUPPORTED;
  }
  out->candidates = C;
  if (hi > C) hi = C;
  if (lo > hi) lo = hi;
  if (threads < 1) threads = 1;
  uint64_t n = hi - lo;
  if ((uint64_t)threads > n) threads = (int32_t)(n ? n : 1);
  worker* ws = (worker*)calloc((size_t)threads, sizeof(worker));
  pthread_t* th = (pthread_t*)calloc((size_t)threads, sizeof(pthread_t));
  uint64_t step = (n + (uint64_t)threads - 1) / (uint64_t)threads;
  for (int t = 0; t < threads; t++) {
    ws[t].B = &B;
    ws[t].lo = lo + step * (uint64_t)t;
    ws[t].hi = ws[t].lo + step;
    if (ws[t].lo > hi) ws[t].lo = hi;
    if (ws[t].hi > hi) ws[t].hi = hi;
    ws[t].totals = totals ? totals + (ws[t].lo - lo) : NULL;
    if (threads > 1) pthread_create(&th[t], NULL, work, &ws[t]);
    else work(&ws[t]);
  }
  for (int t = 0; t < threads; t++) {
    if (threads > 1) pthread_join(th[t], NULL);
    out->valid += ws[t].res.valid;
    if (ws[t].res.has_best &&
        key_less(ws[t].res.best_total, ws[t].res.best_num_split, ws[t].res.best_index, out)) {
      out->has_best = 1;
      out->best_total = ws[t].res.best_total;
      out->best_num_split = ws[t].res.best_num_split;
      out->best_index = ws[t].res.best_index;
    }
  }
  free(ws);
  free(th);
  block_free(&B);
  return SP_OK;
}

/* Routing/cost detail of one candidate, same layout as sp_explain. */
static int explain_core(og* Gp, const int32_t* tmpl, int64_t T, const sp_mesh* M, int64_t mu,
                        int64_t chunk, uint64_t index, sp_explain_out* out);

int oracle_explain(const sp_graph* g, const int32_t* tmpl, int64_t T, const sp_mesh* M, int64_t mu,
                   int64_t chunk, uint64_t index, sp_explain_out* out) {
  og G;
  og_init(&G, g);
  int rc = explain_core(&G, tmpl, T, M, mu, chunk, index, out);
  og_free(&G);
  return rc;
}

int oracle_explain_h(void* h, const int32_t* tmpl, int64_t T, const sp_mesh* M, int64_t mu, int64_t chunk,
                     uint64_t index, sp_explain_out* out) {
  return explain_core((og*)h, tmpl, T, M, mu, chunk, index, out);
}

static int explain_core(og* Gp, const int32_t* tmpl, int64_t T, const sp_mesh* M, int64_t mu,
                        int64_t chunk, uint64_t index, sp_explain_out* out) {
  if (T > SP_EXPLAIN_MAX_T) return SP_ERR_UNSUPPORTED;  /* the fixed-size explain record */
  block_ctx B;
  int rc = block_init(&B, Gp, tmpl, T, M, mu, chunk);
  if (rc != SP_OK) return rc;
  cand_result* R = (cand_result*)calloc(1, sizeof(cand_result));
  eval_candidate(&B, index, R, 1);
  memset(out, 0, sizeof(*out));
  out->valid = R->valid;
  out->T = (int32_t)T;
  out->fail_pos = R->fail_pos;
  if (R->valid) {
    for (int64_t i = 0; i < T; i++) {
      out->pattern[i] = R->pat[i];
      out->state_axis[i] = R->state[i].kind == K_SPLIT ? R->state[i].axis : -1;
      out->exit_axis[i] = R->exit_axis[i];
    }
    out->forward_comm = R->forward;
    out->backward_comm = R->backward;
    out->total = R->total;
    out->bytes_allreduce = R->bytes[C_AR];
    out->bytes_allgather = R->bytes[C_AG];
    out->bytes_reducescatter = R->bytes[C_RS];
    out->bytes_alltoall = R->bytes[C_A2A];
    out->calls_allreduce = R->calls[C_AR];
    out->calls_allgather = R->calls[C_AG];
    out->calls_reducescatter = R->calls[C_RS];
    out->calls_alltoall = R->calls[C_A2A];
    out->collective_calls = R->calls[C_AR] + R->calls[C_AG] + R->calls[C_RS] + R->calls[C_A2A];
  }
  free(R);
  block_free(&B);
  return SP_OK;
}

/* weight slot order (weight_nodes) of a template, for label reconstruction in tests */
int oracle_slots(const sp_graph* g, const int32_t* tmpl, int64_t T, int32_t* slot_pos, int32_t* n_slots) {
  og G;
  og_init(&G, g);
  block_ctx B;
  sp_mesh M;
  memset(&M, 0, sizeof(M));
  M.m = M.n = 1;
  int rc = block_init(&B, &G, tmpl, T, &M, 1, 1);
  if (rc == SP_OK) {
    for (int s = 0; s < B.V; s++) slot_pos[s] = B.slot_pos[s];
    *n_slots = B.V;
    block_free(&B);
  }
  og_free(&G);
  return rc;
}
