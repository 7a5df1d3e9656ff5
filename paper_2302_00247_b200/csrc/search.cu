// Per-block routing tables and batched candidate scoring.
//
// Scoring one candidate in the reference is pattern_routing (search.py:134-224)
// followed by plan_cost (costmodel.py:193-267) and pack_gradients
// (rewrite.py:78-111).  Routing a template node is a pure function of (its
// weight digit, the shard states of its internal producers): node states are
// always one of R / S(0) / S(rank-1).  tables_build evaluates that function
// once per (node, digit, producer-state tuple) on the device and stores the
// chosen pattern and output state in a byte table; the conversion and pattern
// collective costs it needs for the forward longest-path DP go into small
// fp64 tables.  The scoring kernel then resolves a candidate with one byte
// lookup and a few fp64 adds/maxes per node, with everything staged in shared
// memory.  All fp64 arithmetic keeps the reference's operation order
// (round-to-nearest, no contraction), so totals are bit-identical.
#include <cub/cub.cuh>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstdio>
#include <numeric>

#include "patterns.cuh"
#include "sp_internal.h"

namespace sp {

namespace {

constexpr int KMAX = 6;          // internal producers handled by a lookup table
constexpr int MAXT = 256;        // template nodes per block (SP_EXPLAIN_MAX_T)
constexpr int THREADS = 256;     // scoring CTA size
// (-DSP_ITEM_ITERS for A/B builds: 256 / 128 / 64 give c5 32.5 / 31.9 / 31.9 ms --
// a one-GPU search's last wave of items is its tail)
#ifndef SP_ITEM_ITERS
#define SP_ITEM_ITERS 128
#endif
constexpr int ITEM_ITERS_MAX = SP_ITEM_ITERS;  // work item = THREADS * iters candidates
constexpr int ITEM_ITERS_MAX_SKIP = 512;   // ... when prefix skipping is on
// work items per resident CTA a search aims for (a rank's last wave of items is
// its tail: at 8 ranks c5's 65536-candidate items left ~12 per CTA; 8 / 32 / 64 /
// 128 per CTA: 5.65 / 4.90 / 4.71 / 4.72 ms per rank, tools/ab_items.sh)
constexpr int ITEMS_PER_CTA = 64;

__host__ __device__ inline int64_t align16(int64_t x) { return (x + 15) & ~(int64_t)15; }
__host__ __device__ inline uint32_t pow3(int k) {
  uint32_t r = 1;
  for (int i = 0; i < k; i++) r *= 3;
  return r;
}

struct GraphView {
  const uint8_t* op;
  const uint8_t* act_rank;
  const int64_t* act_shape;
  const int64_t* act_bytes;
  const uint8_t* w_rank;
  const int64_t* w_shape;
  const int64_t* w_bytes;
  const uint8_t* w_train;
  const int64_t* in_off;
  const int32_t* in_idx;
};

// Routing of one node for a given digit and internal producer states
// (search.py:153-211).  prod_state[j] indexes R/S0/S(rank-1) of the j-th
// internal producer in GraphNode.inputs order.  Returns the chosen pattern
// (-1 = RoutingFailure) and its output state index; optionally the
// conversion collective on each internal edge.
struct NodeRoute {
  int pattern;
  int state;
  int8_t conv_kind[64];
  int8_t conv_axis[64];
};

__host__ __device__ bool weight_ok(const Pattern& pt, int wrank, const int64_t* wshape, int digit, int64_t d) {
  if (pt.w.kind == K_NONE) return false;  // pattern without a weight spec never matches a weight
  NSpec want;
  if (!normalize(pt.w, wrank, &want)) return false;
  // WEIGHT_OPTIONS_2D/1D (search.py:35-36): replica, split(0), split(1)
  NSpec assigned = digit == 0 ? NSpec{K_R, 0} : NSpec{K_S, (int8_t)(digit - 1)};
  if (!nspec_eq(want, assigned)) return false;
  if (assigned.kind == K_S && (wshape[assigned.axis] % d) != 0) return false;
  return true;
}

__device__ void route_node(const GraphView& G, int32_t n, int32_t blk, const int32_t* node_block,
                           int digit, const int* prod_state, const MeshC& M, NodeRoute* out,
                           bool want_conv) {
  Pattern pats[4];
  const int np = patterns_for(G.op[n], pats);
  const int arank = G.act_rank[n];
  const int64_t* ashape = G.act_shape + (int64_t)n * SP_MAX_RANK;
  int best = -1;
  double best_c = 0.0;
  NSpec best_out{K_R, 0};
  for (int p = 0; p < np; p++) {
    const Pattern& pt = pats[p];
    if (G.w_rank[n] && !weight_ok(pt, G.w_rank[n], G.w_shape + (int64_t)n * SP_MAX_RANK, digit, M.d)) continue;
    double c = 0.0;
    bool feasible = true;
    int j = 0;
    for (int64_t e = G.in_off[n]; e < G.in_off[n + 1]; e++) {
      const int32_t r = G.in_idx[e];
      const bool internal = node_block[r] == blk;
      const int rr = G.act_rank[r];
      const NSpec st = internal ? state_spec(prod_state[j], rr) : NSpec{K_R, 0};
      NSpec req;
      int8_t kind, axis;
      if (!normalize(pt.in, rr, &req) ||
          !convert(st, req, G.act_shape + (int64_t)r * SP_MAX_RANK, M.d, &kind, &axis)) {
        feasible = false;
        break;
      }
      if (kind != C_ID) c = dadd(c, call_cost(kind, G.act_bytes[r], M));
      if (internal) j++;
    }
    if (!feasible) continue;
    NSpec o;
    if (!normalize(pt.out, arank, &o)) continue;
    if (o.kind == K_S && (ashape[o.axis] % M.d) != 0) continue;
    c = dadd(c, call_cost(pt.coll, G.act_bytes[n], M));
    if (best < 0 || c < best_c) {  // min by (cost, pattern index)
      best = p;
      best_c = c;
      best_out = o;
    }
  }
  out->pattern = best;
  if (best < 0) {
    out->state = 0;
    return;
  }
  // apply_collective: the only non-identity pattern collective is AllReduce -> R
  const NSpec fin = pats[best].coll == C_AR ? NSpec{K_R, 0} : best_out;
  out->state = state_index(fin, arank);
  if (want_conv) {
    int j = 0;
    for (int64_t e = G.in_off[n]; e < G.in_off[n + 1]; e++) {
      const int32_t r = G.in_idx[e];
      if (node_block[r] != blk) continue;
      const int rr = G.act_rank[r];
      NSpec req;
      normalize(pats[best].in, rr, &req);
      int8_t kind = C_ID, axis = -1;
      convert(state_spec(prod_state[j], rr), req, G.act_shape + (int64_t)r * SP_MAX_RANK, M.d, &kind, &axis);
      if (j < 64) {
        out->conv_kind[j] = kind;
        out->conv_axis[j] = axis;
      }
      j++;
    }
  }
}

struct EntryLayout {
  int32_t k, nd, out_pool, prod, tab, dbl, train_idx, skip_m;
  uint64_t skip_R;
  int32_t tab4, pad;
};

constexpr int TAB4_PAD = 512;  // failed lanes index past a table by < 3^KMAX / 2 bytes

// Winner re-routing data kept beside the blob (not staged by the scorers):
// per template node its output bytes, op and rank; per internal edge the
// conversion collective and axis for every (pattern, producer state) pair,
// as k_fill's route_node evaluation found them (kind -1: no conversion).
struct XNode {
  int64_t act_bytes;
  uint8_t op, act_rank, pad[6];
};
struct XEdge {
  int8_t kind[4][3], axis[4][3];
};

__global__ void k_mark_blocks(const int64_t* tmpl_off, const int32_t* tmpl_nodes, int64_t nb,
                              int32_t* node_block, int32_t* node_tpos, int32_t* dup) {
  for (int64_t b = blockIdx.x; b < nb; b += gridDim.x)
    for (int64_t e = tmpl_off[b] + threadIdx.x; e < tmpl_off[b + 1]; e += blockDim.x) {
      const int32_t n = tmpl_nodes[e];
      if (atomicExch(&node_block[n], (int32_t)b) != -1) atomicExch(dup, 1);
      node_tpos[n] = (int32_t)(e - tmpl_off[b]);
    }
}

__global__ void k_boundary(GraphView G, int64_t n, const int32_t* node_block, uint8_t* has_cons,
                           uint8_t* ext_cons) {
  for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < n; c += (int64_t)gridDim.x * blockDim.x)
    for (int64_t e = G.in_off[c]; e < G.in_off[c + 1]; e++) {
      const int32_t p = G.in_idx[e];
      has_cons[p] = 1;
      if (node_block[c] != node_block[p] || node_block[p] < 0) ext_cons[p] = 1;
    }
}

// The serial half of a block's layout (k_layout's lane 0, and the host layout
// of small graphs): lays out the blob, assigns pool slots (linear scan; a
// producer's slot is released at its last internal consumer) and derives each
// node's prefix-failure skip (ancestor cone over enumeration positions).
// Per template position i: kk[i] internal fan-in, prodpos[i][] producer
// positions, rel_head[i] -> rel_next[] the producers whose last internal
// consumer is i, slot_of / radix_of its enumeration slot and radix, trainw
// whether it holds a trainable weight.  pool / ancs: scratch of T entries,
// suf: scratch of V + 1.  Every input is read from the caller's (shared)
// arrays: the walk has no global-memory dependency chain.
template <class IDX>
__host__ __device__ inline void layout_serial(int T, const IDX* kk, const int* last, const int16_t (*prodpos)[KMAX],
                                              const int* rel_head, const IDX* rel_next, IDX* pool, uint64_t* ancs,
                                              uint64_t* suf, const int16_t* slot_of, const uint8_t* radix_of,
                                              const uint8_t* trainw, BlobHeader& H, EntryLayout* lay) {
  const int V = H.V;
  int nprod = 0, nt = 0;
  int64_t nent = 0, ndbl = 0, nent4 = 0;
  uint32_t used[MAXT / 32];
  for (int w = 0; w < MAXT / 32; w++) used[w] = 0;
  // suffix products of the enumeration radices: skip_R = suf[skip_m + 1]
  suf[V > 0 ? V : 0] = 1;
  for (int q = V - 1; q >= 0; q--) suf[q] = suf[q + 1] * (((H.radix3 >> q) & 1) ? 3 : 2);
  int npool = 0;
  for (int i = 0; i < T; i++) {
    // release producers whose last internal consumer is i
    for (int j = rel_head[i]; j >= 0; j = rel_next[j])
      if (pool[j] >= 0) used[pool[j] >> 5] &= ~(1u << (pool[j] & 31));
    pool[i] = -1;
    if (last[i] >= 0) {
      int sl = 0;
      for (int w = 0; w < MAXT / 32; w++)
        if (~used[w]) {
#ifdef __CUDA_ARCH__
          sl = w * 32 + __ffs(~used[w]) - 1;
#else
          sl = w * 32 + __builtin_ctz(~used[w]);
#endif
          break;
        }
      used[sl >> 5] |= 1u << (sl & 31);
      pool[i] = (IDX)sl;
      npool = npool > sl + 1 ? npool : sl + 1;
    }
    const int k = kk[i];
    // ancestor cone over enumeration positions (V <= 64)
    uint64_t anc = slot_of[i] >= 0 ? (1ULL << slot_of[i]) : 0ULL;
    for (int j = 0; j < k && j < KMAX; j++) anc |= ancs[prodpos[i][j]];
    ancs[i] = anc;
    EntryLayout L;
    L.k = k;
    L.nd = slot_of[i] >= 0 ? radix_of[i] : 1;
    L.prod = nprod;
    L.tab = (int32_t)nent;
    L.tab4 = (int32_t)nent4;
    L.pad = 0;
    L.dbl = (int32_t)ndbl;
    L.train_idx = trainw[i] ? nt++ : -1;
    L.out_pool = pool[i];
#ifdef __CUDA_ARCH__
    L.skip_m = anc ? 63 - __clzll(anc) : -1;
#else
    L.skip_m = anc ? 63 - __builtin_clzll(anc) : -1;
#endif
    L.skip_R = anc ? (L.skip_m + 1 <= V ? suf[L.skip_m + 1] : 1) : 0;
    nprod += k;
    nent += (int64_t)L.nd * pow3(k < KMAX ? k : KMAX);
    nent4 += 4 * (int64_t)pow3(k < KMAX ? k : KMAX);
    ndbl += 8 + 12 * (int64_t)k;
    lay[i] = L;
  }
  H.T = T;
  H.nt = nt;
  H.npool = npool;
  H.n_prod = nprod;
  int64_t off = sizeof(BlobHeader);
  H.desc_off = (int32_t)off;
  off = align16(off + 16 * (int64_t)T);
  H.skip_off = (int32_t)off;
  off = align16(off + (int64_t)sizeof(NodeSkip) * T);
  H.stride_off = (int32_t)off;
  off = align16(off + 9 * (int64_t)V);
  H.dirty_off = (int32_t)off;
  off = align16(off + 8 * ((int64_t)V + 1));
  H.prod_off = (int32_t)off;
  off = align16(off + 4 * (int64_t)nprod);  // i16 pool slots, then i16 producer positions
  H.tab_off = (int32_t)off;
  off = align16(off + nent);
  H.dbl_off = (int32_t)off;
  off = align16(off + 8 * ndbl);
  H.train_off = (int32_t)off;
  off = align16(off + (int64_t)sizeof(TrainDesc) * nt);
  H.tslot_off = (int32_t)off;
  off = align16(off + 16 * (int64_t)V);
  H.fast_off = (int32_t)off;
  off = align16(off + (int64_t)sizeof(FastNode) * T);
  H.zero_off = (int32_t)off;
  off += 128;
  H.fprod_off = (int32_t)off;
  off = align16(off + 8 * (int64_t)nprod);
  H.tab4_off = (int32_t)off;
  off = align16(off + nent4 + TAB4_PAD);
  H.bytes = (int32_t)off;
}

constexpr int LAYOUT_WARPS = 4;
// One WARP per block: the lanes gather each node's internal fan-in, producer
// positions, last internal consumer, release lists, slot, radix and weight
// flag into shared memory, then lane 0 runs layout_serial on shared memory only.
__global__ void __launch_bounds__(32 * LAYOUT_WARPS) k_layout(GraphView G, const int64_t* tmpl_off,
                                                             const int32_t* tmpl_nodes, int64_t nb,
                                                             const int32_t* node_block, const int32_t* node_tpos,
                                                             const int16_t* slot_of, const uint8_t* radix_of,
                                                             EntryLayout* lay, BlobHeader* hdr, int64_t* blob_bytes,
                                                             int32_t* err) {
  __shared__ int s_last[LAYOUT_WARPS][MAXT], s_head[LAYOUT_WARPS][MAXT];
  __shared__ int16_t s_k[LAYOUT_WARPS][MAXT], s_next[LAYOUT_WARPS][MAXT], s_pool[LAYOUT_WARPS][MAXT];
  __shared__ int16_t s_prodpos[LAYOUT_WARPS][MAXT][KMAX];
  __shared__ uint64_t s_anc[LAYOUT_WARPS][MAXT];
  __shared__ uint64_t s_suf[LAYOUT_WARPS][65];
  __shared__ int16_t s_slot[LAYOUT_WARPS][MAXT];
  __shared__ uint8_t s_rad[LAYOUT_WARPS][MAXT], s_tw[LAYOUT_WARPS][MAXT];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int64_t b = (int64_t)blockIdx.x * LAYOUT_WARPS + w; b < nb; b += (int64_t)gridDim.x * LAYOUT_WARPS) {
    const int64_t e0 = tmpl_off[b];
    const int T = (int)(tmpl_off[b + 1] - e0);
    for (int i = lane; i < T; i += 32) {
      s_last[w][i] = -1;
      s_head[w][i] = -1;
    }
    __syncwarp();
    for (int i = lane; i < T; i += 32) {
      const int32_t n = tmpl_nodes[e0 + i];
      int k = 0;
      for (int64_t e = G.in_off[n]; e < G.in_off[n + 1]; e++) {
        const int32_t r = G.in_idx[e];
        if (node_block[r] != (int32_t)b) continue;
        const int j = node_tpos[r];
        if (j >= i) atomicExch(err, 2);  // template not topologically ordered
        else atomicMax(&s_last[w][j], i);
        if (k < KMAX) s_prodpos[w][i][k] = (int16_t)j;
        k++;
      }
      if (k > KMAX) atomicExch(err, 3);
      s_k[w][i] = (int16_t)k;
      s_slot[w][i] = slot_of[e0 + i];
      s_rad[w][i] = radix_of[e0 + i];
      s_tw[w][i] = (G.w_rank[n] && G.w_train[n]) ? 1 : 0;
    }
    __syncwarp();
    for (int j = lane; j < T; j += 32)
      if (s_last[w][j] >= 0) s_next[w][j] = (int16_t)atomicExch(&s_head[w][s_last[w][j]], j);
    __syncwarp();
    if (lane == 0 && *(volatile int32_t*)err == 0) {
      BlobHeader H = hdr[b];
      layout_serial(T, s_k[w], s_last[w], s_prodpos[w], s_head[w], s_next[w], s_pool[w], s_anc[w], s_suf[w],
                    s_slot[w], s_rad[w], s_tw[w], H, lay + e0);
      hdr[b] = H;
      blob_bytes[b] = H.bytes;
    }
    __syncwarp();
  }
}

// One CTA per block: node descriptors, producer pool slots, fp64 tables and
// the routing byte table (one thread per (node, key)); thread 0 writes the
// header.
__global__ void k_fill(GraphView G, const int64_t* tmpl_off, const int32_t* tmpl_nodes, int64_t nb,
                       const int32_t* node_block, const int32_t* node_tpos, const int16_t* slot_of,
                       const int16_t* ref_slot_of,
                       const EntryLayout* lay, const BlobHeader* hdr_in, const int64_t* blob_off,
                       const uint8_t* has_cons, const uint8_t* ext_cons, sp_mesh mesh, int64_t mu,
                       int64_t chunk, uint8_t* blobs, uint8_t* bound_of, uint8_t* xinfo, const int64_t* xoff) {
  const MeshC M = mesh_consts(mesh);
  __shared__ uint32_t s_kbase[MAXT + 1];
  __shared__ uint32_t s_cnt[MAXT];
  __shared__ int16_t s_outpool[MAXT];
  __shared__ int8_t s_skipm[MAXT], s_rslot[MAXT], s_eslot[MAXT];
  __shared__ uint8_t s_rr[64];
  __shared__ unsigned long long s_tms, s_tmb;  // trainable-weight field masks (BlobHeader)
  for (int64_t b = blockIdx.x; b < nb; b += gridDim.x) {
    const int64_t e0 = tmpl_off[b];
    const int T = (int)(tmpl_off[b + 1] - e0);
    const BlobHeader& H = hdr_in[b];
    uint8_t* blob = blobs + blob_off[b];
    const int V = H.V;
    const uint64_t radix3 = H.radix3;
    // per-node fields staged once (every later pass reads them from shared memory)
    int8_t* perm = (int8_t*)(blob + H.stride_off + 8 * V);  // reference slot -> enumeration position
    for (int i = threadIdx.x; i < T; i += blockDim.x) {
      const EntryLayout L = lay[e0 + i];
      const int rs = ref_slot_of[e0 + i], es = slot_of[e0 + i];
      s_cnt[i] = (uint32_t)L.nd * pow3(L.k);
      s_outpool[i] = (int16_t)L.out_pool;
      s_skipm[i] = (int8_t)L.skip_m;
      s_rslot[i] = (int8_t)rs;
      s_eslot[i] = (int8_t)es;
      if (rs >= 0) {
        s_rr[rs] = ((radix3 >> es) & 1) ? 3 : 2;
        perm[rs] = (int8_t)es;
      }
    }
    for (int q = threadIdx.x; q < 128; q += blockDim.x) blob[H.zero_off + q] = 0;
    if (threadIdx.x == 0) {
      s_tms = s_tmb = 0;
      BlobHeader h = H;
      h.multi_dev = M.d > 1;
      h.setup = M.setup;
      h.c_ar = ddiv(dmul(2.0, (double)(M.d - 1)), (double)M.d);
      h.bw = M.bw;
      h.eff_ar = M.eff[C_AR];
      h.keep_bwd = dadd(1.0, -mesh.overlap_fraction);
      h.mu = mu;
      h.chunk = chunk;
      uint64_t bias = 0;
      for (int q = 0; q < V && V <= 32; q++) bias |= (uint64_t)(((radix3 >> q) & 1) ? 1 : 2) << (2 * (V - 1 - q));
      h.bias = bias;
      h.tmask_small = h.tmask_big = 0;
      h.pad4 = 0;
      *(BlobHeader*)blob = h;
    }
    __syncthreads();
    // reference strides per enumeration position
    uint64_t* stride = (uint64_t*)(blob + H.stride_off);
    for (int i = threadIdx.x; i < T; i += blockDim.x)
      if (s_rslot[i] >= 0) {
        uint64_t st = 1;
        for (int s2 = s_rslot[i] + 1; s2 < V; s2++) st *= s_rr[s2];
        stride[s_eslot[i]] = st;
      }
    // memoised scoring: dirty[q] = nodes to re-route when enumeration positions >= q change
    uint64_t* dirty = (uint64_t*)(blob + H.dirty_off);
    for (int q = threadIdx.x; q <= V; q += blockDim.x) {
      uint64_t mask = 0;
      for (int i = 0; i < T && i < 64; i++)
        if (q == 0 || s_skipm[i] >= q) mask |= 1ULL << i;
      dirty[q] = mask;
    }
    // routing-table key offsets: exclusive scan of nd * 3^k (warp 0)
    if (threadIdx.x < 32) {
      const int lane = threadIdx.x;
      uint32_t acc = 0;
      for (int base = 0; base < T; base += 32) {
        const uint32_t v = base + lane < T ? s_cnt[base + lane] : 0;
        uint32_t x = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
          if (lane >= o) x += y;
        }
        if (base + lane < T) s_kbase[base + lane] = acc + x - v;
        acc += __shfl_sync(0xffffffffu, x, 31);
      }
      if (lane == 0) s_kbase[T] = acc;
    }
    __syncthreads();
    // per-node records
    for (int i = threadIdx.x; i < T; i += blockDim.x) {
      const int64_t e = e0 + i;
      const int32_t n = tmpl_nodes[e];
      const EntryLayout L = lay[e];
      NodeDesc nd;
      nd.slot = slot_of[e];
      nd.k = (uint8_t)L.k;
      nd.nd = (uint8_t)L.nd;
      nd.out_pool = (int16_t)L.out_pool;
      nd.prod = (uint16_t)L.prod;
      nd.tab = (uint32_t)L.tab;
      nd.dbl = (uint32_t)L.dbl;
      ((NodeDesc*)(blob + H.desc_off))[i] = nd;
      {
        // lean-walk record: ready-made smem byte offsets (pool slot p of lane t:
        // reach at pool + (p*THREADS + t)*8, state at pool_states + p*THREADS + t)
        FastNode f;
        f.tab = H.tab4_off + L.tab4;
        f.dbl = H.dbl_off + 8 * L.dbl;
        f.cb0 = L.k >= 1 ? H.dbl_off + 8 * (L.dbl + 8) : H.zero_off;
        f.cb1 = L.k >= 2 ? H.dbl_off + 8 * (L.dbl + 8 + 12) : H.zero_off;
        f.r0 = f.r1 = 0;
        int jj = 0;
        for (int64_t q = G.in_off[n]; q < G.in_off[n + 1]; q++) {
          const int32_t r = G.in_idx[q];
          if (node_block[r] != (int32_t)b) continue;
          const int ps = s_outpool[node_tpos[r]];
          if (L.k <= 2) {
            if (jj == 0) f.r0 = ps * THREADS * 8;
            else f.r1 = ps * THREADS * 8;
          } else {
            int32_t* fp = (int32_t*)(blob + H.fprod_off) + 2 * (L.prod + jj);
            fp[0] = ps * THREADS * 8;
            fp[1] = ps * THREADS;
          }
          jj++;
        }
        if (L.k >= 3) f.r0 = L.prod;
        // -1: no internal consumer (only boundary nodes; the paired walk
        // stores non-boundary results unguarded)
        f.out_r = L.out_pool >= 0 ? L.out_pool * THREADS * 8 : -1;
        const int sh = nd.slot >= 0 && H.V <= 32 ? 2 * (H.V - 1 - nd.slot) : 0;  // (wide blocks: generic walk)
        // kf = k << 16 | boundary << 13 | min(k, 3) << 11 | one-hot class of the
        // three common non-boundary kinds (bit 8: k = 1, bit 9: k = 0, bit 10:
        // k = 2), which the paired walk tests first, in that order of frequency
        // | the digit shift in bits 0..5 (the walk shifts by kf & 63)
        const int bnd = (!has_cons[n] || ext_cons[n]) ? 1 : 0;
        const int kc = L.k < 3 ? L.k : 3;
        f.kf = (L.k << 16) | (bnd << 13) | (kc << 11) |
               ((bnd ? 0 : kc == 1 ? 1 : kc == 0 ? 2 : kc == 2 ? 4 : 0) << 8) | sh;
        ((FastNode*)(blob + H.fast_off))[i] = f;
      }
      ((NodeSkip*)(blob + H.skip_off))[i] = NodeSkip{L.skip_R, L.skip_m, 0};
      XNode* xn = (XNode*)(xinfo + xoff[b]) + i;
      xn->act_bytes = G.act_bytes[n];
      xn->op = G.op[n];
      xn->act_rank = G.act_rank[n];
      XEdge* xe = (XEdge*)(xinfo + xoff[b] + (int64_t)sizeof(XNode) * T) + L.prod;
      int16_t* prod = (int16_t*)(blob + H.prod_off) + L.prod;
      double* dbl = (double*)(blob + H.dbl_off) + L.dbl;
      Pattern pats[4];
      const int np = patterns_for(G.op[n], pats);
      // own[p]: pattern collective call cost on this node's activation
      for (int p = 0; p < 4; p++) dbl[p] = p < np ? call_cost(pats[p].coll, G.act_bytes[n], M) : 0.0;
      // exitc[s]: AllGather back to replica at a subgraph boundary (search.py:213-223)
      const bool boundary = !has_cons[n] || ext_cons[n];
      bound_of[e] = boundary;
      const double ag = boundary ? call_cost(C_AG, G.act_bytes[n], M) : 0.0;
      dbl[4] = 0.0;
      dbl[5] = ag;
      dbl[6] = ag;
      dbl[7] = 0.0;
      // conv[j][p][s]: internal edge conversion cost (0.0 for identity / infeasible)
      int j = 0;
      for (int64_t q = G.in_off[n]; q < G.in_off[n + 1]; q++) {
        const int32_t r = G.in_idx[q];
        if (node_block[r] != (int32_t)b) continue;
        prod[j] = s_outpool[node_tpos[r]];
        ((int16_t*)(blob + H.prod_off))[H.n_prod + L.prod + j] = (int16_t)node_tpos[r];
        const int rr = G.act_rank[r];
        for (int p = 0; p < 4; p++)
          for (int s = 0; s < 3; s++) {
            double c = 0.0;
            NSpec req;
            int8_t kind = C_ID, axis = -1;
            const bool ok = p < np && normalize(pats[p].in, rr, &req) &&
                            convert(state_spec(s, rr), req, G.act_shape + (int64_t)r * SP_MAX_RANK, M.d, &kind, &axis);
            if (ok && kind != C_ID) c = call_cost(kind, G.act_bytes[r], M);
            dbl[8 + (j * 4 + p) * 3 + s] = c;
            xe[j].kind[p][s] = ok ? kind : (int8_t)-1;
            xe[j].axis[p][s] = ok ? axis : (int8_t)-1;
          }
        j++;
      }
      if (L.train_idx >= 0) {
        TrainDesc td;
        td.slot = slot_of[e];
        td.pad = 0;
        td.size = G.w_bytes[n];
        td.uterm = dadd(M.setup, cost_bytes(C_AR, td.size, M));
        ((TrainDesc*)(blob + H.train_off))[L.train_idx] = td;
        if (H.V <= 32 && td.slot >= 0) {
          atomicOr(td.size >= mu ? &s_tmb : &s_tms, 1ULL << (2 * (H.V - 1 - td.slot)));
          ((double*)(blob + H.tslot_off))[td.slot] = td.uterm;
          ((int64_t*)(blob + H.tslot_off + 8 * H.V))[td.slot] = td.size;
        }
      }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      ((BlobHeader*)blob)->tmask_small = s_tms;
      ((BlobHeader*)blob)->tmask_big = s_tmb;
    }
    // routing byte tables: key = Horner(digit, s_0, ..., s_{k-1}) in base 3
    const uint32_t nkeys = s_kbase[T];
    for (uint32_t g = threadIdx.x; g < nkeys; g += blockDim.x) {
      int lo = 0, hi = T;
      while (hi - lo > 1) {
        const int mid = (lo + hi) / 2;
        if (s_kbase[mid] <= g) lo = mid;
        else hi = mid;
      }
      const int i = lo;
      const uint32_t key = g - s_kbase[i];
      const EntryLayout L = lay[e0 + i];
      int ps[KMAX];
      uint32_t x = key;
      for (int jj = L.k - 1; jj >= 0; jj--) {
        ps[jj] = (int)(x % 3);
        x /= 3;
      }
      NodeRoute R;
      route_node(G, tmpl_nodes[e0 + i], (int32_t)b, node_block, (int)x, ps, M, &R, false);
      const uint8_t val = R.pattern < 0 ? (uint8_t)0xFF : (uint8_t)(R.pattern | (R.state << 2));
      blob[H.tab_off + L.tab + key] = val;
      // 4-row table of the lean walk: row = biased digit (x + 4 - nd); byte =
      // pattern * 8 + state (0xFF = RoutingFailure), so the walk's own-cost
      // offset is one mask and the state another
      const uint32_t pk = pow3(L.k), rest = key - x * pk;
      uint8_t* t4 = blob + H.tab4_off + L.tab4 + rest;
      const uint8_t val4 = R.pattern < 0 ? (uint8_t)0xFF : (uint8_t)((R.pattern << 3) | R.state);
      if (slot_of[e0 + i] >= 0) {
        t4[(x + 4 - L.nd) * pk] = val4;
        if (x == 0)
          for (int bb = 0; bb < 4 - L.nd; bb++) t4[bb * pk] = 0xFF;  // unused rows
      } else {
        for (int bb = 0; bb < 4; bb++) t4[bb * pk] = val4;
      }
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// scoring

struct ItemOut {
  unsigned long long total_bits;  // ~0 when the item has no valid candidate
  unsigned long long index;
  uint32_t num_split;
  unsigned long long valid;  // 64-bit: k_score_flow writes one CTA's whole share of a block
};

__device__ __forceinline__ bool key_less(unsigned long long ta, uint32_t na, unsigned long long ia,
                                         unsigned long long tb, uint32_t nb, unsigned long long ib) {
  if (ta != tb) return ta < tb;
  if (na != nb) return na < nb;
  return ia < ib;
}

// max of two non-negative, non-NaN doubles: their bit patterns order like the
// values, so an integer max is exact (and cheaper than DSETP/SEL/FSEL).
__device__ __forceinline__ double dmax_nn(double a, double b) {
  const long long x = __double_as_longlong(a), y = __double_as_longlong(b);
  return __longlong_as_double(x > y ? x : y);
}

__device__ __forceinline__ uint32_t get_digit(uint64_t w0, uint64_t w1, int s) {
  return (uint32_t)(((s < 32 ? w0 : w1) >> ((s & 31) * 2)) & 3);
}

// digits += t in mixed radix (last slot fastest)
__device__ __forceinline__ void mr_add(uint64_t& w0, uint64_t& w1, uint32_t t, int V, uint64_t radix3) {
  for (int s = V - 1; s >= 0 && t; s--) {
    const int sh = (s & 31) * 2;
    uint64_t& w = s < 32 ? w0 : w1;
    const uint32_t d = (uint32_t)((w >> sh) & 3);
    const uint32_t v = d + t;
    uint32_t q, r;
    if ((radix3 >> s) & 1) {
      q = v / 3;
      r = v - q * 3;
    } else {
      q = v >> 1;
      r = v & 1;
    }
    w = (w & ~(3ULL << sh)) | ((uint64_t)r << sh);
    t = q;
  }
}

struct ScorePlan {
  const int64_t* blob_off;
  unsigned long long item_cands;        // candidates per work item
  const unsigned long long* stride;     // per block: index distance between a rank's consecutive items
  const unsigned long long* lo;         // per block start (enumeration index space)
  const unsigned long long* hi;
  const unsigned long long* item_base;  // prefix sum of items per block, [nb+1]
  int64_t nb;
  unsigned long long n_items;
  int skip;                             // exact prefix-failure skipping on/off
  // k_score_flow walk, the final wave: claims from n_main on are sub-items (a
  // 1/split part of one of the rank's last items of block fblk[e], walked in
  // FLOW_SUB warp chunks); item outputs of block b at obase[b] .. obase[b + 1]
  // (its whole items, then its sub-items).  Without a split: n_main = n_items,
  // obase = item_base.
  const unsigned long long* obase = nullptr;
  const unsigned long long* fblk = nullptr;   // [nf] block of each sub-item run (ascending)
  const unsigned long long* fbase = nullptr;  // [nf + 1] claim offsets (from n_main) of the runs
  int64_t nf = 0;
  unsigned long long n_main = ~0ULL;
  unsigned long long split = 1, sub = 0;      // parts per split item, candidates per part
  // k_score_flow: a block's items from cnt1[b] on are a second segment (lo2,
  // hi2, stride2: the relieved tail of the largest block); null: one segment
  const unsigned long long* cnt1 = nullptr;
  const unsigned long long *lo2 = nullptr, *hi2 = nullptr, *stride2 = nullptr;
};

// Pointers into a block's tables staged in shared memory.
struct Tabs {
  const BlobHeader* H;
  const NodeDesc* desc;
  const NodeSkip* skip;
  const uint64_t* stride;  // reference stride per enumeration position
  const int8_t* perm;      // reference slot -> enumeration position
  const int16_t* prodp;
  const uint8_t* tab;
  const double* dbl;
  const TrainDesc* trn;
  const double* tuterm;   // by enumeration position (backward_b)
  const int64_t* tsize;
  double* reach;
  uint8_t* stp;
};

__device__ __forceinline__ Tabs tabs_of(uint8_t* smem) {
  Tabs S;
  S.H = (const BlobHeader*)smem;
  const BlobHeader& H = *S.H;
  S.desc = (const NodeDesc*)(smem + H.desc_off);
  S.skip = (const NodeSkip*)(smem + H.skip_off);
  S.stride = (const uint64_t*)(smem + H.stride_off);
  S.perm = (const int8_t*)(smem + H.stride_off + 8 * H.V);
  S.prodp = (const int16_t*)(smem + H.prod_off);
  S.tab = smem + H.tab_off;
  S.dbl = (const double*)(smem + H.dbl_off);
  S.trn = (const TrainDesc*)(smem + H.train_off);
  S.tuterm = (const double*)(smem + H.tslot_off);
  S.tsize = (const int64_t*)(smem + H.tslot_off + 8 * H.V);
  S.reach = (double*)(smem + ((H.bytes + 15) & ~15));
  S.stp = (uint8_t*)(S.reach + (size_t)H.npool * THREADS);
  return S;
}

// pattern_routing + the forward DP of plan_cost for the lane's candidate
// (digits packed in enumeration order).  Returns -1 when it routes (fwd =
// forward time), else the first failing template position; T when inactive.
// Warp-collective: all 32 lanes call it (uniform node loop, ballot exit).
// Digit encodings: DM_WIDE = 2-bit digits at bits 2q of (w0, w1) (any V <= 64);
// DM_BIASED = one u64, position q at bits 2(V-1-q) holding digit + (4 - radix),
// so a plain integer add carries across mixed-radix positions (V <= 32).
enum : int { DM_WIDE = 1, DM_BIASED = 2 };

template <int DM>
__device__ __forceinline__ int walk(const Tabs& S, uint64_t w0, uint64_t w1, bool active, double& fwd, int tid) {
  // hoist everything loop-invariant into registers (the header lives in smem)
  const int T = S.H->T;
  const int sh_base = 2 * (S.H->V - 1);
  const NodeDesc* __restrict__ desc = S.desc;
  const int16_t* __restrict__ prodp = S.prodp;
  const uint8_t* __restrict__ tab = S.tab;
  const double* __restrict__ dbl = S.dbl;
  double* __restrict__ reach = S.reach + tid;
  uint8_t* __restrict__ stp = S.stp + tid;
  bool ok = active;
  int fail = active ? -1 : T;
  fwd = 0.0;
  for (int i = 0; i < T; i++) {
    const NodeDesc nd = desc[i];
    uint32_t key = 0;
    if (nd.slot >= 0) {
      if (DM == DM_WIDE) key = get_digit(w0, w1, nd.slot);
      else key = (uint32_t)((w0 >> (sh_base - 2 * nd.slot)) & 3) - (4u - nd.nd);
    }
    const double* D = dbl + nd.dbl;
    double r;
    int s;
    uint8_t e;
    // fan-in specialised paths (the node is warp-uniform: no divergence).
    // base = max(0.0, reach[p] + conv) needs no max for one producer: the
    // operands are >= +0.0, so the sum already is the max (bitwise).
    if (nd.k == 0) {
      e = tab[nd.tab + key];
      if (ok && e == 0xFF) { ok = false; fail = i; }
      if (!__any_sync(0xffffffffu, ok)) break;
      s = ok ? (e >> 2) & 3 : 0;
      r = D[e & 3];
    } else if (nd.k == 1) {
      const int ps0 = prodp[nd.prod];
      const int s0 = stp[ps0 * THREADS];
      const double r0 = reach[ps0 * THREADS];
      e = tab[nd.tab + key * 3 + s0];
      if (ok && e == 0xFF) { ok = false; fail = i; }
      if (!__any_sync(0xffffffffu, ok)) break;
      const int p = e & 3;
      s = ok ? (e >> 2) & 3 : 0;
      r = dadd(dadd(r0, D[8 + p * 3 + s0]), D[p]);
    } else if (nd.k == 2) {
      const int ps0 = prodp[nd.prod], ps1 = prodp[nd.prod + 1];
      const int s0 = stp[ps0 * THREADS], s1 = stp[ps1 * THREADS];
      const double r0 = reach[ps0 * THREADS], r1 = reach[ps1 * THREADS];
      e = tab[nd.tab + (key * 3 + s0) * 3 + s1];
      if (ok && e == 0xFF) { ok = false; fail = i; }
      if (!__any_sync(0xffffffffu, ok)) break;
      const int p = e & 3;
      s = ok ? (e >> 2) & 3 : 0;
      r = dadd(dmax_nn(dadd(r0, D[8 + p * 3 + s0]), dadd(r1, D[8 + (4 + p) * 3 + s1])), D[p]);
    } else {
      int sj[KMAX];
      double rj[KMAX];
      for (int j = 0; j < nd.k; j++) {
        const int ps = prodp[nd.prod + j];
        sj[j] = stp[ps * THREADS];
        rj[j] = reach[ps * THREADS];
        key = key * 3 + sj[j];
      }
      e = tab[nd.tab + key];
      if (ok && e == 0xFF) { ok = false; fail = i; }
      if (!__any_sync(0xffffffffu, ok)) break;
      const int p = e & 3;
      s = ok ? (e >> 2) & 3 : 0;
      double bse = 0.0;
      for (int j = 0; j < nd.k; j++) bse = dmax_nn(bse, dadd(rj[j], D[8 + (j * 4 + p) * 3 + sj[j]]));
      r = dadd(bse, D[p]);
    }
    fwd = dmax_nn(fwd, dadd(r, D[4 + s]));
    if (nd.out_pool >= 0) {
      reach[nd.out_pool * THREADS] = r;
      stp[nd.out_pool * THREADS] = (uint8_t)s;
    }
  }
  return ok ? -1 : fail;
}

__device__ __forceinline__ uint32_t opaque_u32(uint32_t x) {
  asm volatile("mov.b32 %0, %0;" : "+r"(x));
  return x;
}

// 32-bit shared-memory accesses (the walk keeps one shared base address in a
// register instead of re-deriving the generic shared window per access).
__device__ __forceinline__ uint32_t lds_u8(uint32_t a) {
  uint32_t v;
  asm volatile("ld.shared.u8 %0, [%1];" : "=r"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ double lds_f64(uint32_t a) {
  double v;
  asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ int32_t lds_s32(uint32_t a) {
  int32_t v;
  asm volatile("ld.shared.s32 %0, [%1];" : "=r"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ int4 lds_v4(uint32_t a) {
  int4 v;
  asm volatile("ld.shared.v4.s32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(a));
  return v;
}
__device__ __forceinline__ void sts_f64(uint32_t a, double v) {
  asm volatile("st.shared.f64 [%0], %1;" ::"r"(a), "d"(v) : "memory");
}
__device__ __forceinline__ void sts_u8(uint32_t a, uint32_t v) {
  asm volatile("st.shared.u8 [%0], %1;" ::"r"(a), "r"(v) : "memory");
}

// Lean walk over FastNode records (biased digit word `w`, V <= 32): the same
// routing + forward DP as walk<>, with every address precomputed by the table
// build and made absolute (shared window) when the blob is staged, so a node
// costs three record loads, one table byte and 1-3 fp64 operands.  `rec` is
// the shared address of FastNode[0], `rb`/`sb` the lane's reach/state pool
// bases.
// Failed or inactive lanes keep executing with masked garbage (pattern 3 /
// state 3 index stays inside the padded tables) until the whole warp has
// failed, exactly like walk<>'s ballot exit.  Only subgraph-boundary nodes
// update the forward max: an interior node's reach never exceeds its internal
// consumer's (conv, own >= 0 and rounding is monotone), so the max over
// boundary nodes is the max over all nodes.
template <bool TRACK>
__device__ __forceinline__ int walk_fast(uint32_t rec, int T, uint64_t w, bool active, double& fwd, uint32_t rb,
                                         uint32_t sb) {
  bool ok = active;
  int fail = active ? -1 : T;
  long long f = 0;  // bit pattern of the forward max (non-negative doubles)
  const uint32_t end = rec + (uint32_t)T * (uint32_t)sizeof(FastNode);
  // table byte e = pattern * 8 + state: pe = e & 0x18 is the own-cost byte
  // offset and 3 * pe the conversion-row offset; failure 0xFF masks to 3 / 3
#define SP_FAIL_CHECK(i)                        \
  {                                             \
    const bool bad = e == 0xFFu;                \
    if (TRACK && ok && bad) fail = (i);         \
    ok = ok && !bad;                            \
    if (!__any_sync(0xffffffffu, ok)) break;    \
  }
  for (int i = 0; rec != end; i++, rec += (uint32_t)sizeof(FastNode)) {
    // A = (tab, dbl, cb0, cb1) absolute, B = (r0, r1, s0, s1), X = (out_r, out_s, sh, kf)
    const int4 A = lds_v4(rec), R = lds_v4(rec + 16);
    // B = (r0, r1, s0, s1), X = (out_r, out_s, sh, kf): state offsets at 1/8 of the reach offsets
    const int4 B = make_int4(R.x, R.y, R.x >> 3, R.y >> 3);
    const int4 X = make_int4(R.z, R.z >> 3, R.w & 63, R.w);  // kf: kind bits tested in place
    const uint32_t b = (uint32_t)(w >> X.z) & 3u;
    const int kc = (X.w >> 11) & 3;  // fan-in, 3 = general
    uint32_t e;
    double r;
    if (kc == 1) {
      const uint32_t s0 = lds_u8(sb + B.z);
      const double r0 = lds_f64(rb + B.x);
      e = lds_u8(A.x + b * 3 + s0);
      SP_FAIL_CHECK(i)
      const uint32_t pe = e & 0x18u;
      r = dadd(dadd(r0, lds_f64(A.z + pe * 3 + s0 * 8)), lds_f64(A.y + pe));
    } else if (kc == 2) {
      const uint32_t s0 = lds_u8(sb + B.z), s1 = lds_u8(sb + B.w);
      const double r0 = lds_f64(rb + B.x), r1 = lds_f64(rb + B.y);
      e = lds_u8(A.x + b * 9 + s0 * 3 + s1);
      SP_FAIL_CHECK(i)
      const uint32_t pe = e & 0x18u;
      r = dadd(dmax_nn(dadd(r0, lds_f64(A.z + pe * 3 + s0 * 8)), dadd(r1, lds_f64(A.w + pe * 3 + s1 * 8))),
               lds_f64(A.y + pe));
    } else if (kc == 0) {
      e = lds_u8(A.x + b);
      SP_FAIL_CHECK(i)
      r = lds_f64(A.y + (e & 0x18u));
    } else {
      const int k = X.w >> 16;
      const uint32_t pp = (uint32_t)B.x;  // absolute address of the (reach, state) offset pairs
      uint32_t key = b;
      for (int j = 0; j < k; j++) key = key * 3 + lds_u8(sb + lds_s32(pp + 8 * j + 4));
      e = lds_u8(A.x + key);
      SP_FAIL_CHECK(i)
      const uint32_t pe = e & 0x18u;
      double bse = 0.0;
      for (int j = 0; j < k; j++) {
        const uint32_t sj = lds_u8(sb + lds_s32(pp + 8 * j + 4));
        bse = dmax_nn(bse, dadd(lds_f64(rb + lds_s32(pp + 8 * j)), lds_f64(A.z + j * 96 + pe * 3 + sj * 8)));
      }
      r = dadd(bse, lds_f64(A.y + pe));
    }
    const uint32_t s = e & 3u;
    if (X.w & (1 << 13)) {
      const long long x = __double_as_longlong(dadd(r, lds_f64(A.y + 32 + s * 8)));
      f = x > f ? x : f;
    }
    if (X.x >= 0) {
      sts_f64(rb + X.x, r);
      sts_u8(sb + X.y, s);
    }
  }
#undef SP_FAIL_CHECK
  fwd = __longlong_as_double(f);
  return ok ? -1 : (TRACK ? fail : T);
}

// Make the staged FastNode table/cost offsets absolute shared addresses.
// With `pair` (two candidates per lane) every pool offset doubles: slot p of
// lane t holds candidate a at (2p*THREADS + t) and b one THREADS further.
__device__ __forceinline__ void patch_fast(uint8_t* smem, bool pair = false) {
  const BlobHeader& H = *(const BlobHeader*)smem;
  const uint32_t base = (uint32_t)__cvta_generic_to_shared(smem);
  FastNode* fn = (FastNode*)(smem + H.fast_off);
  const int32_t m = pair ? 2 : 1;
  for (int i = threadIdx.x; i < H.T; i += blockDim.x) {
    FastNode& f = fn[i];
    f.tab += (int32_t)base;
    f.dbl += (int32_t)base;
    f.cb0 += (int32_t)base;
    f.cb1 += (int32_t)base;
    const int k = f.kf >> 16;
    if (k >= 3) {
      int32_t* pp = (int32_t*)(smem + H.fprod_off) + 2 * f.r0;
      for (int j = 0; j < k; j++) {
        pp[2 * j] *= m;
        pp[2 * j + 1] *= m;
      }
      f.r0 = (int32_t)(base + (uint32_t)H.fprod_off + 8u * (uint32_t)f.r0);
    } else {
      f.r0 *= m;
    }
    f.r1 *= m;
    if (f.out_r >= 0) f.out_r *= m;
  }
}

template <int OFF>
__device__ __forceinline__ uint32_t lds_u8o(uint32_t a) {
  uint32_t v;
  asm volatile("ld.shared.u8 %0, [%1+%2];" : "=r"(v) : "r"(a), "n"(OFF));
  return v;
}
template <int OFF>
__device__ __forceinline__ double lds_f64o(uint32_t a) {
  double v;
  asm volatile("ld.shared.f64 %0, [%1+%2];" : "=d"(v) : "r"(a), "n"(OFF));
  return v;
}
template <int OFF>
__device__ __forceinline__ void sts_f64o(uint32_t a, double v) {
  asm volatile("st.shared.f64 [%0+%2], %1;" ::"r"(a), "d"(v), "n"(OFF) : "memory");
}
template <int OFF>
__device__ __forceinline__ void sts_u8o(uint32_t a, uint32_t v) {
  asm volatile("st.shared.u8 [%0+%2], %1;" ::"r"(a), "r"(v), "n"(OFF) : "memory");
}

// walk_fast for two candidates per lane (brute force): one record load and
// one dispatch per node serve both, and the two dependency chains interleave.
// Candidate b's pool entries sit THREADS entries after candidate a's.  The
// warp leaves when all 64 candidates have failed.  Returns valid bits
// (bit 0 = a, bit 1 = b).
// One node of the paired walk: K = fan-in (3 = general), BND = the node may
// set the forward max.  Returns false when every candidate of the warp failed.
template <int K, bool BND>
__device__ __forceinline__ bool pair_node(const int4& A, const int4& B, const int4& X, uint32_t ba, uint32_t bb,
                                          bool& oka, bool& okb, long long& fa, long long& fb, uint32_t rb,
                                          uint32_t sb) {
  constexpr int RB = THREADS * 8, SB = THREADS;
  uint32_t ea, eb;
  double ra, rx;
  if (K == 1) {
    const uint32_t ps = sb + B.z, pr = rb + B.x;
    const uint32_t s0a = lds_u8o<0>(ps), s0b = lds_u8o<SB>(ps);
    const double r0a = lds_f64o<0>(pr), r0b = lds_f64o<RB>(pr);
    ea = lds_u8(A.x + ba * 3 + s0a);
    eb = lds_u8(A.x + bb * 3 + s0b);
    oka = oka && ea != 0xFFu;
    okb = okb && eb != 0xFFu;
    if (!__any_sync(0xffffffffu, oka || okb)) return false;
    const uint32_t pa = ea & 0x18u, pb = eb & 0x18u;
    ra = dadd(dadd(r0a, lds_f64(A.z + pa * 3 + s0a * 8)), lds_f64(A.y + pa));
    rx = dadd(dadd(r0b, lds_f64(A.z + pb * 3 + s0b * 8)), lds_f64(A.y + pb));
  } else if (K == 2) {
    const uint32_t ps0 = sb + B.z, ps1 = sb + B.w, pr0 = rb + B.x, pr1 = rb + B.y;
    const uint32_t s0a = lds_u8o<0>(ps0), s1a = lds_u8o<0>(ps1);
    const uint32_t s0b = lds_u8o<SB>(ps0), s1b = lds_u8o<SB>(ps1);
    const double r0a = lds_f64o<0>(pr0), r1a = lds_f64o<0>(pr1);
    const double r0b = lds_f64o<RB>(pr0), r1b = lds_f64o<RB>(pr1);
    ea = lds_u8(A.x + ba * 9 + s0a * 3 + s1a);
    eb = lds_u8(A.x + bb * 9 + s0b * 3 + s1b);
    oka = oka && ea != 0xFFu;
    okb = okb && eb != 0xFFu;
    if (!__any_sync(0xffffffffu, oka || okb)) return false;
    const uint32_t pa = ea & 0x18u, pb = eb & 0x18u;
    ra = dadd(dmax_nn(dadd(r0a, lds_f64(A.z + pa * 3 + s0a * 8)), dadd(r1a, lds_f64(A.w + pa * 3 + s1a * 8))),
              lds_f64(A.y + pa));
    rx = dadd(dmax_nn(dadd(r0b, lds_f64(A.z + pb * 3 + s0b * 8)), dadd(r1b, lds_f64(A.w + pb * 3 + s1b * 8))),
              lds_f64(A.y + pb));
  } else if (K == 0) {
    ea = lds_u8(A.x + ba);
    eb = lds_u8(A.x + bb);
    oka = oka && ea != 0xFFu;
    okb = okb && eb != 0xFFu;
    if (!__any_sync(0xffffffffu, oka || okb)) return false;
    ra = lds_f64(A.y + (ea & 0x18u));
    rx = lds_f64(A.y + (eb & 0x18u));
  } else {
    const int k = X.w >> 16;
    const uint32_t pp = (uint32_t)B.x;
    uint32_t ka = ba, kb = bb;
    for (int j = 0; j < k; j++) {
      const uint32_t ps = sb + lds_s32(pp + 8 * j + 4);
      ka = ka * 3 + lds_u8o<0>(ps);
      kb = kb * 3 + lds_u8o<SB>(ps);
    }
    ea = lds_u8(A.x + ka);
    eb = lds_u8(A.x + kb);
    oka = oka && ea != 0xFFu;
    okb = okb && eb != 0xFFu;
    if (!__any_sync(0xffffffffu, oka || okb)) return false;
    const uint32_t pa = ea & 0x18u, pb = eb & 0x18u;
    double xa = 0.0, xb = 0.0;
    for (int j = 0; j < k; j++) {
      const uint32_t ps = sb + lds_s32(pp + 8 * j + 4), pr = rb + lds_s32(pp + 8 * j);
      const uint32_t sja = lds_u8o<0>(ps), sjb = lds_u8o<SB>(ps);
      xa = dmax_nn(xa, dadd(lds_f64o<0>(pr), lds_f64(A.z + j * 96 + pa * 3 + sja * 8)));
      xb = dmax_nn(xb, dadd(lds_f64o<RB>(pr), lds_f64(A.z + j * 96 + pb * 3 + sjb * 8)));
    }
    ra = dadd(xa, lds_f64(A.y + pa));
    rx = dadd(xb, lds_f64(A.y + pb));
  }
  const uint32_t sa = ea & 3u, sx = eb & 3u;
  if (BND) {
    const long long xa = __double_as_longlong(dadd(ra, lds_f64(A.y + 32 + sa * 8)));
    const long long xb = __double_as_longlong(dadd(rx, lds_f64(A.y + 32 + sx * 8)));
    fa = xa > fa ? xa : fa;
    fb = xb > fb ? xb : fb;
  }
  if (!BND || X.x >= 0) {  // a non-boundary node always has an internal consumer
    const uint32_t qr = rb + X.x, qs = sb + X.y;
    sts_f64o<0>(qr, ra);
    sts_f64o<RB>(qr, rx);
    sts_u8o<0>(qs, sa);
    sts_u8o<SB>(qs, sx);
  }
  return true;
}

// walk_fast for two candidates per lane (brute force): one record load and
// one dispatch per node serve both, and the two dependency chains interleave.
// Candidate b's pool entries sit THREADS entries after candidate a's.  The
// warp leaves when all 64 candidates have failed.  Returns valid bits
// (bit 0 = a, bit 1 = b).
__device__ __forceinline__ int walk_pair(uint32_t rec, int T, uint64_t wa, uint64_t wb, bool act_a, bool act_b,
                                         double& fwd_a, double& fwd_b, uint32_t rb, uint32_t sb) {
  bool oka = act_a, okb = act_b;
  long long fa = 0, fb = 0;
  const uint32_t end = rec + (uint32_t)T * (uint32_t)sizeof(FastNode);
  for (; rec != end; rec += (uint32_t)sizeof(FastNode)) {
    // A = (tab, dbl, cb0, cb1) absolute, B = (r0, r1, s0, s1), X = (out_r, out_s, sh, kf)
    const int4 A = lds_v4(rec), R = lds_v4(rec + 16);
    // B = (r0, r1, s0, s1), X = (out_r, out_s, sh, kf): state offsets at 1/8 of the reach offsets
    const int4 B = make_int4(R.x, R.y, R.x >> 3, R.y >> 3);
    const int4 X = make_int4(R.z, R.z >> 3, R.w & 63, R.w);  // kf: kind bits tested in place
    const uint32_t ba = (uint32_t)(wa >> X.z) & 3u, bb = (uint32_t)(wb >> X.z) & 3u;
    bool go;
    // bit tests, most frequent kind first (an if-chain on one value would be
    // turned into a compare tree)
    if (X.w & (1 << 8)) {
      go = pair_node<1, false>(A, B, X, ba, bb, oka, okb, fa, fb, rb, sb);
    } else if (X.w & (1 << 9)) {
      go = pair_node<0, false>(A, B, X, ba, bb, oka, okb, fa, fb, rb, sb);
    } else if (X.w & (1 << 10)) {
      go = pair_node<2, false>(A, B, X, ba, bb, oka, okb, fa, fb, rb, sb);
    } else {
      switch ((X.w >> 11) & 7) {  // min(fan-in, 3) | boundary << 2
        case 5: go = pair_node<1, true>(A, B, X, ba, bb, oka, okb, fa, fb, rb, sb); break;
        case 4: go = pair_node<0, true>(A, B, X, ba, bb, oka, okb, fa, fb, rb, sb); break;
        case 6: go = pair_node<2, true>(A, B, X, ba, bb, oka, okb, fa, fb, rb, sb); break;
        case 7: go = pair_node<3, true>(A, B, X, ba, bb, oka, okb, fa, fb, rb, sb); break;
        default: go = pair_node<3, false>(A, B, X, ba, bb, oka, okb, fa, fb, rb, sb); break;
      }
    }
    if (!go) break;
  }
  fwd_a = __longlong_as_double(fa);
  fwd_b = __longlong_as_double(fb);
  return (oka ? 1 : 0) | (okb ? 2 : 0);
}

// backward of plan_cost: pack_gradients over replicated trainable weights
// (template order), buckets first then unfused, one AllReduce each.
__device__ __forceinline__ double backward(const Tabs& S, uint64_t w0, uint64_t w1) {
  const BlobHeader& H = *S.H;
  double bwd = 0.0;
  if (!H.multi_dev) return bwd;
  long long cur = 0;
  int cur_n = 0;
  for (int q = 0; q < H.nt; q++) {
    const TrainDesc td = S.trn[q];
    if (get_digit(w0, w1, td.slot) != 0 || td.size >= H.mu) continue;
    if (cur + td.size > H.chunk && cur_n) {
      bwd = dadd(bwd, dadd(H.setup, dmul(ddiv(dmul(H.c_ar, (double)cur), H.bw), H.eff_ar)));
      cur = 0;
      cur_n = 0;
    }
    cur += td.size;
    cur_n++;
  }
  if (cur_n) bwd = dadd(bwd, dadd(H.setup, dmul(ddiv(dmul(H.c_ar, (double)cur), H.bw), H.eff_ar)));
  for (int q = 0; q < H.nt; q++) {
    const TrainDesc td = S.trn[q];
    if (get_digit(w0, w1, td.slot) == 0 && td.size >= H.mu) bwd = dadd(bwd, td.uterm);
  }
  return bwd;
}

__device__ __forceinline__ uint32_t num_split_of(uint64_t w0, uint64_t w1) {
  return __popcll((w0 | (w0 >> 1)) & 0x5555555555555555ULL) + __popcll((w1 | (w1 >> 1)) & 0x5555555555555555ULL);
}

// reference index (candidate_by_index order) of enumeration-order digits
__device__ __forceinline__ unsigned long long ref_index(const Tabs& S, uint64_t w0, uint64_t w1) {
  unsigned long long idx = 0;
  for (int q = 0; q < S.H->V; q++) idx += (unsigned long long)get_digit(w0, w1, q) * S.stride[q];
  return idx;
}

__device__ __forceinline__ void decode_enum(const BlobHeader& H, unsigned long long x, uint64_t& w0, uint64_t& w1) {
  w0 = w1 = 0;
  for (int q = H.V - 1; q >= 0; q--) {
    const uint32_t r = ((H.radix3 >> q) & 1) ? 3 : 2;
    const uint32_t d = (uint32_t)(x % r);
    x /= r;
    if (q < 32) w0 |= (uint64_t)d << (q * 2);
    else w1 |= (uint64_t)d << ((q - 32) * 2);
  }
}

// zero every position > m, then +1 at position m (carry upwards)
__device__ __forceinline__ void mr_skip(uint64_t& w0, uint64_t& w1, int m, int V, uint64_t radix3) {
  for (int q = m + 1; q < V; q++) {
    if (q < 32) w0 &= ~(3ULL << (q * 2));
    else w1 &= ~(3ULL << ((q - 32) * 2));
  }
  for (int q = m; q >= 0; q--) {
    uint64_t& w = q < 32 ? w0 : w1;
    const int sh = (q & 31) * 2;
    const uint32_t d = (uint32_t)((w >> sh) & 3) + 1;
    const uint32_t r = ((radix3 >> q) & 1) ? 3 : 2;
    if (d < r) {
      w = (w & ~(3ULL << sh)) | ((uint64_t)d << sh);
      return;
    }
    w &= ~(3ULL << sh);
  }
}

__device__ __forceinline__ unsigned long long shfl_u64(unsigned long long v, int src) {
  const unsigned lo = __shfl_sync(0xffffffffu, (unsigned)v, src);
  const unsigned hi = __shfl_sync(0xffffffffu, (unsigned)(v >> 32), src);
  return ((unsigned long long)hi << 32) | lo;
}

__device__ __forceinline__ unsigned long long warp_max_u64(unsigned long long v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const unsigned long long w = ((unsigned long long)__shfl_xor_sync(0xffffffffu, (unsigned)(v >> 32), o) << 32) |
                                 __shfl_xor_sync(0xffffffffu, (unsigned)v, o);
    v = w > v ? w : v;
  }
  return v;
}

__device__ __forceinline__ void stage_blob(uint8_t* smem, const uint8_t* blobs, int64_t off) {
  const int bytes = ((const BlobHeader*)(blobs + off))->bytes;
  const uint4* src = (const uint4*)(blobs + off);
  uint4* dst = (uint4*)smem;
  for (int q = threadIdx.x; q < bytes / 16; q += blockDim.x) dst[q] = src[q];
}

// ---- biased packed digits (DM_BIASED) --------------------------------------
struct Biased {
  uint64_t B;      // packed biases = the encoding of all-zero digits
  uint64_t NZ;     // bit that is set iff the digit is non-zero, per position
  uint64_t add32;  // unbiased digits of 32 (added to advance a warp by 32)
  uint64_t add64;  // unbiased digits of 64 (paired walk)
};

// y + a where a holds unbiased digits: a field that wraps carries into the next
// slower position by plain binary carry and gets its bias back.
__device__ __forceinline__ uint64_t badd(uint64_t y, uint64_t a, uint64_t B) {
  const uint64_t s = y + a;
  const uint64_t w = ((s ^ y ^ a) >> 2) & 0x5555555555555555ULL;  // carry out of each field
  return s + ((w | (w << 1)) & B);
}

__device__ __forceinline__ uint64_t bencode(const BlobHeader& H, unsigned long long x) {
  uint64_t y = 0;
  for (int q = H.V - 1; q >= 0; q--) {
    const uint32_t r = ((H.radix3 >> q) & 1) ? 3 : 2;
    const uint32_t d = (uint32_t)(x % r);
    x /= r;
    y |= (uint64_t)(d + 4 - r) << (2 * (H.V - 1 - q));
  }
  return y;
}

__device__ __forceinline__ uint32_t bdigit(const BlobHeader& H, uint64_t y, int q) {
  const uint32_t r = ((H.radix3 >> q) & 1) ? 3 : 2;
  return (uint32_t)((y >> (2 * (H.V - 1 - q))) & 3) - (4 - r);
}

// pack_gradients (rewrite.py:78-111) of a replicated-gradient plan on the
// biased digit word: the trainable weights whose digit is 0 come from one
// compare against the all-zero word (bit 2k of z: field k holds digit 0), and
// only those are visited, highest field first -- enumeration order, which is
// template order (the sums' order); sizes and unfused terms are read by
// enumeration position.
__device__ __forceinline__ double backward_b(const Tabs& S, uint64_t y) {
  const BlobHeader& H = *S.H;
  double bwd = 0.0;
  if (!H.multi_dev) return bwd;
  const uint64_t e = y ^ H.bias;
  const uint64_t z = ~(e | (e >> 1)) & 0x5555555555555555ULL;
  const int top = H.V - 1;
  long long cur = 0;
  int cur_n = 0;
  for (uint64_t m = z & H.tmask_small; m;) {
    const int bit = 63 - __clzll(m);
    m &= ~(1ULL << bit);
    const int64_t size = S.tsize[top - (bit >> 1)];
    if (cur + size > H.chunk && cur_n) {
      bwd = dadd(bwd, dadd(H.setup, dmul(ddiv(dmul(H.c_ar, (double)cur), H.bw), H.eff_ar)));
      cur = 0;
      cur_n = 0;
    }
    cur += size;
    cur_n++;
  }
  if (cur_n) bwd = dadd(bwd, dadd(H.setup, dmul(ddiv(dmul(H.c_ar, (double)cur), H.bw), H.eff_ar)));
  for (uint64_t m = z & H.tmask_big; m;) {
    const int bit = 63 - __clzll(m);
    m &= ~(1ULL << bit);
    bwd = dadd(bwd, S.tuterm[top - (bit >> 1)]);
  }
  return bwd;
}

__device__ __forceinline__ unsigned long long ref_index_b(const Tabs& S, uint64_t y) {
  unsigned long long idx = 0;
  for (int q = 0; q < S.H->V; q++) idx += (unsigned long long)bdigit(*S.H, y, q) * S.stride[q];
  return idx;
}

// Batched scorer over ALL blocks of a search in one launch.  Dynamic work
// items (atomic counter) of contiguous enumeration ranges; each warp walks its
// eighth of an item 32 candidates at a time.  With skipping on, a lane whose
// candidate fails at node i proves its whole R-aligned run invalid (R =
// NodeSkip.R), and the warp jumps to the max proven end: the union of the
// lanes' runs is contiguous from the warp's base, so the jump is exact.
#ifndef SP_SCORE_MIN_BLOCKS
#define SP_SCORE_MIN_BLOCKS 4
#endif
template <bool WIDE, bool SKIP>
__global__ void __launch_bounds__(THREADS, SP_SCORE_MIN_BLOCKS) k_score(const uint8_t* __restrict__ blobs, ScorePlan P,
                                                   ItemOut* __restrict__ items,
                                                   unsigned long long* __restrict__ counter) {
  extern __shared__ __align__(16) uint8_t smem[];
  __shared__ unsigned long long s_item;
  __shared__ int64_t s_block;
  __shared__ unsigned long long s_red_t[THREADS / 32], s_red_i[THREADS / 32];
  __shared__ uint32_t s_red_n[THREADS / 32], s_red_v[THREADS / 32];
  __shared__ uint64_t s_lane_add[32];
  __shared__ Biased s_bz;
  constexpr int DM = WIDE ? DM_WIDE : DM_BIASED;
  const int tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;
  int64_t staged = -1;
  while (true) {
    if (tid == 0) s_item = atomicAdd(counter, 1ULL);
    __syncthreads();
    const unsigned long long item = s_item;
    if (item >= P.n_items) break;
    if (tid == 0) {
      int64_t lo = 0, hi = P.nb;
      while (hi - lo > 1) {
        const int64_t mid = (lo + hi) / 2;
        if (P.item_base[mid] <= item) lo = mid;
        else hi = mid;
      }
      s_block = lo;
    }
    __syncthreads();
    const int64_t b = s_block;
    if (b != staged) {
      stage_blob(smem, blobs, P.blob_off[b]);
      if (!WIDE) {
        // per-block constants of the biased encoding
        const BlobHeader* gH = (const BlobHeader*)(blobs + P.blob_off[b]);
        const int V = gH->V;
        const uint64_t r3 = gH->radix3;
        if (tid < 32) {
          uint64_t a = 0;  // unbiased digits of `tid` in the fastest positions
          uint32_t x = (uint32_t)tid;
          for (int q = V - 1; q >= 0 && x; q--) {
            const uint32_t r = ((r3 >> q) & 1) ? 3 : 2;
            a |= (uint64_t)(x % r) << (2 * (V - 1 - q));
            x /= r;
          }
          s_lane_add[tid] = a;
        } else if (tid == 32) {
          Biased z{0, 0, 0, 0};
          uint32_t x = 32;
          for (int q = V - 1; q >= 0; q--) {
            const uint32_t r = ((r3 >> q) & 1) ? 3 : 2;
            const int sh = 2 * (V - 1 - q);
            z.B |= (uint64_t)(4 - r) << sh;
            z.NZ |= (uint64_t)(r == 3 ? 2 : 1) << sh;
            z.add32 |= (uint64_t)(x % r) << sh;
            x /= r;
          }
          s_bz = z;
        }
      }
      staged = b;
    }
    __syncthreads();
    const Tabs S = tabs_of(smem);
    const BlobHeader& H = *S.H;
    const Biased bz = s_bz;
    const unsigned long long ilo = P.lo[b] + (item - P.item_base[b]) * P.stride[b];
    const unsigned long long ihi = min(ilo + P.item_cands, P.hi[b]);
    const unsigned long long span = (ihi - ilo + (THREADS / 32) - 1) / (THREADS / 32);
    const unsigned long long wlo = min(ilo + span * warp, ihi), whi = min(wlo + span, ihi);
    unsigned long long best_t = ~0ULL, best_i = ~0ULL;
    uint32_t best_n = 0xFFFFFFFFu, nvalid = 0;
    if (wlo < whi) {
      uint64_t bw0, bw1 = 0;
      if (WIDE) decode_enum(H, wlo, bw0, bw1);
      else bw0 = bencode(H, wlo);
      const uint64_t lane_add = WIDE ? 0 : s_lane_add[lane];
      unsigned long long base = wlo;
      while (base < whi) {
        const unsigned long long x = base + lane;
        const bool active = x < whi;
        uint64_t w0 = bw0, w1 = bw1;
        if (WIDE) mr_add(w0, w1, (uint32_t)lane, H.V, H.radix3);
        else w0 = badd(bw0, lane_add, bz.B);
        double fwd;
        int fail;
        fail = walk<DM>(S, w0, w1, active, fwd, tid);
        unsigned long long t = x + 1;
        if (fail < 0) {
          const double bwd = WIDE ? backward(S, w0, w1) : backward_b(S, w0);
          const double total = dadd(fwd, dmul(bwd, H.keep_bwd));
          const unsigned long long tb = (unsigned long long)__double_as_longlong(total);
          const uint32_t ns = WIDE ? num_split_of(w0, w1) : (uint32_t)__popcll(w0 & bz.NZ);
          const unsigned long long idx = WIDE ? ref_index(S, w0, w1) : ref_index_b(S, w0);
          nvalid++;
          if (key_less(tb, ns, idx, best_t, best_n, best_i)) {
            best_t = tb;
            best_n = ns;
            best_i = idx;
          }
        } else if (SKIP && active) {
          const NodeSkip sk = S.skip[fail];
          t = sk.R ? (x / sk.R + 1) * sk.R : whi;
        }
        const unsigned long long nb_ = SKIP ? warp_max_u64(t) : base + 32;
        if (nb_ >= whi) break;
        if (nb_ == base + 32) {
          if (WIDE) mr_add(bw0, bw1, 32, H.V, H.radix3);
          else bw0 = badd(bw0, bz.add32, bz.B);
        } else {
          // the lane that proved the longest run provides the next base digits
          const unsigned mask = __ballot_sync(0xffffffffu, t == nb_);
          const int src = __ffs(mask) - 1;
          uint64_t n0 = w0, n1 = w1;
          if (lane == src) {
            const bool jump = fail >= 0 && active && S.skip[fail].R;
            if (WIDE) {
              if (jump) mr_skip(n0, n1, S.skip[fail].m, H.V, H.radix3);
              else mr_add(n0, n1, 1, H.V, H.radix3);
            } else {
              // positions faster than m back to digit 0, then +1 at position m
              const int sh = jump ? 2 * (H.V - 1 - S.skip[fail].m) : 0;
              const uint64_t low = (1ULL << sh) - 1;
              n0 = badd((n0 & ~low) | (bz.B & low), 1ULL << sh, bz.B);
            }
          }
          bw0 = shfl_u64(n0, src);
          if (WIDE) bw1 = shfl_u64(n1, src);
        }
        base = nb_;
      }
    }
    // warp then block argmin of (total, num_split, index) + valid count
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const unsigned long long t2 = __shfl_down_sync(0xffffffffu, best_t, o);
      const unsigned long long i2 = __shfl_down_sync(0xffffffffu, best_i, o);
      const uint32_t n2 = __shfl_down_sync(0xffffffffu, best_n, o);
      nvalid += __shfl_down_sync(0xffffffffu, nvalid, o);
      if (key_less(t2, n2, i2, best_t, best_n, best_i)) {
        best_t = t2;
        best_n = n2;
        best_i = i2;
      }
    }
    if (lane == 0) {
      s_red_t[warp] = best_t;
      s_red_i[warp] = best_i;
      s_red_n[warp] = best_n;
      s_red_v[warp] = nvalid;
    }
    __syncthreads();
    if (tid == 0) {
      ItemOut o{s_red_t[0], s_red_i[0], s_red_n[0], s_red_v[0]};
      for (int w = 1; w < THREADS / 32; w++) {
        o.valid += s_red_v[w];
        if (key_less(s_red_t[w], s_red_n[w], s_red_i[w], o.total_bits, o.num_split, o.index)) {
          o.total_bits = s_red_t[w];
          o.num_split = s_red_n[w];
          o.index = s_red_i[w];
        }
      }
      items[item] = o;
    }
  }
}

// Batched scorer for blocks with <= 32 weight slots (biased digit word): the
// same work decomposition and argmin as k_score, with the lean FastNode walk.
// Each lane carries its own candidate's digit word and advances it by 32 per
// warp step (one carry-fixed add); the warp's remaining count is 32-bit.
// (-DSP_PAIR_CHUNK for A/B builds: 256 / 512 / 1024 / 2048 / 4096 give c5 32.7 / 32.0 /
// 31.7 / 31.65 / 31.8 ms with 32768-candidate items; at 8 ranks 1024 beats 2048,
// 4.28 vs 4.35 ms per share)
#ifndef SP_PAIR_CHUNK
#define SP_PAIR_CHUNK 1024
#endif
constexpr int PAIR_CHUNK = SP_PAIR_CHUNK;  // candidates per warp chunk, walk modes
constexpr int PAIR_MAX_CHUNKS = ITEM_ITERS_MAX * THREADS / PAIR_CHUNK;
#ifndef SP_FLOW_SUB
#define SP_FLOW_SUB 256
#endif
constexpr uint32_t FLOW_SUB = SP_FLOW_SUB;  // warp chunk of k_score_flow's final wave (a multiple of 64)
#ifndef SP_SKIP_CHUNK
#define SP_SKIP_CHUNK 4096
#endif
constexpr int SKIP_CHUNK = SP_SKIP_CHUNK;  // ... with prefix skipping (a chunk costs >= one walk)
constexpr int SKIP_MAX_CHUNKS = ITEM_ITERS_MAX_SKIP * THREADS / SKIP_CHUNK;
#ifndef SP_PAIR_MIN_BLOCKS
#define SP_PAIR_MIN_BLOCKS 4
#endif
// Stage block `off`'s tables into shared memory for k_score_fast / k_score_flow
// (all threads of the CTA): the blob, the lanes' digit offsets, the biased
// digit constants and the digit words of every multiple of `chs` candidates
// up to `maxch` of them; then make the FastNode offsets absolute.  Contains
// the CTA barriers it needs; returns after the last one.
__device__ __forceinline__ void stage_block(uint8_t* smem, const uint8_t* blobs, int64_t off, uint64_t* lane_add,
                                            Biased* bz, uint64_t* cenc, uint32_t chs, int maxch, bool pair,
                                            uint64_t* fenc = nullptr, uint32_t fsub = 0, int nf = 0) {
  const int tid = threadIdx.x;
  stage_blob(smem, blobs, off);
  const BlobHeader* gH = (const BlobHeader*)(blobs + off);
  const int V = gH->V;
  const uint64_t r3 = gH->radix3;
  if (tid < 32) {
    uint64_t a = 0;  // unbiased digits of `tid` in the fastest positions
    uint32_t x = (uint32_t)tid;
    for (int q = V - 1; q >= 0 && x; q--) {
      const uint32_t r = ((r3 >> q) & 1) ? 3 : 2;
      a |= (uint64_t)(x % r) << (2 * (V - 1 - q));
      x /= r;
    }
    lane_add[tid] = a;
  } else if (tid == 32) {
    Biased z{0, 0, 0, 0};
    uint32_t x = 32;
    for (int q = V - 1; q >= 0; q--) {
      const uint32_t r = ((r3 >> q) & 1) ? 3 : 2;
      const int sh = 2 * (V - 1 - q);
      z.B |= (uint64_t)(4 - r) << sh;
      z.NZ |= (uint64_t)(r == 3 ? 2 : 1) << sh;
      z.add32 |= (uint64_t)(x % r) << sh;
      x /= r;
    }
    uint32_t x64 = 64;
    for (int q = V - 1; q >= 0 && x64; q--) {
      const uint32_t r = ((r3 >> q) & 1) ? 3 : 2;
      z.add64 |= (uint64_t)(x64 % r) << (2 * (V - 1 - q));
      x64 /= r;
    }
    *bz = z;
  }
  for (int c = tid - 64; c >= 0 && c < maxch; c += THREADS - 64) {
    uint64_t a = 0;  // unbiased digits of c * chs
    uint64_t x = (uint64_t)c * chs;
    for (int q = V - 1; q >= 0 && x; q--) {
      const uint32_t r = ((r3 >> q) & 1) ? 3 : 2;
      a |= (uint64_t)(x % r) << (2 * (V - 1 - q));
      x /= r;
    }
    cenc[c] = a;
  }
  for (int c = tid - 64 - maxch; c >= 0 && c < nf; c += THREADS - 64 - maxch) {
    uint64_t a = 0;  // unbiased digits of c * fsub
    uint64_t x = (uint64_t)c * fsub;
    for (int q = V - 1; q >= 0 && x; q--) {
      const uint32_t r = ((r3 >> q) & 1) ? 3 : 2;
      a |= (uint64_t)(x % r) << (2 * (V - 1 - q));
      x /= r;
    }
    fenc[c] = a;
  }
  __syncthreads();
  patch_fast(smem, pair);
  __syncthreads();
}

// Per-lane running argmin of a block's valid candidates: (total bits,
// num_split, digits) + valid count; the digits become the reference index
// once, when the result is written (they only break exact ties).
struct LaneBest {
  unsigned long long t = ~0ULL;
  uint32_t n = 0xFFFFFFFFu, valid = 0;
  uint64_t w = 0;
};

// One warp chunk of k_score_fast: `rem` candidates from the lane's digit word
// `w` (lane l holds candidate start + l; with PAIR also start + 32 + l);
// `whi` = the chunk's end in the block's enumeration index space (SKIP).
template <bool SKIP, bool PAIR>
__device__ __forceinline__ void score_chunk(const Tabs& S, const Biased& bz, const uint64_t* lane_add, uint32_t rec0,
                                            uint32_t rb, uint32_t sb, int lane, uint64_t w, uint32_t rem,
                                            unsigned long long whi, LaneBest& lb) {
  const BlobHeader& H = *S.H;
  const int T = H.T;
  auto take = [&](uint64_t wv, double fwd) {
    const double bwd = backward_b(S, wv);
    const double total = dadd(fwd, dmul(bwd, H.keep_bwd));
    const unsigned long long tb = (unsigned long long)__double_as_longlong(total);
    const uint32_t ns = (uint32_t)__popcll(wv & bz.NZ);
    lb.valid++;
    if (tb < lb.t || (tb == lb.t && (ns < lb.n || (ns == lb.n && ref_index_b(S, wv) < ref_index_b(S, lb.w))))) {
      lb.t = tb;
      lb.n = ns;
      lb.w = wv;
    }
  };
  if (PAIR) {
    while (true) {
      const uint64_t wb = badd(w, bz.add32, bz.B);
      double fa, fb;
      const int v = walk_pair(rec0, T, w, wb, (uint32_t)lane < rem, (uint32_t)lane + 32 < rem, fa, fb, rb, sb);
      if (v & 1) take(w, fa);
      if (v & 2) take(wb, fb);
      if (rem <= 64) break;
      rem -= 64;
      w = badd(w, bz.add64, bz.B);
    }
    return;
  }
  // single candidate per lane; with SKIP, lanes prove R-aligned runs invalid
  // and the warp jumps to the furthest proven end (clamped to the chunk)
  unsigned long long base = whi - rem;
  while (true) {
    const bool active = (uint32_t)lane < rem;
    double fwd;
    const int fail = walk_fast<SKIP>(rec0, T, w, active, fwd, rb, sb);
    uint32_t adv = 32;  // SKIP: candidates this lane proves done, from base
    if (fail < 0) {
      take(w, fwd);
      if (SKIP) adv = lane + 1;
    } else if (SKIP) {
      adv = lane + 1;
      if (active) {
        const NodeSkip sk = S.skip[fail];
        const unsigned long long x = base + lane;
        unsigned long long t;
        if (!sk.R) {
          t = whi;
        } else if (whi <= 0xFFFFFFFFull) {  // 32-bit division (the 64-bit one is a long subroutine)
          const uint32_t x32 = (uint32_t)x, r32 = (uint32_t)sk.R;
          t = (unsigned long long)(x32 - x32 % r32) + r32;
        } else {
          t = (x / sk.R + 1) * sk.R;
        }
        adv = (uint32_t)(min(t, whi) - base);
      }
    }
    if (!SKIP) {
      if (rem <= 32) break;
      rem -= 32;
      w = badd(w, bz.add32, bz.B);
    } else {
      // the union of the lanes' proven runs is contiguous from base
      uint32_t m = adv;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
      if (m >= rem) break;
      if (m == 32) {
        w = badd(w, bz.add32, bz.B);
      } else {
        // the lane that proved the longest run provides the next base digits
        const int src = __ffs(__ballot_sync(0xffffffffu, adv == m)) - 1;
        uint64_t n0 = w;
        if (lane == src) {
          const bool jump = fail >= 0 && active && S.skip[fail].R;
          // positions faster than m back to digit 0, then +1 at position m
          const int sh = jump ? 2 * (H.V - 1 - S.skip[fail].m) : 0;
          const uint64_t low = (1ULL << sh) - 1;
          n0 = badd((n0 & ~low) | (bz.B & low), 1ULL << sh, bz.B);
        }
        w = badd(shfl_u64(n0, src), lane_add[lane], bz.B);
      }
      rem -= m;
      base += m;
    }
  }
}

template <bool SKIP, bool PAIR>
__global__ void __launch_bounds__(THREADS, PAIR ? SP_PAIR_MIN_BLOCKS : SP_SCORE_MIN_BLOCKS) k_score_fast(const uint8_t* __restrict__ blobs,
                                                                           ScorePlan P, ItemOut* __restrict__ items,
                                                                           unsigned long long* __restrict__ counter) {
  extern __shared__ __align__(16) uint8_t smem[];
  __shared__ unsigned long long s_item;
  __shared__ int64_t s_block;
  __shared__ unsigned long long s_red_t[THREADS / 32], s_red_i[THREADS / 32];
  __shared__ uint32_t s_red_n[THREADS / 32], s_red_v[THREADS / 32];
  __shared__ uint64_t s_lane_add[32];
  __shared__ Biased s_bz;
  // warps pull CH-candidate chunks of the item from a shared cursor (no
  // static per-warp spans: no barrier idling when walks or skips are skewed)
  constexpr uint32_t CH = SKIP ? SKIP_CHUNK : PAIR_CHUNK;
  // with skipping, a chunk's cost varies most: the last quarter of an item is
  // dealt in quarter-size chunks so the warps reach the item barrier together
  constexpr uint32_t CHS = SKIP ? SKIP_CHUNK / 4 : PAIR_CHUNK;
  constexpr int MAXCH = SKIP ? SKIP_MAX_CHUNKS * 4 : PAIR_MAX_CHUNKS;
  __shared__ uint64_t s_wbase;              // biased digits of the item start
  __shared__ uint64_t s_cenc[MAXCH];        // unbiased digits of j * CHS
  __shared__ uint32_t s_chunk;
  const int tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;
  int64_t staged = -1;
  while (true) {
    if (tid == 0) s_item = atomicAdd(counter, 1ULL);
    __syncthreads();
    const unsigned long long item = s_item;
    if (item >= P.n_items) break;
    if (tid == 0) {
      int64_t lo = 0, hi = P.nb;
      while (hi - lo > 1) {
        const int64_t mid = (lo + hi) / 2;
        if (P.item_base[mid] <= item) lo = mid;
        else hi = mid;
      }
      s_block = lo;
    }
    __syncthreads();
    const int64_t b = s_block;
    if (b != staged) {
      stage_block(smem, blobs, P.blob_off[b], s_lane_add, &s_bz, s_cenc, CHS, MAXCH, PAIR);
      staged = b;
    }
    if (tid == 0) {
      s_wbase = bencode(*(const BlobHeader*)smem, P.lo[b] + (item - P.item_base[b]) * P.stride[b]);
      s_chunk = 0;
    }
    __syncthreads();
    const Tabs S = tabs_of(smem);
    const BlobHeader& H = *S.H;
    const unsigned long long ilo = P.lo[b] + (item - P.item_base[b]) * P.stride[b];
    const unsigned long long ihi = min(ilo + P.item_cands, P.hi[b]);
    unsigned long long best_t = ~0ULL, best_i = ~0ULL;
    uint32_t best_n = 0xFFFFFFFFu, nvalid = 0;
    if (ilo < ihi) {
      // opaque copies keep the shared addresses in registers (ptxas would
      // otherwise re-derive the shared window base at every access)
      const uint32_t rec0 = opaque_u32((uint32_t)__cvta_generic_to_shared(smem) + (uint32_t)H.fast_off);
      // pool: reach[npool][THREADS (x2 paired)] doubles, then the state bytes
      const uint32_t pool = (uint32_t)__cvta_generic_to_shared(S.reach);
      const uint32_t rb = opaque_u32(pool + 8u * (uint32_t)tid);
      const uint32_t sb = opaque_u32(pool + (uint32_t)H.npool * THREADS * (PAIR ? 16u : 8u) + (uint32_t)tid);
      const int T = H.T;
      const uint32_t cnt = (uint32_t)(ihi - ilo);
      LaneBest lb;
      while (true) {
        uint32_t c = 0;
        if (lane == 0) c = atomicAdd(&s_chunk, 1u);
        c = __shfl_sync(0xffffffffu, c, 0);
        // chunk c: CH-sized for the first ~3/4 of the item, CHS-sized after
        const uint32_t nbig = SKIP ? (cnt - cnt / 4) / CH : 0;
        const uint32_t start = c < nbig ? c * CH : nbig * CH + (c - nbig) * CHS;
        if (start >= cnt) break;
        uint32_t rem = min(c < nbig ? CH : CHS, cnt - start);  // candidates left in this chunk
        const uint64_t w = badd(badd(s_wbase, s_cenc[start / CHS], s_bz.B), s_lane_add[lane], s_bz.B);
        score_chunk<SKIP, PAIR>(S, s_bz, s_lane_add, rec0, rb, sb, lane, w, rem, ilo + (unsigned long long)start + rem,
                                lb);
      }
      best_t = lb.t;
      best_n = lb.n;
      nvalid = lb.valid;
      if (best_t != ~0ULL) best_i = ref_index_b(S, lb.w);
    }
    // warp then block argmin of (total, num_split, index) + valid count
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const unsigned long long t2 = __shfl_down_sync(0xffffffffu, best_t, o);
      const unsigned long long i2 = __shfl_down_sync(0xffffffffu, best_i, o);
      const uint32_t n2 = __shfl_down_sync(0xffffffffu, best_n, o);
      nvalid += __shfl_down_sync(0xffffffffu, nvalid, o);
      if (key_less(t2, n2, i2, best_t, best_n, best_i)) {
        best_t = t2;
        best_n = n2;
        best_i = i2;
      }
    }
    if (lane == 0) {
      s_red_t[warp] = best_t;
      s_red_i[warp] = best_i;
      s_red_n[warp] = best_n;
      s_red_v[warp] = nvalid;
    }
    __syncthreads();
    if (tid == 0) {
      ItemOut o{s_red_t[0], s_red_i[0], s_red_n[0], s_red_v[0]};
      for (int w2 = 1; w2 < THREADS / 32; w2++) {
        o.valid += s_red_v[w2];
        if (key_less(s_red_t[w2], s_red_n[w2], s_red_i[w2], o.total_bits, o.num_split, o.index)) {
          o.total_bits = s_red_t[w2];
          o.num_split = s_red_n[w2];
          o.index = s_red_i[w2];
        }
      }
      items[item] = o;
    }
  }
}

// k_score_fast without item barriers.  The CTA keeps two work items in flight
// (slots); warps pull chunks from a slot's cursor, and when a slot runs dry
// each warp moves on to the other slot on its own -- the last warp to leave a
// slot refills it with the next global item.  Warps meet at a barrier only
// when an item belongs to another block (the tables must be restaged) and at
// the end.  Results accumulate per lane over the CTA's whole share of a block
// and are written once into the ItemOut of that share's first item; every
// other item the CTA claims is written empty (k_reduce's min and sum are
// unchanged).  Every warp visits the slots' generations in the same order
// (slot 0 gen 1, slot 1 gen 1, slot 0 gen 2, ...), so a slot's parameters
// are rewritten only after all eight warps have left it.
#ifdef SP_CTA_TRACE
// diagnostics build (-DSP_CTA_TRACE, SP_LIB=...): per CTA of the last k_score_flow
// launch: start, end (globaltimer ns), ns spent closing / staging blocks, stagings
__device__ unsigned long long g_cta_trace[4096][4];
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#endif
struct FlowSlot {
  unsigned long long item, ilo;
  uint64_t wbase;
  int64_t block;
  uint32_t cnt, cursor, retired, gen, fine;
  int state;  // 0: ready (staged block), 1: another block, 2: no more items
};

template <bool SKIP, bool PAIR>
__global__ void __launch_bounds__(THREADS, PAIR ? SP_PAIR_MIN_BLOCKS : SP_SCORE_MIN_BLOCKS) k_score_flow(
    const uint8_t* __restrict__ blobs, ScorePlan P, ItemOut* __restrict__ items,
    unsigned long long* __restrict__ counter) {
  extern __shared__ __align__(16) uint8_t smem[];
  constexpr uint32_t CH = SKIP ? SKIP_CHUNK : PAIR_CHUNK;
  constexpr uint32_t CHS = SKIP ? SKIP_CHUNK / 4 : PAIR_CHUNK;
  constexpr int MAXCH = SKIP ? SKIP_MAX_CHUNKS * 4 : PAIR_MAX_CHUNKS;
  constexpr int NW = THREADS / 32;
  __shared__ uint64_t s_lane_add[32];
  __shared__ Biased s_bz;
  __shared__ uint64_t s_cenc[MAXCH];
  // digits of k * FLOW_SUB (k < CHS / FLOW_SUB): the final wave's finer chunks
  constexpr int NF = SKIP ? 0 : (int)(CHS / FLOW_SUB);
  __shared__ uint64_t s_fenc[NF > 0 ? NF : 1];
  __shared__ FlowSlot s_slot[2];
  __shared__ unsigned long long s_seg;  // item whose ItemOut receives the current share (~0: none yet)
  __shared__ int64_t s_staged;
  __shared__ unsigned long long s_red_t[NW], s_red_i[NW], s_red_v[NW];
  __shared__ uint32_t s_red_n[NW];
  const int tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;

  // one thread: claim the next item into slot x and publish it (gen + 1)
  auto fill = [&](int x) {
    volatile FlowSlot& sl = s_slot[x];
    const unsigned long long it = atomicAdd(counter, 1ULL);
    if (it >= P.n_items) {
      sl.state = 2;
    } else {
      int64_t lo = 0;
      unsigned long long ilo, ihi, out;
      if (SKIP || it < P.n_main) {
        int64_t hi = P.nb;
        while (hi - lo > 1) {
          const int64_t mid = (lo + hi) / 2;
          if (P.item_base[mid] <= it) lo = mid;
          else hi = mid;
        }
        const unsigned long long j = it - P.item_base[lo];
        if (!P.cnt1 || j < P.cnt1[lo]) {
          ilo = P.lo[lo] + j * P.stride[lo];
          ihi = min(ilo + P.item_cands, P.hi[lo]);
        } else {
          ilo = P.lo2[lo] + (j - P.cnt1[lo]) * P.stride2[lo];
          ihi = min(ilo + P.item_cands, P.hi2[lo]);
        }
        out = P.obase ? P.obase[lo] + j : it;
        sl.fine = 0;
      } else {  // sub-item k of run e: part k % split of the block's item nmain + k / split
        const unsigned long long u = it - P.n_main;
        int64_t e = 0, hi = P.nf;
        while (hi - e > 1) {
          const int64_t mid = (e + hi) / 2;
          if (P.fbase[mid] <= u) e = mid;
          else hi = mid;
        }
        lo = (int64_t)P.fblk[e];
        const unsigned long long k = u - P.fbase[e], nmain = P.item_base[lo + 1] - P.item_base[lo];
        const unsigned long long jb = nmain + k / P.split;  // the split item
        unsigned long long blo, bhi;
        if (jb < P.cnt1[lo]) {
          blo = P.lo[lo] + jb * P.stride[lo];
          bhi = min(blo + P.item_cands, P.hi[lo]);
        } else {
          blo = P.lo2[lo] + (jb - P.cnt1[lo]) * P.stride2[lo];
          bhi = min(blo + P.item_cands, P.hi2[lo]);
        }
        ilo = min(blo + (k % P.split) * P.sub, bhi);
        ihi = min(ilo + P.sub, bhi);
        out = P.obase[lo] + nmain + k;
        sl.fine = 1;
      }
      items[out] = ItemOut{~0ULL, ~0ULL, 0xFFFFFFFFu, 0ULL};
      sl.item = out;
      sl.block = lo;
      sl.ilo = ilo;
      sl.cnt = (uint32_t)(ihi - ilo);
      if (lo == s_staged) {
        sl.wbase = bencode(*(const BlobHeader*)smem, ilo);
        sl.state = 0;
      } else {
        sl.state = 1;
      }
    }
    sl.cursor = 0;
    sl.retired = 0;
    __threadfence_block();
    atomicAdd((uint32_t*)&s_slot[x].gen, 1u);
  };
  // warp argmin of the lanes' shares -> s_red[warp]; then (after a barrier)
  // thread 0 writes the CTA's share into s_seg's ItemOut
  auto flush = [&](LaneBest& lb) {
    const Tabs S = tabs_of(smem);
    unsigned long long bt = lb.t, bi = lb.t != ~0ULL ? ref_index_b(S, lb.w) : ~0ULL,
                       nv = lb.valid;
    uint32_t bn = lb.n;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const unsigned long long t2 = __shfl_down_sync(0xffffffffu, bt, o);
      const unsigned long long i2 = __shfl_down_sync(0xffffffffu, bi, o);
      const uint32_t n2 = __shfl_down_sync(0xffffffffu, bn, o);
      nv += __shfl_down_sync(0xffffffffu, nv, o);
      if (key_less(t2, n2, i2, bt, bn, bi)) {
        bt = t2;
        bn = n2;
        bi = i2;
      }
    }
    if (lane == 0) {
      s_red_t[warp] = bt;
      s_red_i[warp] = bi;
      s_red_n[warp] = bn;
      s_red_v[warp] = nv;
    }
    __syncthreads();
    if (tid == 0 && s_seg != ~0ULL) {
      ItemOut o{s_red_t[0], s_red_i[0], s_red_n[0], s_red_v[0]};
      for (int w = 1; w < NW; w++) {
        o.valid += s_red_v[w];
        if (key_less(s_red_t[w], s_red_n[w], s_red_i[w], o.total_bits, o.num_split, o.index)) {
          o.total_bits = s_red_t[w];
          o.num_split = s_red_n[w];
          o.index = s_red_i[w];
        }
      }
      items[s_seg] = o;
    }
    lb = LaneBest{};
  };

#ifdef SP_CTA_TRACE
  unsigned long long tr_t0 = gtimer(), tr_stage = 0, tr_n = 0;
#endif
  if (tid == 0) {
    s_staged = -1;
    s_seg = ~0ULL;
    s_slot[0].gen = s_slot[1].gen = 0;
    fill(0);
    fill(1);
  }
  __syncthreads();
  uint32_t my_gen[2] = {1, 1};
  bool done[2] = {false, false};
  int cur = 0;
  LaneBest lb;
  uint32_t rec0 = 0, rb = 0, sb = 0;
  while (true) {
    if (done[cur]) {
      if (done[cur ^ 1]) break;
      cur ^= 1;
      continue;
    }
    volatile FlowSlot& sl = s_slot[cur];
    if (lane == 0)
      while (*(volatile uint32_t*)&s_slot[cur].gen < my_gen[cur]) __nanosleep(64);
    __syncwarp();
    __threadfence_block();
    const int state = sl.state;
    if (state == 2) {
      done[cur] = true;
      continue;
    }
    if (state == 1) {
      // every warp reaches this slot generation: close the share of the
      // staged block, stage this slot's block
#ifdef SP_CTA_TRACE
      const unsigned long long tr_a = gtimer();
#endif
      flush(lb);
      __syncthreads();
      const int64_t b = sl.block;
      stage_block(smem, blobs, P.blob_off[b], s_lane_add, &s_bz, s_cenc, CHS, MAXCH, PAIR, s_fenc, FLOW_SUB, NF);
      if (tid == 0) {
        s_staged = b;
        s_seg = sl.item;
        sl.wbase = bencode(*(const BlobHeader*)smem, sl.ilo);
        sl.state = 0;
        volatile FlowSlot& ot = s_slot[cur ^ 1];
        if (ot.state == 1 && ot.block == b) {
          ot.wbase = bencode(*(const BlobHeader*)smem, ot.ilo);
          ot.state = 0;
        }
      }
      __syncthreads();
      {
        const Tabs S = tabs_of(smem);
        const BlobHeader& H = *S.H;
        rec0 = opaque_u32((uint32_t)__cvta_generic_to_shared(smem) + (uint32_t)H.fast_off);
        const uint32_t pool = (uint32_t)__cvta_generic_to_shared(S.reach);
        rb = opaque_u32(pool + 8u * (uint32_t)tid);
        sb = opaque_u32(pool + (uint32_t)H.npool * THREADS * (PAIR ? 16u : 8u) + (uint32_t)tid);
      }
#ifdef SP_CTA_TRACE
      tr_stage += gtimer() - tr_a;
      tr_n++;
#endif
      continue;
    }
    uint32_t c = 0;
    if (lane == 0) c = atomicAdd((uint32_t*)&s_slot[cur].cursor, 1u);
    c = __shfl_sync(0xffffffffu, c, 0);
    const uint32_t cnt = sl.cnt;
    // the final wave (sub-items) walks FLOW_SUB-candidate chunks: the kernel
    // ends when the slowest warp's last chunk does
    const bool fine = !SKIP && sl.fine;
    const uint32_t nbig = SKIP ? (cnt - cnt / 4) / CH : 0;
    const uint32_t start = fine ? c * FLOW_SUB : c < nbig ? c * CH : nbig * CH + (c - nbig) * CHS;
    if (start < cnt) {
      const uint32_t rem = min(fine ? FLOW_SUB : c < nbig ? CH : CHS, cnt - start);
      uint64_t w = badd(sl.wbase, s_cenc[start / CHS], s_bz.B);
      if (fine) w = badd(w, s_fenc[(start % CHS) / FLOW_SUB], s_bz.B);
      w = badd(w, s_lane_add[lane], s_bz.B);
      score_chunk<SKIP, PAIR>(tabs_of(smem), s_bz, s_lane_add, rec0, rb, sb, lane, w, rem,
                              sl.ilo + (unsigned long long)start + rem, lb);
      continue;
    }
    // slot dry for this warp: leave it (the last to leave refills it)
    uint32_t r = 0;
    if (lane == 0) {
      r = atomicAdd((uint32_t*)&s_slot[cur].retired, 1u);
      if (r == NW - 1) fill(cur);
    }
    __syncwarp();
    my_gen[cur]++;
    cur ^= 1;
  }
  flush(lb);
#ifdef SP_CTA_TRACE
  if (tid == 0 && blockIdx.x < 4096) {
    g_cta_trace[blockIdx.x][0] = tr_t0;
    g_cta_trace[blockIdx.x][1] = gtimer();
    g_cta_trace[blockIdx.x][2] = tr_stage;
    g_cta_trace[blockIdx.x][3] = tr_n;
  }
#endif
}

// Prefix-skipping scorer without work items: every CTA walks the blocks in
// order, stages a block's tables once, and its warps claim 4096-candidate
// chunks of that block straight from the block's global chunk counter (the
// next claim is issued before the current chunk is walked, so its latency is
// hidden).  A chunk's cost varies by orders of magnitude (a run of proven
// failures costs one walk, a region of valid candidates one walk per 32), so
// balance comes from the whole GPU sharing one counter per block; the CTA
// meets at a barrier only when the block is exhausted.  Each CTA that worked
// on a block appends one record (its warps' argmin + valid count) to the
// block's contribution list; k_reduce_contrib merges them.  Sharded searches
// deal chunk c of a block to rank c mod n_shards.
struct SkipPlan {
  const int64_t* blob_off;
  const unsigned long long* nch;  // this rank's 4096-candidate chunks per block
  unsigned long long* ctr;        // per block: claims (zeroed)
  uint32_t* contrib;              // per block: records appended (zeroed)
  int64_t nb;
  uint32_t shard, n_shards;
  unsigned long long tail;        // the last `tail` chunks of a block are claimed in eighths
};
constexpr uint32_t SKIP_SUB = 8;
constexpr int64_t SKIP_KERNEL_MAX_BLOCKS = 128;

__global__ void __launch_bounds__(THREADS, SP_SCORE_MIN_BLOCKS) k_score_skip(const uint8_t* __restrict__ blobs,
                                                                            SkipPlan P, ItemOut* __restrict__ out) {
  extern __shared__ __align__(16) uint8_t smem[];
  constexpr int NW = THREADS / 32;
  constexpr uint32_t CH = SKIP_CHUNK;
  __shared__ uint64_t s_lane_add[32];
  __shared__ Biased s_bz;
  __shared__ uint64_t s_p2[64];  // unbiased digits of 2^k * CH (mixed radix, wrapping)
  // unbiased digits of j * CH and of j * 1024 * CH (j < 1024): a chunk's start
  // digits in two adds instead of one per set bit of the chunk index
  __shared__ uint64_t s_lo[1024], s_hi[1024];
  __shared__ uint64_t s_sub[SKIP_SUB];  // unbiased digits of k * CH / SKIP_SUB
  // the chunk the CTA claimed before staging block b, in s_first[b & 1]: thread 0
  // writes block b+1's claim while slower threads may still read block b's
  // (the two are separated by block b+1's claim barrier, not by a second one)
  __shared__ unsigned long long s_first[2];
  __shared__ unsigned long long s_red_t[NW], s_red_i[NW], s_red_v[NW];
  __shared__ uint32_t s_red_n[NW];
  const int tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;
  for (int64_t b = 0; b < P.nb; b++) {
    // claims: the first nbig chunks whole, the last `tail` ones in SKIP_SUB
    // parts each (the final wave of a block is short: warps reach the block's
    // end barrier together)
    const unsigned long long nloc = P.nch[b];
    const unsigned long long nsm = min(nloc, P.tail), nbig = nloc - nsm;
    const unsigned long long nclaim = nbig + nsm * SKIP_SUB;
    // claim first: a block whose chunks are gone is neither staged nor visited
    if (tid == 0)
      s_first[b & 1] = *(volatile unsigned long long*)&P.ctr[b] < nclaim ? atomicAdd(&P.ctr[b], 1ULL) : nclaim;
    __syncthreads();
    if (s_first[b & 1] >= nclaim) continue;
    stage_block(smem, blobs, P.blob_off[b], s_lane_add, &s_bz, nullptr, 1, 0, false);
    if (tid == 0) {
      // unbiased digits of 2^k * CH (positions fastest-last, as bencode), by
      // doubling: biased(2x) = badd(biased(x), x), minus the biases
      const BlobHeader& H = *(const BlobHeader*)smem;
      uint64_t a = 0;
      uint32_t x = CH;
      for (int q = H.V - 1; q >= 0 && x; q--) {
        const uint32_t r = ((H.radix3 >> q) & 1) ? 3 : 2;
        a |= (uint64_t)(x % r) << (2 * (H.V - 1 - q));
        x /= r;
      }
      const uint64_t B = s_bz.B;
      for (int k = 0; k < 64; k++) {
        s_p2[k] = a;
        a = badd(badd(B, a, B), a, B) - B;
      }
      uint64_t sub = 0;  // digits of CH / SKIP_SUB, then multiples
      x = CH / SKIP_SUB;
      for (int q = H.V - 1; q >= 0 && x; q--) {
        const uint32_t r = ((H.radix3 >> q) & 1) ? 3 : 2;
        sub |= (uint64_t)(x % r) << (2 * (H.V - 1 - q));
        x /= r;
      }
      uint64_t m = 0;
      for (uint32_t k = 0; k < SKIP_SUB; k++) {
        s_sub[k] = m;
        m = badd(badd(B, m, B), sub, B) - B;
      }
    }
    __syncthreads();
    {
      const uint64_t B = s_bz.B;
      for (int j = tid; j < 1024; j += THREADS) {
        uint64_t lo = 0, hi = 0;
        for (int k = 0; k < 10; k++)
          if ((j >> k) & 1) {
            lo = badd(badd(B, lo, B), s_p2[k], B) - B;
            hi = badd(badd(B, hi, B), s_p2[k + 10], B) - B;
          }
        s_lo[j] = lo;
        s_hi[j] = hi;
      }
    }
    __syncthreads();
    const Tabs S = tabs_of(smem);
    const BlobHeader& H = *S.H;
    const uint32_t rec0 = opaque_u32((uint32_t)__cvta_generic_to_shared(smem) + (uint32_t)H.fast_off);
    const uint32_t pool = (uint32_t)__cvta_generic_to_shared(S.reach);
    const uint32_t rb = opaque_u32(pool + 8u * (uint32_t)tid);
    const uint32_t sb = opaque_u32(pool + (uint32_t)H.npool * THREADS * 8u + (uint32_t)tid);
    const unsigned long long C = H.C;
    LaneBest lb;
    unsigned long long j = 0;
    if (lane == 0) j = warp == 0 ? s_first[b & 1] : atomicAdd(&P.ctr[b], 1ULL);
    j = __shfl_sync(0xffffffffu, j, 0);
    while (j < nclaim) {
      unsigned long long jn = 0;
      if (lane == 0) jn = atomicAdd(&P.ctr[b], 1ULL);  // the next claim, in flight during the walk
      const unsigned long long jl = j < nbig ? j : nbig + (j - nbig) / SKIP_SUB;  // local chunk
      const uint32_t part = j < nbig ? 0u : (uint32_t)((j - nbig) % SKIP_SUB);
      const unsigned long long c = jl * P.n_shards + P.shard;  // the block's chunk
      const unsigned long long cs = c * CH;
      const unsigned long long start = cs + (j < nbig ? 0 : (unsigned long long)part * (CH / SKIP_SUB));
      if (start >= C) {
        j = __shfl_sync(0xffffffffu, jn, 0);
        continue;
      }
      const uint32_t rem = (uint32_t)min((unsigned long long)(j < nbig ? CH : CH / SKIP_SUB), C - start);
      // biased digits of c * CH: the two table entries of its low 20 bits, one add per higher set bit
      uint64_t w = badd(badd(s_bz.B, s_hi[(c >> 10) & 1023], s_bz.B), s_lo[c & 1023], s_bz.B);
      for (unsigned long long m = c >> 20; m; m &= m - 1) w = badd(w, s_p2[20 + __ffsll((long long)m) - 1], s_bz.B);
      w = badd(badd(w, s_sub[part], s_bz.B), s_lane_add[lane], s_bz.B);
      score_chunk<true, false>(S, s_bz, s_lane_add, rec0, rb, sb, lane, w, rem, start + rem, lb);
      j = __shfl_sync(0xffffffffu, jn, 0);
    }
    // the CTA's record for this block
    unsigned long long bt = lb.t, bi = lb.t != ~0ULL ? ref_index_b(S, lb.w) : ~0ULL, nv = lb.valid;
    uint32_t bn = lb.n;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const unsigned long long t2 = __shfl_down_sync(0xffffffffu, bt, o);
      const unsigned long long i2 = __shfl_down_sync(0xffffffffu, bi, o);
      const uint32_t n2 = __shfl_down_sync(0xffffffffu, bn, o);
      nv += __shfl_down_sync(0xffffffffu, nv, o);
      if (key_less(t2, n2, i2, bt, bn, bi)) {
        bt = t2;
        bn = n2;
        bi = i2;
      }
    }
    if (lane == 0) {
      s_red_t[warp] = bt;
      s_red_i[warp] = bi;
      s_red_n[warp] = bn;
      s_red_v[warp] = nv;
    }
    __syncthreads();
    if (tid == 0) {
      ItemOut o{s_red_t[0], s_red_i[0], s_red_n[0], s_red_v[0]};
      for (int w2 = 1; w2 < NW; w2++) {
        o.valid += s_red_v[w2];
        if (key_less(s_red_t[w2], s_red_n[w2], s_red_i[w2], o.total_bits, o.num_split, o.index)) {
          o.total_bits = s_red_t[w2];
          o.num_split = s_red_n[w2];
          o.index = s_red_i[w2];
        }
      }
      const uint32_t k = atomicAdd(&P.contrib[b], 1u);
      out[b * (int64_t)gridDim.x + k] = o;
    }
    __syncthreads();  // the tables of the next block overwrite smem
  }
}

// One CTA per block: merge the contribution records of k_score_skip.
__global__ void k_reduce_contrib(const ItemOut* __restrict__ rec, const uint32_t* __restrict__ contrib, int64_t stride,
                                 int64_t nb, sp_score_out* __restrict__ out) {
  __shared__ ItemOut s[THREADS];
  __shared__ unsigned long long sv[THREADS];
  for (int64_t b = blockIdx.x; b < nb; b += gridDim.x) {
    ItemOut acc{~0ULL, ~0ULL, 0xFFFFFFFFu, 0};
    unsigned long long valid = 0;
    const uint32_t cnt = contrib[b];
    for (uint32_t k = threadIdx.x; k < cnt; k += blockDim.x) {
      const ItemOut o = rec[b * stride + k];
      valid += o.valid;
      if (key_less(o.total_bits, o.num_split, o.index, acc.total_bits, acc.num_split, acc.index)) acc = o;
    }
    s[threadIdx.x] = acc;
    sv[threadIdx.x] = valid;
    __syncthreads();
    for (int st = blockDim.x / 2; st > 0; st >>= 1) {
      if (threadIdx.x < st) {
        const ItemOut o = s[threadIdx.x + st];
        if (key_less(o.total_bits, o.num_split, o.index, s[threadIdx.x].total_bits, s[threadIdx.x].num_split,
                     s[threadIdx.x].index))
          s[threadIdx.x] = o;
        sv[threadIdx.x] += sv[threadIdx.x + st];
      }
      __syncthreads();
    }
    if (threadIdx.x == 0) {
      sp_score_out r;
      r.candidates = 0;
      r.valid = sv[0];
      r.has_best = s[0].index != ~0ULL && sv[0] > 0;
      r.best_index = r.has_best ? s[0].index : 0;
      r.best_total = r.has_best ? __longlong_as_double((long long)s[0].total_bits) : 0.0;
      r.best_num_split = r.has_best ? (int32_t)s[0].num_split : 0;
      out[b] = r;
    }
    __syncthreads();
  }
}

// Memoised brute force: every candidate of the range is visited (32 per warp
// step, consecutive enumeration indices), but a node is re-routed only when a
// digit of its ancestor cone changed since the lane's previous candidate
// (dirty[q0], q0 = first changed enumeration position); every other node keeps
// its cached (reach, state, failed) -- a pure function of those digits, with a
// fixed dummy (state 0, reach 0) after a failure so the cache stays exact.
// Candidates are valid iff no node's failed bit is set.  Templates <= 64 nodes.
constexpr int THREADS_M = 128;

template <bool WIDE>
__global__ void __launch_bounds__(THREADS_M, 4) k_score_memo(const uint8_t* __restrict__ blobs, ScorePlan P,
                                                            ItemOut* __restrict__ items,
                                                            unsigned long long* __restrict__ counter) {
  extern __shared__ __align__(16) uint8_t smem[];
  __shared__ unsigned long long s_item;
  __shared__ int64_t s_block;
  __shared__ unsigned long long s_red_t[THREADS_M / 32], s_red_i[THREADS_M / 32];
  __shared__ uint32_t s_red_n[THREADS_M / 32], s_red_v[THREADS_M / 32];
  const int tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;
  int64_t staged = -1;
  while (true) {
    if (tid == 0) s_item = atomicAdd(counter, 1ULL);
    __syncthreads();
    const unsigned long long item = s_item;
    if (item >= P.n_items) break;
    if (tid == 0) {
      int64_t lo = 0, hi = P.nb;
      while (hi - lo > 1) {
        const int64_t mid = (lo + hi) / 2;
        if (P.item_base[mid] <= item) lo = mid;
        else hi = mid;
      }
      s_block = lo;
    }
    __syncthreads();
    const int64_t b = s_block;
    if (b != staged) {
      stage_blob(smem, blobs, P.blob_off[b]);
      staged = b;
    }
    __syncthreads();
    const BlobHeader& H = *(const BlobHeader*)smem;
    const NodeDesc* desc = (const NodeDesc*)(smem + H.desc_off);
    const int16_t* prodn = (const int16_t*)(smem + H.prod_off) + H.n_prod;
    const uint8_t* tab = smem + H.tab_off;
    const double* dbl = (const double*)(smem + H.dbl_off);
    const uint64_t* dirty = (const uint64_t*)(smem + H.dirty_off);
    double* cache = (double*)(smem + ((H.bytes + 15) & ~15));
    Tabs S = tabs_of(smem);
    const int T = H.T;
    const unsigned long long ilo = P.lo[b] + (item - P.item_base[b]) * P.stride[b];
    const unsigned long long ihi = min(ilo + P.item_cands, P.hi[b]);
    const unsigned long long span = (ihi - ilo + (THREADS_M / 32) - 1) / (THREADS_M / 32);
    const unsigned long long wlo = min(ilo + span * warp, ihi), whi = min(wlo + span, ihi);
    unsigned long long best_t = ~0ULL, best_i = ~0ULL;
    uint32_t best_n = 0xFFFFFFFFu, nvalid = 0;
    if (wlo < whi) {
      uint64_t bw0, bw1;
      decode_enum(H, wlo, bw0, bw1);
      uint64_t pw0 = 0, pw1 = 0, st_lo = 0, st_hi = 0, failmask = 0;
      bool first = true;
      for (unsigned long long base = wlo; base < whi; base += 32) {
        const unsigned long long x = base + lane;
        const bool active = x < whi;
        uint64_t w0 = bw0, w1 = bw1;
        mr_add(w0, w1, (uint32_t)lane, H.V, H.radix3);
        int q = 0;
        if (!first) {
          const uint64_t d0 = pw0 ^ w0, d1 = WIDE ? (pw1 ^ w1) : 0ULL;
          q = d0 ? (__ffsll((long long)d0) - 1) >> 1 : (d1 ? 32 + ((__ffsll((long long)d1) - 1) >> 1) : H.V);
        }
        const int q0 = (int)__reduce_min_sync(0xffffffffu, (unsigned)q);
        uint64_t mask = dirty[q0];
        while (mask) {
          const int i = __ffsll((long long)mask) - 1;
          mask &= mask - 1;
          const NodeDesc nd = desc[i];
          uint32_t key = 0;
          if (nd.slot >= 0) key = WIDE ? get_digit(w0, w1, nd.slot) : (uint32_t)((w0 >> (nd.slot * 2)) & 3);
          const double* D = dbl + nd.dbl;
          double r;
          int p, sj[KMAX];
          double rj[KMAX];
          for (int j = 0; j < nd.k; j++) {
            const int pn = prodn[nd.prod + j];
            sj[j] = (int)(((pn < 32 ? st_lo >> (2 * pn) : st_hi >> (2 * (pn - 32)))) & 3);
            rj[j] = cache[pn * THREADS_M + tid];
            key = key * 3 + sj[j];
          }
          const uint8_t e = tab[nd.tab + key];
          const bool fail = e == 0xFF;
          p = e & 3;
          const int s = fail ? 0 : (e >> 2) & 3;
          if (nd.k == 0) {
            r = D[p];
          } else if (nd.k == 1) {
            r = dadd(dadd(rj[0], D[8 + p * 3 + sj[0]]), D[p]);
          } else {
            double bse = dadd(rj[0], D[8 + p * 3 + sj[0]]);
            for (int j = 1; j < nd.k; j++) bse = dmax_nn(bse, dadd(rj[j], D[8 + (j * 4 + p) * 3 + sj[j]]));
            r = dadd(bse, D[p]);
          }
          if (fail) r = 0.0;
          cache[i * THREADS_M + tid] = r;
          if (i < 32) st_lo = (st_lo & ~(3ULL << (2 * i))) | ((uint64_t)s << (2 * i));
          else st_hi = (st_hi & ~(3ULL << (2 * (i - 32)))) | ((uint64_t)s << (2 * (i - 32)));
          failmask = (failmask & ~(1ULL << i)) | ((uint64_t)fail << i);
        }
        if (active && failmask == 0) {
          // forward = max over nodes of reach + exit AllGather (costmodel.py:239-245)
          double fwd = 0.0;
          for (int i = 0; i < T; i++) {
            const int si = (int)(((i < 32 ? st_lo >> (2 * i) : st_hi >> (2 * (i - 32)))) & 3);
            fwd = dmax_nn(fwd, dadd(cache[i * THREADS_M + tid], dbl[desc[i].dbl + 4 + si]));
          }
          const double total = dadd(fwd, dmul(backward(S, w0, w1), H.keep_bwd));
          const unsigned long long tb = (unsigned long long)__double_as_longlong(total);
          const uint32_t ns = num_split_of(w0, w1);
          const unsigned long long idx = ref_index(S, w0, w1);
          nvalid++;
          if (key_less(tb, ns, idx, best_t, best_n, best_i)) {
            best_t = tb;
            best_n = ns;
            best_i = idx;
          }
        }
        pw0 = w0;
        pw1 = w1;
        first = false;
        mr_add(bw0, bw1, 32, H.V, H.radix3);
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const unsigned long long t2 = __shfl_down_sync(0xffffffffu, best_t, o);
      const unsigned long long i2 = __shfl_down_sync(0xffffffffu, best_i, o);
      const uint32_t n2 = __shfl_down_sync(0xffffffffu, best_n, o);
      nvalid += __shfl_down_sync(0xffffffffu, nvalid, o);
      if (key_less(t2, n2, i2, best_t, best_n, best_i)) {
        best_t = t2;
        best_n = n2;
        best_i = i2;
      }
    }
    if (lane == 0) {
      s_red_t[warp] = best_t;
      s_red_i[warp] = best_i;
      s_red_n[warp] = best_n;
      s_red_v[warp] = nvalid;
    }
    __syncthreads();
    if (tid == 0) {
      ItemOut o{s_red_t[0], s_red_i[0], s_red_n[0], s_red_v[0]};
      for (int w = 1; w < THREADS_M / 32; w++) {
        o.valid += s_red_v[w];
        if (key_less(s_red_t[w], s_red_n[w], s_red_i[w], o.total_bits, o.num_split, o.index)) {
          o.total_bits = s_red_t[w];
          o.num_split = s_red_n[w];
          o.index = s_red_i[w];
        }
      }
      items[item] = o;
    }
  }
}

// Per-candidate totals over a REFERENCE index range [lo, hi) of one block
// (want_table / _eval_range table rows): every candidate walked, NaN = invalid.
__global__ void __launch_bounds__(THREADS) k_score_table(const uint8_t* __restrict__ blobs, int64_t blob_off,
                                                         unsigned long long lo, unsigned long long hi,
                                                         double* __restrict__ totals, ItemOut* __restrict__ cta_out) {
  extern __shared__ __align__(16) uint8_t smem[];
  __shared__ unsigned long long s_red_t[THREADS / 32], s_red_i[THREADS / 32];
  __shared__ uint32_t s_red_n[THREADS / 32], s_red_v[THREADS / 32];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  stage_blob(smem, blobs, blob_off);
  __syncthreads();
  const Tabs S = tabs_of(smem);
  const BlobHeader& H = *S.H;
  unsigned long long best_t = ~0ULL, best_i = ~0ULL;
  uint32_t best_n = 0xFFFFFFFFu, nvalid = 0;
  const unsigned long long stride = (unsigned long long)gridDim.x * THREADS;
  for (unsigned long long base = lo + (unsigned long long)blockIdx.x * THREADS + warp * 32; base < hi; base += stride) {
    const unsigned long long x = base + lane;
    const bool active = x < hi;
    // reference digits -> enumeration positions
    uint64_t w0 = 0, w1 = 0;
    unsigned long long rem = active ? x : 0;
    for (int sidx = H.V - 1; sidx >= 0; sidx--) {
      const uint32_t r = ((H.radix3_ref >> sidx) & 1) ? 3 : 2;
      const uint32_t d = (uint32_t)(rem % r);
      rem /= r;
      const int q = S.perm[sidx];
      if (q < 32) w0 |= (uint64_t)d << (q * 2);
      else w1 |= (uint64_t)d << ((q - 32) * 2);
    }
    double fwd;
    const int fail = walk<DM_WIDE>(S, w0, w1, active, fwd, tid);
    if (fail < 0) {
      const double total = dadd(fwd, dmul(backward(S, w0, w1), H.keep_bwd));
      const unsigned long long tb = (unsigned long long)__double_as_longlong(total);
      const uint32_t ns = num_split_of(w0, w1);
      nvalid++;
      if (key_less(tb, ns, x, best_t, best_n, best_i)) {
        best_t = tb;
        best_n = ns;
        best_i = x;
      }
      if (totals) totals[x - lo] = total;
    } else if (active && totals) {
      totals[x - lo] = __longlong_as_double(0x7ff8000000000000LL);
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const unsigned long long t2 = __shfl_down_sync(0xffffffffu, best_t, o);
    const unsigned long long i2 = __shfl_down_sync(0xffffffffu, best_i, o);
    const uint32_t n2 = __shfl_down_sync(0xffffffffu, best_n, o);
    nvalid += __shfl_down_sync(0xffffffffu, nvalid, o);
    if (key_less(t2, n2, i2, best_t, best_n, best_i)) {
      best_t = t2;
      best_n = n2;
      best_i = i2;
    }
  }
  if (lane == 0) {
    s_red_t[warp] = best_t;
    s_red_i[warp] = best_i;
    s_red_n[warp] = best_n;
    s_red_v[warp] = nvalid;
  }
  __syncthreads();
  if (tid == 0) {
    ItemOut o{s_red_t[0], s_red_i[0], s_red_n[0], s_red_v[0]};
    for (int w = 1; w < THREADS / 32; w++) {
      o.valid += s_red_v[w];
      if (key_less(s_red_t[w], s_red_n[w], s_red_i[w], o.total_bits, o.num_split, o.index)) {
        o.total_bits = s_red_t[w];
        o.num_split = s_red_n[w];
        o.index = s_red_i[w];
      }
    }
    cta_out[blockIdx.x] = o;
  }
}

// One CTA per block: merge its items.
__global__ void k_reduce(const ItemOut* __restrict__ items, const unsigned long long* __restrict__ item_base,
                         int64_t nb, sp_score_out* __restrict__ out) {
  __shared__ ItemOut s[THREADS];
  for (int64_t b = blockIdx.x; b < nb; b += gridDim.x) {
    ItemOut acc{~0ULL, ~0ULL, 0xFFFFFFFFu, 0};
    unsigned long long valid = 0;
    for (unsigned long long it = item_base[b] + threadIdx.x; it < item_base[b + 1]; it += blockDim.x) {
      const ItemOut o = items[it];
      valid += o.valid;
      if (key_less(o.total_bits, o.num_split, o.index, acc.total_bits, acc.num_split, acc.index)) acc = o;
    }
    acc.valid = 0;
    s[threadIdx.x] = acc;
    __shared__ unsigned long long sv[THREADS];
    sv[threadIdx.x] = valid;
    __syncthreads();
    for (int st = blockDim.x / 2; st > 0; st >>= 1) {
      if (threadIdx.x < st) {
        const ItemOut o = s[threadIdx.x + st];
        if (key_less(o.total_bits, o.num_split, o.index, s[threadIdx.x].total_bits, s[threadIdx.x].num_split,
                     s[threadIdx.x].index))
          s[threadIdx.x] = o;
        sv[threadIdx.x] += sv[threadIdx.x + st];
      }
      __syncthreads();
    }
    if (threadIdx.x == 0) {
      sp_score_out r;
      r.candidates = 0;
      r.valid = sv[0];
      r.has_best = s[0].index != ~0ULL && sv[0] > 0;
      r.best_index = r.has_best ? s[0].index : 0;
      r.best_total = r.has_best ? __longlong_as_double((long long)s[0].total_bits) : 0.0;
      r.best_num_split = r.has_best ? (int32_t)s[0].num_split : 0;
      out[b] = r;
    }
    __syncthreads();
  }
}

// First pass of the two-pass item reduction (blocks with many items: one CTA
// reducing a block's 50k items serially cost 0.13 ms on c5): CTA c reduces
// chunk c of REDUCE_CHUNK consecutive items of one block into partial[c]
// (argmin key + summed valid count); k_reduce then merges each block's
// partials (chunk_base[b] .. chunk_base[b + 1]).
constexpr int REDUCE_CHUNK = 1024;
__global__ void __launch_bounds__(THREADS) k_reduce_chunks(const ItemOut* __restrict__ items,
                                                           const unsigned long long* __restrict__ item_base,
                                                           const unsigned long long* __restrict__ chunk_base,
                                                           int64_t nb, unsigned long long n_chunks,
                                                           ItemOut* __restrict__ partial) {
  __shared__ ItemOut s_w[THREADS / 32];
  for (unsigned long long c = blockIdx.x; c < n_chunks; c += gridDim.x) {
    int64_t lo = 0, hi = nb;
    while (hi - lo > 1) {
      const int64_t mid = (lo + hi) / 2;
      if (chunk_base[mid] <= c) lo = mid;
      else hi = mid;
    }
    const unsigned long long i0 = item_base[lo] + (c - chunk_base[lo]) * REDUCE_CHUNK;
    const unsigned long long i1 = min(i0 + REDUCE_CHUNK, item_base[lo + 1]);
    ItemOut acc{~0ULL, ~0ULL, 0xFFFFFFFFu, 0};
    unsigned long long valid = 0;
    for (unsigned long long it = i0 + threadIdx.x; it < i1; it += blockDim.x) {
      const ItemOut o = items[it];
      valid += o.valid;
      if (key_less(o.total_bits, o.num_split, o.index, acc.total_bits, acc.num_split, acc.index)) acc = o;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const unsigned long long t2 = __shfl_down_sync(0xffffffffu, acc.total_bits, o);
      const unsigned long long i2 = __shfl_down_sync(0xffffffffu, acc.index, o);
      const uint32_t n2 = __shfl_down_sync(0xffffffffu, acc.num_split, o);
      valid += __shfl_down_sync(0xffffffffu, valid, o);
      if (key_less(t2, n2, i2, acc.total_bits, acc.num_split, acc.index)) {
        acc.total_bits = t2;
        acc.num_split = n2;
        acc.index = i2;
      }
    }
    if ((threadIdx.x & 31) == 0) {
      acc.valid = valid;
      s_w[threadIdx.x >> 5] = acc;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      ItemOut r = s_w[0];
      for (int w = 1; w < THREADS / 32; w++) {
        r.valid += s_w[w].valid;
        if (key_less(s_w[w].total_bits, s_w[w].num_split, s_w[w].index, r.total_bits, r.num_split, r.index)) {
          r.total_bits = s_w[w].total_bits;
          r.num_split = s_w[w].num_split;
          r.index = s_w[w].index;
        }
      }
      partial[c] = r;
    }
    __syncthreads();
  }
}

// Full detail of one candidate (RoutedPlan + CostReport), single thread.
__global__ void k_explain(GraphView G, const int32_t* tmpl, int T, int32_t blk, const int32_t* node_block,
                          const int32_t* node_tpos, const int16_t* slot_of, const uint8_t* digits,
                          const uint8_t* boundary, sp_mesh mesh, int64_t mu, int64_t chunk,
                          sp_explain_out* out, sp_edge_conv* edges, int32_t max_edges, int32_t* n_edges) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  const MeshC M = mesh_consts(mesh);
  int state[MAXT];

  double reach[MAXT];
  out->valid = 0;
  out->T = T;
  out->fail_pos = -1;
  int ne = 0;
  int64_t bytes[5] = {0, 0, 0, 0, 0}, calls[5] = {0, 0, 0, 0, 0};
  NodeRoute R;
  for (int i = 0; i < T; i++) {
    const int32_t n = tmpl[i];
    int ps[64];
    int k = 0;
    for (int64_t e = G.in_off[n]; e < G.in_off[n + 1]; e++) {
      const int32_t r = G.in_idx[e];
      if (node_block[r] != blk) continue;
      if (k < 64) ps[k] = state[node_tpos[r]];
      k++;
    }
    const int digit = slot_of[i] >= 0 ? digits[slot_of[i]] : 0;
    route_node(G, n, blk, node_block, digit, ps, M, &R, true);
    if (R.pattern < 0) {
      out->fail_pos = i;
      *n_edges = ne;
      return;
    }

    state[i] = R.state;
    Pattern pats[4];
    patterns_for(G.op[n], pats);
    double base = 0.0;
    int j = 0;
    for (int64_t e = G.in_off[n]; e < G.in_off[n + 1]; e++) {
      const int32_t r = G.in_idx[e];
      if (node_block[r] != blk) continue;
      const int kind = R.conv_kind[j];
      double cc = 0.0;
      if (kind != C_ID) {
        cc = call_cost(kind, G.act_bytes[r], M);
        bytes[kind] += G.act_bytes[r];
        calls[kind]++;
        if (ne < max_edges) edges[ne] = sp_edge_conv{i, node_tpos[r], kind, R.conv_axis[j]};
        ne++;
      }
      base = fmax(base, dadd(reach[node_tpos[r]], cc));
      j++;
    }
    const int pc = pats[R.pattern].coll;
    if (pc != C_ID) {
      bytes[pc] += G.act_bytes[n];
      calls[pc]++;
    }
    reach[i] = dadd(base, call_cost(pc, G.act_bytes[n], M));
    out->pattern[i] = R.pattern;
    const NSpec fs = state_spec(R.state, G.act_rank[n]);
    out->state_axis[i] = fs.kind == K_S ? fs.axis : -1;
  }
  double fwd = 0.0;
  for (int i = 0; i < T; i++) {
    const int32_t n = tmpl[i];
    double tail = reach[i];
    out->exit_axis[i] = -1;
    if (boundary[i] && state[i] != 0) {
      tail = dadd(tail, call_cost(C_AG, G.act_bytes[n], M));
      bytes[C_AG] += G.act_bytes[n];
      calls[C_AG]++;
      out->exit_axis[i] = state_spec(state[i], G.act_rank[n]).axis;
    }
    fwd = fmax(fwd, tail);
  }
  double bwd = 0.0;
  if (M.d > 1) {
    int64_t bk[MAXT], uf[MAXT];
    int nbk = 0, nuf = 0, cur_n = 0;
    int64_t cur = 0;
    for (int i = 0; i < T; i++) {
      const int32_t n = tmpl[i];
      if (!G.w_rank[n] || !G.w_train[n] || digits[slot_of[i]] != 0) continue;
      const int64_t sz = G.w_bytes[n];
      if (sz >= mu) {
        uf[nuf++] = sz;
        continue;
      }
      if (cur + sz > chunk && cur_n) {
        bk[nbk++] = cur;
        cur = 0;
        cur_n = 0;
      }
      cur += sz;
      cur_n++;
    }
    if (cur_n) bk[nbk++] = cur;
    for (int q = 0; q < nbk; q++) {
      bwd = dadd(bwd, dadd(M.setup, cost_bytes(C_AR, bk[q], M)));
      bytes[C_AR] += bk[q];
      calls[C_AR]++;
    }
    for (int q = 0; q < nuf; q++) {
      bwd = dadd(bwd, dadd(M.setup, cost_bytes(C_AR, uf[q], M)));
      bytes[C_AR] += uf[q];
      calls[C_AR]++;
    }
  }
  out->valid = 1;
  out->forward_comm = fwd;
  out->backward_comm = bwd;
  out->total = dadd(fwd, dmul(bwd, dadd(1.0, -mesh.overlap_fraction)));
  out->bytes_allreduce = bytes[C_AR];
  out->bytes_allgather = bytes[C_AG];
  out->bytes_reducescatter = bytes[C_RS];
  out->bytes_alltoall = bytes[C_A2A];
  out->calls_allreduce = calls[C_AR];
  out->calls_allgather = calls[C_AG];
  out->calls_reducescatter = calls[C_RS];
  out->calls_alltoall = calls[C_A2A];
  out->collective_calls = calls[C_AR] + calls[C_AG] + calls[C_RS] + calls[C_A2A];
  *n_edges = ne;
}

struct ExplainBlock {
  int32_t valid, fail_pos;
  double forward_comm, backward_comm, total;
  int64_t bytes[4];  // allreduce, allgather, reducescatter, alltoall
  int64_t calls[4];
  int64_t collective_calls;
};
static_assert(sizeof(ExplainBlock) == sizeof(sp_explain_block), "ExplainBlock mirrors sp_explain_block");

// Winner detail for every block in one launch (one thread per block walks
// its template): pattern / state / exit per node, conversion per internal
// edge, forward/backward/total and collective accounting (plan_cost,
// costmodel.py:193-267).  indices[b] == ~0 skips a block.
// k_explain_all from the routing tables instead of re-deriving every pattern
// choice: one warp per block stages the blob into shared memory, then lane 0
// walks the template with the candidate's digits -- the routing byte of each
// node gives its pattern and state (0xFF: the first node that cannot route),
// the fp64 tables its reach (the scoring walk's own operations), and the
// conversion collectives come from the XEdge table k_fill filled with the
// same route_node evaluation.  The backward pass repeats k_explain_all's.
// The winner detail of block b (candidate `index`) by one warp, from its blob
// staged at `smem` (k_explain_fast, and k_search_small after its scoring):
// lane 0 walks the template with the candidate's digits -- the routing byte
// of each node gives its pattern and state (0xFF: the first node that cannot
// route), the fp64 tables its reach (the scoring walk's own operations), and
// the conversion collectives come from the XEdge table k_fill filled with the
// same route_node evaluation.  The backward pass repeats k_explain_all's.
// s_dig: 64 bytes of shared memory, s_ok: one int of shared memory.
// the per-node records explain_warp's lane 0 reads in its serial walk, pulled
// into L1 by the whole warp first (each of those loads would otherwise wait on L2)
__device__ __forceinline__ void explain_prefetch(int64_t b, int64_t e0, int T, const int16_t* ref_slot_of,
                                                 const uint8_t* bound_of, const uint8_t* xinfo, const int64_t* xoff) {
  const int lane = threadIdx.x & 31;
  const uint8_t* xb = xinfo + xoff[b];
  const int64_t xbytes = xoff[b + 1] - xoff[b];
  for (int64_t q = lane * 128; q < xbytes; q += 32 * 128) asm volatile("prefetch.global.L1 [%0];" ::"l"(xb + q));
  for (int q = lane * 128; q < 2 * T; q += 32 * 128)
    asm volatile("prefetch.global.L1 [%0];" ::"l"((const uint8_t*)(ref_slot_of + e0) + q));
  for (int q = lane * 128; q < T; q += 32 * 128) asm volatile("prefetch.global.L1 [%0];" ::"l"(bound_of + e0 + q));
}

__device__ void explain_warp(int64_t b, unsigned long long index, uint8_t* smem, GraphView G, const int64_t* tmpl_off,
                             const int32_t* tmpl_nodes, const int16_t* ref_slot_of, const uint8_t* bound_of,
                             const uint8_t* xinfo, const int64_t* xoff, const int64_t* edge_off, sp_mesh mesh,
                             int64_t mu, int64_t chunk, ExplainBlock* out, int8_t* node_out, int8_t* edge_out,
                             uint8_t* s_dig, int* s_ok_p) {
  const MeshC M = mesh_consts(mesh);
  const int lane = threadIdx.x & 31;
  const int64_t e0 = tmpl_off[b];
  int& s_ok = *s_ok_p;
  const BlobHeader& H = *(const BlobHeader*)smem;
  const NodeDesc* desc = (const NodeDesc*)(smem + H.desc_off);
  const int16_t* prodpos = (const int16_t*)(smem + H.prod_off) + H.n_prod;
  const uint8_t* tab = smem + H.tab_off;
  const double* dbl = (const double*)(smem + H.dbl_off);
  const XNode* xn = (const XNode*)(xinfo + xoff[b]);
  const int T = H.T;
  const XEdge* xe = (const XEdge*)(xinfo + xoff[b] + (int64_t)sizeof(XNode) * T);
  ExplainBlock X;
  X.valid = 0;
  X.fail_pos = -1;
  X.forward_comm = X.backward_comm = X.total = 0.0;
  for (int k = 0; k < 4; k++) X.bytes[k] = X.calls[k] = 0;
  X.collective_calls = 0;
  double fwd = 0.0;
  if (lane == 0) {
    // reference slot order (candidate_by_index, search.py:103-116)
    unsigned long long rem = index;
    for (int q = H.V - 1; q >= 0; q--) {
      const uint32_t r = ((H.radix3_ref >> q) & 1) ? 3 : 2;
      s_dig[q] = (uint8_t)(rem % r);
      rem /= r;
    }
    uint8_t state[MAXT];
    double reach[MAXT];
    int64_t eo = edge_off[b];
    bool ok = true;
    for (int i = 0; i < T; i++) {
      const NodeDesc nd = desc[i];
      const int slot = ref_slot_of[e0 + i];
      uint32_t key = slot >= 0 ? s_dig[slot] : 0;
      for (int j = 0; j < nd.k; j++) key = key * 3 + state[prodpos[nd.prod + j]];
      const uint8_t e = tab[nd.tab + key];
      if (e == 0xFF) {
        X.fail_pos = i;
        ok = false;
        break;
      }
      const int p = e & 3, st = e >> 2;
      state[i] = (uint8_t)st;
      const double* dn = dbl + nd.dbl;
      double base = 0.0;
      for (int j = 0; j < nd.k; j++) {
        const int pp = prodpos[nd.prod + j];
        const int sj = state[pp];
        const int kind = xe[nd.prod + j].kind[p][sj];
        if (kind > 0) {
          X.bytes[kind - 1] += xn[pp].act_bytes;
          X.calls[kind - 1]++;
        }
        edge_out[2 * eo] = (int8_t)kind;
        edge_out[2 * eo + 1] = xe[nd.prod + j].axis[p][sj];
        eo++;
        base = fmax(base, dadd(reach[pp], dn[8 + (j * 4 + p) * 3 + sj]));
      }
      Pattern pats[4];
      patterns_for(xn[i].op, pats);
      const int pc = pats[p].coll;
      if (pc != C_ID) {
        X.bytes[pc - 1] += xn[i].act_bytes;
        X.calls[pc - 1]++;
      }
      reach[i] = dadd(base, dn[p]);
      const NSpec fs = state_spec(st, xn[i].act_rank);
      node_out[4 * (e0 + i)] = (int8_t)p;
      node_out[4 * (e0 + i) + 1] = fs.kind == K_S ? fs.axis : -1;
      node_out[4 * (e0 + i) + 2] = -1;
      node_out[4 * (e0 + i) + 3] = 0;
    }
    if (ok)
      for (int i = 0; i < T; i++) {
        double tail = reach[i];
        if (bound_of[e0 + i] && state[i] != 0) {
          tail = dadd(tail, dbl[desc[i].dbl + 4 + state[i]]);
          X.bytes[C_AG - 1] += xn[i].act_bytes;
          X.calls[C_AG - 1]++;
          node_out[4 * (e0 + i) + 2] = state_spec(state[i], xn[i].act_rank).axis;
        }
        fwd = fmax(fwd, tail);
      }
    s_ok = ok;
  }
  __syncwarp();
  if (!s_ok) {
    if (lane == 0) out[b] = X;
    return;
  }
  double bwd = 0.0;
  if (M.d > 1) {
    // pack_gradients (rewrite.py:78-111): buckets first, then unfused, each one AllReduce.
    // Each trainable weight's byte size (-1: not all-replica / not trainable) is
    // looked up by the warp into shared memory (the blob is no longer read).
    int64_t* szs = (int64_t*)smem;
    for (int i = lane; i < T; i += 32) {
      const int32_t n = tmpl_nodes[e0 + i];
      szs[i] = (!G.w_rank[n] || !G.w_train[n] || s_dig[ref_slot_of[e0 + i]] != 0) ? -1 : G.w_bytes[n];
    }
    __syncwarp();
    if (lane == 0) {
      int64_t cur = 0;
      int cur_n = 0;
      for (int pass = 0; pass < 2; pass++) {
        for (int i = 0; i < T; i++) {
          const int64_t sz = szs[i];
          if (sz < 0) continue;
          if (pass == 0) {
            if (sz >= mu) continue;
            if (cur + sz > chunk && cur_n) {
              bwd = dadd(bwd, dadd(M.setup, cost_bytes(C_AR, cur, M)));
              X.bytes[0] += cur;
              X.calls[0]++;
              cur = 0;
              cur_n = 0;
            }
            cur += sz;
            cur_n++;
          } else if (sz >= mu) {
            bwd = dadd(bwd, dadd(M.setup, cost_bytes(C_AR, sz, M)));
            X.bytes[0] += sz;
            X.calls[0]++;
          }
        }
        if (pass == 0 && cur_n) {
          bwd = dadd(bwd, dadd(M.setup, cost_bytes(C_AR, cur, M)));
          X.bytes[0] += cur;
          X.calls[0]++;
        }
      }
    }
  }
  if (lane == 0) {
    X.valid = 1;
    X.forward_comm = fwd;
    X.backward_comm = bwd;
    X.total = dadd(fwd, dmul(bwd, dadd(1.0, -mesh.overlap_fraction)));
    X.collective_calls = X.calls[0] + X.calls[1] + X.calls[2] + X.calls[3];
    out[b] = X;
  }
}

// k_explain_all from the routing tables instead of re-deriving every pattern
// choice: one warp per block stages the blob into shared memory, then runs
// explain_warp.
__global__ void k_explain_fast(GraphView G, const int64_t* tmpl_off, const int32_t* tmpl_nodes, int64_t nb,
                               const int16_t* ref_slot_of, const uint8_t* bound_of, const uint8_t* blobs,
                               const int64_t* blob_off, const uint8_t* xinfo, const int64_t* xoff,
                               const int64_t* edge_off, const unsigned long long* indices,
                               const sp_score_out* scores, sp_mesh mesh, int64_t mu, int64_t chunk,
                               ExplainBlock* out, int8_t* node_out, int8_t* edge_out) {
  extern __shared__ __align__(16) uint8_t smem[];
  __shared__ uint8_t s_dig[64];
  __shared__ int s_ok;
  const int lane = threadIdx.x & 31;
  for (int64_t b = blockIdx.x; b < nb; b += gridDim.x) {
    const unsigned long long index =
        scores ? (scores[b].has_best ? scores[b].best_index : ~0ULL) : indices[b];
    if (index == ~0ULL) {
      if (lane == 0) {
        ExplainBlock X{};
        X.fail_pos = -1;
        out[b] = X;
      }
      continue;
    }
    const BlobHeader* gH = (const BlobHeader*)(blobs + blob_off[b]);
    const int nbytes = gH->bytes;
    const int64_t e0 = tmpl_off[b];
    __syncwarp();
    for (int q = lane * 16; q < nbytes; q += 32 * 16)
      *(int4*)(smem + q) = *(const int4*)(blobs + blob_off[b] + q);
    explain_prefetch(b, e0, gH->T, ref_slot_of, bound_of, xinfo, xoff);
    __syncwarp();
    explain_warp(b, index, smem, G, tmpl_off, tmpl_nodes, ref_slot_of, bound_of, xinfo, xoff, edge_off, mesh, mu,
                 chunk, out, node_out, edge_out, s_dig, &s_ok);
    __syncwarp();
  }
}

// Searches whose every block is small (<= SMALL_SEARCH_MAX_C candidates: the
// BASELINE configs c1/c3/c4) in ONE kernel: a
// CTA per block stages its tables, its warps walk the block's candidates in
// SMALL_CH-candidate chunks, the CTA reduces the argmin, and warp 0 explains
// the winner from the tables already staged -- instead of the work-item
// scorer, k_reduce and k_explain_fast (three launches, the winner's tables
// staged twice, a global round trip of the per-item records).
// (one CTA walks a whole block: c5's residual group, whose largest blocks hold
// ~2^16 candidates, took 0.67 ms this way against 0.19 ms on the item path)
constexpr unsigned long long SMALL_SEARCH_MAX_C = 8192;
constexpr uint32_t SMALL_CH = 256;
template <bool SKIP>
__global__ void __launch_bounds__(THREADS, SP_SCORE_MIN_BLOCKS) k_search_small(
    const uint8_t* __restrict__ blobs, const int64_t* __restrict__ blob_off, int64_t nb, GraphView G,
    const int64_t* tmpl_off, const int32_t* tmpl_nodes, const int16_t* ref_slot_of, const uint8_t* bound_of,
    const uint8_t* xinfo, const int64_t* xoff, const int64_t* edge_off, sp_mesh mesh, int64_t mu, int64_t chunk,
    sp_score_out* __restrict__ dout, ExplainBlock* xout, int8_t* node_out, int8_t* edge_out) {
  extern __shared__ __align__(16) uint8_t smem[];
  constexpr int NW = THREADS / 32;
  __shared__ uint64_t s_lane_add[32];
  __shared__ Biased s_bz;
  __shared__ unsigned long long s_red_t[NW], s_red_i[NW], s_red_v[NW];
  __shared__ uint32_t s_red_n[NW];
  __shared__ unsigned long long s_best;
  __shared__ uint8_t s_dig[64];
  __shared__ int s_ok;
  const int tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;
  for (int64_t b = blockIdx.x; b < nb; b += gridDim.x) {
    stage_block(smem, blobs, blob_off[b], s_lane_add, &s_bz, nullptr, 1, 0, false);
    const Tabs S = tabs_of(smem);
    const BlobHeader& H = *S.H;
    const uint32_t rec0 = opaque_u32((uint32_t)__cvta_generic_to_shared(smem) + (uint32_t)H.fast_off);
    const uint32_t pool = (uint32_t)__cvta_generic_to_shared(S.reach);
    const uint32_t rb = opaque_u32(pool + 8u * (uint32_t)tid);
    const uint32_t sb = opaque_u32(pool + (uint32_t)H.npool * THREADS * 8u + (uint32_t)tid);
    const unsigned long long C = H.C;
    LaneBest lb;
    for (unsigned long long start = (unsigned long long)warp * SMALL_CH; start < C;
         start += (unsigned long long)NW * SMALL_CH) {
      const uint32_t rem = (uint32_t)min((unsigned long long)SMALL_CH, C - start);
      const uint64_t w = badd(bencode(H, start), s_lane_add[lane], s_bz.B);
      score_chunk<SKIP, false>(S, s_bz, s_lane_add, rec0, rb, sb, lane, w, rem, start + rem, lb);
    }
    // the block's argmin of (total bits, num_split, index) and valid count
    unsigned long long bt = lb.t, bi = lb.t != ~0ULL ? ref_index_b(S, lb.w) : ~0ULL, nv = lb.valid;
    uint32_t bn = lb.n;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const unsigned long long t2 = __shfl_down_sync(0xffffffffu, bt, o);
      const unsigned long long i2 = __shfl_down_sync(0xffffffffu, bi, o);
      const uint32_t n2 = __shfl_down_sync(0xffffffffu, bn, o);
      nv += __shfl_down_sync(0xffffffffu, nv, o);
      if (key_less(t2, n2, i2, bt, bn, bi)) {
        bt = t2;
        bn = n2;
        bi = i2;
      }
    }
    if (lane == 0) {
      s_red_t[warp] = bt;
      s_red_i[warp] = bi;
      s_red_n[warp] = bn;
      s_red_v[warp] = nv;
    }
    __syncthreads();
    if (tid == 0) {
      unsigned long long t = s_red_t[0], i = s_red_i[0], v = s_red_v[0];
      uint32_t n = s_red_n[0];
      for (int w2 = 1; w2 < NW; w2++) {
        v += s_red_v[w2];
        if (key_less(s_red_t[w2], s_red_n[w2], s_red_i[w2], t, n, i)) {
          t = s_red_t[w2];
          n = s_red_n[w2];
          i = s_red_i[w2];
        }
      }
      sp_score_out r;
      r.candidates = C;
      r.valid = v;
      r.has_best = i != ~0ULL && v > 0;
      r.best_index = r.has_best ? i : 0;
      r.best_total = r.has_best ? __longlong_as_double((long long)t) : 0.0;
      r.best_num_split = r.has_best ? (int32_t)n : 0;
      dout[b] = r;
      s_best = r.has_best ? i : ~0ULL;
    }
    __syncthreads();
    if (warp == 0) {
      const unsigned long long index = s_best;
      if (index == ~0ULL) {
        if (lane == 0) {
          ExplainBlock X{};
          X.fail_pos = -1;
          xout[b] = X;
        }
      } else {
        explain_prefetch(b, tmpl_off[b], H.T, ref_slot_of, bound_of, xinfo, xoff);
        __syncwarp();
        explain_warp(b, index, smem, G, tmpl_off, tmpl_nodes, ref_slot_of, bound_of, xinfo, xoff, edge_off, mesh,
                     mu, chunk, xout, node_out, edge_out, s_dig, &s_ok);
      }
    }
    __syncthreads();  // the next block's tables overwrite shared memory
  }
}

__global__ void k_explain_all(GraphView G, const int64_t* tmpl_off, const int32_t* tmpl_nodes, int64_t nb,
                              const int32_t* node_block, const int32_t* node_tpos, const int16_t* slot_of,
                              const uint8_t* bound_of, const uint8_t* blobs, const int64_t* blob_off,
                              const int64_t* edge_off, const unsigned long long* indices,
                              const sp_score_out* scores, sp_mesh mesh,
                              int64_t mu, int64_t chunk, ExplainBlock* out, int8_t* node_out, int8_t* edge_out) {
  const MeshC M = mesh_consts(mesh);
  for (int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; b < nb; b += (int64_t)gridDim.x * blockDim.x) {
    ExplainBlock X;
    X.valid = 0;
    X.fail_pos = -1;
    X.forward_comm = X.backward_comm = X.total = 0.0;
    for (int k = 0; k < 4; k++) X.bytes[k] = X.calls[k] = 0;
    X.collective_calls = 0;
    const unsigned long long index =
        scores ? (scores[b].has_best ? scores[b].best_index : ~0ULL) : indices[b];
    if (index == ~0ULL) {
      out[b] = X;
      continue;
    }
    const BlobHeader* H = (const BlobHeader*)(blobs + blob_off[b]);
    const int V = H->V;
    uint8_t dig[64];  // reference slot order (candidate_by_index, search.py:103-116)
    unsigned long long rem = index;
    for (int s = V - 1; s >= 0; s--) {
      const uint32_t r = ((H->radix3_ref >> s) & 1) ? 3 : 2;
      dig[s] = (uint8_t)(rem % r);
      rem /= r;
    }
    const int64_t e0 = tmpl_off[b];
    const int T = (int)(tmpl_off[b + 1] - e0);
    int state[MAXT];
    double reach[MAXT];
    int64_t eo = edge_off[b];
    NodeRoute R;
    bool ok = true;
    for (int i = 0; i < T && ok; i++) {
      const int32_t n = tmpl_nodes[e0 + i];
      int ps[64];
      int k = 0;
      for (int64_t e = G.in_off[n]; e < G.in_off[n + 1]; e++) {
        const int32_t r = G.in_idx[e];
        if (node_block[r] != (int32_t)b) continue;
        if (k < 64) ps[k] = state[node_tpos[r]];
        k++;
      }
      const int digit = slot_of[e0 + i] >= 0 ? dig[slot_of[e0 + i]] : 0;
      route_node(G, n, (int32_t)b, node_block, digit, ps, M, &R, true);
      if (R.pattern < 0) {
        X.fail_pos = i;
        ok = false;
        break;
      }
      state[i] = R.state;
      Pattern pats[4];
      patterns_for(G.op[n], pats);
      double base = 0.0;
      int j = 0;
      for (int64_t e = G.in_off[n]; e < G.in_off[n + 1]; e++) {
        const int32_t r = G.in_idx[e];
        if (node_block[r] != (int32_t)b) continue;
        const int kind = R.conv_kind[j];
        double cc = 0.0;
        if (kind != C_ID) {
          cc = call_cost(kind, G.act_bytes[r], M);
          X.bytes[kind - 1] += G.act_bytes[r];
          X.calls[kind - 1]++;
        }
        edge_out[2 * eo] = (int8_t)kind;
        edge_out[2 * eo + 1] = R.conv_axis[j];
        eo++;
        base = fmax(base, dadd(reach[node_tpos[r]], cc));
        j++;
      }
      const int pc = pats[R.pattern].coll;
      if (pc != C_ID) {
        X.bytes[pc - 1] += G.act_bytes[n];
        X.calls[pc - 1]++;
      }
      reach[i] = dadd(base, call_cost(pc, G.act_bytes[n], M));
      const NSpec fs = state_spec(R.state, G.act_rank[n]);
      node_out[4 * (e0 + i)] = (int8_t)R.pattern;
      node_out[4 * (e0 + i) + 1] = fs.kind == K_S ? fs.axis : -1;
      node_out[4 * (e0 + i) + 2] = -1;
      node_out[4 * (e0 + i) + 3] = 0;  // unused byte, kept deterministic
    }
    if (!ok) {
      out[b] = X;
      continue;
    }
    double fwd = 0.0;
    for (int i = 0; i < T; i++) {
      const int32_t n = tmpl_nodes[e0 + i];
      double tail = reach[i];
      if (bound_of[e0 + i] && state[i] != 0) {
        tail = dadd(tail, call_cost(C_AG, G.act_bytes[n], M));
        X.bytes[C_AG - 1] += G.act_bytes[n];
        X.calls[C_AG - 1]++;
        node_out[4 * (e0 + i) + 2] = state_spec(state[i], G.act_rank[n]).axis;
      }
      fwd = fmax(fwd, tail);
    }
    double bwd = 0.0;
    if (M.d > 1) {
      // pack_gradients (rewrite.py:78-111): buckets first, then unfused, each one AllReduce
      int64_t cur = 0;
      int cur_n = 0;
      for (int pass = 0; pass < 2; pass++) {
        for (int i = 0; i < T; i++) {
          const int32_t n = tmpl_nodes[e0 + i];
          if (!G.w_rank[n] || !G.w_train[n] || dig[slot_of[e0 + i]] != 0) continue;
          const int64_t sz = G.w_bytes[n];
          if (pass == 0) {
            if (sz >= mu) continue;
            if (cur + sz > chunk && cur_n) {
              bwd = dadd(bwd, dadd(M.setup, cost_bytes(C_AR, cur, M)));
              X.bytes[0] += cur;
              X.calls[0]++;
              cur = 0;
              cur_n = 0;
            }
            cur += sz;
            cur_n++;
          } else if (sz >= mu) {
            bwd = dadd(bwd, dadd(M.setup, cost_bytes(C_AR, sz, M)));
            X.bytes[0] += sz;
            X.calls[0]++;
          }
        }
        if (pass == 0 && cur_n) {
          bwd = dadd(bwd, dadd(M.setup, cost_bytes(C_AR, cur, M)));
          X.bytes[0] += cur;
          X.calls[0]++;
        }
      }
    }
    X.valid = 1;
    X.forward_comm = fwd;
    X.backward_comm = bwd;
    X.total = dadd(fwd, dmul(bwd, dadd(1.0, -mesh.overlap_fraction)));
    X.collective_calls = X.calls[0] + X.calls[1] + X.calls[2] + X.calls[3];
    out[b] = X;
  }
}

inline int grid_for(int64_t n, int sms, int threads = 256) {
  int64_t b = (n + threads - 1) / threads;
  if (b < 1) b = 1;
  const int64_t cap = (int64_t)sms * 16;
  return (int)(b < cap ? b : cap);
}

int strcmp_py(const uint8_t* a, int64_t la, const uint8_t* b, int64_t lb) {
  const int64_t m = la < lb ? la : lb;
  const int c = m ? std::memcmp(a, b, (size_t)m) : 0;
  if (c) return c;
  return (la > lb) - (la < lb);
}

GraphView view_of(sp_dgraph* dg) {
  return GraphView{dg->op.p,      dg->act_rank.p, dg->act_shape.p, dg->act_bytes.p, dg->w_rank.p,
                   dg->w_shape.p, dg->w_bytes.p,  dg->w_train.p,   dg->in_off.p,    dg->in_idx.p};
}

// per-table device state kept for scoring/explain
struct TableDev {
  DevBuf<int32_t> node_block, node_tpos;
  DevBuf<int16_t> slot_of, ref_slot_of;
  DevBuf<uint8_t> has_cons, ext_cons, bound;
  DevBuf<uint8_t> xinfo;  // per block: XNode[T] then XEdge[n_prod] (k_explain_fast)
  DevBuf<int64_t> xoff;   // [nb + 1] byte offsets into xinfo
  DevBuf<int64_t> edge_off;  // [nb + 1] internal-edge offsets (the explain output layout)
};

}  // namespace

// Device buffers of a launched, not yet collected search (sp_score_launch).
// A search in flight.  Its results (and winner detail) are copied into a
// pinned host block right behind the kernels, so several searches can be
// queued on the stream and each collected by its own `done` event.
struct PendingScore {
  bool active = false;
  bool explain = false;
  bool empty = false;  // no work item: nothing was launched
  DevBuf<unsigned long long> dplan;
  DevBuf<ItemOut> items;
  DevBuf<sp_score_out> dout;
  DevBuf<sp_score_out> gath;  // [nranks x nb] records of every lane (multi-GPU exchange)
  bool lane = false;          // a peer lane of a multi-device search: collected by the primary
  DevBuf<ExplainBlock> dblk;
  DevBuf<int8_t> dnode, dedge;
  // single-lane searches: dout | dblk | dnode | dedge as views into one arena
  // laid out like the pinned host block (one D2H copy of the whole result)
  DevBuf<uint8_t> res;
  bool res_packed = false;
  sp_ctx* ctx = nullptr;
  uint8_t* host = nullptr;  // pinned: out | blocks | node | edge
  size_t host_bytes = 0, off_blk = 0, off_node = 0, off_edge = 0;
  // 0 launch, 1 kernel start, 2 kernel end, 3 reduce end, 4 explain end, 5 results on the host
  cudaEvent_t ev[6] = {};
  bool synced = false;  // ev[5] (recorded last, on the same stream) has been waited for
  void events() {  // from the context's pool (cudaEventCreate per search adds up on tiny searches)
    synced = false;
    for (auto& e : ev)
      if (!e) {
        if (!ctx->event_pool.empty()) {
          e = ctx->event_pool.back();
          ctx->event_pool.pop_back();
        } else {
          SP_CUDA(cudaEventCreate(&e));
        }
      }
  }
  void release_host() {
    if (!host) return;
    if (!synced) cudaEventSynchronize(ev[5]);
    ctx->pinned_pool.push_back({host, host_bytes});
    host = nullptr;
    host_bytes = 0;
  }
  ~PendingScore() {
    release_host();
    for (auto& e : ev)
      if (e) {
        if (ctx) {
          if (!synced) cudaEventSynchronize(e);  // recorded work done before another search re-records it
          ctx->event_pool.push_back(e);
        } else {
          cudaEventDestroy(e);
        }
      }
  }
};

struct TablesPriv {
  TableDev dev;
  sp_mesh mesh;
  int64_t mu, chunk;
  PendingScore pending;
  // recorded behind k_fill: work on the auxiliary stream (explain_all) waits
  // for the tables, not for whatever was queued on the main stream since
  cudaEvent_t built = nullptr;
  // packed uploads of the build (one H2D per phase) and their pinned staging;
  // the node maps / boundary flags
  DevBuf<uint8_t> arena, arena2, maps;
  sp_ctx* ctx = nullptr;
  uint8_t* pin = nullptr;
  size_t pin_bytes = 0;
  ~TablesPriv() {
    if (built) {  // back to the context's pool (tables_free waited for it)
      if (ctx) ctx->event_pool.push_back(built);
      else cudaEventDestroy(built);
    }
    if (pin && ctx) pinned_release(ctx, pin, pin_bytes);
  }
  // a pinned block of >= `need` bytes owned by the tables (the stream is
  // synchronised before it is reused or released)
  uint8_t* pinned(size_t need) {
    if (pin && pin_bytes >= need) return pin;
    if (pin) pinned_release(ctx, pin, pin_bytes);
    pin = pinned_acquire(ctx, need, &pin_bytes);
    return pin;
  }
  // ONE H2D of every part of `pk` into `into` (the device arena)
  uint8_t* upload(const PackedUpload& pk, DevBuf<uint8_t>& into, cudaStream_t s) {
    uint8_t* h = pinned(pk.total);
    for (const auto& part : pk.parts)
      if (part.bytes) std::memcpy(h + part.off, part.src, part.bytes);
    into.alloc(std::max<size_t>(pk.total, 16), s);
    if (pk.total) SP_CUDA(cudaMemcpyAsync(into.p, h, pk.total, cudaMemcpyHostToDevice, s));
    g_h2d_bytes += (int64_t)pk.total;
    return into.p;
  }
};

// Winner detail of every block (RoutedPlan/CostReport fields) on stream `s`:
// k_explain_fast from the routing tables, or (SP_EXPLAIN_ROUTE=1, A/B and
// cross-checks) k_explain_all re-deriving each node with route_node.
static void launch_explain(sp_ctx* ctx, sp_tables* t, cudaStream_t s, const int64_t* d_edge_off,
                           const unsigned long long* indices, const sp_score_out* scores, ExplainBlock* blk,
                           int8_t* node, int8_t* edge) {
  TablesPriv* priv = (TablesPriv*)t->priv;
  const int64_t nb = t->n_blocks;
  if (getenv("SP_EXPLAIN_ROUTE")) {
    SP_LAUNCH(ctx, k_explain_all, (int)std::min<int64_t>((nb + 31) / 32, 4096), 32, 0, s, view_of(t->dg),
              t->d_tmpl_off.p, t->d_tmpl_nodes.p, nb, priv->dev.node_block.p, priv->dev.node_tpos.p,
              priv->dev.ref_slot_of.p, priv->dev.bound.p, t->blobs.p, t->d_blob_off.p, d_edge_off, indices, scores,
              priv->mesh, priv->mu, priv->chunk, blk, node, edge);
  } else {
    const size_t smem = (size_t)((t->max_blob + 15) & ~15);
    if (smem > ctx->smem_optin)
      throw Error(SP_ERR_UNSUPPORTED, "block tables exceed shared memory (" + std::to_string(smem) + " bytes)");
    allow_smem(ctx, k_explain_fast, smem);
    SP_LAUNCH(ctx, k_explain_fast, (int)std::min<int64_t>(nb, 4096), 32, smem, s, view_of(t->dg), t->d_tmpl_off.p,
              t->d_tmpl_nodes.p, nb, priv->dev.ref_slot_of.p, priv->dev.bound.p, t->blobs.p, t->d_blob_off.p,
              priv->dev.xinfo.p, priv->dev.xoff.p, d_edge_off, indices, scores, priv->mesh, priv->mu, priv->chunk,
              blk, node, edge);
  }
  SP_CUDA(cudaGetLastError());
}

}  // namespace sp

namespace sp {

void tables_build(sp_ctx* ctx, sp_dgraph* dg, int64_t nb, const int64_t* tmpl_off, const int32_t* tmpl_nodes,
                  const sp_mesh* mesh, int64_t mu, int64_t chunk, sp_tables* out) {
  cudaStream_t s = ctx->stream;
  const int64_t n = dg->n;
  Trace tr("tables");
  if (nb < 0) throw Error(SP_ERR_CONFIG, "negative block count");
  if (mu > chunk) throw Error(SP_ERR_CONFIG, "fusion threshold " + std::to_string(mu) + " exceeds chunk size " +
                                                 std::to_string(chunk));
  out->ctx = ctx;
  out->dg = dg;
  out->n_blocks = nb;
  out->tmpl_off.assign(tmpl_off, tmpl_off + nb + 1);
  const int64_t ne = out->tmpl_off[nb];
  out->tmpl_nodes.assign(tmpl_nodes, tmpl_nodes + ne);
  // host validation + weight slot order (weight_nodes: sorted by name, search.py:85-88)
  std::vector<int16_t> slot_of(ne, -1), ref_slot_of(ne, -1);
  std::vector<uint8_t> radix_of(ne, 1);
  out->slot_pos.assign(nb, {});
  out->hdr.assign(nb, BlobHeader{});
  out->overflow = false;
  out->max_T = 0;
  const uint8_t* names = dg->h_names.data();
  const int64_t* noff = dg->h_name_off.data();
  for (int64_t b = 0; b < nb; b++) {
    const int64_t e0 = out->tmpl_off[b], e1 = out->tmpl_off[b + 1];
    const int64_t T = e1 - e0;
    if (T < 0) throw Error(SP_ERR_CONFIG, "template offsets must be non-decreasing");
    if (T > MAXT) throw Error(SP_ERR_UNSUPPORTED, "template with more than 256 nodes");
    out->max_T = std::max<int32_t>(out->max_T, (int32_t)T);
    std::vector<int64_t> w;
    for (int64_t e = e0; e < e1; e++) {
      const int32_t v = out->tmpl_nodes[e];
      if (v < 0 || v >= n) throw Error(SP_ERR_CONFIG, "template node index out of range");
      Pattern pats[4];
      if (patterns_for(dg->h_op[v], pats) < 0) {
        static const char* labels[] = {"matmul", "elementwise", "layernorm", "softmax", "embedding",
                                       "reshape", "input",  "output",    "auxiliary", "collective"};
        throw Error(SP_ERR_SPEC, std::string(labels[dg->h_op[v] < 10 ? dg->h_op[v] : 9]) +
                                     " is not a shardable compute kind");
      }
      if (dg->h_w_rank[v]) w.push_back(e);
    }
    std::sort(w.begin(), w.end(), [&](int64_t a, int64_t c) {
      const int32_t x = out->tmpl_nodes[a], y = out->tmpl_nodes[c];
      return strcmp_py(names + noff[x], noff[x + 1] - noff[x], names + noff[y], noff[y + 1] - noff[y]) < 0;
    });
    BlobHeader& H = out->hdr[b];
    H.V = (int32_t)w.size();
    H.radix3 = 0;
    H.radix3_ref = 0;
    unsigned __int128 C = 1;
    bool over = w.size() > 64;
    // reference slot order = names sorted (weight_nodes, search.py:85-88); the
    // enumeration order used on the device = template (topological) order, so a
    // failing node's ancestor cone sits in the slow digits (prefix skipping).
    std::vector<int64_t> enum_order(w.begin(), w.end());
    std::sort(enum_order.begin(), enum_order.end());
    for (size_t q = 0; q < enum_order.size() && !over; q++) slot_of[enum_order[q]] = (int16_t)q;
    for (size_t sidx = 0; sidx < w.size(); sidx++) {
      const int64_t e = w[sidx];
      const int r = dg->h_w_rank[out->tmpl_nodes[e]] >= 2 ? 3 : 2;  // _options (search.py:91-93)
      if (!over) {
        ref_slot_of[e] = (int16_t)sidx;
        radix_of[e] = (uint8_t)r;
        if (r == 3) {
          H.radix3_ref |= 1ULL << sidx;
          H.radix3 |= 1ULL << slot_of[e];
        }
      }
      out->slot_pos[b].push_back((int32_t)(e - e0));
      C *= (unsigned)r;
      if (C > (unsigned __int128)UINT64_MAX) over = true;
    }
    H.C = over ? 0 : (uint64_t)C;
    if (over) out->overflow = true;
  }
  tr.mark("host slots");
  TablesPriv* priv = new TablesPriv();
  out->priv = priv;
  priv->ctx = ctx;
  priv->mesh = *mesh;
  priv->mu = mu;
  priv->chunk = chunk;
  TableDev& D = priv->dev;
  const GraphView G = view_of(dg);
  DevBuf<EntryLayout> lay;
  DevBuf<BlobHeader> hdr;
  out->max_blob = 0;
  out->max_pool = 0;
  out->blob_off.assign(nb + 1, 0);
  out->edge_off.assign(nb + 1, 0);
  std::vector<int64_t> xo;
  auto offsets = [&] {
    xo.assign(nb + 1, 0);
    for (int64_t b = 0; b < nb; b++) {
      out->max_blob = std::max<int64_t>(out->max_blob, out->hdr[b].bytes);
      out->max_pool = std::max(out->max_pool, out->hdr[b].npool);
      out->blob_off[b + 1] = out->blob_off[b] + out->hdr[b].bytes;
      out->edge_off[b + 1] = out->edge_off[b] + out->hdr[b].n_prod;
      xo[b + 1] = xo[b] + align16((int64_t)sizeof(XNode) * out->hdr[b].T + (int64_t)sizeof(XEdge) * out->hdr[b].n_prod);
    }
  };
  if (!dg->h_in_off.empty() && ctx->host_layout) {
    // Small graph: node maps, boundary flags and the blob layout on the host
    // (k_mark_blocks / k_boundary / k_layout's work, layout_serial shared), so
    // the build is ONE upload and the fill launch -- no device round trip.
    const int64_t* in_off = dg->h_in_off.data();
    const int32_t* in_idx = dg->h_in_idx.data();
    std::vector<int32_t> nblk(n, -1), ntpos(n, -1);
    std::vector<uint8_t> flags(2 * (size_t)n, 0);  // has_cons | ext_cons
    for (int64_t b = 0; b < nb; b++)
      for (int64_t e = out->tmpl_off[b]; e < out->tmpl_off[b + 1]; e++) {
        const int32_t v = out->tmpl_nodes[e];
        if (nblk[v] != -1) throw Error(SP_ERR_CONFIG, "a node appears in more than one template");
        nblk[v] = (int32_t)b;
        ntpos[v] = (int32_t)(e - out->tmpl_off[b]);
      }
    for (int64_t c = 0; c < n; c++)
      for (int64_t e = in_off[c]; e < in_off[c + 1]; e++) {
        const int32_t p = in_idx[e];
        flags[p] = 1;
        if (nblk[c] != nblk[p] || nblk[p] < 0) flags[n + p] = 1;
      }
    std::vector<EntryLayout> lay_h(std::max<int64_t>(ne, 1));
    std::vector<int> last(MAXT), head(MAXT), kk(MAXT), nxt(MAXT), pool(MAXT);
    std::vector<uint64_t> ancs(MAXT), suf(65);
    std::vector<int16_t> pp((size_t)MAXT * KMAX);
    std::vector<uint8_t> tw(MAXT);
    int err = 0;
    for (int64_t b = 0; b < nb && !err; b++) {
      const int64_t e0 = out->tmpl_off[b];
      const int T = (int)(out->tmpl_off[b + 1] - e0);
      for (int i = 0; i < T; i++) last[i] = head[i] = -1;
      for (int i = 0; i < T; i++) {
        const int32_t v = out->tmpl_nodes[e0 + i];
        int k = 0;
        for (int64_t e = in_off[v]; e < in_off[v + 1]; e++) {
          const int32_t r = in_idx[e];
          if (nblk[r] != (int32_t)b) continue;
          const int j = ntpos[r];
          if (j >= i) err = err ? err : 2;
          else last[j] = std::max(last[j], i);
          if (k < KMAX) pp[(size_t)i * KMAX + k] = (int16_t)j;
          k++;
        }
        if (k > KMAX) err = err ? err : 3;
        kk[i] = k;
        tw[i] = (dg->h_w_rank[v] && dg->h_w_train[v]) ? 1 : 0;
      }
      for (int j = 0; j < T; j++)
        if (last[j] >= 0) {
          nxt[j] = head[last[j]];
          head[last[j]] = j;
        }
      if (!err)
        layout_serial(T, kk.data(), last.data(), (const int16_t(*)[KMAX])pp.data(), head.data(), nxt.data(),
                      pool.data(), ancs.data(), suf.data(), slot_of.data() + e0, radix_of.data() + e0, tw.data(),
                      out->hdr[b], lay_h.data() + e0);
    }
    if (err == 2) throw Error(SP_ERR_CONFIG, "template is not in topological order");
    if (err == 3) throw Error(SP_ERR_UNSUPPORTED, "a template node has more than 6 internal producers");
    offsets();
    tr.mark("host layout");
    PackedUpload pk;
    const size_t o_off = pk.add(out->tmpl_off.data(), (nb + 1) * sizeof(int64_t));
    const size_t o_nodes = pk.add(out->tmpl_nodes.data(), ne * sizeof(int32_t));
    const size_t o_slot = pk.add(slot_of.data(), ne * sizeof(slot_of[0]));
    const size_t o_ref = pk.add(ref_slot_of.data(), ne * sizeof(ref_slot_of[0]));
    const size_t o_hdr = pk.add(out->hdr.data(), nb * sizeof(BlobHeader));
    const size_t o_lay = pk.add(lay_h.data(), ne * sizeof(EntryLayout));
    const size_t o_nb = pk.add(nblk.data(), n * sizeof(int32_t));
    const size_t o_tp = pk.add(ntpos.data(), n * sizeof(int32_t));
    const size_t o_fl = pk.add(flags.data(), 2 * (size_t)n);
    const size_t o_blob = pk.add(out->blob_off.data(), (nb + 1) * sizeof(int64_t));
    const size_t o_x = pk.add(xo.data(), (nb + 1) * sizeof(int64_t));
    const size_t o_e = pk.add(out->edge_off.data(), (nb + 1) * sizeof(int64_t));
    uint8_t* a = priv->upload(pk, priv->arena, s);
    out->d_tmpl_off.set_view((int64_t*)(a + o_off), nb + 1);
    out->d_tmpl_nodes.set_view((int32_t*)(a + o_nodes), ne);
    D.slot_of.set_view((decltype(D.slot_of.p))(a + o_slot), ne);
    D.ref_slot_of.set_view((decltype(D.ref_slot_of.p))(a + o_ref), ne);
    hdr.set_view((BlobHeader*)(a + o_hdr), nb);
    lay.set_view((EntryLayout*)(a + o_lay), ne);
    D.node_block.set_view((int32_t*)(a + o_nb), n);
    D.node_tpos.set_view((int32_t*)(a + o_tp), n);
    D.has_cons.set_view(a + o_fl, n);
    D.ext_cons.set_view(a + o_fl + n, n);
    out->d_blob_off.set_view((int64_t*)(a + o_blob), nb + 1);
    D.xoff.set_view((int64_t*)(a + o_x), nb + 1);
    D.edge_off.set_view((int64_t*)(a + o_e), nb + 1);
    tr.mark("upload");
  } else {
  // the host-built arrays in one H2D (pinned staging, packed arena)
  DevBuf<uint8_t> radix_d;
  {
    PackedUpload pk;
    const size_t o_off = pk.add(out->tmpl_off.data(), (nb + 1) * sizeof(int64_t));
    const size_t o_nodes = pk.add(out->tmpl_nodes.data(), ne * sizeof(int32_t));
    const size_t o_slot = pk.add(slot_of.data(), ne * sizeof(slot_of[0]));
    const size_t o_ref = pk.add(ref_slot_of.data(), ne * sizeof(ref_slot_of[0]));
    const size_t o_radix = pk.add(radix_of.data(), ne);
    const size_t o_hdr = pk.add(out->hdr.data(), nb * sizeof(BlobHeader));
    uint8_t* a = priv->upload(pk, priv->arena, s);
    out->d_tmpl_off.set_view((int64_t*)(a + o_off), nb + 1);
    out->d_tmpl_nodes.set_view((int32_t*)(a + o_nodes), ne);
    D.slot_of.set_view((decltype(D.slot_of.p))(a + o_slot), ne);
    D.ref_slot_of.set_view((decltype(D.ref_slot_of.p))(a + o_ref), ne);
    radix_d.set_view(a + o_radix, ne);
    hdr.set_view((BlobHeader*)(a + o_hdr), nb);
  }
  tr.mark("upload");
  // node maps (-1) and boundary flags + error words (0) in one arena: two memsets
  const size_t nm_bytes = ((size_t)n * 8 + 15) & ~(size_t)15;
  priv->maps.alloc(nm_bytes + (((size_t)2 * n + 15) & ~(size_t)15) + 16, s);
  D.node_block.set_view((int32_t*)priv->maps.p, n);
  D.node_tpos.set_view((int32_t*)priv->maps.p + n, n);
  D.has_cons.set_view(priv->maps.p + nm_bytes, n);
  D.ext_cons.set_view(priv->maps.p + nm_bytes + n, n);
  int32_t* err = (int32_t*)(priv->maps.p + nm_bytes + (((size_t)2 * n + 15) & ~(size_t)15));
  SP_CUDA(cudaMemsetAsync(priv->maps.p, 0xff, (size_t)n * 8, s));
  SP_CUDA(cudaMemsetAsync(priv->maps.p + nm_bytes, 0, priv->maps.n - nm_bytes, s));
  if (nb > 0)
    SP_LAUNCH(ctx, k_mark_blocks, (int)std::min<int64_t>(nb, 65535), 128, 0, s, out->d_tmpl_off.p, out->d_tmpl_nodes.p, nb,
                                                                  D.node_block.p, D.node_tpos.p, err);
  SP_LAUNCH(ctx, k_boundary, grid_for(n, ctx->sm_count), 256, 0, s, G, n, D.node_block.p, D.has_cons.p, D.ext_cons.p);
  tr.mark("mark+boundary");
  DevBuf<int64_t> blob_bytes;
  lay.alloc(ne, s);
  blob_bytes.alloc(nb + 1, s);
  const int gb = (int)std::min<int64_t>(std::max<int64_t>(nb, 1), 65535);
  if (nb > 0)
    SP_LAUNCH(ctx, k_layout, (int)std::min<int64_t>((nb + LAYOUT_WARPS - 1) / LAYOUT_WARPS, 65535), 32 * LAYOUT_WARPS,
              0, s, G, out->d_tmpl_off.p, out->d_tmpl_nodes.p, nb, D.node_block.p,
              D.node_tpos.p, D.slot_of.p, radix_d.p, lay.p, hdr.p, blob_bytes.p, err);
  // errors + the laid-out headers back in one pinned block (the staging block is
  // free again: its H2D is ordered before these copies)
  tr.mark("layout launch");
  int32_t err_h[2];
  {
    const size_t hb = (size_t)nb * sizeof(BlobHeader);
    uint8_t* h = priv->pinned(hb + 16);
    SP_CUDA(cudaMemcpyAsync(h, err, 2 * sizeof(int32_t), cudaMemcpyDeviceToHost, s));
    if (nb) SP_CUDA(cudaMemcpyAsync(h + 16, hdr.p, hb, cudaMemcpyDeviceToHost, s));
    g_d2h_bytes += (int64_t)(8 + hb);
    SP_CUDA(cudaStreamSynchronize(s));
    std::memcpy(err_h, h, sizeof(err_h));
    if (nb) std::memcpy(out->hdr.data(), h + 16, hb);
  }
  tr.mark("layout sync");
  if (err_h[0] == 1) throw Error(SP_ERR_CONFIG, "a node appears in more than one template");
  if (err_h[0] == 2) throw Error(SP_ERR_CONFIG, "template is not in topological order");
  if (err_h[0] == 3)
    throw Error(SP_ERR_UNSUPPORTED, "a template node has more than 6 internal producers");
  offsets();
  PackedUpload pk;
  const size_t o_blob = pk.add(out->blob_off.data(), (nb + 1) * sizeof(int64_t));
  const size_t o_x = pk.add(xo.data(), (nb + 1) * sizeof(int64_t));
  const size_t o_e = pk.add(out->edge_off.data(), (nb + 1) * sizeof(int64_t));
  uint8_t* a = priv->upload(pk, priv->arena2, s);
  out->d_blob_off.set_view((int64_t*)(a + o_blob), nb + 1);
  D.xoff.set_view((int64_t*)(a + o_x), nb + 1);
  D.edge_off.set_view((int64_t*)(a + o_e), nb + 1);
  }
  tr.mark("offsets");
  out->blobs.alloc(std::max<int64_t>(out->blob_off[nb], 16), s);
  D.bound.alloc(ne, s);
  D.xinfo.alloc(std::max<int64_t>(xo[nb], 16), s);
  tr.mark("alloc+upload2");
  if (nb > 0)
    SP_LAUNCH(ctx, k_fill, (int)std::min<int64_t>(nb, 65535), 128, 0, s, G, out->d_tmpl_off.p, out->d_tmpl_nodes.p, nb, D.node_block.p,
              D.node_tpos.p, D.slot_of.p, D.ref_slot_of.p, lay.p, hdr.p, out->d_blob_off.p, D.has_cons.p, D.ext_cons.p, *mesh, mu,
              chunk, out->blobs.p, D.bound.p, D.xinfo.p, D.xoff.p);
  SP_CUDA(cudaGetLastError());
  {
    TablesPriv* tp = (TablesPriv*)out->priv;
    if (!tp->built) {
      if (!ctx->event_pool.empty()) {
        tp->built = ctx->event_pool.back();
        ctx->event_pool.pop_back();
      } else {
        SP_CUDA(cudaEventCreate(&tp->built));
      }
    }
    SP_CUDA(cudaEventRecord(tp->built, s));
  }
  tr.mark("fill launch");
}

static size_t score_smem(const sp_tables* t) {
  return (size_t)((t->max_blob + 15) & ~15) + (size_t)t->max_pool * THREADS * 9 + 16;
}

struct FusedExplain {
  void* blocks;
  int8_t* node;
  int8_t* edge;
};

// Byte layout of a search's results in the pinned host block (and, for a
// packed single-lane search, in its device arena): out | blocks | node | edge.
struct ResultLayout {
  size_t off_blk, off_node, off_edge, need;
};
static ResultLayout result_layout(const sp_tables* t, bool explain) {
  const int64_t nb = t->n_blocks;
  const int64_t ne = t->tmpl_off[nb], nedge = t->edge_off[nb];
  ResultLayout L;
  L.off_blk = ((size_t)nb * sizeof(sp_score_out) + 63) & ~(size_t)63;
  L.off_node = L.off_blk + (explain ? (((size_t)nb * sizeof(ExplainBlock) + 63) & ~(size_t)63) : 0);
  L.off_edge = L.off_node + (explain ? (((size_t)4 * ne + 63) & ~(size_t)63) : 0);
  L.need = L.off_edge + (explain ? (size_t)2 * nedge : 0);
  return L;
}

// The per-block result records of a search (pd.dout); a single-lane search
// with winner detail gets them packed with the detail outputs in one arena.
static void alloc_dout(PendingScore& pd, const sp_tables* t, cudaStream_t s, bool lane) {
  const int64_t nb = t->n_blocks;
  pd.res_packed = pd.explain && !lane;
  if (!pd.res_packed) {
    pd.dout.alloc(nb, s);
    return;
  }
  const ResultLayout L = result_layout(t, true);
  pd.res.alloc(std::max<size_t>(L.need, 16), s);
  const int64_t ne = t->tmpl_off[nb], nedge = t->edge_off[nb];
  pd.dout.set_view((sp_score_out*)pd.res.p, nb);
  pd.dblk.set_view((ExplainBlock*)(pd.res.p + L.off_blk), nb);
  pd.dnode.set_view((int8_t*)(pd.res.p + L.off_node), 4 * ne);
  pd.dedge.set_view((int8_t*)(pd.res.p + L.off_edge), 2 * nedge);
}

// Enqueue scoring (+ k_reduce, + winner detail when `explain`) of
// [lo[b], hi[b]) for every block; the buffers stay in the tables' pending
// slot until score_finish collects them.
// Returns false when this shard has no work item and `must_out` is false
// (nothing launched); with `must_out` (a lane of a multi-GPU exchange) an
// empty shard still produces its all-empty records.
static bool score_items(sp_ctx* ctx, sp_tables* t, int32_t shard, int32_t n_shards, bool must_out) {
  cudaStream_t s = ctx->stream;
  Trace tr("score_items");
  const int64_t nb = t->n_blocks;
  TablesPriv* priv = (TablesPriv*)t->priv;
  PendingScore& pd = priv->pending;
  pd.empty = false;
  const size_t smem = score_smem(t);
  if (smem > ctx->smem_optin)
    throw Error(SP_ERR_UNSUPPORTED, "block tables exceed shared memory (" + std::to_string(smem) + " bytes)");
  // any block with more than 32 weight slots needs the two-word digit encoding
  // (SP_FORCE_WIDE=1 selects it everywhere: tests cross-check both encodings)
  bool wide = getenv("SP_FORCE_WIDE") != nullptr;
  for (int64_t b = 0; b < nb; b++) wide = wide || t->hdr[b].V > 32;
  // memoised brute force needs every template <= 64 nodes (bitmask state)
  const bool memo = !ctx->skip && ctx->memo && t->max_T <= 64;
  const int threads = memo ? THREADS_M : THREADS;
  // SP_SCORE_GENERIC=1 selects the generic walk for narrow blocks (A/B checks)
  const bool generic = getenv("SP_SCORE_GENERIC") != nullptr;
  // brute force on narrow blocks walks two candidates per lane (SP_SCORE_SINGLE=1: one)
  const bool pair = !generic && !wide && !memo && !ctx->skip && getenv("SP_SCORE_SINGLE") == nullptr;
  // the brute-force FastNode walks run barrier-free (k_score_flow, c5: 35.7
  // -> 35.3 ms); with prefix skipping an item often takes microseconds and
  // the per-item hand-over costs more than the barrier it saves (8.0 -> 8.7
  // ms), so skipping keeps k_score_fast.  SP_SCORE_ITEMS=1 / SP_SCORE_FLOW=1
  // force either version (A/B checks).
  const bool items_mode = getenv("SP_SCORE_ITEMS") != nullptr;
  const bool flow_skip = getenv("SP_SCORE_FLOW") != nullptr;
  auto fast_skip = flow_skip ? k_score_flow<true, false> : k_score_fast<true, false>;
  auto fast_pair = items_mode ? k_score_fast<false, true> : k_score_flow<false, true>;
  auto fast_one = items_mode ? k_score_fast<false, false> : k_score_flow<false, false>;
  auto kern = memo ? (wide ? k_score_memo<true> : k_score_memo<false>)
              : ctx->skip ? (wide ? k_score<true, true> : generic ? k_score<false, true> : fast_skip)
                          : (wide ? k_score<true, false>
                                  : generic ? k_score<false, false> : pair ? fast_pair : fast_one);
  const size_t smem_k = memo   ? (size_t)((t->max_blob + 15) & ~15) + (size_t)t->max_T * THREADS_M * 8 + 16
                       : pair ? (size_t)((t->max_blob + 15) & ~15) + (size_t)t->max_pool * THREADS * 18 + 16
                              : smem;
  if (smem_k > ctx->smem_optin)
    throw Error(SP_ERR_UNSUPPORTED, "block tables exceed shared memory (" + std::to_string(smem_k) + " bytes)");
  // prefix skipping on narrow blocks: per-block chunk counters, no work items
  // (SP_SCORE_ITEMS=1 / SP_SKIP_ITEMS=1 select the item kernels: A/B checks)
  // Every CTA of k_score_skip visits every block of the search in order (one
  // claim + barrier per block), so a search of many cheap blocks (c5's ~1000
  // residual singletons: 0.85 ms) runs on the item kernel instead (0.10 ms).
  if (ctx->skip && !wide && !generic && !memo && !items_mode && !flow_skip && nb <= SKIP_KERNEL_MAX_BLOCKS &&
      getenv("SP_SKIP_ITEMS") == nullptr) {
    allow_smem(ctx, k_score_skip, smem);
    int per = resident_ctas(ctx, k_score_skip, THREADS, smem);
    if (per < 1) per = 1;
    const int64_t grid = (int64_t)ctx->sm_count * per;
    const unsigned long long N = (unsigned long long)n_shards, r = (unsigned long long)shard;
    std::vector<unsigned long long> plan(3 * nb, 0);
    unsigned long long any = 0;
    for (int64_t b = 0; b < nb; b++) {
      const unsigned long long C = t->hdr[b].C;
      const unsigned long long nc = C / SKIP_CHUNK + (C % SKIP_CHUNK ? 1 : 0);
      plan[b] = nc > r ? (nc - 1 - r) / N + 1 : 0;
      any += plan[b];
    }
    if (any == 0) {
      if (!must_out) return false;
      alloc_dout(pd, t, s, must_out);
      SP_CUDA(cudaMemsetAsync(pd.dout.p, 0, (size_t)nb * sizeof(sp_score_out), s));
      SP_CUDA(cudaEventRecord(pd.ev[1], s));
      SP_CUDA(cudaEventRecord(pd.ev[2], s));
      SP_CUDA(cudaEventRecord(pd.ev[3], s));
      return true;
    }
    pd.dplan.upload(plan.data(), plan.size(), s);  // nch | ctr | contrib
    SP_CUDA(cudaMemsetAsync(pd.dplan.p + nb, 0, (size_t)2 * nb * sizeof(unsigned long long), s));
    pd.items.alloc((size_t)nb * grid, s);
    alloc_dout(pd, t, s, must_out);
    // SP_SKIP_TAIL=k: claim the last k chunks of a block in eighths (a shorter
    // final wave before the block's end barrier); measured no gain on c5
    // (7.38 ms at 0, 7.41-7.52 ms at 296-2000), so off by default
    const char* tail_env = getenv("SP_SKIP_TAIL");
    const unsigned long long tail = tail_env ? strtoull(tail_env, nullptr, 10) : 0ULL;
    SkipPlan SPn{t->d_blob_off.p, pd.dplan.p, pd.dplan.p + nb, (uint32_t*)(pd.dplan.p + 2 * nb), nb, (uint32_t)shard,
                 (uint32_t)n_shards, tail};
    SP_CUDA(cudaEventRecord(pd.ev[1], s));
    SP_LAUNCH(ctx, k_score_skip, (unsigned)grid, THREADS, smem, s, t->blobs.p, SPn, pd.items.p);
    SP_CUDA(cudaEventRecord(pd.ev[2], s));
    SP_LAUNCH(ctx, k_reduce_contrib, (unsigned)std::min<int64_t>(nb, 4096), THREADS, 0, s, pd.items.p, SPn.contrib,
              grid, nb, pd.dout.p);
    SP_CUDA(cudaGetLastError());
    SP_CUDA(cudaEventRecord(pd.ev[3], s));
    return true;
  }
  tr.mark("kernel choice");
  allow_smem(ctx, kern, smem_k);
  int per_sm = resident_ctas(ctx, kern, threads, smem_k);
  if (per_sm < 1) per_sm = 1;
  const unsigned long long slots = (unsigned long long)ctx->sm_count * per_sm;
  // size work items so each rank's grid gets ~ITEMS_PER_CTA items per resident CTA
  // (dynamic balance); with prefix skipping a candidate costs far less, so
  // items may grow larger.  Ranks deal the items of every block round-robin
  // (the global item sequence, item g to rank g mod n_shards): early-exit
  // cost varies along a block's index range, so contiguous slices would
  // leave one rank with the expensive end.  The merge is an exact
  // lexicographic min, so any partition gives the same result.  The sizing
  // depends only on the tables and n_shards: every rank derives the same
  // items.
  tr.mark("smem+occupancy");
  const unsigned long long N = (unsigned long long)n_shards, r = (unsigned long long)shard;
  unsigned long long total = 0;
  for (int64_t b = 0; b < nb; b++) total += t->hdr[b].C;
  const unsigned long long cap = ctx->skip ? ITEM_ITERS_MAX_SKIP : ITEM_ITERS_MAX;
  const unsigned long long per_rank = total / N + (total % N ? 1 : 0);
  static const unsigned long long ipc = getenv("SP_ITEMS_PER_CTA") ? strtoull(getenv("SP_ITEMS_PER_CTA"), nullptr, 10)
                                                                   : ITEMS_PER_CTA;  // (A/B override)
  unsigned long long iters = (per_rank + slots * ipc * THREADS - 1) / (slots * ipc * THREADS);
  iters = std::max<unsigned long long>(1, std::min<unsigned long long>(iters, memo ? ITEM_ITERS_MAX_SKIP : cap));
  // the paired walk hands items out in PAIR_CHUNK-candidate warp chunks: an item
  // smaller than one chunk per warp leaves warps idle (8-rank c5 share: 13k-
  // candidate items, 4.30 -> 4.42 ms) -- unless the search is too small to
  // give every CTA such an item
  const unsigned long long min_iters = (unsigned long long)(THREADS / 32) * PAIR_CHUNK / THREADS;
  if (pair && iters < min_iters && per_rank >= slots * min_iters * THREADS) iters = min_iters;
  const unsigned long long item_cands = iters * THREADS;
  // rank 0 assembles the report after its share (root_only): at 4+ ranks it is
  // relieved of whole blocks worth <= SP_ROOT_RELIEF% (default 14) of an 8-rank share --
  // the second-largest blocks down -- dealt over ranks 1..N-1 instead; with the
  // brute-force walk, what is left of the budget comes off the largest block:
  // its last items (from item J on) are dealt over ranks 1..N-1 as a second
  // segment of that block on each of them
  const bool flow_walk = kern == fast_pair || kern == fast_one;
  std::vector<char> excl(nb, 0);
  int64_t big = -1;
  unsigned long long big_J = 0;
  {
    const long relief_pct = getenv("SP_ROOT_RELIEF") ? strtol(getenv("SP_ROOT_RELIEF"), nullptr, 10) : 14;
    if (N >= 4 && relief_pct > 0) {
      std::vector<int64_t> order(nb);
      for (int64_t b = 0; b < nb; b++) order[b] = b;
      std::sort(order.begin(), order.end(), [&](int64_t a, int64_t c) {
        return t->hdr[a].C != t->hdr[c].C ? t->hdr[a].C > t->hdr[c].C : a < c;
      });
      // rank 0's extra host work (report assembly, the cheap group) is about
      // constant, so is the work it sheds: a share of an 8-rank search
      const double budget = (double)relief_pct / 100.0 * (double)total / 8.0;
      double used = 0.0;
      for (size_t k = 1; k < order.size(); k++) {
        const double share = (double)t->hdr[order[k]].C / (double)N;
        if (used + share <= budget) {
          excl[order[k]] = 1;
          used += share;
        }
      }
      const unsigned long long Cb = t->hdr[order[0]].C, nchb = Cb / item_cands + (Cb % item_cands ? 1 : 0);
      const unsigned long long moved = (unsigned long long)((budget - used) * (double)N / (double)item_cands);
      if (flow_walk && !items_mode && nb > 0 && moved > 0 && !getenv("SP_NO_PARTIAL_RELIEF")) {
        big = order[0];
        big_J = nchb - std::min(moved, nchb);
      }
    }
  }
  std::vector<unsigned long long> lo(nb), hi(nb), base(nb + 1, 0), stride(nb);
  // second segments (the relieved tail of the largest block): items cnt1[b] on
  std::vector<unsigned long long> cnt1(nb), lo2(nb), hi2(nb), stride2(nb, item_cands);
  unsigned long long gbase = 0, gex = 0;
  for (int64_t b = 0; b < nb; b++) {
    const unsigned long long C = t->hdr[b].C;
    unsigned long long nch = C / item_cands + (C % item_cands ? 1 : 0);
    unsigned long long j0, cnt, M;
    lo2[b] = hi2[b] = C;
    unsigned long long cnt2 = 0;
    if (b == big) {  // items >= big_J over ranks 1..N-1, then the rest as usual
      const unsigned long long j2 = big_J + (r == 0 ? 0 : r - 1);
      if (r > 0 && j2 < nch) {
        cnt2 = (nch - 1 - j2) / (N - 1) + 1;
        lo2[b] = j2 * item_cands;
      }
      stride2[b] = (N - 1) * item_cands;
      nch = big_J;
    }
    if (excl[b]) {  // dealt over ranks 1..N-1
      M = N - 1;
      j0 = r == 0 ? nch : (r - 1 + M - gex % M) % M;
      gex += nch;
    } else {
      M = N;
      j0 = (r + N - gbase % N) % N;  // first item of block b dealt to this rank
      gbase += nch;
    }
    cnt = j0 < nch ? (nch - 1 - j0) / M + 1 : 0;
    lo[b] = j0 < nch ? j0 * item_cands : C;
    hi[b] = std::min(C, nch * item_cands);
    stride[b] = M * item_cands;
    cnt1[b] = cnt;
    base[b + 1] = base[b] + cnt + cnt2;
  }
  const unsigned long long n_items = base[nb];
  // the final wave of the brute-force walk (k_score_flow): the rank's last
  // SP_FLOW_TAIL (default 4) items per resident CTA -- the last items of the
  // item order -- are claimed last, each in SP_FLOW_SPLIT (default 4) parts.
  // An item of the costliest region outlasts the average one several times,
  // and the kernel ends with its last CTA (c5, CTA end times from a
  // -DSP_CTA_TRACE build: first-to-last spread 1.0 -> 0.22 ms, kernel 31.70
  // -> 31.26 ms; 8-rank share 4.33 -> 4.2 ms).
  std::vector<unsigned long long> nsplit(nb, 0), obase(nb + 1, 0), fblk, fbase{0};
  const unsigned long long split_w = getenv("SP_FLOW_SPLIT") ? strtoull(getenv("SP_FLOW_SPLIT"), nullptr, 10) : 4;
  const unsigned long long tail_w = getenv("SP_FLOW_TAIL") ? strtoull(getenv("SP_FLOW_TAIL"), nullptr, 10) : 4;
  const unsigned long long split = flow_walk && !items_mode && split_w > 1 ? split_w : 1;
  if (split > 1) {
    unsigned long long quota = tail_w * slots;
    for (int64_t b = nb - 1; b >= 0 && quota; b--) {
      nsplit[b] = std::min(base[b + 1] - base[b], quota);
      quota -= nsplit[b];
    }
    // runs in ascending block order: the split blocks are the last ones, so
    // the claim sequence stays block-monotone (a CTA's claims never return
    // to a block it has left: its share of a block is flushed only once)
    for (int64_t b = 0; b < nb; b++)
      if (nsplit[b]) {
        fblk.push_back((unsigned long long)b);
        fbase.push_back(fbase.back() + nsplit[b] * split);
      }
  }
  {  // claim bases without the split items; output bases with their parts
    unsigned long long m = 0;
    for (int64_t b = 0; b < nb; b++) {
      const unsigned long long cnt = base[b + 1] - base[b];
      base[b] = m;
      m += cnt - nsplit[b];
      obase[b + 1] = obase[b] + cnt - nsplit[b] + nsplit[b] * split;
    }
    base[nb] = m;
  }
  const unsigned long long n_main = base[nb];
  const int64_t nf = (int64_t)fblk.size();
  const unsigned long long n_claims = obase[nb];  // = n_main + every part of the split items
  if (n_items == 0) {
    if (!must_out) return false;
    alloc_dout(pd, t, s, must_out);
    SP_CUDA(cudaMemsetAsync(pd.dout.p, 0, (size_t)nb * sizeof(sp_score_out), s));  // valid 0, has_best 0
    SP_CUDA(cudaEventRecord(pd.ev[1], s));
    SP_CUDA(cudaEventRecord(pd.ev[2], s));
    SP_CUDA(cudaEventRecord(pd.ev[3], s));
    return true;
  }
  // blocks with many items reduce in two passes (chunks of REDUCE_CHUNK items, then per block)
  unsigned long long max_items = 0;
  for (int64_t b = 0; b < nb; b++) max_items = std::max(max_items, obase[b + 1] - obase[b]);
  const bool two_pass = max_items > 2 * REDUCE_CHUNK;
  // one small H2D for the plan: lo | hi | base | counter | stride | obase | fblk | fbase (| chunk_base)
  const size_t o_obase = 4 * nb + 2, o_fblk = o_obase + nb + 1, o_fbase = o_fblk + nf, o_seg = o_fbase + nf + 1,
               o_cb = o_seg + 4 * nb;
  std::vector<unsigned long long> plan(o_cb + (two_pass ? nb + 1 : 0), 0);
  std::copy(lo.begin(), lo.end(), plan.begin());
  std::copy(hi.begin(), hi.end(), plan.begin() + nb);
  std::copy(base.begin(), base.end(), plan.begin() + 2 * nb);
  std::copy(stride.begin(), stride.end(), plan.begin() + 3 * nb + 2);
  std::copy(obase.begin(), obase.end(), plan.begin() + o_obase);
  std::copy(fblk.begin(), fblk.end(), plan.begin() + o_fblk);
  std::copy(fbase.begin(), fbase.end(), plan.begin() + o_fbase);
  std::copy(cnt1.begin(), cnt1.end(), plan.begin() + o_seg);
  std::copy(lo2.begin(), lo2.end(), plan.begin() + o_seg + nb);
  std::copy(hi2.begin(), hi2.end(), plan.begin() + o_seg + 2 * nb);
  std::copy(stride2.begin(), stride2.end(), plan.begin() + o_seg + 3 * nb);
  unsigned long long n_chunks = 0;
  if (two_pass) {
    unsigned long long* cb = plan.data() + o_cb;
    for (int64_t b = 0; b < nb; b++) {
      cb[b] = n_chunks;
      n_chunks += (obase[b + 1] - obase[b] + REDUCE_CHUNK - 1) / REDUCE_CHUNK;
    }
    cb[nb] = n_chunks;
  }
  DevBuf<unsigned long long>& dplan = pd.dplan;
  DevBuf<ItemOut>& items = pd.items;
  DevBuf<sp_score_out>& dout = pd.dout;
  tr.mark("plan");
  dplan.upload(plan.data(), plan.size(), s);
  items.alloc(n_claims + n_chunks, s);  // (partials of the two-pass reduction behind the items)
  alloc_dout(pd, t, s, must_out);
  tr.mark("upload+alloc");
  unsigned long long* counter = dplan.p + 3 * nb + 1;
  ScorePlan P{t->d_blob_off.p, item_cands, dplan.p + 3 * nb + 2, dplan.p, dplan.p + nb, dplan.p + 2 * nb, nb,
              n_claims, ctx->skip};
  P.obase = dplan.p + o_obase;
  P.fblk = dplan.p + o_fblk;
  P.fbase = dplan.p + o_fbase;
  P.cnt1 = dplan.p + o_seg;
  P.lo2 = dplan.p + o_seg + nb;
  P.hi2 = dplan.p + o_seg + 2 * nb;
  P.stride2 = dplan.p + o_seg + 3 * nb;
  P.nf = nf;
  P.n_main = n_main;
  P.split = split;
  P.sub = (item_cands + split - 1) / split;
  const unsigned long long grid = std::min<unsigned long long>(n_claims, slots);
  SP_CUDA(cudaEventRecord(pd.ev[1], s));
  SP_LAUNCH(ctx, kern, (unsigned)grid, threads, smem_k, s, t->blobs.p, P, items.p, counter);
  SP_CUDA(cudaEventRecord(pd.ev[2], s));
  tr.mark("score launch");
  if (two_pass) {
    const unsigned long long* d_cb = dplan.p + o_cb;
    SP_LAUNCH(ctx, k_reduce_chunks, (unsigned)std::min<unsigned long long>(n_chunks, 65535), THREADS, 0, s, items.p,
              dplan.p + o_obase, d_cb, nb, n_chunks, items.p + n_claims);
    SP_LAUNCH(ctx, k_reduce, (unsigned)std::min<int64_t>(nb, 4096), THREADS, 0, s, items.p + n_claims, d_cb, nb,
              dout.p);
  } else {
    SP_LAUNCH(ctx, k_reduce, (unsigned)std::min<int64_t>(nb, 4096), THREADS, 0, s, items.p, dplan.p + o_obase, nb,
              dout.p);
  }
  SP_CUDA(cudaGetLastError());
  SP_CUDA(cudaEventRecord(pd.ev[3], s));
  return true;
}

// Enqueue the winner detail (when `explain`) and the copy of the per-block
// results (+ detail) into a pinned host block behind pd.dout.
// SP_OPT_SIM_SHARD only: blocks without a valid candidate in this share take
// the all-replica plan (index 0)
__global__ void k_sim_replica(int64_t nb, sp_score_out* __restrict__ out) {
  for (int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; b < nb; b += (int64_t)gridDim.x * blockDim.x)
    if (!out[b].has_best) {
      out[b].has_best = 1;
      out[b].best_index = 0;
      out[b].best_num_split = 0;
      out[b].best_total = -1.0;  // k_sim_totals: the all-replica plan's total from its detail
    }
}
__global__ void k_sim_totals(int64_t nb, const ExplainBlock* __restrict__ x, sp_score_out* __restrict__ out) {
  for (int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; b < nb; b += (int64_t)gridDim.x * blockDim.x)
    if (out[b].best_total < 0.0) out[b].best_total = x[b].total;
}

static void score_results(sp_ctx* ctx, sp_tables* t, bool explain, bool explained = false) {
  cudaStream_t s = ctx->stream;
  const int64_t nb = t->n_blocks;
  TablesPriv* priv = (TablesPriv*)t->priv;
  PendingScore& pd = priv->pending;
  const bool packed = pd.res_packed && explain;
  pd.explain = explain;
  DevBuf<sp_score_out>& dout = pd.dout;
  const int64_t ne = t->tmpl_off[nb], nedge = t->edge_off[nb];
  if (explain && !explained) {
    // winner detail straight from the device-side argmin: no host round trip
    if (!packed) {
      pd.dblk.alloc(nb, s);
      pd.dnode.alloc(4 * std::max<int64_t>(ne, 1), s);
      pd.dedge.alloc(2 * std::max<int64_t>(nedge, 1), s);
    }
    launch_explain(ctx, t, s, priv->dev.edge_off.p, nullptr, dout.p, pd.dblk.p, pd.dnode.p, pd.dedge.p);
    if (ctx->sim_nranks > 1)
      SP_LAUNCH(ctx, k_sim_totals, (unsigned)std::max<int64_t>(1, std::min<int64_t>((nb + 255) / 256, 1024)), 256, 0,
                s, nb, pd.dblk.p, dout.p);
  }
  SP_CUDA(cudaEventRecord(pd.ev[4], s));
  // results (and winner detail) to the pinned block now: collecting this
  // search later does not wait for whatever is queued behind it
  const ResultLayout L = result_layout(t, explain);
  pd.off_blk = L.off_blk;
  pd.off_node = L.off_node;
  pd.off_edge = L.off_edge;
  pd.host = pinned_acquire(ctx, L.need, &pd.host_bytes);
  if (packed) {
    SP_CUDA(cudaMemcpyAsync(pd.host, pd.res.p, L.need, cudaMemcpyDeviceToHost, s));
  } else {
    SP_CUDA(cudaMemcpyAsync(pd.host, dout.p, (size_t)nb * sizeof(sp_score_out), cudaMemcpyDeviceToHost, s));
    if (explain) {
      SP_CUDA(cudaMemcpyAsync(pd.host + pd.off_blk, pd.dblk.p, (size_t)nb * sizeof(ExplainBlock),
                              cudaMemcpyDeviceToHost, s));
      if (ne) SP_CUDA(cudaMemcpyAsync(pd.host + pd.off_node, pd.dnode.p, (size_t)4 * ne, cudaMemcpyDeviceToHost, s));
      if (nedge)
        SP_CUDA(cudaMemcpyAsync(pd.host + pd.off_edge, pd.dedge.p, (size_t)2 * nedge, cudaMemcpyDeviceToHost, s));
    }
  }
  g_d2h_bytes += (int64_t)(nb * sizeof(sp_score_out)) +
                 (explain ? (int64_t)(nb * sizeof(ExplainBlock)) + 4 * ne + 2 * nedge : 0);
  SP_CUDA(cudaEventRecord(pd.ev[5], s));
  pd.active = true;
}

// Single-lane search (no exchange, or the caller exchanges on the host).
// One-kernel search + winner detail when every block is small (k_search_small).
// Returns false (nothing launched) when the search does not qualify.
static bool score_small(sp_ctx* ctx, sp_tables* t) {
  const int64_t nb = t->n_blocks;
  if (nb < 1 || getenv("SP_SEARCH_SMALL_OFF") || getenv("SP_EXPLAIN_ROUTE") || getenv("SP_FORCE_WIDE") ||
      getenv("SP_SCORE_GENERIC") || getenv("SP_SCORE_ITEMS"))
    return false;
  if (!ctx->skip && ctx->memo) return false;
  for (int64_t b = 0; b < nb; b++)
    if (t->hdr[b].C > SMALL_SEARCH_MAX_C || t->hdr[b].V > 32) return false;
  const size_t smem = score_smem(t);
  if (smem > ctx->smem_optin) return false;
  cudaStream_t s = ctx->stream;
  TablesPriv* priv = (TablesPriv*)t->priv;
  PendingScore& pd = priv->pending;
  pd.empty = false;
  pd.explain = true;
  alloc_dout(pd, t, s, false);
  if (!pd.res_packed) {
    pd.dblk.alloc(nb, s);
    pd.dnode.alloc(4 * std::max<int64_t>(t->tmpl_off[nb], 1), s);
    pd.dedge.alloc(2 * std::max<int64_t>(t->edge_off[nb], 1), s);
  }
  auto kern = ctx->skip ? k_search_small<true> : k_search_small<false>;
  allow_smem(ctx, kern, smem);
  int per = resident_ctas(ctx, kern, THREADS, smem);
  if (per < 1) per = 1;
  const unsigned grid = (unsigned)std::min<int64_t>(nb, (int64_t)ctx->sm_count * per);
  SP_CUDA(cudaEventRecord(pd.ev[1], s));
  SP_LAUNCH(ctx, kern, grid, THREADS, smem, s, t->blobs.p, t->d_blob_off.p, nb, view_of(t->dg), t->d_tmpl_off.p,
            t->d_tmpl_nodes.p, priv->dev.ref_slot_of.p, priv->dev.bound.p, priv->dev.xinfo.p, priv->dev.xoff.p,
            priv->dev.edge_off.p, priv->mesh, priv->mu, priv->chunk, pd.dout.p, pd.dblk.p, pd.dnode.p, pd.dedge.p);
  SP_CUDA(cudaGetLastError());
  SP_CUDA(cudaEventRecord(pd.ev[2], s));
  SP_CUDA(cudaEventRecord(pd.ev[3], s));
  score_results(ctx, t, true, true);
  return true;
}

static void score_enqueue(sp_ctx* ctx, sp_tables* t, int32_t shard, int32_t n_shards, bool explain) {
  PendingScore& pd = ((TablesPriv*)t->priv)->pending;
  if (explain && n_shards == 1 && score_small(ctx, t)) return;
  pd.explain = explain;
  if (!score_items(ctx, t, shard, n_shards, false)) {
    pd.empty = true;
    pd.active = true;
    SP_CUDA(cudaEventRecord(pd.ev[5], ctx->stream));
    return;
  }
  score_results(ctx, t, explain);
}

// Exact merge of the lanes' per-block records (search.py:337-343): the
// lexicographic (total, num_split, index) minimum over the lanes that routed a
// candidate (non-negative doubles order like their bit patterns), valid
// counts summed.  One thread per block.
__global__ void k_merge_ranks(const sp_score_out* __restrict__ gath, int32_t n, int64_t nb,
                              sp_score_out* __restrict__ out) {
  for (int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; b < nb; b += (int64_t)gridDim.x * blockDim.x) {
    sp_score_out acc{};
    for (int32_t r = 0; r < n; r++) {
      const sp_score_out o = gath[(int64_t)r * nb + b];
      acc.valid += o.valid;
      if (!o.has_best) continue;
      if (!acc.has_best ||
          key_less((unsigned long long)__double_as_longlong(o.best_total), (uint32_t)o.best_num_split, o.best_index,
                   (unsigned long long)__double_as_longlong(acc.best_total), (uint32_t)acc.best_num_split,
                   acc.best_index)) {
        acc.best_total = o.best_total;
        acc.best_num_split = o.best_num_split;
        acc.best_index = o.best_index;
        acc.has_best = 1;
      }
    }
    out[b] = acc;
  }
}

static void pending_begin(sp_ctx* ctx, sp_tables* t) {
  PendingScore& pd = ((TablesPriv*)t->priv)->pending;
  if (pd.active) throw Error(SP_ERR_CONFIG, "a search on these tables is already in flight");
  pd.ctx = ctx;
  pd.events();
  pd.release_host();
  pd.lane = false;
  SP_CUDA(cudaEventRecord(pd.ev[0], ctx->stream));
}

// Multi-GPU search: lane i scores shard rank_i of n, the lanes' records are
// exchanged (one ncclAllGather, or peer copies onto the primary when the lanes
// share a GPU) and merged on the device; the merged records get the winner
// detail and go to the host on lanes[0]'s stream (and, with NCCL, on every
// lane of `merge_all`: every rank of a process-per-GPU job ends with the
// merged result).
static void score_enqueue_lanes(const std::vector<sp_ctx*>& lanes, const std::vector<sp_tables*>& tl,
                                const std::vector<int32_t>& ranks, int32_t n, bool explain) {
  const int64_t nb = tl[0]->n_blocks;
  const size_t rec = (size_t)nb * sizeof(sp_score_out);
  for (size_t i = 0; i < lanes.size(); i++) {
    SP_CUDA(cudaSetDevice(lanes[i]->device));
    score_items(lanes[i], tl[i], ranks[i], n, true);
  }
  sp_ctx* P = lanes[0];
  PendingScore& pp = ((TablesPriv*)tl[0]->priv)->pending;
  if (P->transport == SP_TRANSPORT_NCCL) {
    for (size_t i = 0; i < lanes.size(); i++) {
      SP_CUDA(cudaSetDevice(lanes[i]->device));
      PendingScore& pd = ((TablesPriv*)tl[i]->priv)->pending;
      pd.gath.alloc((size_t)n * nb, lanes[i]->stream);
    }
    nccl_group_start();
    for (size_t i = 0; i < lanes.size(); i++) {
      PendingScore& pd = ((TablesPriv*)tl[i]->priv)->pending;
      nccl_allgather(lanes[i], pd.dout.p, pd.gath.p, rec);
    }
    nccl_group_end();
  } else {  // SP_TRANSPORT_P2P: lanes of this process, records copied onto the primary
    SP_CUDA(cudaSetDevice(P->device));
    pp.gath.alloc((size_t)n * nb, P->stream);
    for (size_t i = 0; i < lanes.size(); i++) {
      PendingScore& pd = ((TablesPriv*)tl[i]->priv)->pending;
      if (i) SP_CUDA(cudaStreamWaitEvent(P->stream, pd.ev[3], 0));
      SP_CUDA(cudaMemcpyPeerAsync(pp.gath.p + (size_t)ranks[i] * nb, P->device, pd.dout.p, lanes[i]->device, rec,
                                  P->stream));
    }
  }
  SP_CUDA(cudaSetDevice(P->device));
  const unsigned grid = (unsigned)std::max<int64_t>(1, std::min<int64_t>((nb + THREADS - 1) / THREADS, 1024));
  SP_LAUNCH(P, k_merge_ranks, grid, THREADS, 0, P->stream, pp.gath.p, n, nb, pp.dout.p);
  SP_CUDA(cudaGetLastError());
  score_results(P, tl[0], explain);
  for (size_t i = 1; i < lanes.size(); i++) {  // peer lanes: collected with the primary
    PendingScore& pd = ((TablesPriv*)tl[i]->priv)->pending;
    pd.lane = true;
    pd.active = true;
  }
}

// Collect an enqueued search: wait for its own `done` event, then copy the
// per-block results (and winner detail into fx when it was enqueued) out of
// its pinned block.
static void score_finish(sp_ctx* ctx, sp_tables* t, std::vector<sp_score_out>& res, const FusedExplain* fx) {
  const int64_t nb = t->n_blocks;
  TablesPriv* priv = (TablesPriv*)t->priv;
  PendingScore& pd = priv->pending;
  if (!pd.active) throw Error(SP_ERR_CONFIG, "no search in flight on these tables");
  pd.active = false;
  res.assign(nb, sp_score_out{});
  SP_CUDA(cudaEventSynchronize(pd.ev[5]));
  pd.synced = true;
  if (pd.empty) return;
  if (fx && !pd.explain) throw Error(SP_ERR_CONFIG, "winner detail requested but not enqueued");
  std::memcpy(res.data(), pd.host, (size_t)nb * sizeof(sp_score_out));
  if (fx) {
    const int64_t ne = t->tmpl_off[nb], nedge = t->edge_off[nb];
    std::memcpy(fx->blocks, pd.host + pd.off_blk, (size_t)nb * sizeof(ExplainBlock));
    if (ne) std::memcpy(fx->node, pd.host + pd.off_node, (size_t)4 * ne);
    if (nedge) std::memcpy(fx->edge, pd.host + pd.off_edge, (size_t)2 * nedge);
  }
  float ms = 0;
  SP_CUDA(cudaEventElapsedTime(&ms, pd.ev[1], pd.ev[2]));
  ctx->score_kernel_ms = ms;
  if (getenv("SP_SCORE_TRACE")) {
    float a = 0, b = 0, c = 0, d = 0;
    cudaEventElapsedTime(&a, pd.ev[0], pd.ev[1]);
    cudaEventElapsedTime(&b, pd.ev[2], pd.ev[3]);
    cudaEventElapsedTime(&c, pd.ev[3], pd.ev[4]);
    cudaEventElapsedTime(&d, pd.ev[4], pd.ev[5]);
    fprintf(stderr, "[score] nb %lld: launch->kernel %.3f ms, kernel %.3f, reduce %.3f, explain %.3f, d2h %.3f\n",
            (long long)nb, a, ms, b, c, d);
#ifdef SP_CTA_TRACE
    static unsigned long long h[4096][4];
    cudaMemcpyFromSymbol(h, g_cta_trace, sizeof(h));
    std::vector<unsigned long long> st, en;
    double stg = 0, nst = 0;
    int n = 0;
    for (int i = 0; i < 4096 && h[i][0]; i++, n++) {
      st.push_back(h[i][0]);
      en.push_back(h[i][1]);
      stg += h[i][2];
      nst += h[i][3];
    }
    if (n) {
      const unsigned long long t0 = *std::min_element(st.begin(), st.end());
      std::sort(st.begin(), st.end());
      std::sort(en.begin(), en.end());
      auto us = [&](unsigned long long x) { return (x - t0) / 1e3; };
      fprintf(stderr, "[cta] %d CTAs: start max %.1f us; end p0 %.1f p10 %.1f p50 %.1f p90 %.1f max %.1f us; "
                      "per CTA %.1f stagings, %.1f us closing+staging\n",
              n, us(st.back()), us(en[0]), us(en[n / 10]), us(en[n / 2]), us(en[n * 9 / 10]), us(en.back()), nst / n,
              stg / n / 1e3);
    }
    std::memset(h, 0, sizeof(h));
    cudaMemcpyToSymbol(g_cta_trace, h, sizeof(h));
#endif
  }
  pd.release_host();
}

void score_launch(sp_ctx* ctx, sp_tables* t, int32_t shard, int32_t n_shards, bool explain, bool local) {
  if (n_shards < 1 || shard < 0 || shard >= n_shards) throw Error(SP_ERR_CONFIG, "bad shard / n_shards");
  if (t->overflow) throw Error(SP_ERR_UNSUPPORTED, "a block has more than 2**64 candidates");
  if (local) {  // SP_SCORE_LOCAL: the whole search on this device, no exchange, no peer lanes
    pending_begin(ctx, t);
    score_enqueue(ctx, t, 0, 1, explain);
    return;
  }
  if (!ctx->peers.empty()) {  // this process drives several devices
    if (t->peers.size() != ctx->peers.size()) throw Error(SP_ERR_CONFIG, "tables were not built on every device");
    std::vector<sp_ctx*> lanes{ctx};
    std::vector<sp_tables*> tl{t};
    std::vector<int32_t> ranks{0};
    for (size_t i = 0; i < ctx->peers.size(); i++) {
      lanes.push_back(ctx->peers[i]);
      tl.push_back(t->peers[i]);
      ranks.push_back((int32_t)i + 1);
    }
    for (size_t i = 0; i < lanes.size(); i++) {
      SP_CUDA(cudaSetDevice(lanes[i]->device));
      pending_begin(lanes[i], tl[i]);
    }
    score_enqueue_lanes(lanes, tl, ranks, (int32_t)lanes.size(), explain);
    return;
  }
  pending_begin(ctx, t);
  // a search of small blocks only runs whole on every rank (one kernel, tens of
  // microseconds): no share to exchange, every rank ends with the same records
  if (explain && n_shards == 1 && (ctx->comm || ctx->sim_nranks > 1) && score_small(ctx, t)) return;
  if (ctx->comm) {  // one process per GPU: this rank's share, NCCL exchange (also at nranks 1)
    score_enqueue_lanes({ctx}, {t}, {ctx->rank}, ctx->nranks, explain);
    return;
  }
  if (ctx->sim_nranks > 1 && n_shards == 1) {
    // measurement (tools/shard_sim.py): this rank's share of an sim_nranks-rank
    // search, then what the NCCL form does after its all-gather -- here a copy
    // of this rank's records stands in for the gathered ones -- k_merge_ranks
    // and the winner detail chained on the device.  A block this share has no
    // valid candidate for takes the all-replica plan (index 0, which always
    // routes) so the host assembles a report as rank 0 would.
    PendingScore& pd = ((TablesPriv*)t->priv)->pending;
    pd.explain = explain;
    score_items(ctx, t, ctx->sim_rank, ctx->sim_nranks, true);
    const int64_t nb = t->n_blocks;
    pd.gath.alloc((size_t)std::max<int64_t>(nb, 1), ctx->stream);
    SP_CUDA(cudaMemcpyAsync(pd.gath.p, pd.dout.p, (size_t)nb * sizeof(sp_score_out), cudaMemcpyDeviceToDevice,
                            ctx->stream));
    const unsigned grid = (unsigned)std::max<int64_t>(1, std::min<int64_t>((nb + THREADS - 1) / THREADS, 1024));
    SP_LAUNCH(ctx, k_merge_ranks, grid, THREADS, 0, ctx->stream, pd.gath.p, 1, nb, pd.dout.p);
    SP_LAUNCH(ctx, k_sim_replica, grid, THREADS, 0, ctx->stream, nb, pd.dout.p);
    SP_CUDA(cudaGetLastError());
    score_results(ctx, t, explain);
    return;
  }
  score_enqueue(ctx, t, shard, n_shards, explain);
}

void score_wait(sp_ctx* ctx, sp_tables* t, sp_score_out* out, void* xblocks, int8_t* xnode, int8_t* xedge) {
  const int64_t nb = t->n_blocks;
  std::vector<sp_score_out> res;
  FusedExplain fx{xblocks, xnode, xedge};
  PendingScore& pd = ((TablesPriv*)t->priv)->pending;
  score_finish(ctx, t, res, xblocks ? &fx : nullptr);
  float ms = 0;
  SP_CUDA(cudaEventElapsedTime(&ms, pd.ev[0], pd.ev[5]));
  ctx->score_ms = ms;
  // peer lanes finished before the primary's records were merged; the search's
  // kernel time is the slowest lane's
  for (size_t i = 0; i < t->peers.size(); i++) {
    PendingScore& pl = ((TablesPriv*)t->peers[i]->priv)->pending;
    if (!pl.active || !pl.lane) continue;
    pl.active = false;
    pl.lane = false;
    SP_CUDA(cudaSetDevice(ctx->peers[i]->device));
    SP_CUDA(cudaEventSynchronize(pl.ev[2]));
    float k = 0;
    SP_CUDA(cudaEventElapsedTime(&k, pl.ev[1], pl.ev[2]));
    ctx->score_kernel_ms = std::max<double>(ctx->score_kernel_ms, k);
  }
  SP_CUDA(cudaSetDevice(ctx->device));
  for (int64_t b = 0; b < nb; b++) {
    out[b] = res.empty() ? sp_score_out{} : res[b];
    out[b].candidates = t->hdr[b].C;
  }
}

void score_all(sp_ctx* ctx, sp_tables* t, int32_t shard, int32_t n_shards, sp_score_out* out, void* xblocks,
               int8_t* xnode, int8_t* xedge) {
  score_launch(ctx, t, shard, n_shards, xblocks != nullptr);
  score_wait(ctx, t, out, xblocks, xnode, xedge);
}

void score_range(sp_ctx* ctx, sp_tables* t, int64_t block, uint64_t lo, uint64_t hi, double* totals,
                 sp_score_out* out) {
  if (block < 0 || block >= t->n_blocks) throw Error(SP_ERR_CONFIG, "block index out of range");
  const BlobHeader& H = t->hdr[block];
  if (H.C == 0) throw Error(SP_ERR_UNSUPPORTED, "block has more than 2**64 candidates");
  if (hi > H.C) hi = H.C;
  if (lo > hi) lo = hi;
  cudaStream_t s = ctx->stream;
  *out = sp_score_out{};
  out->candidates = H.C;
  if (hi == lo) return;
  const size_t smem = score_smem(t);
  if (smem > ctx->smem_optin)
    throw Error(SP_ERR_UNSUPPORTED, "block tables exceed shared memory (" + std::to_string(smem) + " bytes)");
  allow_smem(ctx, k_score_table, smem);
  const unsigned long long n = hi - lo;
  const unsigned grid = (unsigned)std::min<unsigned long long>((n + THREADS - 1) / THREADS, 4ULL * ctx->sm_count);
  DevBuf<double> dt;
  DevBuf<ItemOut> cta;
  if (totals) dt.alloc(n, s);
  cta.alloc(grid, s);
  SP_LAUNCH(ctx, k_score_table, grid, THREADS, smem, s, t->blobs.p, t->blob_off[block], lo, hi,
            totals ? dt.p : nullptr, cta.p);
  SP_CUDA(cudaGetLastError());
  std::vector<ItemOut> h(grid);
  cta.download(h.data(), grid, s);
  if (totals) dt.download(totals, n, s);
  SP_CUDA(cudaStreamSynchronize(s));
  for (const ItemOut& o : h) {
    out->valid += o.valid;
    if (o.valid == 0) continue;
    sp_score_out c{};
    c.has_best = 1;
    c.best_total = __builtin_bit_cast(double, o.total_bits);
    c.best_num_split = (int32_t)o.num_split;
    c.best_index = o.index;
    c.valid = 0;
    merge_key(out, &c);
  }
}

void explain(sp_ctx* ctx, sp_tables* t, int64_t block, uint64_t index, sp_explain_out* out, sp_edge_conv* edges,
             int32_t max_edges, int32_t* n_edges) {
  if (block < 0 || block >= t->n_blocks) throw Error(SP_ERR_CONFIG, "block index out of range");
  cudaStream_t s = ctx->stream;
  const BlobHeader& H = t->hdr[block];
  if (H.C == 0) throw Error(SP_ERR_UNSUPPORTED, "block has more than 2**64 candidates");
  if (index >= H.C) throw Error(SP_ERR_CONFIG, "candidate index out of range");
  const int V = H.V;
  std::vector<uint8_t> digits(std::max(V, 1), 0);
  uint64_t rem = index;
  for (int sidx = V - 1; sidx >= 0; sidx--) {
    const uint64_t r = ((H.radix3_ref >> sidx) & 1) ? 3 : 2;
    digits[sidx] = (uint8_t)(rem % r);
    rem /= r;
  }
  TablesPriv* priv = (TablesPriv*)t->priv;
  const int64_t e0 = t->tmpl_off[block];
  const int T = (int)(t->tmpl_off[block + 1] - e0);
  DevBuf<uint8_t> ddig;
  ddig.upload(digits.data(), digits.size(), s);
  DevBuf<sp_explain_out> dout;
  DevBuf<sp_edge_conv> dedges;
  DevBuf<int32_t> dne;
  dout.alloc(1, s);
  dedges.alloc(std::max(max_edges, 1), s);
  dne.alloc(1, s);
  SP_LAUNCH(ctx, k_explain, 1, 1, 0, s, view_of(t->dg), t->d_tmpl_nodes.p + e0, T, (int32_t)block, priv->dev.node_block.p,
                            priv->dev.node_tpos.p, priv->dev.ref_slot_of.p + e0, ddig.p, priv->dev.bound.p + e0, priv->mesh, priv->mu,
                            priv->chunk, dout.p, dedges.p, max_edges, dne.p);
  SP_CUDA(cudaGetLastError());
  dout.download(out, 1, s);
  int32_t ne = 0;
  dne.download(&ne, 1, s);
  SP_CUDA(cudaStreamSynchronize(s));
  *n_edges = ne;
  if (edges && ne > 0) {
    dedges.download(edges, std::min(ne, max_edges), s);
    SP_CUDA(cudaStreamSynchronize(s));
  }
}

void explain_all(sp_ctx* ctx, sp_tables* t, const uint64_t* indices, void* blocks_out, int8_t* node_out,
                 int8_t* edge_out) {
  // on the auxiliary stream, after the tables only: a search queued on the
  // main stream meanwhile (the expensive block group) does not delay it
  cudaStream_t s = ctx->aux;
  const int64_t nb = t->n_blocks;
  if (nb == 0) return;
  TablesPriv* priv = (TablesPriv*)t->priv;
  SP_CUDA(cudaStreamWaitEvent(s, priv->built, 0));
  const int64_t ne = t->tmpl_off[nb];
  const int64_t nedge = t->edge_off[nb];
  // one H2D (indices + edge offsets), one D2H per output array
  std::vector<unsigned long long> up(2 * nb + 1);
  for (int64_t b = 0; b < nb; b++) up[b] = indices[b];
  for (int64_t b = 0; b <= nb; b++) up[nb + b] = (unsigned long long)t->edge_off[b];
  DevBuf<unsigned long long> dup;
  dup.upload(up.data(), up.size(), s);
  DevBuf<ExplainBlock> dblk;
  DevBuf<int8_t> dnode, dedge;
  dblk.alloc(nb, s);
  dnode.alloc(4 * std::max<int64_t>(ne, 1), s);
  dedge.alloc(2 * std::max<int64_t>(nedge, 1), s);
  launch_explain(ctx, t, s, (const int64_t*)(dup.p + nb), dup.p, nullptr, dblk.p, dnode.p, dedge.p);
  dblk.download((ExplainBlock*)blocks_out, nb, s);
  dnode.download(node_out, 4 * ne, s);
  dedge.download(edge_out, 2 * nedge, s);
  SP_CUDA(cudaStreamSynchronize(s));
}


// ---------------------------------------------------------------------------
// Route search: blocks beyond the table path's limits (more than MAXT template
// nodes, a node with more than KMAX internal producers, or tables larger than
// shared memory) are searched without routing tables -- every candidate is
// routed node by node with route_node (the reference's per-node pattern
// choice, search.py:134-224) and costed like plan_cost (costmodel.py:193-267),
// per-thread reach/state kept in a global scratch ([T][threads], coalesced).
// Same outputs as the table path (per-block argmin records, winner detail).
namespace {

struct RouteBlock {
  int64_t e0, T;
  unsigned long long C;
  uint64_t radix3_ref;  // bit s: reference slot s has 3 options
  int32_t V, pad;
};

constexpr int ROUTE_THREADS = 128;
constexpr int ROUTE_MAXK = 64;  // internal producers of one node (route_node's conversion arrays)

// one candidate of block `B` by reference index: valid?, total, num_split
__device__ bool route_candidate(const GraphView& G, const RouteBlock& B, int32_t b, const int32_t* tmpl_nodes,
                                const int16_t* ref_slot, const int32_t* node_block, const int32_t* node_tpos,
                                const uint8_t* bound, const MeshC& M, const sp_mesh& mesh, int64_t mu,
                                int64_t chunk, unsigned long long index, uint8_t* st, double* rc, int64_t stride,
                                double* total, uint32_t* nsplit, int* fail_pos) {
  uint8_t dig[64];
  unsigned long long rem = index;
  uint32_t ns = 0;
  for (int s = B.V - 1; s >= 0; s--) {
    const uint32_t r = ((B.radix3_ref >> s) & 1) ? 3 : 2;
    dig[s] = (uint8_t)(rem % r);
    rem /= r;
    ns += dig[s] != 0;
  }
  NodeRoute R;
  int ps[ROUTE_MAXK];
  for (int64_t i = 0; i < B.T; i++) {
    const int32_t n = tmpl_nodes[B.e0 + i];
    int k = 0;
    for (int64_t e = G.in_off[n]; e < G.in_off[n + 1]; e++) {
      const int32_t r = G.in_idx[e];
      if (node_block[r] != b) continue;
      if (k < ROUTE_MAXK) ps[k] = st[node_tpos[r] * stride];
      k++;
    }
    if (k > ROUTE_MAXK) {  // flagged by k_route_bound; the search is abandoned
      *fail_pos = (int)i;
      return false;
    }
    const int slot = ref_slot[B.e0 + i];
    route_node(G, n, b, node_block, slot >= 0 ? dig[slot] : 0, ps, M, &R, true);
    if (R.pattern < 0) {
      *fail_pos = (int)i;
      return false;
    }
    st[i * stride] = (uint8_t)R.state;
    Pattern pats[4];
    patterns_for(G.op[n], pats);
    double base = 0.0;
    int j = 0;
    for (int64_t e = G.in_off[n]; e < G.in_off[n + 1]; e++) {
      const int32_t r = G.in_idx[e];
      if (node_block[r] != b) continue;
      const int kind = R.conv_kind[j];
      const double cc = kind != C_ID ? call_cost(kind, G.act_bytes[r], M) : 0.0;
      base = fmax(base, dadd(rc[node_tpos[r] * stride], cc));
      j++;
    }
    rc[i * stride] = dadd(base, call_cost(pats[R.pattern].coll, G.act_bytes[n], M));
  }
  double fwd = 0.0;
  for (int64_t i = 0; i < B.T; i++) {
    double tail = rc[i * stride];
    const int s = st[i * stride];
    if (bound[B.e0 + i] && s != 0) tail = dadd(tail, call_cost(C_AG, G.act_bytes[tmpl_nodes[B.e0 + i]], M));
    fwd = fmax(fwd, tail);
  }
  double bwd = 0.0;
  if (M.d > 1) {  // pack_gradients (rewrite.py:78-111): buckets, then unfused; one AllReduce each
    int64_t cur = 0;
    int cur_n = 0;
    for (int pass = 0; pass < 2; pass++) {
      for (int64_t i = 0; i < B.T; i++) {
        const int32_t n = tmpl_nodes[B.e0 + i];
        if (!G.w_rank[n] || !G.w_train[n] || dig[ref_slot[B.e0 + i]] != 0) continue;
        const int64_t sz = G.w_bytes[n];
        if (pass == 0) {
          if (sz >= mu) continue;
          if (cur + sz > chunk && cur_n) {
            bwd = dadd(bwd, dadd(M.setup, cost_bytes(C_AR, cur, M)));
            cur = 0;
            cur_n = 0;
          }
          cur += sz;
          cur_n++;
        } else if (sz >= mu) {
          bwd = dadd(bwd, dadd(M.setup, cost_bytes(C_AR, sz, M)));
        }
      }
      if (pass == 0 && cur_n) bwd = dadd(bwd, dadd(M.setup, cost_bytes(C_AR, cur, M)));
    }
  }
  *total = dadd(fwd, dmul(bwd, dadd(1.0, -mesh.overlap_fraction)));
  *nsplit = ns;
  return true;
}

__global__ void __launch_bounds__(ROUTE_THREADS) k_score_route(GraphView G, const RouteBlock* __restrict__ blocks,
                                                               int64_t nb, const int32_t* tmpl_nodes,
                                                               const int16_t* ref_slot, const int32_t* node_block,
                                                               const int32_t* node_tpos, const uint8_t* bound,
                                                               sp_mesh mesh, int64_t mu, int64_t chunk,
                                                               uint8_t* st_scr, double* rc_scr,
                                                               ItemOut* __restrict__ out, uint32_t* contrib) {
  const MeshC M = mesh_consts(mesh);
  const int64_t NT = (int64_t)gridDim.x * blockDim.x;
  const int64_t gt = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  constexpr int NW = ROUTE_THREADS / 32;
  __shared__ unsigned long long s_t[NW], s_i[NW], s_v[NW];
  __shared__ uint32_t s_n[NW];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int64_t b = 0; b < nb; b++) {
    const RouteBlock B = blocks[b];
    unsigned long long bt = ~0ULL, bi = ~0ULL, nv = 0;
    uint32_t bn = 0xFFFFFFFFu;
    for (unsigned long long x = (unsigned long long)gt; x < B.C; x += (unsigned long long)NT) {
      double tot;
      uint32_t ns;
      int fp;
      if (!route_candidate(G, B, (int32_t)b, tmpl_nodes, ref_slot, node_block, node_tpos, bound, M, mesh, mu, chunk,
                           x, st_scr + gt, rc_scr + gt, NT, &tot, &ns, &fp))
        continue;
      nv++;
      const unsigned long long tb = (unsigned long long)__double_as_longlong(tot);
      if (key_less(tb, ns, x, bt, bn, bi)) {
        bt = tb;
        bn = ns;
        bi = x;
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const unsigned long long t2 = __shfl_down_sync(0xffffffffu, bt, o);
      const unsigned long long i2 = __shfl_down_sync(0xffffffffu, bi, o);
      const uint32_t n2 = __shfl_down_sync(0xffffffffu, bn, o);
      nv += __shfl_down_sync(0xffffffffu, nv, o);
      if (key_less(t2, n2, i2, bt, bn, bi)) {
        bt = t2;
        bn = n2;
        bi = i2;
      }
    }
    if (lane == 0) {
      s_t[warp] = bt;
      s_i[warp] = bi;
      s_n[warp] = bn;
      s_v[warp] = nv;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      ItemOut o{s_t[0], s_i[0], s_n[0], s_v[0]};
      for (int w = 1; w < NW; w++) {
        o.valid += s_v[w];
        if (key_less(s_t[w], s_n[w], s_i[w], o.total_bits, o.num_split, o.index)) {
          o.total_bits = s_t[w];
          o.num_split = s_n[w];
          o.index = s_i[w];
        }
      }
      if (o.valid) out[b * (int64_t)gridDim.x + atomicAdd(&contrib[b], 1u)] = o;
    }
    __syncthreads();
  }
}

// winner detail of the route blocks (the fields of k_explain_all): one thread per block
__global__ void k_explain_route(GraphView G, const RouteBlock* __restrict__ blocks, int64_t nb,
                                const int32_t* tmpl_nodes, const int16_t* ref_slot, const int32_t* node_block,
                                const int32_t* node_tpos, const uint8_t* bound, const int64_t* edge_off,
                                const unsigned long long* indices, const sp_score_out* scores, sp_mesh mesh,
                                int64_t mu, int64_t chunk, uint8_t* st_scr, double* rc_scr, ExplainBlock* out,
                                int8_t* node_out, int8_t* edge_out) {
  const MeshC M = mesh_consts(mesh);
  for (int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; b < nb; b += (int64_t)gridDim.x * blockDim.x) {
    const RouteBlock B = blocks[b];
    ExplainBlock X;
    X.valid = 0;
    X.fail_pos = -1;
    X.forward_comm = X.backward_comm = X.total = 0.0;
    for (int k = 0; k < 4; k++) X.bytes[k] = X.calls[k] = 0;
    X.collective_calls = 0;
    const unsigned long long index = scores ? (scores[b].has_best ? scores[b].best_index : ~0ULL) : indices[b];
    if (index == ~0ULL || index >= B.C) {
      out[b] = X;
      continue;
    }
    uint8_t* st = st_scr + B.e0;  // ΣT scratch: block b's template range
    double* rc = rc_scr + B.e0;
    uint8_t dig[64];
    unsigned long long rem = index;
    for (int s = B.V - 1; s >= 0; s--) {
      const uint32_t r = ((B.radix3_ref >> s) & 1) ? 3 : 2;
      dig[s] = (uint8_t)(rem % r);
      rem /= r;
    }
    int64_t eo = edge_off[b];
    NodeRoute R;
    int ps[ROUTE_MAXK];
    bool ok = true;
    for (int64_t i = 0; i < B.T && ok; i++) {
      const int32_t n = tmpl_nodes[B.e0 + i];
      int k = 0;
      for (int64_t e = G.in_off[n]; e < G.in_off[n + 1]; e++) {
        const int32_t r = G.in_idx[e];
        if (node_block[r] != (int32_t)b) continue;
        if (k < ROUTE_MAXK) ps[k] = st[node_tpos[r]];
        k++;
      }
      const int slot = ref_slot[B.e0 + i];
      route_node(G, n, (int32_t)b, node_block, slot >= 0 ? dig[slot] : 0, ps, M, &R, true);
      if (R.pattern < 0) {
        X.fail_pos = (int)i;
        ok = false;
        break;
      }
      st[i] = (uint8_t)R.state;
      Pattern pats[4];
      patterns_for(G.op[n], pats);
      double base = 0.0;
      int j = 0;
      for (int64_t e = G.in_off[n]; e < G.in_off[n + 1]; e++) {
        const int32_t r = G.in_idx[e];
        if (node_block[r] != (int32_t)b) continue;
        const int kind = R.conv_kind[j];
        double cc = 0.0;
        if (kind != C_ID) {
          cc = call_cost(kind, G.act_bytes[r], M);
          X.bytes[kind - 1] += G.act_bytes[r];
          X.calls[kind - 1]++;
        }
        edge_out[2 * eo] = (int8_t)kind;
        edge_out[2 * eo + 1] = R.conv_axis[j];
        eo++;
        base = fmax(base, dadd(rc[node_tpos[r]], cc));
        j++;
      }
      const int pc = pats[R.pattern].coll;
      if (pc != C_ID) {
        X.bytes[pc - 1] += G.act_bytes[n];
        X.calls[pc - 1]++;
      }
      rc[i] = dadd(base, call_cost(pc, G.act_bytes[n], M));
      const NSpec fs = state_spec(R.state, G.act_rank[n]);
      node_out[4 * (B.e0 + i)] = (int8_t)R.pattern;
      node_out[4 * (B.e0 + i) + 1] = fs.kind == K_S ? fs.axis : -1;
      node_out[4 * (B.e0 + i) + 2] = -1;
      node_out[4 * (B.e0 + i) + 3] = 0;
    }
    if (!ok) {
      out[b] = X;
      continue;
    }
    double fwd = 0.0;
    for (int64_t i = 0; i < B.T; i++) {
      const int32_t n = tmpl_nodes[B.e0 + i];
      double tail = rc[i];
      if (bound[B.e0 + i] && st[i] != 0) {
        tail = dadd(tail, call_cost(C_AG, G.act_bytes[n], M));
        X.bytes[C_AG - 1] += G.act_bytes[n];
        X.calls[C_AG - 1]++;
        node_out[4 * (B.e0 + i) + 2] = state_spec(st[i], G.act_rank[n]).axis;
      }
      fwd = fmax(fwd, tail);
    }
    double bwd = 0.0;
    if (M.d > 1) {
      int64_t cur = 0;
      int cur_n = 0;
      for (int pass = 0; pass < 2; pass++) {
        for (int64_t i = 0; i < B.T; i++) {
          const int32_t n = tmpl_nodes[B.e0 + i];
          if (!G.w_rank[n] || !G.w_train[n] || dig[ref_slot[B.e0 + i]] != 0) continue;
          const int64_t sz = G.w_bytes[n];
          if (pass == 0) {
            if (sz >= mu) continue;
            if (cur + sz > chunk && cur_n) {
              bwd = dadd(bwd, dadd(M.setup, cost_bytes(C_AR, cur, M)));
              X.bytes[0] += cur;
              X.calls[0]++;
              cur = 0;
              cur_n = 0;
            }
            cur += sz;
            cur_n++;
          } else if (sz >= mu) {
            bwd = dadd(bwd, dadd(M.setup, cost_bytes(C_AR, sz, M)));
            X.bytes[0] += sz;
            X.calls[0]++;
          }
        }
        if (pass == 0 && cur_n) {
          bwd = dadd(bwd, dadd(M.setup, cost_bytes(C_AR, cur, M)));
          X.bytes[0] += cur;
          X.calls[0]++;
        }
      }
    }
    X.valid = 1;
    X.forward_comm = fwd;
    X.backward_comm = bwd;
    X.total = dadd(fwd, dmul(bwd, dadd(1.0, -mesh.overlap_fraction)));
    X.collective_calls = X.calls[0] + X.calls[1] + X.calls[2] + X.calls[3];
    out[b] = X;
  }
}

// internal producers per template entry and the boundary flag, for the route blocks
__global__ void k_route_bound(GraphView G, const int64_t* tmpl_off, const int32_t* tmpl_nodes, int64_t nb,
                              const int32_t* node_block, const int32_t* node_tpos, const uint8_t* has_cons,
                              const uint8_t* ext_cons, uint8_t* bound, int32_t* err) {
  for (int64_t b = blockIdx.x; b < nb; b += gridDim.x)
    for (int64_t e = tmpl_off[b] + threadIdx.x; e < tmpl_off[b + 1]; e += blockDim.x) {
      const int32_t n = tmpl_nodes[e];
      bound[e] = !has_cons[n] || ext_cons[n];
      int k = 0;
      for (int64_t q = G.in_off[n]; q < G.in_off[n + 1]; q++) {
        const int32_t r = G.in_idx[q];
        if (node_block[r] != (int32_t)b) continue;
        k++;
        if (node_tpos[r] >= e - tmpl_off[b]) atomicExch(err, 2);  // template not topologically ordered
      }
      if (k > ROUTE_MAXK) atomicExch(err, 3);
    }
}

}  // namespace

// The route search of `nb` blocks (templates in tmpl_off/tmpl_nodes, reference
// slot of every template entry or -1, radix 2/3 per entry, internal-edge
// offsets per block): scores (argmin records) unless `indices` is given, then
// the winner (or the given candidate) detail of every block.
void route_search(sp_ctx* ctx, sp_dgraph* dg, int64_t nb, const int64_t* tmpl_off, const int32_t* tmpl_nodes,
                  const int16_t* ref_slot, const uint8_t* radix, const int64_t* edge_off, const sp_mesh* mesh,
                  int64_t mu, int64_t chunk, const uint64_t* indices, sp_score_out* scores, void* xblocks,
                  int8_t* xnode, int8_t* xedge) {
  cudaStream_t s = ctx->stream;
  if (mu > chunk)
    throw Error(SP_ERR_CONFIG, "fusion threshold " + std::to_string(mu) + " exceeds chunk size " + std::to_string(chunk));
  const int64_t n = dg->n, ne = tmpl_off[nb];
  std::vector<RouteBlock> rb(nb);
  int64_t maxT = 1;
  for (int64_t b = 0; b < nb; b++) {
    RouteBlock& B = rb[b];
    B.e0 = tmpl_off[b];
    B.T = tmpl_off[b + 1] - tmpl_off[b];
    maxT = std::max(maxT, B.T);
    unsigned __int128 C = 1;
    int V = 0;
    uint64_t r3 = 0;
    for (int64_t e = B.e0; e < B.e0 + B.T; e++) {
      if (ref_slot[e] < 0) continue;
      if (ref_slot[e] >= 64) throw Error(SP_ERR_UNSUPPORTED, "a block has more than 2**64 candidates");
      V = std::max(V, ref_slot[e] + 1);
      if (radix[e] == 3) r3 |= 1ULL << ref_slot[e];
      C *= radix[e];
      if (C > (unsigned __int128)UINT64_MAX) throw Error(SP_ERR_UNSUPPORTED, "a block has more than 2**64 candidates");
    }
    B.C = (unsigned long long)C;
    B.V = V;
    B.radix3_ref = r3;
  }
  const int64_t nedge = edge_off[nb];
  PackedUpload pk;
  const size_t o_off = pk.add(tmpl_off, (nb + 1) * 8), o_nodes = pk.add(tmpl_nodes, ne * 4),
               o_slot = pk.add(ref_slot, ne * 2), o_eoff = pk.add(edge_off, (nb + 1) * 8),
               o_rb = pk.add(rb.data(), nb * sizeof(RouteBlock)),
               o_idx = indices ? pk.add(indices, nb * 8) : 0;
  size_t pin_bytes = 0;
  uint8_t* pin = pinned_acquire(ctx, std::max<size_t>(pk.total, nb * sizeof(sp_score_out) + 64), &pin_bytes);
  struct Release {
    sp_ctx* ctx;
    uint8_t* p;
    size_t n;
    ~Release() { pinned_release(ctx, p, n); }
  } rel{ctx, pin, pin_bytes};
  for (const auto& part : pk.parts)
    if (part.bytes) std::memcpy(pin + part.off, part.src, part.bytes);
  DevBuf<uint8_t> arena;
  arena.alloc(std::max<size_t>(pk.total, 16), s);
  SP_CUDA(cudaMemcpyAsync(arena.p, pin, pk.total, cudaMemcpyHostToDevice, s));
  g_h2d_bytes += (int64_t)pk.total;
  const int64_t* d_off = (const int64_t*)(arena.p + o_off);
  const int32_t* d_nodes = (const int32_t*)(arena.p + o_nodes);
  const int16_t* d_slot = (const int16_t*)(arena.p + o_slot);
  const int64_t* d_eoff = (const int64_t*)(arena.p + o_eoff);
  const RouteBlock* d_rb = (const RouteBlock*)(arena.p + o_rb);
  DevBuf<int32_t> node_block, node_tpos, err;
  DevBuf<uint8_t> has_cons, ext_cons, bound;
  node_block.alloc(n, s);
  node_tpos.alloc(n, s);
  err.alloc(2, s);
  has_cons.alloc(n, s);
  ext_cons.alloc(n, s);
  bound.alloc(std::max<int64_t>(ne, 1), s);
  SP_CUDA(cudaMemsetAsync(node_block.p, 0xff, n * 4, s));
  SP_CUDA(cudaMemsetAsync(node_tpos.p, 0xff, n * 4, s));
  SP_CUDA(cudaMemsetAsync(err.p, 0, 8, s));
  SP_CUDA(cudaMemsetAsync(has_cons.p, 0, n, s));
  SP_CUDA(cudaMemsetAsync(ext_cons.p, 0, n, s));
  const GraphView G = view_of(dg);
  const int gb = (int)std::min<int64_t>(std::max<int64_t>(nb, 1), 65535);
  if (nb > 0) SP_LAUNCH(ctx, k_mark_blocks, gb, 128, 0, s, d_off, d_nodes, nb, node_block.p, node_tpos.p, err.p);
  SP_LAUNCH(ctx, k_boundary, grid_for(n, ctx->sm_count), 256, 0, s, G, n, node_block.p, has_cons.p, ext_cons.p);
  if (nb > 0)
    SP_LAUNCH(ctx, k_route_bound, gb, 128, 0, s, G, d_off, d_nodes, nb, node_block.p, node_tpos.p, has_cons.p,
              ext_cons.p, bound.p, err.p);
  DevBuf<sp_score_out> dout;
  dout.alloc(std::max<int64_t>(nb, 1), s);
  const int grid = ctx->sm_count * 2;
  const int64_t NT = (int64_t)grid * ROUTE_THREADS;
  DevBuf<uint8_t> st;
  DevBuf<double> rc;
  if (!indices) {
    DevBuf<ItemOut> rec;
    DevBuf<uint32_t> contrib;
    st.alloc((size_t)maxT * NT, s);
    rc.alloc((size_t)maxT * NT, s);
    rec.alloc((size_t)std::max<int64_t>(nb, 1) * grid, s);
    contrib.alloc(std::max<int64_t>(nb, 1), s);
    SP_CUDA(cudaMemsetAsync(contrib.p, 0, std::max<int64_t>(nb, 1) * 4, s));
    SP_LAUNCH(ctx, k_score_route, grid, ROUTE_THREADS, 0, s, G, d_rb, nb, d_nodes, d_slot, node_block.p, node_tpos.p,
              bound.p, *mesh, mu, chunk, st.p, rc.p, rec.p, contrib.p);
    SP_LAUNCH(ctx, k_reduce_contrib, (unsigned)std::min<int64_t>(std::max<int64_t>(nb, 1), 4096), THREADS, 0, s, rec.p,
              contrib.p, (int64_t)grid, nb, dout.p);
    SP_CUDA(cudaGetLastError());
  }
  DevBuf<ExplainBlock> dblk;
  DevBuf<int8_t> dnode, dedge;
  dblk.alloc(std::max<int64_t>(nb, 1), s);
  dnode.alloc(4 * std::max<int64_t>(ne, 1), s);
  dedge.alloc(2 * std::max<int64_t>(nedge, 1), s);
  SP_CUDA(cudaMemsetAsync(dnode.p, 0, 4 * std::max<int64_t>(ne, 1), s));
  if (st.n < (size_t)ne) st.alloc(std::max<int64_t>(ne, 1), s);
  if (rc.n < (size_t)ne) rc.alloc(std::max<int64_t>(ne, 1), s);
  SP_LAUNCH(ctx, k_explain_route, (int)std::max<int64_t>(1, std::min<int64_t>((nb + 63) / 64, 1024)), 64, 0, s, G,
            d_rb, nb, d_nodes, d_slot, node_block.p, node_tpos.p, bound.p, d_eoff,
            indices ? (const unsigned long long*)(arena.p + o_idx) : nullptr, indices ? nullptr : dout.p, *mesh, mu,
            chunk, st.p, rc.p, dblk.p, dnode.p, dedge.p);
  SP_CUDA(cudaGetLastError());
  int32_t err_h[2];
  SP_CUDA(cudaMemcpyAsync(err_h, err.p, 8, cudaMemcpyDeviceToHost, s));
  if (scores && !indices) SP_CUDA(cudaMemcpyAsync(scores, dout.p, nb * sizeof(sp_score_out), cudaMemcpyDeviceToHost, s));
  if (xblocks) SP_CUDA(cudaMemcpyAsync(xblocks, dblk.p, nb * sizeof(ExplainBlock), cudaMemcpyDeviceToHost, s));
  if (xnode && ne) SP_CUDA(cudaMemcpyAsync(xnode, dnode.p, 4 * ne, cudaMemcpyDeviceToHost, s));
  if (xedge && nedge) SP_CUDA(cudaMemcpyAsync(xedge, dedge.p, 2 * nedge, cudaMemcpyDeviceToHost, s));
  g_d2h_bytes += 8 + (int64_t)(nb * (sizeof(sp_score_out) + sizeof(ExplainBlock)) + 4 * ne + 2 * nedge);
  SP_CUDA(cudaStreamSynchronize(s));
  if (err_h[0] == 1) throw Error(SP_ERR_CONFIG, "a node appears in more than one template");
  if (err_h[0] == 2) throw Error(SP_ERR_CONFIG, "template is not in topological order");
  if (err_h[0] == 3) throw Error(SP_ERR_UNSUPPORTED, "a template node has more than 64 internal producers");
  if (scores)
    for (int64_t b = 0; b < nb; b++) {
      if (indices) scores[b] = sp_score_out{};
      scores[b].candidates = rb[b].C;
    }
}

void tables_wait_built(sp_tables* t) {
  TablesPriv* priv = (TablesPriv*)t->priv;
  if (priv && priv->built) cudaEventSynchronize(priv->built);
  else if (t->ctx) cudaStreamSynchronize(t->ctx->stream);
}

void tables_free_priv(sp_tables* t) {
  delete (TablesPriv*)t->priv;
  t->priv = nullptr;
}

void merge_key(sp_score_out* acc, const sp_score_out* o) {
  acc->valid += o->valid;
  if (!o->has_best) return;
  bool take = !acc->has_best;
  if (!take) {
    if (o->best_total != acc->best_total) take = o->best_total < acc->best_total;
    else if (o->best_num_split != acc->best_num_split) take = o->best_num_split < acc->best_num_split;
    else take = o->best_index < acc->best_index;
  }
  if (take) {
    acc->has_best = 1;
    acc->best_total = o->best_total;
    acc->best_num_split = o->best_num_split;
    acc->best_index = o->best_index;
  }
}

}  // namespace sp
