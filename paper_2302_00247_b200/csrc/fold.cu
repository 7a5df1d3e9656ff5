// Graph upload and shared-subgraph folding on the device.
//
// Reference semantics (pruning.py:123-201): siblings are grouped by their
// depth-d name prefix; among the children of one parent, groups whose exact
// template key (_template_key, pruning.py:97-111) occurs >= min_dup times are
// accepted as one Subgraph; the rest descend one level, and members that end
// at depth d become residual singletons.  Whether a group is still "active"
// at level d depends only on its ancestors, so the recursion is executed
// level-synchronously over all sibling sets at once:
//
//   per level d (all kernels grid-stride over the active nodes / groups)
//     1. sort active nodes by (prefix_d hash, rel-name hash)   [CUB radix]
//        -> groups = runs of equal prefix hash, members in canonical order
//     2. 1-round WL entry hash per node: rel name, op, weight, multiset of
//        internal producers' rel names; group key = commutative sum
//     3. sort groups by (parent group, key)                     [CUB radix]
//        -> classes = runs of equal (parent, key)
//     4. exact verification: every node's prefix bytes against its group
//        head, every group member-by-member against its class head (rel
//        bytes, op, weight, internal-producer positions).  Any mismatch is a
//        hash collision: the whole fold reruns with a new seed, so the
//        partition is exact, not probabilistic.
//     5. classes with >= min_dup groups are accepted; the rest split into
//        residuals (depth == d) and next-level actives.
//
// The host then orders the result the way the reference's string sorts do
// (instances and blocks by prefix string, template by topological rank).
#include <cub/cub.cuh>
#include <cuda_pipeline.h>

#include <algorithm>
#include <atomic>
#include <thread>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <numeric>

#include <functional>
#include <condition_variable>
#include <mutex>
#include <unistd.h>
#include "sp_internal.h"

namespace sp {

namespace {

constexpr uint64_t kPolyB = 0x100000001b3ULL;  // odd polynomial base

__host__ __device__ __forceinline__ uint64_t fmix64(uint64_t k) {
  k ^= k >> 33;
  k *= 0xff51afd7ed558ccdULL;
  k ^= k >> 33;
  k *= 0xc4ceb9fe1a85ec53ULL;
  k ^= k >> 33;
  return k;
}


__global__ void k_depth(const int64_t* __restrict__ off, const uint8_t* __restrict__ s, int64_t n,
                        int32_t* __restrict__ depth, int32_t* __restrict__ maxd) {
  int32_t local = 1;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    int32_t d = 1;
    for (int64_t k = off[i]; k < off[i + 1]; k++) d += s[k] == '/';
    depth[i] = d;
    local = max(local, d);
  }
  atomicMax(maxd, local);
}

// Per node and depth d: prefix end, prefix hash, rel-name hash.
// Output element of (node i, depth dd) at i*si + dd*sd: node-major (si = D,
// sd = 1) or level-major (si = 1, sd = n: one depth's values of all nodes are
// contiguous, so a level pass reads them coalesced).
__device__ __forceinline__ void name_hash_one(int64_t i, const int64_t* __restrict__ off, const uint8_t* __restrict__ s, int64_t n,
                            int32_t D, uint64_t seed, int32_t* __restrict__ pend,
                            uint64_t* __restrict__ ph, uint64_t* __restrict__ rh, int64_t si, int64_t sd) {
  const uint8_t* p = s + off[i];
  const int64_t L = off[i + 1] - off[i];
  // forward: prefix ends and prefix hashes (h = poly(p[0:k])), straight to the
  // outputs at each '/' (no per-thread arrays)
  uint64_t h = 0;
  int d = 0;
  for (int64_t k = 0; k <= L; k++) {
    if (k == L || p[k] == '/') {
      if (d < D) {
        pend[i * si + d * sd] = (int32_t)k;
        ph[i * si + d * sd] = fmix64(h ^ fmix64(seed + (uint64_t)k));
      }
      d++;
      if (k == L) break;
    }
    h = h * kPolyB + (uint64_t)p[k] + 1;
  }
  const int dn = d;  // node depth
  const uint64_t seed_r = seed ^ 0x9e3779b97f4a7c15ULL;
  // backward: rel = the suffix after each prefix (r = poly of p[k+1:L] read
  // backwards), the node itself (rel "") at its own depth
  if (dn - 1 < D) rh[i * si + (dn - 1) * sd] = fmix64(fmix64(seed_r));
  uint64_t r = 0;
  int slash = dn - 1;
  for (int64_t k = L - 1; k >= 0; k--) {
    if (p[k] == '/') {
      slash--;
      if (slash < D) rh[i * si + slash * sd] = fmix64(r ^ fmix64(seed_r + (uint64_t)(L - 1 - k)));
    }
    r = r * kPolyB + (uint64_t)p[k] + 1;
  }
  for (int dd = dn; dd < D; dd++) {  // deeper than the node: never grouped
    pend[i * si + dd * sd] = (int32_t)L;
    ph[i * si + dd * sd] = 0;
    rh[i * si + dd * sd] = 0;
  }
}

__global__ void k_name_hash(const int64_t* __restrict__ off, const uint8_t* __restrict__ s, int64_t n,
                            int32_t D, uint64_t seed, int32_t* __restrict__ pend,
                            uint64_t* __restrict__ ph, uint64_t* __restrict__ rh) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    name_hash_one(i, off, s, n, D, seed, pend, ph, rh, D, 1);
}

__global__ void k_gather_keys(const int32_t* __restrict__ act, int64_t nA, const uint64_t* __restrict__ src,
                              int32_t D, int32_t dd, uint64_t* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nA;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = src[(int64_t)act[i] * D + dd];
}

__global__ void k_heads_u64(const uint64_t* __restrict__ k, int64_t n, int32_t* __restrict__ head) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    head[i] = (i == 0 || k[i] != k[i - 1]) ? 1 : 0;
}

// groups: cur[node] = stamp|gid, gstart[gid] = first sorted position,
// inv[node] = sorted position (when inv is given)
__global__ void k_group_setup(const int32_t* __restrict__ sorted, const int32_t* __restrict__ gid,
                              int64_t nA, int64_t stamp, int64_t* __restrict__ cur,
                              int32_t* __restrict__ gstart, int32_t* __restrict__ inv) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nA;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int32_t g = gid[i] - 1;  // inclusive scan of heads
    const int32_t v = sorted[i];
    cur[v] = stamp | (int64_t)g;
    if (inv) inv[v] = (int32_t)i;
    if (i == 0 || gid[i - 1] != gid[i]) gstart[g] = (int32_t)i;
  }
}

__device__ __forceinline__ uint64_t weight_hash(int64_t n, const uint8_t* w_rank, const int64_t* w_shape,
                                                const uint8_t* w_train) {
  const int r = w_rank[n];
  if (!r) return 0x51ed270b27a8f1a3ULL;
  uint64_t h = fmix64(0x2545f4914f6cdd1dULL + (uint64_t)r * 31 + (uint64_t)w_train[n]);
  for (int k = 0; k < r; k++) h = fmix64(h ^ (uint64_t)w_shape[n * SP_MAX_RANK + k] * 0x9e3779b97f4a7c15ULL);
  return h;
}

// Entry hash (template key entry) and group key sums; positions in group.
__device__ __forceinline__ void entry_one(int64_t i, const int32_t* __restrict__ sorted, const int32_t* __restrict__ gid, int64_t nA,
                        const int32_t* __restrict__ gstart, const int64_t* __restrict__ cur,
                        const uint64_t* __restrict__ rh, int32_t D, int32_t dd,
                        const uint8_t* __restrict__ op, const uint8_t* __restrict__ w_rank,
                        const int64_t* __restrict__ w_shape, const uint8_t* __restrict__ w_train,
                        const int64_t* __restrict__ in_off, const int32_t* __restrict__ in_idx,
                        int32_t* __restrict__ pos, unsigned long long* __restrict__ gkey) {
  const int32_t n = sorted[i];
  const int32_t g = gid[i] - 1;
  pos[n] = (int32_t)(i - gstart[g]);
  const int64_t me = cur[n];
  uint64_t prod = 0;
  for (int64_t e = in_off[n]; e < in_off[n + 1]; e++) {
    const int32_t r = in_idx[e];
    if (cur[r] == me) prod += fmix64(rh[(int64_t)r * D + dd] ^ 0x6a09e667f3bcc909ULL);
  }
  uint64_t h = fmix64(rh[(int64_t)n * D + dd] + 0x3c6ef372fe94f82bULL * (uint64_t)(op[n] + 1));
  h = fmix64(h ^ weight_hash(n, w_rank, w_shape, w_train));
  h = fmix64(h + fmix64(prod ^ 0xbb67ae8584caa73bULL));
  const uint64_t val = fmix64(h ^ 0xa54ff53a5f1d36f1ULL);
  // lanes of one group (consecutive in sorted order) add their terms in three
  // 22-bit slices, one 64-bit atomic per group per warp (a shared-memory 64-bit
  // atomicAdd is a CAS loop: every member of a group retrying it serialised)
  const unsigned mask = __match_any_sync(__activemask(), g);
  const uint64_t s0 = __reduce_add_sync(mask, (unsigned)(val & 0x3fffff));
  const uint64_t s1 = __reduce_add_sync(mask, (unsigned)((val >> 22) & 0x3fffff));
  const uint64_t s2 = __reduce_add_sync(mask, (unsigned)(val >> 44));
  if ((int)(threadIdx.x & 31) == __ffs(mask) - 1)
    atomicAdd(&gkey[g], (unsigned long long)(s0 + (s1 << 22) + (s2 << 44)));
}

// k_entry in NODE order (multi-kernel path): a node's own arrays and its
// producers' (topological neighbours) are read coalesced instead of in the
// prefix-hash order of the sort; nodes not active at this level are skipped.
__global__ void k_entry_nodes(int64_t n, int64_t stamp, const int64_t* __restrict__ cur,
                              const int32_t* __restrict__ inv, const int32_t* __restrict__ gstart,
                              const uint64_t* __restrict__ rh, int32_t D, int32_t dd,
                              const uint8_t* __restrict__ op, const uint8_t* __restrict__ w_rank,
                              const int64_t* __restrict__ w_shape, const uint8_t* __restrict__ w_train,
                              const int64_t* __restrict__ in_off, const int32_t* __restrict__ in_idx,
                              int32_t* __restrict__ pos, unsigned long long* __restrict__ gkey) {
  const int lane = threadIdx.x & 31;
  // warp-uniform trip count: the group-key sums are aggregated per warp
  for (int64_t base = blockIdx.x * (int64_t)blockDim.x + (threadIdx.x & ~31); base < n;
       base += (int64_t)gridDim.x * blockDim.x) {
    const int64_t v = base + lane;
    const int64_t me = v < n ? cur[v] : -1;
    const bool act = v < n && (me & ~(int64_t)0xffffffff) == stamp;
    const int32_t g = (int32_t)(me & 0xffffffff);
    uint64_t val = 0;
    if (act) {
      pos[v] = inv[v] - gstart[g];
      uint64_t prod = 0;
      for (int64_t e = in_off[v]; e < in_off[v + 1]; e++) {
        const int32_t r = in_idx[e];
        if (cur[r] == me) prod += fmix64(rh[(int64_t)r * D + dd] ^ 0x6a09e667f3bcc909ULL);
      }
      uint64_t h = fmix64(rh[v * D + dd] + 0x3c6ef372fe94f82bULL * (uint64_t)(op[v] + 1));
      h = fmix64(h ^ weight_hash(v, w_rank, w_shape, w_train));
      h = fmix64(h + fmix64(prod ^ 0xbb67ae8584caa73bULL));
      val = fmix64(h ^ 0xa54ff53a5f1d36f1ULL);
    }
    // lanes of one group (consecutive nodes usually share it) add their u64
    // terms in three 22-bit slices (each slice sum fits 32 bits), one atomic per group
    const unsigned mask = __match_any_sync(0xffffffffu, act ? g : -1 - lane);
    const uint64_t s0 = __reduce_add_sync(mask, (unsigned)(val & 0x3fffff));
    const uint64_t s1 = __reduce_add_sync(mask, (unsigned)((val >> 22) & 0x3fffff));
    const uint64_t s2 = __reduce_add_sync(mask, (unsigned)(val >> 44));
    if (act && lane == __ffs(mask) - 1)
      atomicAdd(&gkey[g], (unsigned long long)(s0 + (s1 << 22) + (s2 << 44)));
  }
}

__global__ void k_class_keys(int64_t nG, int64_t nA, const int32_t* __restrict__ gstart,
                             const int32_t* __restrict__ sorted, const unsigned long long* __restrict__ gkey,
                             const int32_t* __restrict__ gparent, uint64_t* __restrict__ ck,
                             uint32_t* __restrict__ par, int32_t* __restrict__ gidx) {
  for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < nG;
       g += (int64_t)gridDim.x * blockDim.x) {
    const int64_t s0 = gstart[g];
    const int64_t s1 = g + 1 < nG ? gstart[g + 1] : nA;
    ck[g] = fmix64((uint64_t)gkey[g] ^ fmix64((uint64_t)(s1 - s0) + 0x1f83d9abfb41bd6bULL));
    par[g] = (uint32_t)gparent[sorted[s0]];
    gidx[g] = (int32_t)g;
  }
}

__global__ void k_class_heads(const uint32_t* __restrict__ par, const uint64_t* __restrict__ ck,
                              int64_t nG, int32_t* __restrict__ head) {
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < nG;
       j += (int64_t)gridDim.x * blockDim.x)
    head[j] = (j == 0 || par[j] != par[j - 1] || ck[j] != ck[j - 1]) ? 1 : 0;
}

// class of every group, class starts over the class-ordered group list
__global__ void k_class_setup(const int32_t* __restrict__ order, const int32_t* __restrict__ cid,
                              int64_t nG, int32_t* __restrict__ gclass, int32_t* __restrict__ cstart) {
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < nG;
       j += (int64_t)gridDim.x * blockDim.x) {
    const int32_t c = cid[j] - 1;
    gclass[order[j]] = c;
    if (j == 0 || cid[j - 1] != cid[j]) cstart[c] = (int32_t)j;
  }
}

__device__ __forceinline__ bool bytes_eq(const uint8_t* a, const uint8_t* b, int64_t n) {
  for (int64_t k = 0; k < n; k++)
    if (a[k] != b[k]) return false;
  return true;
}

__device__ void sort_small(int32_t* v, int n) {
  for (int i = 1; i < n; i++) {
    int32_t x = v[i];
    int j = i - 1;
    while (j >= 0 && v[j] > x) {
      v[j + 1] = v[j];
      j--;
    }
    v[j + 1] = x;
  }
}

// Exact checks: prefix bytes vs group head, distinct rel hashes inside a
// group, and member-by-member template-key equality vs the class head group.
__device__ __forceinline__ void verify_one(int64_t i, const int32_t* __restrict__ sorted, const int32_t* __restrict__ gid, int64_t nA,
                         int64_t nG, const int32_t* __restrict__ gstart, const int32_t* __restrict__ gclass,
                         const int32_t* __restrict__ cstart, const int32_t* __restrict__ corder,
                         const int64_t* __restrict__ cur, const int32_t* __restrict__ pos,
                         const int32_t* __restrict__ pend, const uint64_t* __restrict__ rh, int32_t D,
                         int32_t dd, const int64_t* __restrict__ name_off, const uint8_t* __restrict__ names,
                         const uint8_t* __restrict__ op, const uint8_t* __restrict__ w_rank,
                         const int64_t* __restrict__ w_shape, const uint8_t* __restrict__ w_train,
                         const int64_t* __restrict__ in_off, const int32_t* __restrict__ in_idx,
                         int32_t* __restrict__ collision) {
  const int32_t n = sorted[i];
  const int32_t g = gid[i] - 1;
  const int64_t s0 = gstart[g];
  const int64_t gsz = (g + 1 < nG ? gstart[g + 1] : nA) - s0;
  bool bad = false;
  // (a) same prefix string as the group head
  const int32_t h = sorted[s0];
  const int32_t pl = pend[(int64_t)n * D + dd];
  if (pl != pend[(int64_t)h * D + dd] || !bytes_eq(names + name_off[n], names + name_off[h], pl)) bad = true;
  // (b) rel hashes strictly distinct inside a group (canonical order well defined)
  if (i > s0 && rh[(int64_t)sorted[i - 1] * D + dd] == rh[(int64_t)n * D + dd]) bad = true;
  // (c) template key equality with the class head group at the same canonical position
  const int32_t c = gclass[g];
  const int32_t hg = corder[cstart[c]];
  if (hg != g) {
    const int64_t h0 = gstart[hg];
    const int64_t hsz = (hg + 1 < nG ? gstart[hg + 1] : nA) - h0;
    const int64_t j = i - s0;
    if (hsz != gsz) {
      bad = true;
    } else {
      const int32_t b = sorted[h0 + j];
      const int64_t la = name_off[n + 1] - name_off[n];
      const int64_t lb = name_off[b + 1] - name_off[b];
      int64_t sa = pl > 0 ? pl + 1 : 0;
      const int32_t plb = pend[(int64_t)b * D + dd];
      int64_t sb = plb > 0 ? plb + 1 : 0;
      sa = sa > la ? la : sa;
      sb = sb > lb ? lb : sb;
      if (la - sa != lb - sb || !bytes_eq(names + name_off[n] + sa, names + name_off[b] + sb, la - sa))
        bad = true;
      if (op[n] != op[b] || w_rank[n] != w_rank[b] || w_train[n] != w_train[b]) bad = true;
      for (int k = 0; k < w_rank[n] && !bad; k++)
        if (w_shape[(int64_t)n * SP_MAX_RANK + k] != w_shape[(int64_t)b * SP_MAX_RANK + k]) bad = true;
      // internal producers as canonical positions
      int32_t pa[16], pb[16];
      int ka = 0, kb = 0;
      bool over = false;
      for (int64_t e = in_off[n]; e < in_off[n + 1]; e++)
        if (cur[in_idx[e]] == cur[n]) {
          if (ka < 16) pa[ka] = pos[in_idx[e]];
          ka++;
        }
      for (int64_t e = in_off[b]; e < in_off[b + 1]; e++)
        if (cur[in_idx[e]] == cur[b]) {
          if (kb < 16) pb[kb] = pos[in_idx[e]];
          kb++;
        }
      if (ka != kb) bad = true;
      if (!bad && ka > 16) over = true;
      if (!bad && !over) {
        sort_small(pa, ka);
        sort_small(pb, kb);
        for (int k = 0; k < ka; k++)
          if (pa[k] != pb[k]) bad = true;
      }
      if (!bad && over) {
        // wide fan-in: quadratic multiset comparison (rare)
        for (int64_t e = in_off[n]; e < in_off[n + 1] && !bad; e++) {
          const int32_t r = in_idx[e];
          if (cur[r] != cur[n]) continue;
          int ca = 0, cb = 0;
          for (int64_t f = in_off[n]; f < in_off[n + 1]; f++)
            ca += cur[in_idx[f]] == cur[n] && pos[in_idx[f]] == pos[r];
          for (int64_t f = in_off[b]; f < in_off[b + 1]; f++)
            cb += cur[in_idx[f]] == cur[b] && pos[in_idx[f]] == pos[r];
          if (ca != cb) bad = true;
        }
      }
    }
  }
  if (bad) atomicExch(collision, 1);
}

// k_verify in node order (multi-kernel path): node v is checked at its sorted
// position inv[v]; its own name and producer reads are coalesced.
__global__ void k_verify_nodes(int64_t n, int64_t stamp, const int32_t* __restrict__ inv, const int32_t* __restrict__ sorted,
                               const int32_t* __restrict__ gid, int64_t nA, int64_t nG,
                               const int32_t* __restrict__ gstart, const int32_t* __restrict__ gclass,
                               const int32_t* __restrict__ cstart, const int32_t* __restrict__ corder,
                               const int64_t* __restrict__ cur, const int32_t* __restrict__ pos,
                               const int32_t* __restrict__ pend, const uint64_t* __restrict__ rh, int32_t D,
                               int32_t dd, const int64_t* __restrict__ name_off, const uint8_t* __restrict__ names,
                               const uint8_t* __restrict__ op, const uint8_t* __restrict__ w_rank,
                               const int64_t* __restrict__ w_shape, const uint8_t* __restrict__ w_train,
                               const int64_t* __restrict__ in_off, const int32_t* __restrict__ in_idx,
                               int32_t* __restrict__ collision) {
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x) {
    if ((cur[v] & ~(int64_t)0xffffffff) != stamp) continue;
    verify_one(inv[v], sorted, gid, nA, nG, gstart, gclass, cstart, corder, cur, pos, pend, rh, D, dd, name_off, names,
               op, w_rank, w_shape, w_train, in_off, in_idx, collision);
  }
}

// accept / residual / descend for every active node
__device__ __forceinline__ void accept_one(int64_t i, const int32_t* __restrict__ sorted, const int32_t* __restrict__ gid, int64_t nA,
                         int64_t nC, int64_t nG, const int32_t* __restrict__ gclass,
                         const int32_t* __restrict__ cstart, const int32_t* __restrict__ depth,
                         int32_t level, int32_t min_dup, int32_t* __restrict__ gparent,
                         uint8_t* __restrict__ next_flag, uint8_t* __restrict__ residual,
                         uint8_t* __restrict__ gaccept) {
  const int32_t n = sorted[i];
  const int32_t g = gid[i] - 1;
  const int32_t c = gclass[g];
  const int64_t csz = (c + 1 < nC ? cstart[c + 1] : nG) - cstart[c];
  const bool acc = csz >= min_dup;
  if (i == 0 || gid[i - 1] != gid[i]) gaccept[g] = acc;
  next_flag[i] = 0;
  if (acc) return;
  if (depth[n] <= level) {
    residual[n] = 1;
  } else {
    next_flag[i] = 1;
    gparent[n] = g;
  }
}

__global__ void k_accept(const int32_t* __restrict__ sorted, const int32_t* __restrict__ gid, int64_t nA,
                         int64_t nC, int64_t nG, const int32_t* __restrict__ gclass,
                         const int32_t* __restrict__ cstart, const int32_t* __restrict__ depth,
                         int32_t level, int32_t min_dup, int32_t* __restrict__ gparent,
                         uint8_t* __restrict__ next_flag, uint8_t* __restrict__ residual,
                         uint8_t* __restrict__ gaccept) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nA;
       i += (int64_t)gridDim.x * blockDim.x)
    accept_one(i, sorted, gid, nA, nC, nG, gclass, cstart, depth, level, min_dup, gparent, next_flag, residual, gaccept);
}

// ---------------------------------------------------------------------------
// Single-CTA fold for graphs up to SMALL_MAX nodes: the same level algorithm
// with block-wide bitonic sorts and scans in shared memory, so the whole
// prune_graph is one launch and one device->host copy.

constexpr int SMALL_THREADS = 1024;
constexpr int64_t SMALL_MAX = 8192;

__device__ int32_t block_inclusive_scan(int32_t* a, int n, int32_t* s_warp) {
  const int NT = blockDim.x, tid = threadIdx.x;
  const int per = (n + NT - 1) / NT;
  const int lo = min(n, tid * per), hi = min(n, lo + per);
  int32_t sum = 0;
  for (int i = lo; i < hi; i++) sum += a[i];
  const int lane = tid & 31, w = tid >> 5;
  int32_t x = sum;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int32_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) s_warp[w] = x;
  __syncthreads();
  if (w == 0) {
    int32_t v = lane < (NT >> 5) ? s_warp[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int32_t y = __shfl_up_sync(0xffffffffu, v, o);
      if (lane >= o) v += y;
    }
    s_warp[lane] = v;
  }
  __syncthreads();
  int32_t run = x - sum + (w > 0 ? s_warp[w - 1] : 0);
  for (int i = lo; i < hi; i++) {
    run += a[i];
    a[i] = run;
  }
  const int32_t total = s_warp[(NT >> 5) - 1];
  __syncthreads();
  return total;
}

// ascending by (K1, K2, V); P2 a power of two
__device__ void block_bitonic(uint64_t* K1, uint64_t* K2, int32_t* V, int P2) {
  for (int size = 2; size <= P2; size <<= 1)
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      for (int t = threadIdx.x; t < (P2 >> 1); t += blockDim.x) {
        const int i = ((t & ~(stride - 1)) << 1) | (t & (stride - 1));
        const int j = i + stride;
        const bool gt = K1[i] != K1[j] ? K1[i] > K1[j] : (K2[i] != K2[j] ? K2[i] > K2[j] : V[i] > V[j]);
        const bool up = (i & size) == 0;
        if (gt == up) {
          const uint64_t a = K1[i], b = K2[i];
          const int32_t c = V[i];
          K1[i] = K1[j];
          K2[i] = K2[j];
          V[i] = V[j];
          K1[j] = a;
          K2[j] = b;
          V[j] = c;
        }
      }
      __syncthreads();
    }
}

__device__ __forceinline__ int pow2ceil(int x) {
  int p = 1;
  while (p < x) p <<= 1;
  return p;
}

struct SmallArgs {
  const int64_t* name_off;
  const uint8_t* names;
  const uint8_t* op;
  const uint8_t* w_rank;
  const int64_t* w_shape;
  const uint8_t* w_train;
  const int64_t* in_off;
  const int32_t* in_idx;
  int64_t n;
  int32_t D;
  int32_t min_dup;
  uint64_t seed;
  int32_t *depth, *pend, *pos, *gparent, *gclass, *act, *flag, *cid;
  uint64_t *ph, *rh;
  int64_t* cur;
  unsigned long long* gkey;
  int32_t *sorted, *gstart, *corder, *cstart, *info, *collision;
  uint8_t *gaccept, *residual, *next_flag;
  // shared-memory staging (k_fold_small<true>): byte offsets into the dynamic
  // shared memory of the per-node scratch and of the graph arrays the level
  // loop reads, so its dependent accesses hit shared memory, not L2 / DRAM
  int32_t o_depth, o_pos, o_gparent, o_gclass, o_act, o_flag, o_cid, o_ph, o_rh, o_cur, o_gkey, o_next;
  int32_t o_name_off, o_names, o_op, o_w_rank, o_w_train, o_w_shape, o_in_off, o_in_idx;
  int64_t name_bytes, n_edges;
  long long* prof;  // SP_FOLD_PROF: clock64() at each phase boundary (thread 0), else null
  uint8_t* hcache;  // the graph's name-hash cache (ph | rh | pend | depth | level-1 order), or null
  int32_t hc_ready; // 1: hcache holds this seed's hashes (read them), 0: compute and fill it
};

// cooperative global -> shared copy (16-byte words when both ends allow it)
__device__ void copy_in(uint8_t* dst, const uint8_t* src, size_t bytes) {
  if ((((uintptr_t)src | (uintptr_t)dst) & 15) == 0) {
    const size_t w = bytes >> 4;
    for (size_t i = threadIdx.x; i < w; i += blockDim.x) ((uint4*)dst)[i] = ((const uint4*)src)[i];
    for (size_t i = (w << 4) + threadIdx.x; i < bytes; i += blockDim.x) dst[i] = src[i];
  } else if ((((uintptr_t)src | (uintptr_t)dst) & 3) == 0) {
    const size_t w = bytes >> 2;
    for (size_t i = threadIdx.x; i < w; i += blockDim.x) ((uint32_t*)dst)[i] = ((const uint32_t*)src)[i];
    for (size_t i = (w << 2) + threadIdx.x; i < bytes; i += blockDim.x) dst[i] = src[i];
  } else {
    for (size_t i = threadIdx.x; i < bytes; i += blockDim.x) dst[i] = src[i];
  }
}

#ifndef SP_FOLD_NOREG
#define SP_FOLD_NOREG 0
#endif
// global -> shared copy issued as asynchronous 16-byte copies (LDGSTS) when
// both ends are 16-byte aligned, so the staging copies of several arrays are
// all in flight together (one memory latency, not one per array); the caller
// commits and waits (copy_in_wait).  Unaligned copies fall back to copy_in.
__device__ void copy_in_async(uint8_t* dst, const uint8_t* src, size_t bytes) {
  if ((((uintptr_t)src | (uintptr_t)dst) & 15) != 0) {
    copy_in(dst, src, bytes);
    return;
  }
  const size_t w = bytes >> 4;
  for (size_t i = threadIdx.x; i < w; i += blockDim.x) __pipeline_memcpy_async(dst + 16 * i, src + 16 * i, 16);
  for (size_t i = (w << 4) + threadIdx.x; i < bytes; i += blockDim.x) dst[i] = src[i];
}
__device__ __forceinline__ void copy_in_wait() {
  __pipeline_commit();
  __pipeline_wait_prior(0);
  __syncthreads();
}

constexpr int RANK_SORT_MAX = 256;  // n^2 compares beat the bitonic network's barriers up to here
// Ascending (K1, K2, V) order of n <= blockDim.x distinct entries by rank
// counting: thread i counts the entries below its own (broadcast shared reads,
// no barrier per step) and writes its entry to that rank.  One pass and two
// barriers instead of the bitonic network's log^2 stages, each with a barrier.
__device__ void block_rank_sort(uint64_t* K1, uint64_t* K2, int32_t* V, int n) {
  const int i = threadIdx.x;
  uint64_t a = 0, b = 0;
  int32_t c = 0, r = 0;
  if (i < n) {
    a = K1[i];
    b = K2[i];
    c = V[i];
#pragma unroll 4
    for (int j = 0; j < n; j++) {
      const uint64_t x = K1[j], y = K2[j];
      r += (int)((x < a) | ((x == a) & ((y < b) | ((y == b) & (V[j] < c)))));
    }
  }
  __syncthreads();
  if (i < n) {
    K1[r] = a;
    K2[r] = b;
    V[r] = c;
  }
  __syncthreads();
}

__device__ __forceinline__ bool key3_less(uint64_t a1, uint64_t a2, int32_t av, uint64_t b1, uint64_t b2, int32_t bv) {
  return a1 != b1 ? a1 < b1 : (a2 != b2 ? a2 < b2 : av < bv);
}

// The bitonic network with every stage of stride < 64 in registers: a warp
// loads a 64-entry chunk (lane l: entries 64c + l and 64c + l + 32), stride 32
// is an in-thread exchange and strides < 32 are warp shuffles, so only stages
// of stride >= 64 go through shared memory with a barrier (1024 entries: 10
// barrier stages instead of 55).  Item: the entry's keys; load(i) / store(i, x)
// read / write entry i, less(x, y) orders two entries (all distinct), shfl(x,
// m) is __shfl_xor_sync of every field.  Any P2 >= 64 (a power of two), any
// block size that is a multiple of 32.
template <class Item, class Load, class Store, class Less, class Shfl>
__device__ void bitonic_sort_reg(int P2, Load load, Store store, Less less, Shfl shfl) {
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5, nw = blockDim.x >> 5;
  const int nch = P2 >> 6;
  auto stages = [&](Item& a, Item& b, int i0, int size, int smax) {
    for (int stride = smax; stride > 0; stride >>= 1) {
      if (stride == 32) {
        if (less(b, a) == ((i0 & size) == 0)) {
          const Item x = a;
          a = b;
          b = x;
        }
      } else {
        const bool lower = (lane & stride) == 0;
        const Item ya = shfl(a, stride), yb = shfl(b, stride);
        const bool up_a = (i0 & size) == 0, up_b = ((i0 + 32) & size) == 0;
        const bool lta = less(ya, a), ltb = less(yb, b);
        if (lower == up_a ? lta : !lta) a = ya;
        if (lower == up_b ? ltb : !ltb) b = yb;
      }
    }
  };
  for (int c = warp; c < nch; c += nw) {  // every size up to 64 inside each chunk
    const int i0 = c * 64 + lane;
    Item a = load(i0), b = load(i0 + 32);
    for (int size = 2; size <= 64; size <<= 1) stages(a, b, i0, size, size >> 1);
    store(i0, a);
    store(i0 + 32, b);
  }
  __syncthreads();
  for (int size = 128; size <= P2; size <<= 1) {
    for (int stride = size >> 1; stride >= 64; stride >>= 1) {
      for (int q = t; q < (P2 >> 1); q += blockDim.x) {
        const int i = ((q & ~(stride - 1)) << 1) | (q & (stride - 1));
        const int j = i + stride;
        const Item x = load(i), y = load(j);
        if (less(y, x) == ((i & size) == 0)) {
          store(i, y);
          store(j, x);
        }
      }
      __syncthreads();
    }
    for (int c = warp; c < nch; c += nw) {
      const int i0 = c * 64 + lane;
      Item a = load(i0), b = load(i0 + 32);
      stages(a, b, i0, size, 32);
      store(i0, a);
      store(i0 + 32, b);
    }
    __syncthreads();
  }
}

struct Key3 {
  uint64_t k1, k2;
  int32_t v;
};

// ascending by (K1, K2, V): rank counting when every entry has a thread, else
// the bitonic network over P2 (a power of two >= n, padded with ~0 keys),
// register-resident below stride 64 (bitonic_sort_reg)
__device__ void block_sort(uint64_t* K1, uint64_t* K2, int32_t* V, int n, int P2) {
  if (n <= RANK_SORT_MAX && n <= (int)blockDim.x) block_rank_sort(K1, K2, V, n);
  else if (P2 >= 64 && !SP_FOLD_NOREG)
    bitonic_sort_reg<Key3>(
        P2, [&](int i) { return Key3{K1[i], K2[i], V[i]}; },
        [&](int i, const Key3& x) {
          K1[i] = x.k1;
          K2[i] = x.k2;
          V[i] = x.v;
        },
        [](const Key3& x, const Key3& y) { return key3_less(x.k1, x.k2, x.v, y.k1, y.k2, y.v); },
        [](const Key3& x, int m) {
          return Key3{__shfl_xor_sync(0xffffffffu, x.k1, m), __shfl_xor_sync(0xffffffffu, x.k2, m),
                      __shfl_xor_sync(0xffffffffu, x.v, m)};
        });
  else block_bitonic(K1, K2, V, P2);
}

template <bool STG>
__global__ void __launch_bounds__(SMALL_THREADS) k_fold_small(SmallArgs a) {
  extern __shared__ __align__(16) uint8_t sm[];
  __shared__ int32_t s_warp[32];
  int np_ = 0;
#define PROF()                                                       \
  do {                                                               \
    if (a.prof && threadIdx.x == 0) {                                \
      a.prof[np_] = clock64();                                       \
      unsigned long long g_;                                         \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g_));         \
      a.prof[128 + np_] = (long long)g_;                             \
    }                                                                \
    np_++;                                                           \
  } while (0)
  PROF();
  const int tid = threadIdx.x, NT = blockDim.x;
  const int n = (int)a.n, D = a.D;
  const int P2max = pow2ceil(n);
  uint64_t* K1 = (uint64_t*)sm;
  uint64_t* K2 = K1 + P2max;
  int32_t* V = (int32_t*)(K2 + P2max);
#define SMALL_PTR(T, f) T const f = STG ? (T)(sm + a.o_##f) : a.f
  SMALL_PTR(int32_t*, depth);
  SMALL_PTR(int32_t*, pos);
  SMALL_PTR(int32_t*, gparent);
  SMALL_PTR(int32_t*, gclass);
  SMALL_PTR(int32_t*, act);
  SMALL_PTR(int32_t*, flag);
  SMALL_PTR(int32_t*, cid);
  SMALL_PTR(uint64_t*, ph);
  SMALL_PTR(uint64_t*, rh);
  SMALL_PTR(int64_t*, cur);
  SMALL_PTR(unsigned long long*, gkey);
  uint8_t* const next_flag = STG ? sm + a.o_next : a.next_flag;
  SMALL_PTR(const int64_t*, name_off);
  SMALL_PTR(const uint8_t*, names);
  SMALL_PTR(const uint8_t*, op);
  SMALL_PTR(const uint8_t*, w_rank);
  SMALL_PTR(const uint8_t*, w_train);
  SMALL_PTR(const int64_t*, w_shape);
  SMALL_PTR(const int64_t*, in_off);
  SMALL_PTR(const int32_t*, in_idx);
#undef SMALL_PTR
  if (STG) {
    copy_in_async((uint8_t*)name_off, (const uint8_t*)a.name_off, (size_t)(n + 1) * 8);
    copy_in_async((uint8_t*)names, a.names, (size_t)a.name_bytes);
    copy_in_async((uint8_t*)op, a.op, (size_t)n);
    copy_in_async((uint8_t*)w_rank, a.w_rank, (size_t)n);
    copy_in_async((uint8_t*)w_train, a.w_train, (size_t)n);
    copy_in_async((uint8_t*)w_shape, (const uint8_t*)a.w_shape, (size_t)n * SP_MAX_RANK * 8);
    copy_in_async((uint8_t*)in_off, (const uint8_t*)a.in_off, (size_t)(n + 1) * 8);
    copy_in_async((uint8_t*)in_idx, (const uint8_t*)a.in_idx, (size_t)a.n_edges * 4);
    if (a.hc_ready) {
      copy_in_async((uint8_t*)ph, a.hcache, (size_t)n * D * 8);
      copy_in_async((uint8_t*)rh, a.hcache + (size_t)n * D * 8, (size_t)n * D * 8);
      copy_in_async((uint8_t*)depth, a.hcache + (size_t)n * D * 20, (size_t)n * 4);
    }
    copy_in_wait();
  } else if (a.hc_ready) {
    copy_in((uint8_t*)ph, a.hcache, (size_t)n * D * 8);
    copy_in((uint8_t*)rh, a.hcache + (size_t)n * D * 8, (size_t)n * D * 8);
    copy_in((uint8_t*)depth, a.hcache + (size_t)n * D * 20, (size_t)n * 4);
  }
  PROF();
  const int64_t nD = (int64_t)n * D;
  if (a.hc_ready) {  // the names' hashes from the graph's first search
    const int32_t* hp = (const int32_t*)(a.hcache + nD * 16);
    for (int64_t k = tid; k < nD; k += NT) a.pend[k] = hp[k];
  }
  for (int i = tid; i < n; i += NT) {
    if (!a.hc_ready) {
      int32_t d = 1;
      for (int64_t k = name_off[i]; k < name_off[i + 1]; k++) d += names[k] == '/';
      depth[i] = d;
      name_hash_one(i, name_off, names, a.n, D, a.seed, a.pend, ph, rh, D, 1);
    }
    gparent[i] = 0;
    a.residual[i] = 0;
    cur[i] = -1;
    act[i] = i;
  }
  __syncthreads();
  if (!a.hc_ready && a.hcache) {  // keep them for the graph's next searches
    uint64_t* hph = (uint64_t*)a.hcache;
    int32_t* hp = (int32_t*)(a.hcache + nD * 16);
    for (int64_t k = tid; k < nD; k += NT) {
      hph[k] = ph[k];
      hph[nD + k] = rh[k];
      hp[k] = a.pend[k];
    }
    for (int i = tid; i < n; i += NT) hp[nD + i] = depth[i];
  }
  PROF();
  int nA = n;
  int level = 1;
  for (; nA > 0 && level <= D; level++) {
    const int dd = level - 1;
    int32_t* srt = a.sorted + (int64_t)dd * n;
    int32_t* gs = a.gstart + (int64_t)dd * (n + 1);
    int32_t* co = a.corder + (int64_t)dd * n;
    int32_t* cs = a.cstart + (int64_t)dd * (n + 1);
    uint8_t* ga = a.gaccept + (int64_t)dd * n;
    // 1. sort active nodes by (prefix hash, rel hash); level 1 sorts every
    // node, a function of the names and the seed: its order comes from the
    // name-hash cache after the graph's first search
    const int P2 = pow2ceil(nA);
    int32_t* const hsorted = a.hcache ? (int32_t*)(a.hcache + (int64_t)n * D * 20 + (int64_t)n * 4) : nullptr;
    if (level == 1 && a.hc_ready) {
      for (int i = tid; i < nA; i += NT) {
        const int32_t v = hsorted[i];
        K1[i] = ph[(int64_t)v * D];
        K2[i] = rh[(int64_t)v * D];
        V[i] = v;
      }
      __syncthreads();
      PROF();
      PROF();
    } else {
      const int nfill = nA <= NT && nA <= RANK_SORT_MAX ? nA : P2;
      for (int i = tid; i < nfill; i += NT) {
        if (i < nA) {
          const int32_t v = act[i];
          K1[i] = ph[(int64_t)v * D + dd];
          K2[i] = rh[(int64_t)v * D + dd];
          V[i] = v;
        } else {
          K1[i] = K2[i] = ~0ULL;
          V[i] = 0x7fffffff;
        }
      }
      __syncthreads();
      PROF();
      block_sort(K1, K2, V, nA, P2);
      PROF();
      if (level == 1 && hsorted)
        for (int i = tid; i < nA; i += NT) hsorted[i] = V[i];
    }
    for (int i = tid; i < nA; i += NT) {
      srt[i] = V[i];
      flag[i] = (i == 0 || K1[i] != K1[i - 1]) ? 1 : 0;
    }
    __syncthreads();
    const int nG = block_inclusive_scan(flag, nA, s_warp);
    const int64_t stamp = ((int64_t)level) << 32;
    for (int i = tid; i < nA; i += NT) {
      const int32_t g = flag[i] - 1;
      cur[srt[i]] = stamp | (int64_t)g;
      if (i == 0 || flag[i - 1] != flag[i]) gs[g] = i;
    }
    for (int g = tid; g < nG; g += NT) gkey[g] = 0;
    if (tid == 0) gs[nG] = nA;
    __syncthreads();
    PROF();
    // 2. entry hashes / group keys
    for (int i = tid; i < nA; i += NT)
      entry_one(i, srt, flag, nA, gs, cur, rh, D, dd, op, w_rank, w_shape, w_train, in_off, in_idx, pos, gkey);
    __syncthreads();
    PROF();
    // 3. classes: sort groups by (parent, key)
    const int P2g = pow2ceil(nG);
    const int gfill = nG <= NT && nG <= RANK_SORT_MAX ? nG : P2g;
    for (int g = tid; g < gfill; g += NT) {
      if (g < nG) {
        K1[g] = (uint64_t)(uint32_t)gparent[srt[gs[g]]];
        K2[g] = fmix64((uint64_t)gkey[g] ^ fmix64((uint64_t)(gs[g + 1] - gs[g]) + 0x1f83d9abfb41bd6bULL));
        V[g] = g;
      } else {
        K1[g] = K2[g] = ~0ULL;
        V[g] = 0x7fffffff;
      }
    }
    __syncthreads();
    block_sort(K1, K2, V, nG, P2g);
    PROF();
    for (int j = tid; j < nG; j += NT) {
      co[j] = V[j];
      cid[j] = (j == 0 || K1[j] != K1[j - 1] || K2[j] != K2[j - 1]) ? 1 : 0;
    }
    __syncthreads();
    const int nC = block_inclusive_scan(cid, nG, s_warp);
    for (int j = tid; j < nG; j += NT) {
      const int32_t c = cid[j] - 1;
      gclass[co[j]] = c;
      if (j == 0 || cid[j - 1] != cid[j]) cs[c] = j;
    }
    if (tid == 0) cs[nC] = nG;
    __syncthreads();
    PROF();
    // 4. exact verification, 5. accept / residual / descend
    for (int i = tid; i < nA; i += NT)
      verify_one(i, srt, flag, nA, nG, gs, gclass, cs, co, cur, pos, a.pend, rh, D, dd, name_off, names, op, w_rank,
                 w_shape, w_train, in_off, in_idx, a.collision);
    __syncthreads();
    PROF();
    for (int i = tid; i < nA; i += NT)
      accept_one(i, srt, flag, nA, nC, nG, gclass, cs, depth, level, a.min_dup, gparent, next_flag, a.residual, ga);
    __syncthreads();
    for (int i = tid; i < nA; i += NT) cid[i] = next_flag[i];
    __syncthreads();
    const int nNext = block_inclusive_scan(cid, nA, s_warp);
    for (int i = tid; i < nA; i += NT)
      if (next_flag[i]) act[cid[i] - 1] = srt[i];
    if (tid == 0) {
      a.info[dd * 4 + 0] = nA;
      a.info[dd * 4 + 1] = nG;
      a.info[dd * 4 + 2] = nC;
    }
    nA = nNext;
    __syncthreads();
    PROF();
  }
  if (tid == 0) a.info[D * 4] = nA > 0 ? -1 : level - 1;
  PROF();
#undef PROF
}

inline int grid_for(int64_t n, int sms) {
  int64_t b = (n + 255) / 256;
  if (b < 1) b = 1;
  int64_t cap = (int64_t)sms * 16;
  return (int)(b < cap ? b : cap);
}

struct LevelOut {
  int32_t level;
  std::vector<int32_t> sorted, gstart, corder, cstart;
  std::vector<uint8_t> gaccept;
};

int strcmp_py(const uint8_t* a, int64_t la, const uint8_t* b, int64_t lb) {
  int64_t m = la < lb ? la : lb;
  int c = m ? std::memcmp(a, b, (size_t)m) : 0;
  if (c) return c;
  return (la > lb) - (la < lb);
}

}  // namespace

// int32 [n x R] shapes -> int64 [n x SP_MAX_RANK] (unused dims 0); identity topo ranks
__global__ void k_expand_graph(int64_t n, int R, const int32_t* __restrict__ a32, const int32_t* __restrict__ w32,
                               int64_t* __restrict__ a64, int64_t* __restrict__ w64, int64_t* __restrict__ topo) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n * SP_MAX_RANK;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t row = i / SP_MAX_RANK;
    const int k = (int)(i % SP_MAX_RANK);
    if (a64) {
      a64[i] = k < R ? a32[row * R + k] : 0;
      w64[i] = k < R ? w32[row * R + k] : 0;
    }
    if (topo && k == 0) topo[row] = row;
  }
}

// Host-side fan-out for graph_upload's byte work (validation scans, the
// name depth scan, copies into the pinned staging buffer): ~20 MB at 10^5
// nodes, memory-bound, so spread over a few threads.
// Persistent workers for host_parallel: spawning up to 15 std::threads per call
// cost ~0.3 ms per call (three calls per graph upload).  Workers sleep on a
// condition variable between jobs; one job at a time (callers serialise on
// run_mu).  The pool is never destroyed (its threads block until exit).
struct HostPool {
  std::mutex run_mu, mu;
  std::condition_variable cv;
  std::vector<std::thread> th;
  const std::function<void(int)>* job = nullptr;
  int active = 0;
  uint64_t gen = 0;
  std::atomic<int> done{0};
  explicit HostPool(int workers) {
    for (int t = 1; t <= workers; t++)
      th.emplace_back([this, t] {
        uint64_t seen = 0;
        std::unique_lock<std::mutex> lk(mu);
        for (;;) {
          cv.wait(lk, [&] { return gen != seen; });
          seen = gen;
          const std::function<void(int)>* f = job;
          const int a = active;
          lk.unlock();
          if (t < a) (*f)(t);
          done.fetch_add(1, std::memory_order_acq_rel);
          lk.lock();
        }
      });
  }
  void run(int T, const std::function<void(int)>& f) {
    std::lock_guard<std::mutex> serial(run_mu);
    const int workers = (int)th.size();
    done.store(0, std::memory_order_relaxed);
    {
      std::lock_guard<std::mutex> lk(mu);
      job = &f;
      active = T;
      gen++;
    }
    cv.notify_all();
    f(0);
    for (unsigned spins = 0; done.load(std::memory_order_acquire) < workers; spins++)
      if (spins > 2048) std::this_thread::yield();
  }
};
inline HostPool& host_pool() {
  static HostPool* p = new HostPool((int)std::min(15u, std::max(1u, std::thread::hardware_concurrency()) - 1));
  return *p;
}

template <class F>
void host_parallel(int64_t n, int64_t grain, F&& f) {
  static const int hw = std::max(1u, std::thread::hardware_concurrency());
  const int T = (int)std::max<int64_t>(1, std::min<int64_t>({(int64_t)hw, 16, n / std::max<int64_t>(1, grain)}));
  if (T <= 1) {
    f(0, n, 0);
    return;
  }
  const std::function<void(int)> job = [&](int t) { f(n * t / T, n * (t + 1) / T, t); };
  static const pid_t owner = getpid();
  if (getpid() != owner) {  // a forked child has none of the pool's threads
    for (int t = 0; t < T; t++) job(t);
    return;
  }
  host_pool().run(T, job);
}

void graph_upload(sp_ctx* ctx, const sp_graph* g, sp_dgraph* dg) {
  const int64_t n = g->n_nodes;
  if (n < 1) throw Error(SP_ERR_CONFIG, "graph has no nodes");
  if (n >= (int64_t)INT32_MAX) throw Error(SP_ERR_UNSUPPORTED, "more than 2^31 nodes");
  cudaStream_t s = ctx->stream;
  static const bool trace = std::getenv("SP_UPLOAD_TRACE") != nullptr;
  const auto tu0 = std::chrono::steady_clock::now();
  auto ms_since = [&](std::chrono::steady_clock::time_point a) {
    return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - a).count();
  };
  dg->ctx = ctx;
  dg->n = n;
  dg->E = g->in_off[n];
  const int64_t nb = g->name_off[n];
  const int64_t E = dg->E;
  // validation + depth (1 + number of '/') per node, one pass per thread slice
  std::atomic<int> bad_rank{0}, bad_edge{0}, wide{0}, permuted{0}, max_rank{1};
  std::atomic<int32_t> maxd{1};
  host_parallel(n, 8192, [&](int64_t lo, int64_t hi, int) {
    int32_t md = 1;
    int mr = 1;
    bool br = false, be = false, pm = false;
    for (int64_t i = lo; i < hi; i++) {
      br |= g->act_rank[i] < 1 || g->act_rank[i] > SP_MAX_RANK || g->w_rank[i] > SP_MAX_RANK;
      mr = std::max(mr, (int)std::max(g->act_rank[i], g->w_rank[i]));
      pm |= g->topo_rank[i] != i;
      const uint8_t* a = g->name_bytes + g->name_off[i];
      const int64_t L = g->name_off[i + 1] - g->name_off[i];
      int32_t d = 1;
      for (int64_t k = 0; k < L; k++) d += a[k] == '/';
      md = std::max(md, d);
    }
    const int64_t elo = E * lo / n, ehi = E * hi / n;
    for (int64_t e = elo; e < ehi; e++) be |= g->in_idx[e] < 0 || g->in_idx[e] >= n;
    if (br) bad_rank = 1;
    if (be) bad_edge = 1;
    if (pm) permuted = 1;
    int cr = max_rank.load();
    while (mr > cr && !max_rank.compare_exchange_weak(cr, mr)) {
    }
    int32_t cur = maxd.load();
    while (md > cur && !maxd.compare_exchange_weak(cur, md)) {
    }
  });
  if (bad_rank) throw Error(SP_ERR_UNSUPPORTED, "tensor rank outside 1..SP_MAX_RANK");
  if (bad_edge) throw Error(SP_ERR_CONFIG, "producer index out of range");
  dg->max_depth = maxd;
  const double tu_check = ms_since(tu0);
  // every array in ONE pinned staging buffer and ONE host->device copy
  struct Part {
    const void* src;
    size_t bytes;
    size_t off;
  };
  // H2D bytes: shapes travel as int32 [n x R] (R = the graph's largest rank)
  // when every dim fits, an identity topo_rank not at all; k_expand_graph
  // rebuilds the int64 [n x SP_MAX_RANK] layouts on the device
  // shapes are packed optimistically: the pack pass itself detects a dim
  // past int32 (one read of the shapes instead of two) and the copy is then
  // redone with the int64 layout
  for (bool pack = true;; pack = false) {
    const bool iota = !permuted;
    const int R = max_rank;
    const size_t shape_bytes = pack ? (size_t)n * R * 4 : (size_t)n * SP_MAX_RANK * 8;
    Part parts[13] = {
        {g->name_bytes, (size_t)nb, 0},
        {g->name_off, (size_t)(n + 1) * 8, 0},
        {g->topo_rank, iota ? 0 : (size_t)n * 8, 0},
        {g->op, (size_t)n, 0},
        {g->act_rank, (size_t)n, 0},
        {g->w_rank, (size_t)n, 0},
        {g->w_trainable, (size_t)n, 0},
        {pack ? nullptr : g->act_shape, shape_bytes, 0},
        {pack ? nullptr : g->w_shape, shape_bytes, 0},
        {g->act_bytes, (size_t)n * 8, 0},
        {g->w_bytes, (size_t)n * 8, 0},
        {g->in_off, (size_t)(n + 1) * 8, 0},
        {g->in_idx, (size_t)E * 4, 0},
    };
    size_t total = 0;
    for (Part& p : parts) {
      p.off = total;
      total += (p.bytes + 255) & ~(size_t)255;
    }
    if (ctx->staging_bytes < total) {
      if (ctx->staging) cudaFreeHost(ctx->staging);
      ctx->staging = nullptr;
      SP_CUDA(cudaHostAlloc(&ctx->staging, total, cudaHostAllocDefault));
      ctx->staging_bytes = total;
    }
    // host copies the library itself needs (string order, slot order, op validity),
    // in vectors a freed graph of this context left behind when there is one
    if (!ctx->host_copies.empty()) {
      HostGraphCopies& hc = ctx->host_copies.back();
      dg->h_names.swap(hc.names);
      dg->h_op.swap(hc.op);
      dg->h_w_rank.swap(hc.w_rank);
      dg->h_w_train.swap(hc.w_train);
      dg->h_name_off.swap(hc.name_off);
      dg->h_topo.swap(hc.topo);
      dg->h_in_off.swap(hc.in_off);
      dg->h_in_idx.swap(hc.in_idx);
      ctx->host_copies.pop_back();
    }
    dg->h_names.resize((size_t)nb);
    dg->h_name_off.resize((size_t)n + 1);
    dg->h_topo.resize((size_t)n);
    dg->h_op.resize((size_t)n);
    dg->h_w_rank.resize((size_t)n);
    const bool host_csr = n <= SP_HOST_LAYOUT_MAX;
    dg->h_in_off.resize(host_csr ? (size_t)n + 1 : 0);
    dg->h_in_idx.resize(host_csr ? (size_t)E : 0);
    dg->h_w_train.resize(host_csr ? (size_t)n : 0);
    const double tu_alloc = ms_since(tu0);
    // the previous upload may still be reading the staging buffer
    SP_CUDA(cudaStreamSynchronize(s));
    const double tu_sync = ms_since(tu0);
    uint8_t* st = (uint8_t*)ctx->staging;
    struct Copy {
      void* dst;
      const void* src;
      size_t bytes;
    };
    std::vector<Copy> copies;
    for (const Part& p : parts)
      if (p.bytes && p.src) copies.push_back({st + p.off, p.src, p.bytes});
    copies.push_back({dg->h_names.data(), g->name_bytes, (size_t)nb});
    copies.push_back({dg->h_name_off.data(), g->name_off, (size_t)(n + 1) * 8});
    copies.push_back({dg->h_topo.data(), g->topo_rank, (size_t)n * 8});
    copies.push_back({dg->h_op.data(), g->op, (size_t)n});
    copies.push_back({dg->h_w_rank.data(), g->w_rank, (size_t)n});
    if (host_csr) {
      copies.push_back({dg->h_in_off.data(), g->in_off, (size_t)(n + 1) * 8});
      copies.push_back({dg->h_in_idx.data(), g->in_idx, (size_t)E * 4});
      copies.push_back({dg->h_w_train.data(), g->w_trainable, (size_t)n});
    }
    std::vector<size_t> cstart(copies.size() + 1, 0);
    for (size_t k = 0; k < copies.size(); k++) cstart[k + 1] = cstart[k] + copies[k].bytes;
    // byte range [lo, hi) of the concatenated copies per thread
    host_parallel((int64_t)cstart.back(), 1 << 20, [&](int64_t lo, int64_t hi, int) {
      size_t k = std::upper_bound(cstart.begin(), cstart.end(), (size_t)lo) - cstart.begin() - 1;
      for (size_t pos = (size_t)lo; pos < (size_t)hi && k < copies.size(); k++) {
        const size_t a = pos - cstart[k], b = std::min(copies[k].bytes, (size_t)hi - cstart[k]);
        if (b > a) std::memcpy((uint8_t*)copies[k].dst + a, (const uint8_t*)copies[k].src + a, b - a);
        pos = cstart[k + 1];
      }
    });
    if (pack) {
      host_parallel(n, 16384, [&](int64_t lo, int64_t hi, int) {
        int32_t* a32 = (int32_t*)(st + parts[7].off);
        int32_t* w32 = (int32_t*)(st + parts[8].off);
        uint64_t big = 0;
        for (int64_t i = lo; i < hi; i++)
          for (int k = 0; k < R; k++) {
            const uint64_t a = (uint64_t)g->act_shape[i * SP_MAX_RANK + k], w = (uint64_t)g->w_shape[i * SP_MAX_RANK + k];
            big |= (a | w) & ~(uint64_t)INT32_MAX;
            a32[i * R + k] = (int32_t)a;
            w32[i * R + k] = (int32_t)w;
          }
        // unused dims (k >= R) must be 0 by the sp_graph contract
        for (int64_t i = lo; i < hi && !big; i++)
          for (int k = R; k < SP_MAX_RANK; k++)
            big |= (uint64_t)(g->act_shape[i * SP_MAX_RANK + k] | g->w_shape[i * SP_MAX_RANK + k]);
        if (big) wide = 1;
      });
      if (wide) continue;  // a dim past int32 (or a non-zero unused dim): full layout
    }
    const double tu_copy = ms_since(tu0);
    // device arena: the staged bytes, then the expanded arrays
    const size_t exp_shape = pack ? (size_t)n * SP_MAX_RANK * 8 : 0, exp_topo = iota ? (size_t)n * 8 : 0;
    const size_t off_a = total, off_w = off_a + ((exp_shape + 255) & ~(size_t)255),
                 off_t = off_w + ((exp_shape + 255) & ~(size_t)255);
    dg->arena.alloc(off_t + exp_topo, s);
    g_h2d_bytes += (int64_t)total;
    SP_CUDA(cudaMemcpyAsync(dg->arena.p, st, total, cudaMemcpyHostToDevice, s));
    uint8_t* dbase = dg->arena.p;
    if (pack || iota) {
      SP_LAUNCH(ctx, k_expand_graph, 2 * 148, 256, 0, s, n, R,
                pack ? (const int32_t*)(dbase + parts[7].off) : nullptr,
                pack ? (const int32_t*)(dbase + parts[8].off) : nullptr, pack ? (int64_t*)(dbase + off_a) : nullptr,
                pack ? (int64_t*)(dbase + off_w) : nullptr, iota ? (int64_t*)(dbase + off_t) : nullptr);
      SP_CUDA(cudaGetLastError());
    }
    if (trace)
      std::fprintf(stderr, "[upload] check %.3f alloc %.3f sync %.3f copy %.3f issue %.3f ms (%zu B)\n", tu_check,
                   tu_alloc, tu_sync, tu_copy, ms_since(tu0), total);
    uint8_t* base = dg->arena.p;
    dg->names.p = base + parts[0].off;
    dg->name_off.p = (int64_t*)(base + parts[1].off);
    dg->topo.p = (int64_t*)(base + (iota ? off_t : parts[2].off));
    dg->op.p = base + parts[3].off;
    dg->act_rank.p = base + parts[4].off;
    dg->w_rank.p = base + parts[5].off;
    dg->w_train.p = base + parts[6].off;
    dg->act_shape.p = (int64_t*)(base + (pack ? off_a : parts[7].off));
    dg->w_shape.p = (int64_t*)(base + (pack ? off_w : parts[8].off));
    dg->act_bytes.p = (int64_t*)(base + parts[9].off);
    dg->w_bytes.p = (int64_t*)(base + parts[10].off);
    dg->in_off.p = (int64_t*)(base + parts[11].off);
    dg->in_idx.p = (int32_t*)(base + parts[12].off);
    return;
  }
}

__global__ void k_iota(int32_t* __restrict__ out, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = (int32_t)i;
}

template <class T>
__global__ void k_gather(const int32_t* __restrict__ idx, int64_t m, const T* __restrict__ src,
                         T* __restrict__ dst) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m;
       i += (int64_t)gridDim.x * blockDim.x)
    dst[i] = src[idx[i]];
}

// ---------------------------------------------------------------------------
// Device-side block assembly (accept, pruning.py:136-148) for the multi-kernel
// fold: every accepted class of a level becomes one block whose instances are
// its groups ordered by prefix string and whose template is the first of them,
// members in the template's topological order.  Siblings of one class share
// their parent prefix, so ordering the instance prefixes is ordering their
// last path components: a radix sort on (class, first 16 component bytes),
// exact unless two components of one class agree on 16 bytes (then the tie
// flag sends the whole fold to the host ordering below).


__global__ void k_acc_keys(const int32_t* __restrict__ accG, int64_t Ga, const int32_t* __restrict__ sorted,
                           const int32_t* __restrict__ gstart, const int32_t* __restrict__ gclass,
                           const int32_t* __restrict__ pend, int64_t ps, int64_t pd, int32_t dd,
                           const int64_t* __restrict__ name_off, const uint8_t* __restrict__ names,
                           uint64_t* __restrict__ k0, uint64_t* __restrict__ k1, uint32_t* __restrict__ kc,
                           uint8_t* __restrict__ longc, int32_t* __restrict__ idx) {
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < Ga; j += (int64_t)gridDim.x * blockDim.x) {
    const int32_t g = accG[j];
    const int32_t h = sorted[gstart[g]];
    const int64_t pe = pend[(int64_t)h * ps + dd * pd];
    const int64_t p0 = dd > 0 ? (int64_t)pend[(int64_t)h * ps + (dd - 1) * pd] + 1 : 0;
    const int64_t len = pe > p0 ? pe - p0 : 0;
    const uint8_t* c = names + name_off[h] + p0;
    // first 16 component bytes, big-endian, zero padded.  (A shift-accumulate
    // helper called twice, `k = k << 8 | (b < len ? p[b] : 0)`, came out of
    // nvcc 12.9 -O3 for sm_100a with stray copies of bytes 2..4 in bytes 4..6
    // for some inputs -- instance orders flipped; tools/diag_fold.py A/B.)
    uint64_t a = 0, b = 0;
    const int64_t m = len < 16 ? len : 16;
    for (int64_t q = 0; q < m; q++) {
      const uint64_t x = c[q];
      if (q < 8) a |= x << (56 - 8 * q);
      else b |= x << (120 - 8 * q);
    }
    k0[j] = a;
    k1[j] = b;
    kc[j] = (uint32_t)gclass[g];
    longc[j] = len > 16;
    idx[j] = (int32_t)j;
  }
}

template <class T>
__global__ void k_gather_idx(const int32_t* __restrict__ idx, int64_t m, const T* __restrict__ src,
                             T* __restrict__ dst) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x)
    dst[i] = src[idx[i]];
}

// class heads over the sorted accepted groups + tie detection
__global__ void k_acc_heads(const uint32_t* __restrict__ kc, const uint64_t* __restrict__ k0s,
                            const uint64_t* __restrict__ k1s, int64_t Ga, int32_t* __restrict__ head,
                            int32_t* __restrict__ tie) {
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < Ga; p += (int64_t)gridDim.x * blockDim.x) {
    const bool h = p == 0 || kc[p] != kc[p - 1];
    head[p] = h;
    if (!h && k0s[p] == k0s[p - 1] && k1s[p] == k1s[p - 1]) atomicExch(tie, 1);
  }
}

// per class: start position, R, T, template group
__global__ void k_acc_classes(const int32_t* __restrict__ head_scan, int64_t Ga, const int32_t* __restrict__ order,
                              const int32_t* __restrict__ accG, const int32_t* __restrict__ gstart, int64_t nG,
                              int64_t nA, int32_t* __restrict__ cls_start, int32_t* __restrict__ cls_R,
                              int32_t* __restrict__ cls_T) {
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < Ga; p += (int64_t)gridDim.x * blockDim.x) {
    const int32_t k = head_scan[p] - 1;
    const bool first = p == 0 || head_scan[p - 1] != head_scan[p];
    const bool last = p + 1 == Ga || head_scan[p + 1] != head_scan[p];
    if (first) {
      cls_start[k] = (int32_t)p;
      const int32_t g = accG[order[p]];
      cls_T[k] = (int32_t)((g + 1 < nG ? gstart[g + 1] : nA) - gstart[g]);
    }
    if (last) cls_R[k] = (int32_t)(p + 1);  // run end (exclusive); R = end - start in k_acc_fix
  }
}

__global__ void k_acc_fix(int64_t K, const int32_t* __restrict__ cls_start, int32_t* __restrict__ cls_R,
                          const int32_t* __restrict__ cls_T, int64_t* __restrict__ cls_RT, int64_t* __restrict__ cls_Tl) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < K; k += (int64_t)gridDim.x * blockDim.x) {
    cls_R[k] -= cls_start[k];
    cls_RT[k] = (int64_t)cls_R[k] * cls_T[k];
    cls_Tl[k] = cls_T[k];
  }
}

__device__ __forceinline__ int64_t upper_off(const int64_t* off, int64_t K, int64_t e) {
  // largest k with off[k] <= e (off exclusive scan, off[0] = 0)
  int64_t lo = 0, hi = K;
  while (hi - lo > 1) {
    const int64_t mid = (lo + hi) / 2;
    if (off[mid] <= e) lo = mid;
    else hi = mid;
  }
  return lo;
}

// canonical keys: (class, topo rank of the template group's member) -> position in group
__global__ void k_canon_keys(int64_t total, int64_t K, const int64_t* __restrict__ coff,
                             const int32_t* __restrict__ cls_start, const int32_t* __restrict__ order,
                             const int32_t* __restrict__ accG, const int32_t* __restrict__ gstart,
                             const int32_t* __restrict__ sorted, const int64_t* __restrict__ topo,
                             uint64_t* __restrict__ key, int32_t* __restrict__ val) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t k = upper_off(coff, K, e);
    const int64_t t = e - coff[k];
    const int32_t g = accG[order[cls_start[k]]];
    key[e] = ((uint64_t)k << 32) | (uint64_t)(uint32_t)topo[sorted[gstart[g] + t]];
    val[e] = (int32_t)t;
  }
}

__global__ void k_acc_members(int64_t total, int64_t K, const int64_t* __restrict__ moff,
                              const int64_t* __restrict__ coff, const int32_t* __restrict__ cls_start,
                              const int32_t* __restrict__ cls_T, const int32_t* __restrict__ order,
                              const int32_t* __restrict__ accG, const int32_t* __restrict__ gstart,
                              const int32_t* __restrict__ sorted, const int32_t* __restrict__ canon,
                              int32_t* __restrict__ members) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t k = upper_off(moff, K, e);
    const int64_t local = e - moff[k];
    const int64_t T = cls_T[k];
    const int64_t i = local / T, t = local - i * T;
    const int32_t g = accG[order[cls_start[k] + i]];
    members[e] = sorted[gstart[g] + canon[coff[k] + t]];
  }
}

__global__ void k_acc_insts(int64_t Ga, const int32_t* __restrict__ order, const int32_t* __restrict__ accG,
                            const int32_t* __restrict__ gstart, const int32_t* __restrict__ sorted,
                            const int32_t* __restrict__ pend, int64_t ps, int64_t pd, int32_t dd,
                            int32_t* __restrict__ inode, int32_t* __restrict__ ilen) {
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < Ga; p += (int64_t)gridDim.x * blockDim.x) {
    const int32_t h = sorted[gstart[accG[order[p]]]];
    inode[p] = h;
    ilen[p] = pend[(int64_t)h * ps + dd * pd];
  }
}

// Single-CTA block assembly of one level (levels with at most LS_CAP accepted
// groups, e.g. c5's 3,476): the work of level_blocks' ~25 CUB / helper
// launches and two host round trips in ONE launch -- accepted groups in id
// order (ballot scan), instance keys, a bitonic sort by (class, first 16
// component bytes), class heads + tie check, per-class start / R / T, member
// and template offsets, and the canonical (class, topological rank) order of
// the template members (when they fit, else counts[3] asks the host for the
// CUB path).  counts = {K, M, CT, too_big}.
constexpr int LS_CAP = 4096;
constexpr int64_t LS_MAX_GROUPS = 1 << 20;  // nG scanned by one CTA

struct Key4 {
  uint64_t a0, a1;
  uint32_t c;
  int32_t ix;
};

__device__ __forceinline__ bool ls_less(uint32_t ca, uint64_t a0, uint64_t a1, int32_t ia, uint32_t cb, uint64_t b0,
                                        uint64_t b1, int32_t ib) {
  if (ca != cb) return ca < cb;
  if (a0 != b0) return a0 < b0;
  if (a1 != b1) return a1 < b1;
  return ia < ib;
}

__global__ void __launch_bounds__(1024) k_level_small(
    int64_t nG, int64_t nA, const uint8_t* __restrict__ gaccept, const int32_t* __restrict__ sorted,
    const int32_t* __restrict__ gstart, const int32_t* __restrict__ gclass, const int32_t* __restrict__ pend,
    int64_t ps, int64_t pd, int32_t dd, const int64_t* __restrict__ name_off, const uint8_t* __restrict__ names,
    const int64_t* __restrict__ topo, int32_t* __restrict__ tie, int32_t* __restrict__ accG_o,
    int32_t* __restrict__ order_o, int32_t* __restrict__ cls_start, int32_t* __restrict__ cls_R,
    int32_t* __restrict__ cls_T, int64_t* __restrict__ moff, int64_t* __restrict__ coff, int32_t* __restrict__ canon,
    int64_t* __restrict__ counts) {
  extern __shared__ __align__(16) uint8_t sm[];
  __shared__ int32_t s_warp[32];
  uint64_t* K0 = (uint64_t*)sm;
  uint64_t* K1 = K0 + LS_CAP;
  uint32_t* KC = (uint32_t*)(K1 + LS_CAP);
  int32_t* IX = (int32_t*)(KC + LS_CAP);
  int32_t* ACC = IX + LS_CAP;
  int32_t* HD = ACC + LS_CAP;
  const int tid = threadIdx.x, NT = blockDim.x, lane = tid & 31, w = tid >> 5, NW = NT >> 5;
  // 1. accepted groups in group-id order
  int base = 0;
  for (int64_t g0 = 0; g0 < nG; g0 += NT) {
    const int64_t g = g0 + tid;
    const bool f = g < nG && gaccept[g];
    const unsigned bal = __ballot_sync(0xffffffffu, f);
    if (lane == 0) s_warp[w] = __popc(bal);
    __syncthreads();
    if (w == 0) {
      int v = lane < NW ? s_warp[lane] : 0;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v += y;
      }
      s_warp[lane] = v;
    }
    __syncthreads();
    const int pos = base + (w ? s_warp[w - 1] : 0) + __popc(bal & ((1u << lane) - 1u));
    if (f && pos < LS_CAP) ACC[pos] = (int32_t)g;
    base += s_warp[NW - 1];
    __syncthreads();
  }
  const int Ga = base;
  if (Ga > LS_CAP) {  // the host bounds Ga by the level's accepted count: cannot happen
    if (tid == 0) counts[3] = 1;
    return;
  }
  // 2. instance keys: class, first 16 bytes of the last component (big-endian)
  const int P2 = pow2ceil(Ga > 0 ? Ga : 1);
  for (int j = tid; j < P2; j += NT) {
    if (j < Ga) {
      const int32_t g = ACC[j];
      const int32_t h = sorted[gstart[g]];
      const int64_t pe = pend[(int64_t)h * ps + dd * pd];
      const int64_t p0 = dd > 0 ? (int64_t)pend[(int64_t)h * ps + (dd - 1) * pd] + 1 : 0;
      const int64_t len = pe > p0 ? pe - p0 : 0;
      const uint8_t* c = names + name_off[h] + p0;
      uint64_t a = 0, b = 0;
      const int64_t m = len < 16 ? len : 16;
      for (int64_t q = 0; q < m; q++) {
        const uint64_t x = c[q];
        if (q < 8) a |= x << (56 - 8 * q);
        else b |= x << (120 - 8 * q);
      }
      K0[j] = a;
      K1[j] = b;
      KC[j] = (uint32_t)gclass[g];
      IX[j] = j;
    } else {
      K0[j] = K1[j] = ~0ULL;
      KC[j] = 0xffffffffu;
      IX[j] = 0x7fffffff;
    }
  }
  __syncthreads();
  // 3. bitonic sort by (class, k0, k1, j)
  if (P2 >= 64) {
    bitonic_sort_reg<Key4>(
        P2, [&](int i) { return Key4{K0[i], K1[i], KC[i], IX[i]}; },
        [&](int i, const Key4& x) {
          KC[i] = x.c;
          K0[i] = x.a0;
          K1[i] = x.a1;
          IX[i] = x.ix;
        },
        [](const Key4& x, const Key4& y) { return ls_less(x.c, x.a0, x.a1, x.ix, y.c, y.a0, y.a1, y.ix); },
        [](const Key4& x, int m) {
          return Key4{__shfl_xor_sync(0xffffffffu, x.a0, m), __shfl_xor_sync(0xffffffffu, x.a1, m),
                      __shfl_xor_sync(0xffffffffu, x.c, m), __shfl_xor_sync(0xffffffffu, x.ix, m)};
        });
  } else {
  for (int size = 2; size <= P2; size <<= 1)
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      for (int t = tid; t < (P2 >> 1); t += NT) {
        const int i = ((t & ~(stride - 1)) << 1) | (t & (stride - 1));
        const int j = i + stride;
        const bool gt = ls_less(KC[j], K0[j], K1[j], IX[j], KC[i], K0[i], K1[i], IX[i]);
        if (gt == ((i & size) == 0)) {
          const uint32_t c0 = KC[i];
          const uint64_t a = K0[i], b = K1[i];
          const int32_t x = IX[i];
          KC[i] = KC[j]; K0[i] = K0[j]; K1[i] = K1[j]; IX[i] = IX[j];
          KC[j] = c0; K0[j] = a; K1[j] = b; IX[j] = x;
        }
      }
      __syncthreads();
    }
  }
  // 4. class heads, tie check (two instance components of a class equal on 16 bytes)
  for (int p = tid; p < Ga; p += NT) {
    const bool hd = p == 0 || KC[p] != KC[p - 1];
    HD[p] = hd;
    if (!hd && K0[p] == K0[p - 1] && K1[p] == K1[p - 1]) atomicExch(tie, 1);
    accG_o[p] = ACC[p];
    order_o[p] = IX[p];
  }
  __syncthreads();
  const int K = block_inclusive_scan(HD, Ga, s_warp);
  // 5. per class: start, R, T
  for (int p = tid; p < Ga; p += NT) {
    const int32_t k = HD[p] - 1;
    if (p == 0 || HD[p - 1] != HD[p]) {
      cls_start[k] = p;
      const int32_t g = ACC[IX[p]];
      cls_T[k] = (int32_t)((g + 1 < nG ? gstart[g + 1] : nA) - gstart[g]);
    }
    if (p + 1 == Ga || HD[p + 1] != HD[p]) cls_R[k] = p + 1;
  }
  __syncthreads();
  // member / template offsets (exclusive scans; KC / HD reused)
  for (int k = tid; k < K; k += NT) {
    cls_R[k] -= cls_start[k];
    KC[k] = (uint32_t)(cls_R[k] * cls_T[k]);
    HD[k] = cls_T[k];
  }
  __syncthreads();
  const int M = block_inclusive_scan((int32_t*)KC, K, s_warp);
  const int CT = block_inclusive_scan(HD, K, s_warp);
  for (int k = tid; k < K; k += NT) {
    moff[k] = (int64_t)KC[k] - (int64_t)cls_R[k] * cls_T[k];
    coff[k] = (int64_t)HD[k] - cls_T[k];
  }
  if (tid == 0) {
    moff[K] = M;
    coff[K] = CT;
    counts[0] = K;
    counts[1] = M;
    counts[2] = CT;
    counts[3] = CT > LS_CAP;
  }
  __syncthreads();
  if (CT > LS_CAP) return;
  // 6. canonical order of every class's template members: sort (class, topo rank)
  const int P2c = pow2ceil(CT > 0 ? CT : 1);
  for (int e = tid; e < P2c; e += NT) {
    if (e < CT) {
      int lo = 0, hi = K;  // largest k with coff[k] <= e
      while (hi - lo > 1) {
        const int mid = (lo + hi) >> 1;
        if (coff[mid] <= e) lo = mid;
        else hi = mid;
      }
      const int t = e - (int)coff[lo];
      const int32_t g = ACC[IX[cls_start[lo]]];
      K0[e] = ((uint64_t)lo << 32) | (uint64_t)(uint32_t)topo[sorted[gstart[g] + t]];
      K1[e] = 0;
      HD[e] = t;
    } else {
      K0[e] = K1[e] = ~0ULL;
      HD[e] = 0x7fffffff;
    }
  }
  __syncthreads();
  block_sort(K0, K1, HD, CT, P2c);
  for (int e = tid; e < CT; e += NT) canon[e] = HD[e];
}

// One level's blocks, still on the device (downloaded once after the loop).
struct LevelBlocks {
  int64_t K = 0, Ga = 0, M = 0;
  DevBuf<int32_t> cls_T, cls_R, cls_start, inode, ilen, members;
};

// SP_FOLD_TRACE=1: host-side phase times of the multi-kernel fold on stderr
struct FoldTrace {
  bool on = getenv("SP_FOLD_TRACE") != nullptr;
  std::chrono::steady_clock::time_point t0 = std::chrono::steady_clock::now(), last = t0;
  void mark(const char* what) {
    if (!on) return;
    const auto now = std::chrono::steady_clock::now();
    fprintf(stderr, "[fold] %-28s %9.3f ms (total %9.3f)\n", what,
            std::chrono::duration<double, std::milli>(now - last).count(),
            std::chrono::duration<double, std::milli>(now - t0).count());
    last = now;
  }
};

template <class T>
static T d2h_scalar(const T* p, cudaStream_t s) {
  T v{};
  g_d2h_bytes += (int64_t)sizeof(T);
  SP_CUDA(cudaMemcpyAsync(&v, p, sizeof(T), cudaMemcpyDeviceToHost, s));
  SP_CUDA(cudaStreamSynchronize(s));
  return v;
}

// Accepted classes of one level -> blocks (device arrays); sets *tie when two
// instance components of one class agree on their first 16 bytes.
// pend of (node h, depth d) at h*ps + d*pd (node- or level-major, see name_hash_one).
static void level_blocks(sp_ctx* ctx, sp_dgraph* dg, int32_t dd, int64_t nA, int64_t nG, const int32_t* sorted,
                         const int32_t* gstart, const int32_t* gclass, const uint8_t* gaccept, const int32_t* pend,
                         int64_t ps, int64_t pd, int32_t* d_tie, LevelBlocks& L, int64_t nacc = -1) {
  cudaStream_t s = ctx->stream;
  const int sms = ctx->sm_count;
  if (nacc >= 0 && nacc <= LS_CAP && nG <= LS_MAX_GROUPS && !getenv("SP_FOLD_LEVEL_CUB")) {
    // one CTA assembles the level; one host round trip for the counts
    const int64_t Ga = nacc;
    DevBuf<int32_t> accG, order, canon;
    DevBuf<int64_t> offs;  // moff [Ga+1] | coff [Ga+1] | counts [4]
    accG.alloc(std::max<int64_t>(Ga, 1), s);
    order.alloc(std::max<int64_t>(Ga, 1), s);
    canon.alloc(LS_CAP, s);
    offs.alloc(2 * (Ga + 1) + 4, s);
    L.cls_T.alloc(std::max<int64_t>(Ga, 1), s);
    L.cls_R.alloc(std::max<int64_t>(Ga, 1), s);
    L.cls_start.alloc(std::max<int64_t>(Ga, 1), s);
    int64_t* moff = offs.p;
    int64_t* coff = offs.p + Ga + 1;
    int64_t* dcnt = offs.p + 2 * (Ga + 1);
    const size_t smem = (size_t)LS_CAP * 32;
    allow_smem(ctx, k_level_small, smem);
    SP_LAUNCH(ctx, k_level_small, 1, 1024, smem, s, nG, nA, gaccept, sorted, gstart, gclass, pend, ps, pd, dd,
              dg->name_off.p, dg->names.p, dg->topo.p, d_tie, accG.p, order.p, L.cls_start.p, L.cls_R.p, L.cls_T.p,
              moff, coff, canon.p, dcnt);
    int64_t cnt[4];
    g_d2h_bytes += sizeof(cnt);
    SP_CUDA(cudaMemcpyAsync(cnt, dcnt, sizeof(cnt), cudaMemcpyDeviceToHost, s));
    SP_CUDA(cudaStreamSynchronize(s));
    if (!cnt[3]) {
      const int64_t K = cnt[0], M = cnt[1];
      L.Ga = Ga;
      L.K = K;
      L.M = M;
      L.members.alloc(std::max<int64_t>(M, 1), s);
      L.inode.alloc(std::max<int64_t>(Ga, 1), s);
      L.ilen.alloc(std::max<int64_t>(Ga, 1), s);
      if (M)
        SP_LAUNCH(ctx, k_acc_members, grid_for(M, sms), 256, 0, s, M, K, moff, coff, L.cls_start.p, L.cls_T.p,
                  order.p, accG.p, gstart, sorted, canon.p, L.members.p);
      if (Ga)
        SP_LAUNCH(ctx, k_acc_insts, grid_for(Ga, sms), 256, 0, s, Ga, order.p, accG.p, gstart, sorted, pend, ps, pd,
                  dd, L.inode.p, L.ilen.p);
      return;
    }
    // templates too large for the one-CTA canonical sort: the CUB path below
  }
  DevBuf<int32_t> iota, accG, nsel;
  iota.alloc(nG, s);
  accG.alloc(nG, s);
  nsel.alloc(1, s);
  SP_LAUNCH(ctx, k_iota, grid_for(nG, sms), 256, 0, s, iota.p, nG);
  DevBuf<uint8_t> tmp;
  size_t tb = 0;
  ctx->cub_calls++;
  SP_CUDA(cub::DeviceSelect::Flagged(nullptr, tb, iota.p, gaccept, accG.p, nsel.p, (int)nG, s));
  tmp.alloc(tb, s);
  SP_CUDA(cub::DeviceSelect::Flagged(tmp.p, tb, iota.p, gaccept, accG.p, nsel.p, (int)nG, s));
  const int64_t Ga = d2h_scalar(nsel.p, s);
  L.Ga = Ga;
  if (Ga == 0) return;
  DevBuf<uint64_t> k0, k1, k0s, k1s, t64;
  DevBuf<uint32_t> kc, kcs, t32;
  DevBuf<uint8_t> longc;
  DevBuf<int32_t> idx, o1, o2;
  k0.alloc(Ga, s); k1.alloc(Ga, s); k0s.alloc(Ga, s); k1s.alloc(Ga, s); t64.alloc(Ga, s);
  kc.alloc(Ga, s); kcs.alloc(Ga, s); t32.alloc(Ga, s);
  longc.alloc(Ga, s);
  idx.alloc(Ga, s); o1.alloc(Ga, s); o2.alloc(Ga, s);
  const int gA = grid_for(Ga, sms);
  SP_LAUNCH(ctx, k_acc_keys, gA, 256, 0, s, accG.p, Ga, sorted, gstart, gclass, pend, ps, pd, dd, dg->name_off.p,
            dg->names.p, k0.p, k1.p, kc.p, longc.p, idx.p);
  // LSD: component bytes 8..15, then 0..7, then class (stable)
  auto sort_pairs = [&](auto* kin, auto* kout, const int32_t* vin, int32_t* vout, int bits) {
    size_t b = 0;
    ctx->cub_calls++;
    SP_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, b, kin, kout, vin, vout, (int)Ga, 0, bits, s));
    if (b > tmp.n) tmp.alloc(b, s);
    b = tmp.n;
    SP_CUDA(cub::DeviceRadixSort::SortPairs(tmp.p, b, kin, kout, vin, vout, (int)Ga, 0, bits, s));
  };
  sort_pairs(k1.p, k1s.p, idx.p, o1.p, 64);
  SP_LAUNCH(ctx, k_gather_idx<uint64_t>, gA, 256, 0, s, o1.p, Ga, k0.p, t64.p);
  sort_pairs(t64.p, k0s.p, o1.p, o2.p, 64);
  SP_LAUNCH(ctx, k_gather_idx<uint32_t>, gA, 256, 0, s, o2.p, Ga, kc.p, t32.p);
  sort_pairs(t32.p, kcs.p, o2.p, o1.p, 32);
  int32_t* order = o1.p;  // sorted position -> index into accG
  // keys in final order for the tie check
  SP_LAUNCH(ctx, k_gather_idx<uint64_t>, gA, 256, 0, s, order, Ga, k0.p, k0s.p);
  SP_LAUNCH(ctx, k_gather_idx<uint64_t>, gA, 256, 0, s, order, Ga, k1.p, k1s.p);
  DevBuf<int32_t> head;
  head.alloc(Ga, s);
  SP_LAUNCH(ctx, k_acc_heads, gA, 256, 0, s, kcs.p, k0s.p, k1s.p, Ga, head.p, d_tie);
  {
    size_t b = 0;
    ctx->cub_calls++;
    SP_CUDA(cub::DeviceScan::InclusiveSum(nullptr, b, head.p, head.p, (int)Ga, s));
    if (b > tmp.n) tmp.alloc(b, s);
    b = tmp.n;
    SP_CUDA(cub::DeviceScan::InclusiveSum(tmp.p, b, head.p, head.p, (int)Ga, s));
  }
  const int64_t K = d2h_scalar(head.p + Ga - 1, s);
  L.K = K;
  L.cls_T.alloc(K, s);
  L.cls_R.alloc(K, s);
  L.cls_start.alloc(K, s);
  DevBuf<int64_t> moff, coff;
  moff.alloc(K + 1, s);
  coff.alloc(K + 1, s);
  SP_LAUNCH(ctx, k_acc_classes, gA, 256, 0, s, head.p, Ga, order, accG.p, gstart, nG, nA, L.cls_start.p, L.cls_R.p,
            L.cls_T.p);
  SP_CUDA(cudaMemsetAsync(moff.p + K, 0, sizeof(int64_t), s));
  SP_CUDA(cudaMemsetAsync(coff.p + K, 0, sizeof(int64_t), s));
  SP_LAUNCH(ctx, k_acc_fix, grid_for(K, sms), 256, 0, s, K, L.cls_start.p, L.cls_R.p, L.cls_T.p, moff.p, coff.p);
  for (DevBuf<int64_t>* o : {&moff, &coff}) {
    size_t b = 0;
    ctx->cub_calls++;
    SP_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, b, o->p, o->p, (int)(K + 1), s));
    if (b > tmp.n) tmp.alloc(b, s);
    b = tmp.n;
    SP_CUDA(cub::DeviceScan::ExclusiveSum(tmp.p, b, o->p, o->p, (int)(K + 1), s));
  }
  int64_t tot[2];
  g_d2h_bytes += 16;
  SP_CUDA(cudaMemcpyAsync(&tot[0], moff.p + K, 8, cudaMemcpyDeviceToHost, s));
  SP_CUDA(cudaMemcpyAsync(&tot[1], coff.p + K, 8, cudaMemcpyDeviceToHost, s));
  SP_CUDA(cudaStreamSynchronize(s));
  const int64_t M = tot[0], CT = tot[1];
  L.M = M;
  // canonical order of the template members: sort (class, topo rank)
  DevBuf<uint64_t> ck, cks;
  DevBuf<int32_t> cv, canon;
  ck.alloc(CT, s); cks.alloc(CT, s); cv.alloc(CT, s); canon.alloc(CT, s);
  SP_LAUNCH(ctx, k_canon_keys, grid_for(CT, sms), 256, 0, s, CT, K, coff.p, L.cls_start.p, order, accG.p, gstart,
            sorted, dg->topo.p, ck.p, cv.p);
  {
    size_t b = 0;
    ctx->cub_calls++;
    SP_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, b, ck.p, cks.p, cv.p, canon.p, (int)CT, 0, 64, s));
    if (b > tmp.n) tmp.alloc(b, s);
    b = tmp.n;
    SP_CUDA(cub::DeviceRadixSort::SortPairs(tmp.p, b, ck.p, cks.p, cv.p, canon.p, (int)CT, 0, 64, s));
  }
  L.members.alloc(M, s);
  L.inode.alloc(Ga, s);
  L.ilen.alloc(Ga, s);
  SP_LAUNCH(ctx, k_acc_members, grid_for(M, sms), 256, 0, s, M, K, moff.p, coff.p, L.cls_start.p, L.cls_T.p, order,
            accG.p, gstart, sorted, canon.p, L.members.p);
  SP_LAUNCH(ctx, k_acc_insts, gA, 256, 0, s, Ga, order, accG.p, gstart, sorted, pend, ps, pd, dd, L.inode.p, L.ilen.p);
}

// Host ordering: the string-order decisions of pruning.py:136-148, 200 over
// the device partition (instances and blocks by prefix string, template by
// topological rank).  O(accepted groups log) string compares.
static void fold_finalize(sp_dgraph* dg, const std::vector<LevelOut>& levels, const std::vector<uint8_t>& resid_h,
                          const std::vector<int32_t>& pend_h, int32_t D, sp_fold* out) {
  const int64_t n = dg->n;
  const uint8_t* names = dg->h_names.data();
  const int64_t* noff = dg->h_name_off.data();
  const int64_t* topo = dg->h_topo.data();
  struct Block {
    int64_t pnode, plen;
    std::vector<int64_t> inst_node, inst_len;
    std::vector<int32_t> members;  // instance-major
    int64_t T;
  };
  std::vector<Block> blocks;
  for (const LevelOut& lv : levels) {
    const int64_t dd = lv.level - 1;
    const int64_t nC = (int64_t)lv.cstart.size() - 1;
    for (int64_t c = 0; c < nC; c++) {
      const int32_t g0 = lv.corder[lv.cstart[c]];
      if (!lv.gaccept[g0]) continue;
      std::vector<int32_t> gs(lv.corder.begin() + lv.cstart[c], lv.corder.begin() + lv.cstart[c + 1]);
      auto gprefix = [&](int32_t g, int64_t* node, int64_t* len) {
        *node = lv.sorted[lv.gstart[g]];
        *len = pend_h[(size_t)(*node) * D + dd];
      };
      std::sort(gs.begin(), gs.end(), [&](int32_t a, int32_t b) {
        int64_t na, la, nb, lb;
        gprefix(a, &na, &la);
        gprefix(b, &nb, &lb);
        return strcmp_py(names + noff[na], la, names + noff[nb], lb) < 0;
      });
      const int32_t tg = gs[0];
      const int64_t T = lv.gstart[tg + 1] - lv.gstart[tg];
      std::vector<int32_t> canon(T);  // template position -> canonical position
      std::iota(canon.begin(), canon.end(), 0);
      std::sort(canon.begin(), canon.end(), [&](int32_t a, int32_t b) {
        return topo[lv.sorted[lv.gstart[tg] + a]] < topo[lv.sorted[lv.gstart[tg] + b]];
      });
      Block B;
      gprefix(tg, &B.pnode, &B.plen);
      B.T = T;
      for (int32_t g : gs) {
        int64_t pn, pl;
        gprefix(g, &pn, &pl);
        B.inst_node.push_back(pn);
        B.inst_len.push_back(pl);
        for (int64_t tpos = 0; tpos < T; tpos++) B.members.push_back(lv.sorted[lv.gstart[g] + canon[tpos]]);
      }
      blocks.push_back(std::move(B));
    }
  }
  for (int64_t i = 0; i < n; i++) {
    if (!resid_h[i]) continue;
    Block B;
    B.pnode = i;
    B.plen = noff[i + 1] - noff[i];
    B.T = 1;
    B.inst_node.push_back(i);
    B.inst_len.push_back(B.plen);
    B.members.push_back((int32_t)i);
    blocks.push_back(std::move(B));
  }
  std::vector<int64_t> order(blocks.size());
  std::iota(order.begin(), order.end(), 0);
  std::sort(order.begin(), order.end(), [&](int64_t a, int64_t b) {
    const Block& A = blocks[a];
    const Block& Bb = blocks[b];
    return strcmp_py(names + noff[A.pnode], A.plen, names + noff[Bb.pnode], Bb.plen) < 0;
  });
  out->block_T.clear();
  out->block_inst_off.assign(1, 0);
  out->block_member_off.assign(1, 0);
  out->inst_prefix_node.clear();
  out->inst_prefix_len.clear();
  out->members.clear();
  for (int64_t bi : order) {
    const Block& B = blocks[bi];
    out->block_T.push_back(B.T);
    out->inst_prefix_node.insert(out->inst_prefix_node.end(), B.inst_node.begin(), B.inst_node.end());
    out->inst_prefix_len.insert(out->inst_prefix_len.end(), B.inst_len.begin(), B.inst_len.end());
    out->members.insert(out->members.end(), B.members.begin(), B.members.end());
    out->block_inst_off.push_back((int64_t)out->inst_prefix_node.size());
    out->block_member_off.push_back((int64_t)out->members.size());
  }
  if ((int64_t)out->members.size() != n) throw Error(SP_ERR_CUDA, "fold did not cover every node exactly once");
  sp_blocks& v = out->view;
  v.n_blocks = (int64_t)out->block_T.size();
  v.n_instances = (int64_t)out->inst_prefix_node.size();
  v.n_members = (int64_t)out->members.size();
  v.block_T = out->block_T.data();
  v.block_inst_off = out->block_inst_off.data();
  v.block_member_off = out->block_member_off.data();
  v.inst_prefix_node = out->inst_prefix_node.data();
  v.inst_prefix_len = out->inst_prefix_len.data();
  v.members = out->members.data();
}

// Blocks from the device-side assembly: download each level's blocks and the
// residual singletons, order all blocks by template prefix string
// (pruning.py:200) and concatenate.  Host work is O(blocks log blocks) string
// compares plus one pass over the members.
// With d_rlist, the residual list (d_nr entries) comes from the device in the
// same copy, and with d_flags the fold's collision / tie words too (h_flags;
// when either is set nothing is finalised): one host round trip in all.
static void fold_finalize_blocks(sp_dgraph* dg, std::vector<LevelBlocks>& lv, const std::vector<int32_t>& resid_in,
                                 cudaStream_t s, sp_fold* out, const int32_t* d_rlist = nullptr, int64_t d_nr = 0,
                                 const int32_t* d_coll = nullptr, const int32_t* d_tie = nullptr,
                                 int32_t* h_flags = nullptr) {
  const uint8_t* names = dg->h_names.data();
  const int64_t* noff = dg->h_name_off.data();
  std::vector<int32_t> resid_from_device;
  const std::vector<int32_t>& resid = d_rlist ? resid_from_device : resid_in;
  // every level's class arrays to ONE pinned block (10^7-node folds move
  // ~50 MB here: pageable copies and zero-filled vectors cost 30+ ms)
  struct Host {
    const int32_t *T, *R, *start, *inode, *ilen, *members;
    int64_t K = 0;
    std::vector<int64_t> moff;
  };
  std::vector<Host> h(lv.size());
  size_t total = 16 + (size_t)(d_rlist ? d_nr : 0) * 4;
  for (const LevelBlocks& L : lv) total += (size_t)(3 * L.K + 2 * L.Ga + L.M) * 4;
  size_t got = 0;
  uint8_t* pin = total ? sp::pinned_acquire(dg->ctx, total, &got) : nullptr;
  struct Release {
    sp_ctx* ctx;
    uint8_t* p;
    size_t n;
    ~Release() { sp::pinned_release(ctx, p, n); }
  } rel{dg->ctx, pin, got};
  {
    int32_t* q = (int32_t*)pin;
    auto get = [&](const DevBuf<int32_t>& d, int64_t cnt) {
      int32_t* at = q;
      if (cnt) SP_CUDA(cudaMemcpyAsync(at, d.p, (size_t)cnt * 4, cudaMemcpyDeviceToHost, s));
      g_d2h_bytes += cnt * 4;
      q += cnt;
      return (const int32_t*)at;
    };
    int32_t* flags_at = q;
    q += 4;
    if (d_coll) SP_CUDA(cudaMemcpyAsync(flags_at, d_coll, 4, cudaMemcpyDeviceToHost, s));
    if (d_tie) SP_CUDA(cudaMemcpyAsync(flags_at + 1, d_tie, 4, cudaMemcpyDeviceToHost, s));
    for (size_t l = 0; l < lv.size(); l++) {
      LevelBlocks& L = lv[l];
      Host& H = h[l];
      H.K = L.K;
      if (!L.K) continue;
      H.T = get(L.cls_T, L.K);
      H.R = get(L.cls_R, L.K);
      H.start = get(L.cls_start, L.K);
      H.inode = get(L.inode, L.Ga);
      H.ilen = get(L.ilen, L.Ga);
      H.members = get(L.members, L.M);
    }
    const int32_t* rl = q;
    if (d_rlist && d_nr) {
      SP_CUDA(cudaMemcpyAsync(q, d_rlist, (size_t)d_nr * 4, cudaMemcpyDeviceToHost, s));
      g_d2h_bytes += d_nr * 4;
    }
    SP_CUDA(cudaStreamSynchronize(s));
    if (h_flags) {
      h_flags[0] = d_coll ? flags_at[0] : 0;
      h_flags[1] = d_tie ? flags_at[1] : 0;
      if (h_flags[0] || h_flags[1]) return;
    }
    if (d_rlist) resid_from_device.assign(rl, rl + d_nr);
  }
  struct Ref {
    int64_t pnode, plen;
    int32_t level;  // -1: residual singleton
    int32_t k;      // class (or residual node)
  };
  std::vector<Ref> blocks;
  for (size_t l = 0; l < lv.size(); l++) {
    Host& H = h[l];
    H.moff.assign(H.K + 1, 0);
    for (int64_t k = 0; k < H.K; k++) {
      H.moff[k + 1] = H.moff[k] + (int64_t)H.R[k] * H.T[k];
      const int32_t p0 = H.start[k];
      blocks.push_back({H.inode[p0], H.ilen[p0], (int32_t)l, (int32_t)k});
    }
  }
  for (int32_t v : resid) blocks.push_back({v, noff[v + 1] - noff[v], -1, v});
  std::sort(blocks.begin(), blocks.end(), [&](const Ref& a, const Ref& b) {
    return strcmp_py(names + noff[a.pnode], a.plen, names + noff[b.pnode], b.plen) < 0;
  });
  const int64_t nb = (int64_t)blocks.size();
  out->block_T.resize(nb);
  out->block_inst_off.assign(nb + 1, 0);
  out->block_member_off.assign(nb + 1, 0);
  for (int64_t b = 0; b < nb; b++) {
    const Ref& r = blocks[b];
    const int64_t T = r.level < 0 ? 1 : h[r.level].T[r.k];
    const int64_t R = r.level < 0 ? 1 : h[r.level].R[r.k];
    out->block_T[b] = T;
    out->block_inst_off[b + 1] = out->block_inst_off[b] + R;
    out->block_member_off[b + 1] = out->block_member_off[b] + R * T;
  }
  if (out->block_member_off[nb] != dg->n) throw Error(SP_ERR_CUDA, "fold did not cover every node exactly once");
  const int64_t ni = out->block_inst_off[nb];
  out->inst_prefix_node.resize(ni);
  out->inst_prefix_len.resize(ni);
  out->members.resize(dg->n);
  // members: one contiguous segment per class; instances widened to int64.
  // Both split over host threads by element ranges of the output.
  host_parallel(ni, 1 << 16, [&](int64_t lo, int64_t hi, int) {
    int64_t b = std::upper_bound(out->block_inst_off.begin(), out->block_inst_off.end(), lo) -
                out->block_inst_off.begin() - 1;
    for (int64_t j = lo; j < hi; b++) {
      const Ref& r = blocks[b];
      const int64_t io = out->block_inst_off[b], e = std::min(hi, out->block_inst_off[b + 1]);
      if (r.level < 0) {
        out->inst_prefix_node[j] = r.pnode;
        out->inst_prefix_len[j] = r.plen;
      } else {
        const Host& H = h[r.level];
        const int64_t p0 = H.start[r.k];
        for (int64_t i = j; i < e; i++) {
          out->inst_prefix_node[i] = H.inode[p0 + (i - io)];
          out->inst_prefix_len[i] = H.ilen[p0 + (i - io)];
        }
      }
      j = e;
    }
  });
  host_parallel(dg->n, 1 << 18, [&](int64_t lo, int64_t hi, int) {
    int64_t b = std::upper_bound(out->block_member_off.begin(), out->block_member_off.end(), lo) -
                out->block_member_off.begin() - 1;
    for (int64_t j = lo; j < hi; b++) {
      const Ref& r = blocks[b];
      const int64_t mo = out->block_member_off[b], e = std::min(hi, out->block_member_off[b + 1]);
      if (r.level < 0) {
        out->members[j] = r.k;
      } else {
        const Host& H = h[r.level];
        std::memcpy(out->members.data() + j, H.members + H.moff[r.k] + (j - mo), sizeof(int32_t) * (size_t)(e - j));
      }
      j = e;
    }
  });
  sp_blocks& v = out->view;
  v.n_blocks = nb;
  v.n_instances = (int64_t)out->inst_prefix_node.size();
  v.n_members = (int64_t)out->members.size();
  v.block_T = out->block_T.data();
  v.block_inst_off = out->block_inst_off.data();
  v.block_member_off = out->block_member_off.data();
  v.inst_prefix_node = out->inst_prefix_node.data();
  v.inst_prefix_len = out->inst_prefix_len.data();
  v.members = out->members.data();
}

// One launch + one device->host copy for graphs of <= SMALL_MAX nodes.
static void fold_once_small(sp_ctx* ctx, sp_dgraph* dg, int32_t min_dup, uint64_t seed, sp_fold* out,
                            bool* collided) {
  cudaStream_t s = ctx->stream;
  Trace tr("fold_small");
  const int64_t n = dg->n;
  const int32_t D = dg->max_depth;
  // one arena for scratch + outputs
  const size_t nd = (size_t)n * D, nd1 = (size_t)(n + 1) * D;
  DevBuf<int32_t> i32;
  DevBuf<uint64_t> u64;
  // i32: depth pos gparent gclass act flag cid | sorted gstart corder cstart info collision pend |
  // then (bytes) gaccept residual next_flag: everything the host reads is one
  // contiguous range (one D2H)
  const size_t i32_scratch = 7 * (size_t)n;
  const size_t i32_out = nd + nd1 + nd + nd1 + (size_t)(4 * D + 4) + 1 + nd;
  const size_t u8_words = (nd + 2 * (size_t)n + 3) / 4;
  i32.alloc(i32_scratch + i32_out + u8_words, s);
  u64.alloc(2 * nd + 2 * (size_t)n, s);  // ph rh cur gkey
  SmallArgs A;
  A.name_off = dg->name_off.p;
  A.names = dg->names.p;
  A.op = dg->op.p;
  A.w_rank = dg->w_rank.p;
  A.w_shape = dg->w_shape.p;
  A.w_train = dg->w_train.p;
  A.in_off = dg->in_off.p;
  A.in_idx = dg->in_idx.p;
  A.n = n;
  A.D = D;
  A.min_dup = min_dup;
  A.seed = seed;
  int32_t* p = i32.p;
  A.depth = p; p += n;
  A.pos = p; p += n;
  A.gparent = p; p += n;
  A.gclass = p; p += n;
  A.act = p; p += n;
  A.flag = p; p += n;
  A.cid = p; p += n;
  int32_t* out0 = p;
  A.sorted = p; p += nd;
  A.gstart = p; p += nd1;
  A.corder = p; p += nd;
  A.cstart = p; p += nd1;
  A.info = p; p += 4 * D + 4;
  A.collision = p; p += 1;
  A.pend = p; p += nd;
  uint8_t* u8p = (uint8_t*)p;
  A.ph = u64.p;
  A.rh = u64.p + nd;
  A.cur = (int64_t*)(u64.p + 2 * nd);
  A.gkey = (unsigned long long*)(u64.p + 2 * nd + n);
  A.gaccept = u8p;
  A.residual = u8p + nd;
  A.next_flag = u8p + nd + n;
  SP_CUDA(cudaMemsetAsync(A.collision, 0, sizeof(int32_t), s));
  const int P2 = [&] { int q = 1; while (q < n) q <<= 1; return q; }();
  // stage the per-node scratch and the graph arrays in shared memory when they fit
  A.name_bytes = dg->h_name_off[n];
  A.n_edges = dg->E;
  size_t smem = 0;
  auto take = [&](size_t bytes) {
    const int32_t o = (int32_t)smem;
    smem += (bytes + 15) & ~(size_t)15;
    return o;
  };
  take((size_t)P2 * 20);
  const size_t base = smem;
  A.o_depth = take((size_t)n * 4);
  A.o_pos = take((size_t)n * 4);
  A.o_gparent = take((size_t)n * 4);
  A.o_gclass = take((size_t)n * 4);
  A.o_act = take((size_t)n * 4);
  A.o_flag = take((size_t)n * 4);
  A.o_cid = take((size_t)n * 4);
  A.o_ph = take((size_t)n * D * 8);
  A.o_rh = take((size_t)n * D * 8);
  A.o_cur = take((size_t)n * 8);
  A.o_gkey = take((size_t)n * 8);
  A.o_next = take((size_t)n);
  A.o_name_off = take((size_t)(n + 1) * 8);
  A.o_names = take((size_t)A.name_bytes);
  A.o_op = take((size_t)n);
  A.o_w_rank = take((size_t)n);
  A.o_w_train = take((size_t)n);
  A.o_w_shape = take((size_t)n * SP_MAX_RANK * 8);
  A.o_in_off = take((size_t)(n + 1) * 8);
  A.o_in_idx = take((size_t)A.n_edges * 4);
  const bool stage = smem <= std::min<size_t>(ctx->smem_optin, 200 << 10) && !getenv("SP_FOLD_NOSTAGE");
  if (!stage) smem = base;
  auto kern = stage ? k_fold_small<true> : k_fold_small<false>;
  allow_smem(ctx, kern, smem);
  SP_CUDA(cudaEventRecord(ctx->ev[6], s));
  // one thread per node (rank-counting sorts, one node per thread in the
  // per-node passes), or one per bitonic compare-exchange beyond 1024 nodes
  const int threads = n <= RANK_SORT_MAX ? std::max(64, (int)((n + 31) / 32 * 32)) : std::min(SMALL_THREADS, P2 / 2);
  tr.mark("setup");
  {  // name hashes: computed by the graph's first search at this seed, then read
    const bool hit = dg->name_hash.p && dg->name_hash_seed == seed && dg->name_hash_D == D &&
                     !getenv("SP_FOLD_NOHASHCACHE");
    if (!hit) {
      dg->name_hash.alloc(nd * 20 + (size_t)n * 8, s);  // + the level-1 sort order
      dg->name_hash_seed = seed;
      dg->name_hash_D = D;
    }
    A.hcache = dg->name_hash.p;
    A.hc_ready = hit ? 1 : 0;
  }
  static const bool prof = getenv("SP_FOLD_PROF") != nullptr;
  DevBuf<long long> profb;
  A.prof = nullptr;
  if (prof) {
    profb.alloc(256, s);
    SP_CUDA(cudaMemsetAsync(profb.p, 0, 256 * sizeof(long long), s));
    A.prof = profb.p;
  }
  SP_LAUNCH(ctx, kern, 1, threads, smem, s, A);
  if (prof) {
    long long h[256];
    SP_CUDA(cudaMemcpyAsync(h, profb.p, sizeof(h), cudaMemcpyDeviceToHost, s));
    SP_CUDA(cudaStreamSynchronize(s));
    fprintf(stderr, "[fold_small prof] n=%lld threads=%d: cycles", (long long)n, threads);
    for (int i = 1; i < 128 && h[i]; i++) fprintf(stderr, " %lld", h[i] - h[i - 1]);
    int last = 1;
    while (last < 128 && h[128 + last]) last++;
    fprintf(stderr, "; %lld ns, %.0f MHz\n", h[128 + last - 1] - h[128],
            (double)(h[last - 1] - h[0]) * 1e3 / (double)std::max(1LL, h[128 + last - 1] - h[128]));
  }
  SP_CUDA(cudaGetLastError());
  SP_CUDA(cudaEventRecord(ctx->ev[7], s));
  // outputs, pend, gaccept + residual: one contiguous range, one pinned block, one copy
  const size_t b_out = (i32_out - nd) * 4, b_pend = nd * 4, b_u8 = nd + n;
  size_t pin_bytes = 0;
  uint8_t* pin = pinned_acquire(ctx, b_out + b_pend + b_u8, &pin_bytes);
  struct Release {
    sp_ctx* ctx;
    uint8_t* p;
    size_t n;
    ~Release() { pinned_release(ctx, p, n); }
  } rel{ctx, pin, pin_bytes};
  g_d2h_bytes += (int64_t)(b_out + b_pend + b_u8);
  SP_CUDA(cudaMemcpyAsync(pin, out0, b_out + b_pend + b_u8, cudaMemcpyDeviceToHost, s));
  SP_CUDA(cudaStreamSynchronize(s));
  tr.mark("launch+d2h sync");
  const int32_t* h_out_p = (const int32_t*)pin;
  std::vector<int32_t> pend_h((const int32_t*)(pin + b_out), (const int32_t*)(pin + b_out) + nd);
  const uint8_t* h_u8 = pin + b_out + b_pend;
  {
    float ms = 0;
    SP_CUDA(cudaEventElapsedTime(&ms, ctx->ev[6], ctx->ev[7]));
    ctx->fold_device_ms = ms;
  }
  const int32_t* h_sorted = h_out_p;
  const int32_t* h_gstart = h_sorted + nd;
  const int32_t* h_corder = h_gstart + nd1;
  const int32_t* h_cstart = h_corder + nd;
  const int32_t* h_info = h_cstart + nd1;
  const int32_t coll = h_info[4 * D + 4];
  *collided = coll != 0;
  if (*collided) return;
  const int32_t nlev = h_info[4 * D];
  if (nlev < 0) throw Error(SP_ERR_CUDA, "fold did not terminate");
  ctx->fold_levels = nlev;
  std::vector<LevelOut> levels;
  for (int32_t dd = 0; dd < nlev; dd++) {
    const int32_t nA = h_info[dd * 4], nG = h_info[dd * 4 + 1], nC = h_info[dd * 4 + 2];
    LevelOut lv;
    lv.level = dd + 1;
    lv.sorted.assign(h_sorted + (size_t)dd * n, h_sorted + (size_t)dd * n + nA);
    lv.gstart.assign(h_gstart + (size_t)dd * (n + 1), h_gstart + (size_t)dd * (n + 1) + nG + 1);
    lv.corder.assign(h_corder + (size_t)dd * n, h_corder + (size_t)dd * n + nG);
    lv.cstart.assign(h_cstart + (size_t)dd * (n + 1), h_cstart + (size_t)dd * (n + 1) + nC + 1);
    lv.gaccept.assign(h_u8 + (size_t)dd * n, h_u8 + (size_t)dd * n + nG);
    levels.push_back(std::move(lv));
  }
  std::vector<uint8_t> resid_h(h_u8 + nd, h_u8 + nd + n);
  tr.mark("unpack");
  fold_finalize(dg, levels, resid_h, pend_h, D, out);
  tr.mark("finalize");
}

static void fold_once(sp_ctx* ctx, sp_dgraph* dg, int32_t min_dup, uint64_t seed, sp_fold* out,
                      bool* collided) {
  cudaStream_t s = ctx->stream;
  const int sms = ctx->sm_count;
  const int64_t n = dg->n;
  const int32_t D = dg->max_depth;
  FoldTrace tr;

  DevBuf<int32_t> depth, maxd, pend, act, sorted1, sorted2, gidv, gstart, pos, gparent, gclass, corder,
      corder2, corder3, cid, cstart, collision, nsel;
  DevBuf<uint64_t> ph, rh, k1, k1s, k2, k2s, ck, cks, cks2;
  DevBuf<uint32_t> par, par2, pars;
  DevBuf<int64_t> cur;
  DevBuf<unsigned long long> gkey;
  DevBuf<uint8_t> next_flag, residual, gaccept;
  DevBuf<int32_t> inv;
  inv.alloc(n, s);
  depth.alloc(n, s);
  maxd.alloc(1, s);
  pend.alloc((size_t)n * D, s);
  ph.alloc((size_t)n * D, s);
  rh.alloc((size_t)n * D, s);
  act.alloc(n, s);
  sorted1.alloc(n, s);
  sorted2.alloc(n, s);
  gidv.alloc(n, s);
  gstart.alloc(n, s);
  pos.alloc(n, s);
  gparent.alloc(n, s);
  gclass.alloc(n, s);
  corder.alloc(n, s);
  corder2.alloc(n, s);
  corder3.alloc(n, s);
  cid.alloc(n, s);
  cstart.alloc(n, s);
  collision.alloc(1, s);
  nsel.alloc(1, s);
  k1.alloc(n, s);
  k1s.alloc(n, s);
  k2.alloc(n, s);
  k2s.alloc(n, s);
  ck.alloc(n, s);
  cks.alloc(n, s);
  cks2.alloc(n, s);
  par.alloc(n, s);
  par2.alloc(n, s);
  pars.alloc(n, s);
  cur.alloc(n, s);
  gkey.alloc(n, s);
  next_flag.alloc(n, s);
  residual.alloc(n, s);
  gaccept.alloc(n, s);

  // per-level outputs stay on the device until the loop ends (one download)
  DevBuf<int32_t> st_sorted, st_gstart, st_corder, st_cstart;
  DevBuf<uint8_t> st_gaccept;
  size_t st_cap = (size_t)n * 2;
  st_sorted.alloc(st_cap, s);
  st_gstart.alloc(st_cap, s);
  st_corder.alloc(st_cap, s);
  st_cstart.alloc(st_cap, s);
  st_gaccept.alloc(st_cap, s);

  tr.mark("alloc");
  SP_CUDA(cudaEventRecord(ctx->ev[6], s));
  SP_CUDA(cudaMemsetAsync(maxd.p, 0, sizeof(int32_t), s));
  SP_LAUNCH(ctx, k_depth, grid_for(n, sms), 256, 0, s, dg->name_off.p, dg->names.p, n, depth.p, maxd.p);
  SP_LAUNCH(ctx, k_name_hash, grid_for(n, sms), 128, 0, s, dg->name_off.p, dg->names.p, n, D, seed, pend.p, ph.p, rh.p);
  SP_CUDA(cudaMemsetAsync(gparent.p, 0, n * sizeof(int32_t), s));
  SP_CUDA(cudaMemsetAsync(residual.p, 0, n, s));
  SP_CUDA(cudaMemsetAsync(collision.p, 0, sizeof(int32_t), s));
  SP_CUDA(cudaMemsetAsync(cur.p, 0xff, n * sizeof(int64_t), s));
  SP_LAUNCH(ctx, k_iota, grid_for(n, sms), 256, 0, s, act.p, n);

  // CUB scratch sized for the largest call
  size_t tmp_bytes = 0, t = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, t, k1.p, k1s.p, act.p, sorted1.p, (int)n, 0, 64, s);
  tmp_bytes = std::max(tmp_bytes, t);
  cub::DeviceRadixSort::SortPairs(nullptr, t, par.p, pars.p, corder.p, corder2.p, (int)n, 0, 32, s);
  tmp_bytes = std::max(tmp_bytes, t);
  cub::DeviceScan::InclusiveSum(nullptr, t, gidv.p, gidv.p, (int)n, s);
  tmp_bytes = std::max(tmp_bytes, t);
  cub::DeviceSelect::Flagged(nullptr, t, sorted2.p, next_flag.p, act.p, nsel.p, (int)n, s);
  tmp_bytes = std::max(tmp_bytes, t);
  ctx->cub_tmp.alloc(tmp_bytes, s);
  void* tmp = ctx->cub_tmp.p;

  struct LevelSize {
    int64_t nA, nG, nC;
    size_t off_a, off_g, off_c;
  };
  std::vector<LevelSize> sizes;
  size_t used_a = 0, used_g = 0, used_c = 0;
  // grow the level store (stream-ordered; only when the bound n*2 is exceeded)
  auto reserve = [&](auto& buf, size_t used, size_t need) {
    if (used + need <= buf.n) return;
    using T = std::remove_reference_t<decltype(*buf.p)>;
    DevBuf<T> bigger;
    bigger.alloc(std::max(buf.n * 2, used + need), s);
    if (used) SP_CUDA(cudaMemcpyAsync(bigger.p, buf.p, used * sizeof(T), cudaMemcpyDeviceToDevice, s));
    buf = std::move(bigger);
  };
  // device-side block assembly (SP_FOLD_HOST_ORDER=1: the host ordering of fold_finalize)
  const bool device_blocks = getenv("SP_FOLD_HOST_ORDER") == nullptr;
  std::vector<LevelBlocks> lblocks;
  DevBuf<int32_t> tie;
  tie.alloc(1, s);
  SP_CUDA(cudaMemsetAsync(tie.p, 0, sizeof(int32_t), s));
  int64_t nA = n;
  for (int32_t level = 1; nA > 0; level++) {
    if (level > D) throw Error(SP_ERR_CUDA, "fold did not terminate");
    const int32_t dd = level - 1;
    const int g1 = grid_for(nA, sms);
    // 1. sort active nodes by (prefix hash, rel hash): rel first, then prefix (stable
    //    LSD).  The rel-hash pass only orders members inside a group, so its low
    //    32 bits suffice: a 32-bit tie that misaligns two groups of a class fails
    //    the exact verification and the fold reruns with a new seed.
    SP_LAUNCH(ctx, k_gather_keys, g1, 256, 0, s, act.p, nA, rh.p, D, dd, k2.p);
    t = tmp_bytes;
    ctx->cub_calls++;
    SP_CUDA(cub::DeviceRadixSort::SortPairs(tmp, t, k2.p, k2s.p, act.p, sorted1.p, (int)nA, 0, 32, s));
    SP_LAUNCH(ctx, k_gather_keys, g1, 256, 0, s, sorted1.p, nA, ph.p, D, dd, k1.p);
    t = tmp_bytes;
    ctx->cub_calls++;
    SP_CUDA(cub::DeviceRadixSort::SortPairs(tmp, t, k1.p, k1s.p, sorted1.p, sorted2.p, (int)nA, 0, 64, s));
    SP_LAUNCH(ctx, k_heads_u64, g1, 256, 0, s, k1s.p, nA, gidv.p);
    t = tmp_bytes;
    ctx->cub_calls++;
    SP_CUDA(cub::DeviceScan::InclusiveSum(tmp, t, gidv.p, gidv.p, (int)nA, s));
    int32_t nG32 = 0;
    g_d2h_bytes += 4;
    SP_CUDA(cudaMemcpyAsync(&nG32, gidv.p + nA - 1, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
    SP_CUDA(cudaStreamSynchronize(s));
    const int64_t nG = nG32;
    const int64_t stamp = ((int64_t)level) << 32;
    SP_LAUNCH(ctx, k_group_setup, g1, 256, 0, s, sorted2.p, gidv.p, nA, stamp, cur.p, gstart.p, inv.p);
    // 2. entry hashes and group keys (node order: coalesced reads)
    SP_CUDA(cudaMemsetAsync(gkey.p, 0, nG * sizeof(unsigned long long), s));
    SP_LAUNCH(ctx, k_entry_nodes, grid_for(n, sms), 256, 0, s, n, stamp, cur.p, inv.p, gstart.p, rh.p, D, dd, dg->op.p,
              dg->w_rank.p, dg->w_shape.p, dg->w_train.p, dg->in_off.p, dg->in_idx.p, pos.p, gkey.p);
    // 3. classes: sort groups by (parent, key) -- key first, then parent (stable)
    const int gG = grid_for(nG, sms);
    SP_LAUNCH(ctx, k_class_keys, gG, 256, 0, s, nG, nA, gstart.p, sorted2.p, gkey.p, gparent.p, ck.p, par.p, corder.p);
    t = tmp_bytes;
    ctx->cub_calls++;
    SP_CUDA(cub::DeviceRadixSort::SortPairs(tmp, t, ck.p, cks.p, corder.p, corder2.p, (int)nG, 0, 64, s));
    SP_LAUNCH(ctx, k_gather<uint32_t>, gG, 256, 0, s, corder2.p, nG, par.p, par2.p);
    t = tmp_bytes;
    ctx->cub_calls++;
    SP_CUDA(cub::DeviceRadixSort::SortPairs(tmp, t, par2.p, pars.p, corder2.p, corder3.p, (int)nG, 0, 32, s));
    SP_LAUNCH(ctx, k_gather<uint64_t>, gG, 256, 0, s, corder3.p, nG, ck.p, cks2.p);
    SP_LAUNCH(ctx, k_class_heads, gG, 256, 0, s, pars.p, cks2.p, nG, cid.p);
    t = tmp_bytes;
    ctx->cub_calls++;
    SP_CUDA(cub::DeviceScan::InclusiveSum(tmp, t, cid.p, cid.p, (int)nG, s));
    int32_t nC32 = 0;
    g_d2h_bytes += 4;
    SP_CUDA(cudaMemcpyAsync(&nC32, cid.p + nG - 1, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
    SP_CUDA(cudaStreamSynchronize(s));
    const int64_t nC = nC32;
    SP_LAUNCH(ctx, k_class_setup, gG, 256, 0, s, corder3.p, cid.p, nG, gclass.p, cstart.p);
    // 4. exact verification against group and class heads
    SP_LAUNCH(ctx, k_verify_nodes, grid_for(n, sms), 128, 0, s, n, stamp, inv.p, sorted2.p, gidv.p, nA, nG, gstart.p,
              gclass.p, cstart.p, corder3.p, cur.p, pos.p, pend.p, rh.p, D, dd, dg->name_off.p, dg->names.p,
              dg->op.p, dg->w_rank.p, dg->w_shape.p, dg->w_train.p, dg->in_off.p, dg->in_idx.p, collision.p);
    // 5. accept / residual / descend
    SP_LAUNCH(ctx, k_accept, g1, 256, 0, s, sorted2.p, gidv.p, nA, nC, nG, gclass.p, cstart.p, depth.p, level, min_dup,
                                gparent.p, next_flag.p, residual.p, gaccept.p);
    tr.mark("level: group/class/verify");
    // accepted classes -> blocks, assembled on the device
    if (device_blocks) {
      lblocks.emplace_back();
      level_blocks(ctx, dg, dd, nA, nG, sorted2.p, gstart.p, gclass.p, gaccept.p, pend.p, D, 1, tie.p, lblocks.back());
      tr.mark("level: blocks");
    }
    reserve(st_sorted, used_a, nA);
    reserve(st_gstart, used_g, nG);
    reserve(st_corder, used_g, nG);
    reserve(st_gaccept, used_g, nG);
    reserve(st_cstart, used_c, nC);
    SP_CUDA(cudaMemcpyAsync(st_sorted.p + used_a, sorted2.p, nA * 4, cudaMemcpyDeviceToDevice, s));
    SP_CUDA(cudaMemcpyAsync(st_gstart.p + used_g, gstart.p, nG * 4, cudaMemcpyDeviceToDevice, s));
    SP_CUDA(cudaMemcpyAsync(st_corder.p + used_g, corder3.p, nG * 4, cudaMemcpyDeviceToDevice, s));
    SP_CUDA(cudaMemcpyAsync(st_gaccept.p + used_g, gaccept.p, nG, cudaMemcpyDeviceToDevice, s));
    SP_CUDA(cudaMemcpyAsync(st_cstart.p + used_c, cstart.p, nC * 4, cudaMemcpyDeviceToDevice, s));
    sizes.push_back({nA, nG, nC, used_a, used_g, used_c});
    used_a += nA;
    used_g += nG;
    used_c += nC;
    t = tmp_bytes;
    ctx->cub_calls++;
    SP_CUDA(cub::DeviceSelect::Flagged(tmp, t, sorted2.p, next_flag.p, act.p, nsel.p, (int)nA, s));
    int32_t nsel_h = 0;
    g_d2h_bytes += 4;
    SP_CUDA(cudaMemcpyAsync(&nsel_h, nsel.p, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
    SP_CUDA(cudaStreamSynchronize(s));
    nA = nsel_h;
  }
  SP_CUDA(cudaEventRecord(ctx->ev[7], s));
  int32_t coll_h = 0;
  g_d2h_bytes += 4;
  SP_CUDA(cudaMemcpyAsync(&coll_h, collision.p, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
  SP_CUDA(cudaStreamSynchronize(s));
  {
    float ms = 0;
    SP_CUDA(cudaEventElapsedTime(&ms, ctx->ev[6], ctx->ev[7]));
    ctx->fold_device_ms = ms;
    ctx->fold_levels = (int32_t)sizes.size();
  }
  *collided = coll_h != 0;
  if (*collided) return;
  tr.mark("loop end");
  if (device_blocks && d2h_scalar(tie.p, s) == 0) {
    // residual singletons, compacted on the device
    DevBuf<int32_t> iota, rlist, nsel2;
    iota.alloc(n, s);
    rlist.alloc(n, s);
    nsel2.alloc(1, s);
    SP_LAUNCH(ctx, k_iota, grid_for(n, sms), 256, 0, s, iota.p, n);
    size_t tb = 0;
    ctx->cub_calls++;
    SP_CUDA(cub::DeviceSelect::Flagged(nullptr, tb, iota.p, residual.p, rlist.p, nsel2.p, (int)n, s));
    DevBuf<uint8_t> tmp2;
    tmp2.alloc(tb, s);
    SP_CUDA(cub::DeviceSelect::Flagged(tmp2.p, tb, iota.p, residual.p, rlist.p, nsel2.p, (int)n, s));
    const int64_t nr = d2h_scalar(nsel2.p, s);
    std::vector<int32_t> resid(nr);
    rlist.download(resid.data(), nr, s);
    tr.mark("residuals");
    fold_finalize_blocks(dg, lblocks, resid, s, out);
    tr.mark("finalize");
    return;
  }
  std::vector<uint8_t> resid_h(n);
  std::vector<int32_t> pend_h((size_t)n * D);
  std::vector<int32_t> h_sorted(used_a), h_gstart(used_g), h_corder(used_g), h_cstart(used_c);
  std::vector<uint8_t> h_gaccept(used_g);
  residual.download(resid_h.data(), n, s);
  pend.download(pend_h.data(), (size_t)n * D, s);
  st_sorted.download(h_sorted.data(), used_a, s);
  st_gstart.download(h_gstart.data(), used_g, s);
  st_corder.download(h_corder.data(), used_g, s);
  st_gaccept.download(h_gaccept.data(), used_g, s);
  st_cstart.download(h_cstart.data(), used_c, s);
  SP_CUDA(cudaStreamSynchronize(s));
  std::vector<LevelOut> levels(sizes.size());
  for (size_t l = 0; l < sizes.size(); l++) {
    const LevelSize& z = sizes[l];
    LevelOut& lv = levels[l];
    lv.level = (int32_t)l + 1;
    lv.sorted.assign(h_sorted.begin() + z.off_a, h_sorted.begin() + z.off_a + z.nA);
    lv.gstart.assign(h_gstart.begin() + z.off_g, h_gstart.begin() + z.off_g + z.nG);
    lv.gstart.push_back((int32_t)z.nA);
    lv.corder.assign(h_corder.begin() + z.off_g, h_corder.begin() + z.off_g + z.nG);
    lv.gaccept.assign(h_gaccept.begin() + z.off_g, h_gaccept.begin() + z.off_g + z.nG);
    lv.cstart.assign(h_cstart.begin() + z.off_c, h_cstart.begin() + z.off_c + z.nC);
    lv.cstart.push_back((int32_t)z.nG);
  }

  fold_finalize(dg, levels, resid_h, pend_h, D, out);
}


// ---------------------------------------------------------------------------
// Hash-grouped fold (multi-kernel path).  The level algorithm above with its
// sorts replaced by hash tables, every node pass in node order (coalesced):
//   * groups: open-addressing table keyed by the level's 64-bit prefix hash
//     (k_hg_insert; the CAS winner is the group's head), sizes and template-key
//     sums aggregated per warp (k_hg_entry), compact group ids by a scan of the
//     head flags in node order (k_hg_ids);
//   * classes: a second table keyed by (parent group, key sum, size)
//     (k_hc_insert / k_hc_count);
//   * member segments (a counting scatter) and the canonical member order
//     (rank of the relative-name hash inside the group, k_hg_rank) only for
//     groups whose class has >= 2 groups or is accepted -- the huge top-level
//     groups of a deep graph are neither;
//   * exact verification (prefix bytes vs the group head; member by member vs
//     the class head group, including the parent) and accept/descend in one
//     node pass each.
// Hash collisions are detected exactly as before (the fold reruns with a new
// seed); a multi-group class with groups larger than RANK_MAX falls back to
// the sort-based path.  Per level: two host syncs (the group count after the
// insert, the level's counters after accept).

// Name hashing of the hash fold, in two 32-bit polynomial lanes packed in a u64
// (32-bit IMADs are full rate; a 64-bit multiply is several instructions).
// Only consistency matters: equal byte strings hash equal, and every grouping
// decision is re-checked on the bytes.
constexpr uint32_t kP1 = 0x01000193u, kP2 = 0x5bd1e995u;

__device__ __forceinline__ uint64_t poly_step(uint64_t h, uint32_t c) {
  return ((uint64_t)((uint32_t)(h >> 32) * kP1 + c) << 32) | (uint32_t)((uint32_t)h * kP2 + c);
}
__device__ __forceinline__ uint32_t upow32(uint32_t b, int64_t e) {
  uint32_t r = 1;
  while (e) {
    if (e & 1) r *= b;
    b *= b;
    e >>= 1;
  }
  return r;
}
// poly(s) = hall - poly(prefix) * B^(len(s)), lane-wise mod 2^32
__device__ __forceinline__ uint64_t poly_suffix(uint64_t hall, uint64_t hpre, int64_t e) {
  const uint32_t a = (uint32_t)(hall >> 32) - (uint32_t)(hpre >> 32) * upow32(kP1, e);
  const uint32_t b = (uint32_t)hall - (uint32_t)hpre * upow32(kP2, e);
  return ((uint64_t)a << 32) | b;
}

// Per node, once per fold (hash path): depth, the polynomial hash of the whole
// name, and the static part of the template-key entry (op, weight shape,
// trainable).  The names of a block's 256 nodes are staged through shared
// memory with coalesced loads when they fit.
constexpr int PREP_SMEM = 16384;
__global__ void __launch_bounds__(256) k_hg_prep(const int64_t* __restrict__ off, const uint8_t* __restrict__ names,
                                                 int64_t n, const uint8_t* __restrict__ op,
                                                 const uint8_t* __restrict__ w_rank, const int64_t* __restrict__ w_shape,
                                                 const uint8_t* __restrict__ w_train, int32_t* __restrict__ depth,
                                                 uint64_t* __restrict__ hall, uint64_t* __restrict__ sh) {
  __shared__ __align__(16) uint32_t swords[PREP_SMEM / 4 + 2];
  const uint8_t* sbuf = (const uint8_t*)swords;
  const int64_t total = off[n];
  const bool aligned = ((uintptr_t)names & 3) == 0;
  for (int64_t b0 = (int64_t)blockIdx.x * blockDim.x; b0 < n; b0 += (int64_t)gridDim.x * blockDim.x) {
    const int64_t e = b0 + blockDim.x < n ? b0 + blockDim.x : n;
    const int64_t lo = off[b0], hi = off[e];
    // 4-byte words [lo/4, ceil(hi/4)) -- coalesced, every load in flight at once
    const int64_t w0 = lo >> 2, w1 = (hi + 3) >> 2;
    const bool staged = aligned && (w1 - w0) * 4 <= PREP_SMEM;
    if (staged) {
      const uint32_t* gw = (const uint32_t*)names;
      const int64_t last = (total + 3) >> 2;  // words holding name bytes (the arena continues past them)
#pragma unroll 4
      for (int64_t w = w0 + threadIdx.x; w < w1; w += blockDim.x) swords[w - w0] = w < last ? gw[w] : 0u;
    }
    __syncthreads();
    const int64_t v = b0 + threadIdx.x;
    if (v < n) {
      const int64_t a = off[v], L = off[v + 1] - a;
      const uint8_t* p = staged ? sbuf + (a - (w0 << 2)) : names + a;
      uint64_t h = 0;
      int d = 1;
      for (int64_t k = 0; k < L; k++) {
        const uint32_t c = p[k];
        d += c == '/';
        h = poly_step(h, c + 1);
      }
      depth[v] = d;
      hall[v] = h;
      sh[v] = fmix64(weight_hash(v, w_rank, w_shape, w_train) + 0x3c6ef372fe94f82bULL * (uint64_t)(op[v] + 1));
    }
    __syncthreads();
  }
}

// The keys of one level for the nodes active at it: extend the node's prefix
// polynomial by one component (pend of the previous depth -> this one), then
// prefix hash, prefix end (level-major pend, read again by the block
// assembly) and the relative-name hash (suffix = whole name minus prefix).
// The keys of depth dd for node v: extend the node's prefix polynomial by one
// component (pend of the previous depth -> this one), then the prefix hash,
// the prefix end (level-major pend, read again by the block assembly) and the
// relative-name hash (suffix = whole name minus prefix).  Returns the prefix hash.
__device__ __forceinline__ uint64_t node_keys(int64_t v, int64_t n, int32_t dd, const int64_t* __restrict__ off,
                                              const uint8_t* __restrict__ names, uint64_t seed,
                                              const uint64_t* __restrict__ hall, uint64_t* __restrict__ ppoly,
                                              int32_t* __restrict__ pend, uint64_t* __restrict__ ph,
                                              uint64_t* __restrict__ rh) {
  const int64_t a = off[v], L = off[v + 1] - a;
  const uint8_t* p = names + a;
  int64_t k = dd ? pend[(int64_t)(dd - 1) * n + v] : 0;
  uint64_t h = dd ? ppoly[v] : 0;
  if (dd && k < L) h = poly_step(h, '/' + 1), k++;  // the separator closing the previous prefix
  for (; k < L && p[k] != '/'; k++) h = poly_step(h, (uint32_t)p[k] + 1);
  const int64_t q = k;
  pend[(int64_t)dd * n + v] = (int32_t)q;
  ppoly[v] = h;
  const uint64_t key = fmix64(h ^ fmix64(seed + (uint64_t)q));
  ph[v] = key;
  int64_t start = q > 0 ? q + 1 : 0;
  if (start > L) start = L;
  uint64_t hrel = 0;
  if (q < L) hrel = poly_suffix(hall[v], start > 0 ? poly_step(h, '/' + 1) : 0, L - start);
  rh[v] = fmix64(hrel ^ fmix64((seed ^ 0x9e3779b97f4a7c15ULL) + (uint64_t)(L - start)));
  return key;
}

// Upper bound of the number of distinct prefix hashes among the lanes with
// `act`: boundaries between consecutive lanes (every distinct key has one at
// its first occurrence in node order), lane 0 always counting.  Lane 0 returns
// the warp's count.
__device__ __forceinline__ int32_t warp_boundaries(bool act, uint64_t key) {
  const int lane = threadIdx.x & 31;
  const uint64_t pk = __shfl_up_sync(0xffffffffu, key, 1);
  const bool pa = __shfl_up_sync(0xffffffffu, act, 1);
  const bool bnd = act && (lane == 0 || !pa || pk != key);
  return __popc(__ballot_sync(0xffffffffu, bnd));
}

__device__ __forceinline__ void block_add(int32_t x, int32_t* __restrict__ dst) {
  __shared__ int32_t s_w[32];
  x = __reduce_add_sync(0xffffffffu, (unsigned)x);
  if ((threadIdx.x & 31) == 0) s_w[threadIdx.x >> 5] = x;
  __syncthreads();
  if (threadIdx.x == 0) {
    int32_t t = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); w++) t += s_w[w];
    if (t) atomicAdd(dst, t);
  }
  __syncthreads();
}

constexpr int64_t RANK_MAX = 1024;

struct HashStats {  // device counters of one level
  int32_t nG, overflow, nC, nnext, nacc, big, est, nres;
};

// level-1 keys of every node + the group-count bound
__global__ void __launch_bounds__(256) k_hg_keys1(int64_t n, const int64_t* __restrict__ off,
                                                  const uint8_t* __restrict__ names, uint64_t seed,
                                                  const uint64_t* __restrict__ hall, uint64_t* __restrict__ ppoly,
                                                  int32_t* __restrict__ pend, uint64_t* __restrict__ ph,
                                                  uint64_t* __restrict__ rh, HashStats* __restrict__ st) {
  int32_t est = 0;
  for (int64_t base = blockIdx.x * (int64_t)blockDim.x + (threadIdx.x & ~31); base < n;
       base += (int64_t)gridDim.x * blockDim.x) {
    const int64_t v = base + (threadIdx.x & 31);
    const bool act = v < n;
    const uint64_t key = act ? node_keys(v, n, 0, off, names, seed, hall, ppoly, pend, ph, rh) : 0;
    const int32_t c = warp_boundaries(act, key);
    if ((threadIdx.x & 31) == 0) est += c;
  }
  block_add(est, &st->est);
}


__device__ __forceinline__ uint64_t nz64(uint64_t k) { return k ? k : 0x9e3779b97f4a7c15ULL; }

// one pass over the nodes active at `level`: find-or-insert the prefix hash
// Overflow (more keys than half the capacity, or a probe run longer than
// max_probe) stops every thread at its next node: the host retries the level
// with a table of 2 x the active count.
// Lanes of a warp that carry the same key (consecutive members of one group)
// probe once: the lowest such lane finds or inserts, the others take its slot.
__global__ void __launch_bounds__(256) k_hg_insert(int64_t n, const uint8_t* __restrict__ alive, int32_t level,
                                                   const uint64_t* __restrict__ ph,
                                                   unsigned long long* __restrict__ tkey, int32_t* __restrict__ thead,
                                                   uint32_t mask, uint32_t max_probe, uint32_t* __restrict__ nslot,
                                                   HashStats* __restrict__ st) {
  volatile int32_t* overflow = &st->overflow;
  const int lane = threadIdx.x & 31;
  for (int64_t base = blockIdx.x * (int64_t)blockDim.x + (threadIdx.x & ~31); base < n;
       base += (int64_t)gridDim.x * blockDim.x) {
    const int64_t v = base + lane;
    const bool act = v < n && alive[v] == level;
    const unsigned long long key = act ? nz64(ph[v]) : 0;
    const unsigned same = __match_any_sync(0xffffffffu, key);
    const int leader = __ffs(same) - 1;
    uint32_t h = (uint32_t)(key >> 17) & mask;
    bool gave_up = false;
    if (act && lane == leader) {
      for (uint32_t probe = 0;; probe++) {
        unsigned long long k = tkey[h];
        if (k == 0) {
          k = atomicCAS(&tkey[h], 0ULL, key);
          if (k == 0) {
            thead[h] = (int32_t)v;
            if ((uint32_t)atomicAdd(&st->nG, 1) >= (mask + 1) / 2) *overflow = 1;
            break;
          }
        }
        if (k == key) break;
        h = (h + 1) & mask;
        if (probe >= max_probe || (probe == 8 && *overflow)) {  // the flag is read on long runs only
          *overflow = 1;
          gave_up = true;
          break;
        }
      }
    }
    h = __shfl_sync(0xffffffffu, h, leader);
    gave_up = __shfl_sync(0xffffffffu, gave_up, leader);
    if (act && !gave_up) nslot[v] = h;
  }
}

// template-key entry hash per node (rel name, op, weight, internal producers'
// rel names), summed per group slot; group sizes counted alongside.  Lanes of
// a warp that share a slot add in three 22-bit slices (each slice sum fits 32
// bits): one atomic per slot per warp.
__global__ void __launch_bounds__(256) k_hg_entry(int64_t n, const uint8_t* __restrict__ alive, int32_t level,
                                                  const uint32_t* __restrict__ nslot, const uint64_t* __restrict__ rh,
                                                  const uint64_t* __restrict__ sh, const int64_t* __restrict__ in_off,
                                                  const int32_t* __restrict__ in_idx,
                                                  const int32_t* __restrict__ thead, int32_t* __restrict__ hf,
                                                  unsigned long long* __restrict__ tgkey, int32_t* __restrict__ tcnt) {
  // the slot of the block's first node is usually every lane's (huge top-level
  // groups): its sum goes through shared memory, one global atomic per block
  __shared__ unsigned long long s_sum;
  __shared__ int32_t s_cnt;
  __shared__ uint32_t s_hot;
  const int lane = threadIdx.x & 31;
  for (int64_t b0 = (int64_t)blockIdx.x * blockDim.x; b0 < n; b0 += (int64_t)gridDim.x * blockDim.x) {
    const int64_t v = b0 + threadIdx.x;
    const bool act = v < n && alive[v] == level;
    const uint32_t sl = act ? nslot[v] : 0xffffffffu;
    if (v < n) hf[v] = act && thead[sl] == (int32_t)v;  // group heads (compact ids by their scan)
    if (threadIdx.x == 0) {
      s_hot = sl;
      s_sum = 0;
      s_cnt = 0;
    }
    uint64_t val = 0;
    if (act) {
      uint64_t prod = 0;
      for (int64_t e = in_off[v]; e < in_off[v + 1]; e++) {
        const int32_t r = in_idx[e];
        if (alive[r] == level && nslot[r] == sl) prod += fmix64(rh[r] ^ 0x6a09e667f3bcc909ULL);
      }
      uint64_t h = fmix64(rh[v] ^ sh[v]);
      h = fmix64(h + fmix64(prod ^ 0xbb67ae8584caa73bULL));
      val = fmix64(h ^ 0xa54ff53a5f1d36f1ULL);
    }
    __syncthreads();
    const unsigned mask = __match_any_sync(0xffffffffu, act ? (int)sl : -1 - lane);
    const uint64_t s0 = __reduce_add_sync(mask, (unsigned)(val & 0x3fffff));
    const uint64_t s1 = __reduce_add_sync(mask, (unsigned)((val >> 22) & 0x3fffff));
    const uint64_t s2 = __reduce_add_sync(mask, (unsigned)(val >> 44));
    if (act && lane == __ffs(mask) - 1) {
      const unsigned long long part = (unsigned long long)(s0 + (s1 << 22) + (s2 << 44));
      if (sl == s_hot) {
        atomicAdd(&s_sum, part);
        atomicAdd(&s_cnt, __popc(mask));
      } else {
        atomicAdd(&tgkey[sl], part);
        atomicAdd(&tcnt[sl], __popc(mask));
      }
    }
    __syncthreads();
    if (threadIdx.x == 0 && s_cnt) {
      atomicAdd(&tgkey[s_hot], s_sum);
      atomicAdd(&tcnt[s_hot], s_cnt);
    }
  }
}

// compact group ids in node order of the heads; per-group arrays
__global__ void k_hg_ids(int64_t n, const int32_t* __restrict__ hf, const int32_t* __restrict__ hs,
                         const uint32_t* __restrict__ nslot, const unsigned long long* __restrict__ tgkey,
                         const int32_t* __restrict__ tcnt, const int32_t* __restrict__ gparent,
                         int32_t* __restrict__ tgid, int32_t* __restrict__ gnode, int32_t* __restrict__ gsize,
                         unsigned long long* __restrict__ gkey, int32_t* __restrict__ gpar) {
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x) {
    if (!hf[v]) continue;
    const int32_t g = hs[v] - 1;
    const uint32_t sl = nslot[v];
    tgid[sl] = g;
    gnode[g] = (int32_t)v;
    gsize[g] = tcnt[sl];
    gkey[g] = tgkey[sl];
    gpar[g] = gparent[v];
  }
}

// classes: find-or-insert (parent, key sum, size) per group
__global__ void k_hc_insert(int64_t gmax, const int32_t* __restrict__ d_nG, const unsigned long long* __restrict__ gkey,
                            const int32_t* __restrict__ gsize,
                            const int32_t* __restrict__ gpar, unsigned long long* __restrict__ ckey,
                            int32_t* __restrict__ chead, uint32_t mask, uint32_t* __restrict__ gcs,
                            HashStats* __restrict__ st) {
  const int64_t nG = *d_nG < gmax ? *d_nG : gmax;
  for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < nG; g += (int64_t)gridDim.x * blockDim.x) {
    const unsigned long long key =
        nz64(fmix64((uint64_t)gkey[g] ^ fmix64((uint64_t)gsize[g] + 0x1f83d9abfb41bd6bULL) ^
                    fmix64((uint64_t)(uint32_t)gpar[g] * 0x9e3779b97f4a7c15ULL + 0x5be0cd19137e2179ULL)));
    uint32_t h = (uint32_t)(key >> 13) & mask;
    for (uint32_t probe = 0;; probe++) {
      unsigned long long k = ckey[h];
      if (k == 0) {
        k = atomicCAS(&ckey[h], 0ULL, key);
        if (k == 0) {
          chead[h] = (int32_t)g;
          atomicAdd(&st->nC, 1);
          break;
        }
      }
      if (k == key) break;
      h = (h + 1) & mask;
      if (probe > mask) {  // cannot happen: capacity >= 2 nG
        st->overflow = 1;
        break;
      }
    }
    gcs[g] = h;
  }
}

__global__ void k_hc_count(int64_t gmax, const int32_t* __restrict__ d_nG, const uint32_t* __restrict__ gcs,
                           int32_t* __restrict__ ccnt) {
  const int64_t nG = *d_nG < gmax ? *d_nG : gmax;
  const int lane = threadIdx.x & 31;
  for (int64_t base = blockIdx.x * (int64_t)blockDim.x + (threadIdx.x & ~31); base < nG;
       base += (int64_t)gridDim.x * blockDim.x) {
    const int64_t g = base + lane;
    const bool ok = g < nG;
    const uint32_t c = ok ? gcs[g] : 0;
    const unsigned mask = __match_any_sync(0xffffffffu, ok ? (int)c : -1 - lane);
    if (ok && lane == __ffs(mask) - 1) atomicAdd(&ccnt[c], __popc(mask));
  }
}

// member segments (counting scatter) for groups whose class is multi-group or accepted
__global__ void k_hg_place(int64_t n, const uint8_t* __restrict__ alive, int32_t level,
                           const uint32_t* __restrict__ nslot, const int32_t* __restrict__ tgid,
                           const uint32_t* __restrict__ gcs, const int32_t* __restrict__ ccnt, int32_t min_dup,
                           const int32_t* __restrict__ gstart, int32_t* __restrict__ gfill,
                           int32_t* __restrict__ seg, int32_t* __restrict__ li) {
  const int lane = threadIdx.x & 31;
  for (int64_t base = blockIdx.x * (int64_t)blockDim.x + (threadIdx.x & ~31); base < n;
       base += (int64_t)gridDim.x * blockDim.x) {
    const int64_t v = base + lane;
    bool need = false;
    int32_t g = 0;
    if (v < n && alive[v] == level) {
      g = tgid[nslot[v]];
      const int32_t cs = ccnt[gcs[g]];
      need = cs >= 2 || cs >= min_dup;
    }
    const unsigned mask = __match_any_sync(0xffffffffu, need ? g : -1 - lane);
    int32_t b = 0;
    const int leader = __ffs(mask) - 1;
    if (need && lane == leader) b = atomicAdd(&gfill[g], __popc(mask));
    b = __shfl_sync(mask, b, leader);
    if (need) {
      const int32_t l = b + __popc(mask & ((1u << lane) - 1));
      li[v] = l;
      seg[gstart[g] + l] = (int32_t)v;
    }
  }
}

// canonical member order: rank of the rel hash inside the group (multi-group
// classes); accepted single-group classes keep the segment order
__global__ void k_hg_rank(int64_t n, const uint8_t* __restrict__ alive, int32_t level,
                          const uint32_t* __restrict__ nslot, const int32_t* __restrict__ tgid,
                          const uint32_t* __restrict__ gcs, const int32_t* __restrict__ ccnt, int32_t min_dup,
                          const int32_t* __restrict__ gstart, const int32_t* __restrict__ gsize,
                          const int32_t* __restrict__ seg, const int32_t* __restrict__ li,
                          const uint64_t* __restrict__ rh, int32_t* __restrict__ sorted, int32_t* __restrict__ pos,
                          int32_t* __restrict__ collision, HashStats* __restrict__ st) {
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x) {
    if (alive[v] != level) continue;
    const int32_t g = tgid[nslot[v]];
    const int32_t cs = ccnt[gcs[g]];
    if (cs < 2 && cs < min_dup) continue;
    const int32_t s0 = gstart[g], sz = gsize[g];
    int32_t r = li[v];
    if (cs >= 2) {
      if (sz > RANK_MAX) {
        st->big = 1;
        continue;
      }
      const uint64_t me = rh[v];
      r = 0;
      for (int32_t k = 0; k < sz; k++) {
        const int32_t u = seg[s0 + k];
        const uint64_t x = rh[u];
        r += x < me;
        if (x == me && u != (int32_t)v) atomicExch(collision, 1);  // equal rel hashes in one group
      }
    }
    sorted[s0 + r] = (int32_t)v;
    pos[v] = r;
  }
}

// The end of a level, one pass over its active nodes: (1) exact checks --
// prefix bytes vs the group head, and for multi-group classes member-by-member
// equality with the class head group at the same canonical position (rel
// bytes, op, weight, internal producers as canonical positions) with equal
// parent and size; (2) accept / residual / descend, written to the NEXT
// level's state array (this level's stays read-only, so the internal-producer
// tests of other threads see it unchanged); (3) the next level's keys for the
// nodes that descend, and its group-count bound.
__global__ void __launch_bounds__(128) k_hg_finish(
    int64_t n, const uint8_t* __restrict__ alive, uint8_t* __restrict__ alive_next, int32_t level, int32_t D,
    const uint32_t* __restrict__ nslot, const int32_t* __restrict__ tgid, const uint32_t* __restrict__ gcs,
    const int32_t* __restrict__ ccnt, const int32_t* __restrict__ chead, const int32_t* __restrict__ gnode,
    const int32_t* __restrict__ gsize, const int32_t* __restrict__ gpar, const int32_t* __restrict__ gstart,
    const int32_t* __restrict__ sorted, const int32_t* __restrict__ pos, int32_t* __restrict__ pend,
    const int64_t* __restrict__ name_off, const uint8_t* __restrict__ names, const uint8_t* __restrict__ op,
    const uint8_t* __restrict__ w_rank, const int64_t* __restrict__ w_shape, const uint8_t* __restrict__ w_train,
    const int64_t* __restrict__ in_off, const int32_t* __restrict__ in_idx, const int32_t* __restrict__ depth,
    int32_t min_dup, int32_t* __restrict__ gparent, uint8_t* __restrict__ residual, uint8_t* __restrict__ gaccept,
    uint64_t seed, const uint64_t* __restrict__ hall, uint64_t* __restrict__ ppoly, uint64_t* __restrict__ ph,
    uint64_t* __restrict__ rh, int32_t* __restrict__ collision, HashStats* __restrict__ st) {
  const int32_t* pend_l = pend + (int64_t)(level - 1) * n;
  int32_t nnext = 0, nacc = 0, est = 0, nres = 0;
  bool bad = false;
  for (int64_t base = blockIdx.x * (int64_t)blockDim.x + (threadIdx.x & ~31); base < n;
       base += (int64_t)gridDim.x * blockDim.x) {
    const int64_t v = base + (threadIdx.x & 31);
    bool next = false;
    uint64_t key = 0;
    if (v < n && alive[v] == level) {
      const uint32_t sl = nslot[v];
      const int32_t g = tgid[sl];
      const int32_t h = gnode[g];
      const int32_t pl = pend_l[v];
      // same prefix string as the group head: the same parent group (whose
      // prefixes the previous level verified) and the same last component
      {
        const int32_t phd = pend_l[h];
        const int64_t cv = level > 1 ? (int64_t)pend_l[v - n] + 1 : 0;
        const int64_t ch = level > 1 ? (int64_t)pend_l[h - n] + 1 : 0;
        if (gparent[v] != gpar[g] || pl - cv != phd - ch ||
            !bytes_eq(names + name_off[v] + cv, names + name_off[h] + ch, pl - cv))
          bad = true;
      }
      const uint32_t cs = gcs[g];
      const int32_t hg = chead[cs];
      const int32_t csz = ccnt[cs];
      if (csz >= 2 && hg != g) {
        if (gsize[g] != gsize[hg] || gpar[g] != gpar[hg]) {
          bad = true;
        } else {
          const int32_t b = sorted[gstart[hg] + pos[v]];
          const uint32_t slb = nslot[b];
          const int64_t la = name_off[v + 1] - name_off[v];
          const int64_t lb = name_off[b + 1] - name_off[b];
          const int32_t plb = pend_l[b];
          int64_t sa = pl > 0 ? pl + 1 : 0, sb = plb > 0 ? plb + 1 : 0;
          sa = sa > la ? la : sa;
          sb = sb > lb ? lb : sb;
          if (la - sa != lb - sb || !bytes_eq(names + name_off[v] + sa, names + name_off[b] + sb, la - sa)) bad = true;
          if (op[v] != op[b] || w_rank[v] != w_rank[b] || w_train[v] != w_train[b]) bad = true;
          for (int k = 0; k < w_rank[v]; k++)
            if (w_shape[v * SP_MAX_RANK + k] != w_shape[(int64_t)b * SP_MAX_RANK + k]) bad = true;
          // internal producers (deduplicated inputs) as canonical positions: equal sets
          int ka = 0, kb = 0;
          for (int64_t e = in_off[b]; e < in_off[b + 1]; e++) {
            const int32_t r = in_idx[e];
            kb += alive[r] == level && nslot[r] == slb;
          }
          for (int64_t e = in_off[v]; e < in_off[v + 1]; e++) {
            const int32_t r = in_idx[e];
            if (alive[r] != level || nslot[r] != sl) continue;
            ka++;
            const int32_t pr = pos[r];
            bool found = false;
            for (int64_t f = in_off[b]; f < in_off[b + 1] && !found; f++) {
              const int32_t q = in_idx[f];
              found = alive[q] == level && nslot[q] == slb && pos[q] == pr;
            }
            bad = bad || !found;
          }
          bad = bad || ka != kb;
        }
      }
      const bool acc = csz >= min_dup;
      if (h == (int32_t)v) {
        gaccept[g] = acc;
        nacc += acc;
      }
      if (acc) {
        alive_next[v] = 0;
      } else if (depth[v] <= level) {
        residual[v] = 1;
        nres++;
        alive_next[v] = 0;
      } else {
        alive_next[v] = (uint8_t)(level + 1);
        gparent[v] = g;
        nnext++;
        next = level < D;
        if (next) key = node_keys(v, n, level, name_off, names, seed, hall, ppoly, pend, ph, rh);
      }
    }
    const int32_t c = warp_boundaries(next, key);
    if ((threadIdx.x & 31) == 0) est += c;
  }
  if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicExch(collision, 1);
  block_add(nnext, &st->nnext);
  block_add(nacc, &st->nacc);
  block_add(est, &st->est);
  block_add(nres, &st->nres);
}

static uint32_t table_cap(int64_t need) {
  uint64_t c = 1024;
  while (c < (uint64_t)need * 2) c <<= 1;
  return (uint32_t)c;
}

// one attempt of the hash-grouped fold; *collided on a hash collision, *fallback
// when a multi-group class has groups too large to rank in place, or when two
// instance prefixes of a class tie on 16 bytes (both rerun on the sort path)
static void fold_once_hash(sp_ctx* ctx, sp_dgraph* dg, int32_t min_dup, uint64_t seed, sp_fold* out,
                           bool* collided, bool* fallback) {
  cudaStream_t s = ctx->stream;
  const int sms = ctx->sm_count;
  const int64_t n = dg->n;
  const int32_t D = dg->max_depth;
  FoldTrace tr;
  *collided = *fallback = false;
  if (D > 250) {  // levels are stamped in one byte
    *fallback = true;
    return;
  }
  DevBuf<int32_t> depth, pend, hf, hs, tgid, gnode, gsize, gpar, gstart, gfill, seg, li, sorted, pos, gparent, tcnt,
      chead, ccnt, thead, collision, tie;
  DevBuf<uint32_t> nslot, gcs;
  DevBuf<uint64_t> ph, rh, sh, hall, ppoly;
  DevBuf<unsigned long long> tkey, tgkey, gkey, ckey;
  DevBuf<uint8_t> alive, alive2, residual, gaccept;
  DevBuf<HashStats> st;
  depth.alloc(n, s);
  pend.alloc((size_t)n * D, s);  // level-major; depth dd written at level dd + 1
  ph.alloc(n, s);                 // the current level's keys
  rh.alloc(n, s);
  hall.alloc(n, s);
  ppoly.alloc(n, s);
  sh.alloc(n, s);
  hf.alloc(n, s);
  hs.alloc(n, s);
  nslot.alloc(n, s);
  li.alloc(n, s);
  pos.alloc(n, s);
  seg.alloc(n, s);
  sorted.alloc(n, s);
  gparent.alloc(n, s);
  alive.alloc(n, s);
  alive2.alloc(n, s);
  residual.alloc(n, s);
  collision.alloc(1, s);
  tie.alloc(1, s);
  st.alloc(1, s);
  size_t tmp_bytes = 0;
  cub::DeviceScan::InclusiveSum(nullptr, tmp_bytes, hf.p, hs.p, (int)n, s);
  ctx->cub_tmp.alloc(tmp_bytes, s);
  HashStats* hst = (HashStats*)pinned_acquire(ctx, sizeof(HashStats), &tmp_bytes);
  struct Release {
    sp_ctx* ctx;
    void* p;
    size_t n;
    ~Release() { pinned_release(ctx, p, n); }
  } rel{ctx, hst, tmp_bytes};
  tr.mark("alloc");
  const int gn = grid_for(n, sms);
  SP_CUDA(cudaEventRecord(ctx->ev[6], s));
  SP_LAUNCH(ctx, k_hg_prep, gn, 256, 0, s, dg->name_off.p, dg->names.p, n, dg->op.p, dg->w_rank.p, dg->w_shape.p,
            dg->w_train.p, depth.p, hall.p, sh.p);
  SP_CUDA(cudaMemsetAsync(gparent.p, 0, n * sizeof(int32_t), s));
  SP_CUDA(cudaMemsetAsync(residual.p, 0, n, s));
  SP_CUDA(cudaMemsetAsync(alive.p, 1, n, s));
  SP_CUDA(cudaMemsetAsync(collision.p, 0, sizeof(int32_t), s));
  SP_CUDA(cudaMemsetAsync(tie.p, 0, sizeof(int32_t), s));
  // level 1's group-count bound; later levels get theirs with the previous level's counters
  SP_CUDA(cudaMemsetAsync(st.p, 0, sizeof(HashStats), s));
  SP_LAUNCH(ctx, k_hg_keys1, gn, 256, 0, s, n, dg->name_off.p, dg->names.p, seed, hall.p, ppoly.p, pend.p, ph.p, rh.p,
            st.p);
  SP_CUDA(cudaMemcpyAsync(hst, st.p, sizeof(HashStats), cudaMemcpyDeviceToHost, s));
  SP_CUDA(cudaStreamSynchronize(s));
  g_d2h_bytes += sizeof(HashStats);
  tr.mark("prep+keys1");
  int64_t est = hst->est;
  std::vector<LevelBlocks> lblocks;
  int64_t nA = n;
  int32_t levels = 0;
  int64_t n_resid = 0;
  // the level's node states are read-only while the level runs; its end writes
  // the next level's into the other buffer (stale entries are older levels)
  uint8_t* cur = alive.p;
  uint8_t* nxt = alive2.p;
  for (int32_t level = 1; nA > 0; level++, std::swap(cur, nxt)) {
    if (level > D) throw Error(SP_ERR_CUDA, "fold did not terminate");
    const int32_t dd = level - 1;
    const uint64_t* ph_l = ph.p;
    const uint64_t* rh_l = rh.p;
    // 1. groups: find-or-insert the prefix hash into a table of >= 2 x the
    //    group-count bound (no overflow possible; every later per-group array
    //    and the class table are sized by the bound, the exact count stays on
    //    the device until the level's one host sync)
    const int64_t gmax = std::max<int64_t>(1, std::min<int64_t>(est, nA));
    const uint32_t cap = table_cap(gmax);
    tkey.alloc(cap, s);
    thead.alloc(cap, s);
    tgkey.alloc(cap, s);
    tcnt.alloc(cap, s);
    tgid.alloc(cap, s);
    SP_CUDA(cudaMemsetAsync(tkey.p, 0, (size_t)cap * 8, s));
    SP_CUDA(cudaMemsetAsync(tgkey.p, 0, (size_t)cap * 8, s));
    SP_CUDA(cudaMemsetAsync(tcnt.p, 0, (size_t)cap * 4, s));
    SP_CUDA(cudaMemsetAsync(st.p, 0, sizeof(HashStats), s));
    tr.mark("level alloc");
    SP_LAUNCH(ctx, k_hg_insert, gn, 256, 0, s, n, cur, level, ph_l, tkey.p, thead.p, cap - 1, cap, nslot.p, st.p);
    // 2. group sizes and template-key sums per slot; head flags
    SP_LAUNCH(ctx, k_hg_entry, gn, 256, 0, s, n, cur, level, nslot.p, rh_l, sh.p, dg->in_off.p, dg->in_idx.p, thead.p,
              hf.p, tgkey.p, tcnt.p);
    // 3. compact group ids (heads in node order) and per-group arrays
    {
      size_t t = ctx->cub_tmp.n;
      ctx->cub_calls++;
      SP_CUDA(cub::DeviceScan::InclusiveSum(ctx->cub_tmp.p, t, hf.p, hs.p, (int)n, s));
    }
    gnode.alloc(gmax, s);
    gsize.alloc(gmax + 1, s);
    gkey.alloc(gmax, s);
    gpar.alloc(gmax, s);
    gstart.alloc(gmax + 1, s);
    gfill.alloc(gmax, s);
    gcs.alloc(gmax, s);
    gaccept.alloc(gmax, s);
    SP_CUDA(cudaMemsetAsync(gsize.p, 0, (size_t)(gmax + 1) * 4, s));
    SP_LAUNCH(ctx, k_hg_ids, gn, 256, 0, s, n, hf.p, hs.p, nslot.p, tgkey.p, tcnt.p, gparent.p, tgid.p, gnode.p,
              gsize.p, gkey.p, gpar.p);
    {
      size_t t = 0;
      cub::DeviceScan::ExclusiveSum(nullptr, t, gsize.p, gstart.p, (int)(gmax + 1), s);
      if (t > ctx->cub_tmp.n) ctx->cub_tmp.alloc(t, s);
      t = ctx->cub_tmp.n;
      ctx->cub_calls++;
      SP_CUDA(cub::DeviceScan::ExclusiveSum(ctx->cub_tmp.p, t, gsize.p, gstart.p, (int)(gmax + 1), s));
    }
    // 4. classes (over the groups g < nG, the count read on the device)
    const uint32_t ccap = table_cap(gmax);
    ckey.alloc(ccap, s);
    chead.alloc(ccap, s);
    ccnt.alloc(ccap, s);
    SP_CUDA(cudaMemsetAsync(ckey.p, 0, (size_t)ccap * 8, s));
    SP_CUDA(cudaMemsetAsync(ccnt.p, 0, (size_t)ccap * 4, s));
    const int gg = grid_for(gmax, sms);
    SP_LAUNCH(ctx, k_hc_insert, gg, 256, 0, s, gmax, &st.p->nG, gkey.p, gsize.p, gpar.p, ckey.p, chead.p, ccap - 1,
              gcs.p, st.p);
    SP_LAUNCH(ctx, k_hc_count, gg, 256, 0, s, gmax, &st.p->nG, gcs.p, ccnt.p);
    // 5. member segments + canonical order (multi-group / accepted classes only)
    SP_CUDA(cudaMemsetAsync(gfill.p, 0, (size_t)gmax * 4, s));
    SP_LAUNCH(ctx, k_hg_place, gn, 256, 0, s, n, cur, level, nslot.p, tgid.p, gcs.p, ccnt.p, min_dup, gstart.p,
              gfill.p, seg.p, li.p);
    SP_LAUNCH(ctx, k_hg_rank, gn, 256, 0, s, n, cur, level, nslot.p, tgid.p, gcs.p, ccnt.p, min_dup, gstart.p,
              gsize.p, seg.p, li.p, rh_l, sorted.p, pos.p, collision.p, st.p);
    // 6. exact verification, accept / residual / descend, the next level's keys
    SP_LAUNCH(ctx, k_hg_finish, gn, 128, 0, s, n, cur, nxt, level, D, nslot.p, tgid.p, gcs.p, ccnt.p, chead.p,
              gnode.p, gsize.p, gpar.p, gstart.p, sorted.p, pos.p, pend.p, dg->name_off.p, dg->names.p, dg->op.p,
              dg->w_rank.p, dg->w_shape.p, dg->w_train.p, dg->in_off.p, dg->in_idx.p, depth.p, min_dup, gparent.p,
              residual.p, gaccept.p, seed, hall.p, ppoly.p, ph.p, rh.p, collision.p, st.p);
    tr.mark("level enqueue");
    SP_CUDA(cudaMemcpyAsync(hst, st.p, sizeof(HashStats), cudaMemcpyDeviceToHost, s));
    SP_CUDA(cudaStreamSynchronize(s));
    g_d2h_bytes += sizeof(HashStats);
    tr.mark("level sync");
    levels++;
    if (hst->overflow) throw Error(SP_ERR_CUDA, "fold group table overflow");
    if (hst->big) {
      *fallback = true;
      return;
    }
    const int64_t nG = hst->nG;
    // accepted classes -> blocks (gclass = class table slot: any unique id works)
    if (hst->nacc) {
      lblocks.emplace_back();
      level_blocks(ctx, dg, dd, nA, nG, sorted.p, gstart.p, (const int32_t*)gcs.p, gaccept.p, pend.p, 1, n, tie.p,
                   lblocks.back(), hst->nacc);
      if (tr.on)
        fprintf(stderr, "[fold] level %d: nA %lld nG %lld nacc %d -> K %lld Ga %lld M %lld\n", level, (long long)nA,
                (long long)nG, hst->nacc, (long long)lblocks.back().K, (long long)lblocks.back().Ga,
                (long long)lblocks.back().M);
      tr.mark("level: blocks");
    }
    nA = hst->nnext;
    est = hst->est;
    n_resid += hst->nres;
  }
  SP_CUDA(cudaEventRecord(ctx->ev[7], s));
  // residual singletons compacted on the device (their count is the levels'
  // sum), then ONE copy of everything the host needs, flags included
  DevBuf<int32_t> iota, rlist, nsel2;
  iota.alloc(n, s);
  rlist.alloc(n, s);
  nsel2.alloc(1, s);
  SP_LAUNCH(ctx, k_iota, grid_for(n, sms), 256, 0, s, iota.p, n);
  size_t tb = 0;
  ctx->cub_calls++;
  SP_CUDA(cub::DeviceSelect::Flagged(nullptr, tb, iota.p, residual.p, rlist.p, nsel2.p, (int)n, s));
  DevBuf<uint8_t> tmp2;
  tmp2.alloc(tb, s);
  SP_CUDA(cub::DeviceSelect::Flagged(tmp2.p, tb, iota.p, residual.p, rlist.p, nsel2.p, (int)n, s));
  tr.mark("residuals");
  int32_t flags[2] = {0, 0};
  fold_finalize_blocks(dg, lblocks, {}, s, out, rlist.p, n_resid, collision.p, tie.p, flags);
  {
    float ms = 0;
    SP_CUDA(cudaEventElapsedTime(&ms, ctx->ev[6], ctx->ev[7]));
    ctx->fold_device_ms = ms;
    ctx->fold_levels = levels;
  }
  *collided = flags[0] != 0;
  if (!*collided && flags[1]) *fallback = true;
  tr.mark("finalize");
}

void fold_run(sp_ctx* ctx, sp_dgraph* dg, int32_t min_dup, sp_fold* out) {
  if (min_dup < 1) throw Error(SP_ERR_CONFIG, "min_duplicates must be >= 1");
  bool collided = false;
  for (int attempt = 0; attempt < 8; attempt++) {
    const uint64_t seed = 0x243f6a8885a308d3ULL + 0x9e3779b97f4a7c15ULL * (uint64_t)attempt;
    if (dg->n <= SMALL_MAX && dg->max_depth <= 64 && !getenv("SP_FOLD_MULTI")) {
      fold_once_small(ctx, dg, min_dup, seed, out, &collided);
    } else {
      // the hash-grouped path; SP_FOLD_SORT=1 selects the sort-based one (A/B, fallback)
      bool fallback = getenv("SP_FOLD_SORT") != nullptr;
      if (!fallback) fold_once_hash(ctx, dg, min_dup, seed, out, &collided, &fallback);
      if (fallback && !collided) fold_once(ctx, dg, min_dup, seed, out, &collided);
    }
    if (!collided) return;
  }
  throw Error(SP_ERR_CUDA, "fold hash verification failed on every seed");
}

}  // namespace sp
