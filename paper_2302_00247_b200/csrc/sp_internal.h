// Internal declarations shared by the backend translation units.
#pragma once

#include <cuda_runtime.h>

#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <memory>
#include <mutex>
#include <string>
#include <utility>
#include <vector>

#include "../../include/shardsearch.h"

namespace sp {

// Host-side phase timer of an entry point (SP_TRACE=1): one stderr line per mark.
struct Trace {
  const char* tag;
  bool on;
  std::chrono::steady_clock::time_point t0, last;
  explicit Trace(const char* t) : tag(t), on(getenv("SP_TRACE") != nullptr) {
    if (on) t0 = last = std::chrono::steady_clock::now();
  }
  void mark(const char* what) {
    if (!on) return;
    const auto now = std::chrono::steady_clock::now();
    fprintf(stderr, "[%s] %-24s %8.1f us (total %8.1f)\n", tag, what,
            std::chrono::duration<double, std::micro>(now - last).count(),
            std::chrono::duration<double, std::micro>(now - t0).count());
    last = now;
  }
};

// Error carrying an sp_status code; converted at the C boundary (capi.cu).
struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

#define SP_CUDA(call)                                                                     \
  do {                                                                                    \
    cudaError_t e_ = (call);                                                              \
    if (e_ != cudaSuccess)                                                                \
      throw ::sp::Error(SP_ERR_CUDA, std::string(#call) + ": " + cudaGetErrorString(e_)); \
  } while (0)

// Host<->device bytes moved by the library (bench `e2e` h2d/d2h accounting).
inline std::atomic<int64_t> g_h2d_bytes{0}, g_d2h_bytes{0};

// Kernel launch that also counts toward sp_launch_counts (bench `gpu_launches`).
#define SP_LAUNCH(ctx, kernel, grid, block, smem, stream, ...) \
  do {                                                           \
    (ctx)->own_launches++;                                       \
    kernel<<<grid, block, smem, stream>>>(__VA_ARGS__);          \
  } while (0)

// Stream-ordered cache of small device blocks (<= 1 MiB, power-of-two size
// classes): a block released on stream s is handed to the next allocation of
// its class on s -- work queued on s after the release is ordered after the
// work that used it, exactly the guarantee cudaFreeAsync + cudaMallocAsync on
// s give -- without a CUDA API call.  A tiny search allocates and frees ~20
// scratch buffers per call (~1 us of driver time each); large buffers still
// go through the stream-ordered pool.  Blocks are returned with
// devcache_drop(stream) before the stream is destroyed.
constexpr int DEVCACHE_MIN_LOG = 8, DEVCACHE_MAX_LOG = 20;
struct DevCache {
  struct Entry {
    cudaStream_t s;
    std::vector<void*> free_[DEVCACHE_MAX_LOG - DEVCACHE_MIN_LOG + 1];
  };
  std::mutex m;
  std::vector<Entry> streams;
  Entry& of(cudaStream_t s) {
    for (auto& e : streams)
      if (e.s == s) return e;
    streams.push_back(Entry{s, {}});
    return streams.back();
  }
};
inline DevCache& devcache() {
  static DevCache* c = new DevCache();  // never destroyed: released per stream
  return *c;
}
inline int devcache_class(size_t bytes) {
  if (bytes > ((size_t)1 << DEVCACHE_MAX_LOG)) return -1;
  int c = DEVCACHE_MIN_LOG;
  while (((size_t)1 << c) < bytes) c++;
  return c - DEVCACHE_MIN_LOG;
}
inline void* devcache_get(cudaStream_t s, int cls) {
  DevCache& c = devcache();
  std::lock_guard<std::mutex> lock(c.m);
  auto& v = c.of(s).free_[cls];
  if (v.empty()) return nullptr;
  void* p = v.back();
  v.pop_back();
  return p;
}
inline void devcache_put(cudaStream_t s, int cls, void* p) {
  DevCache& c = devcache();
  std::lock_guard<std::mutex> lock(c.m);
  c.of(s).free_[cls].push_back(p);
}
inline void devcache_drop(cudaStream_t s) {
  DevCache& c = devcache();
  std::lock_guard<std::mutex> lock(c.m);
  for (size_t i = 0; i < c.streams.size(); i++)
    if (c.streams[i].s == s) {
      for (auto& v : c.streams[i].free_)
        for (void* p : v) cudaFreeAsync(p, s);
      c.streams.erase(c.streams.begin() + (std::ptrdiff_t)i);
      return;
    }
}

// Owning device allocation (cudaMallocAsync on the context stream, small ones
// through DevCache).
template <class T>
struct DevBuf {
  T* p = nullptr;
  size_t n = 0;
  cudaStream_t s = nullptr;
  bool view = false;  // p points into memory another buffer owns
  int8_t cls = -1;    // DevCache size class of p, -1: from the pool
  DevBuf() = default;
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  DevBuf(DevBuf&& o) noexcept : p(o.p), n(o.n), s(o.s), view(o.view), cls(o.cls) {
    o.p = nullptr; o.n = 0; o.view = false; o.cls = -1;
  }
  DevBuf& operator=(DevBuf&& o) noexcept {
    if (this != &o) {
      release();
      p = o.p; n = o.n; s = o.s; view = o.view; cls = o.cls;
      o.p = nullptr; o.n = 0; o.view = false; o.cls = -1;
    }
    return *this;
  }
  ~DevBuf() { release(); }
  void release() {
    if (p && !view) {
      if (cls >= 0) devcache_put(s, cls, p);
      else cudaFreeAsync(p, s);
    }
    p = nullptr;
    n = 0;
    view = false;
    cls = -1;
  }
  // view `count` elements at `at` (owned elsewhere, e.g. a packed upload arena)
  void set_view(T* at, size_t count) {
    release();
    p = at;
    n = count;
    view = true;
  }
  void alloc(size_t count, cudaStream_t stream) {
    if (count <= n && p && !view) return;
    release();
    s = stream;
    n = count;
    const size_t bytes = (count ? count : 1) * sizeof(T);
    const int c = devcache_class(bytes);
    if (c >= 0) {
      p = (T*)devcache_get(stream, c);
      if (!p) SP_CUDA(cudaMallocAsync(&p, (size_t)1 << (c + DEVCACHE_MIN_LOG), stream));
      cls = (int8_t)c;
      return;
    }
    SP_CUDA(cudaMallocAsync(&p, bytes, stream));
  }
  void upload(const T* h, size_t count, cudaStream_t stream) {
    alloc(count, stream);
    g_h2d_bytes += (int64_t)(count * sizeof(T));
    if (count) SP_CUDA(cudaMemcpyAsync(p, h, count * sizeof(T), cudaMemcpyHostToDevice, stream));
  }
  void download(T* h, size_t count, cudaStream_t stream) const {
    g_d2h_bytes += (int64_t)(count * sizeof(T));
    if (count) SP_CUDA(cudaMemcpyAsync(h, p, count * sizeof(T), cudaMemcpyDeviceToHost, stream));
  }
  void zero(cudaStream_t stream) {
    if (n) SP_CUDA(cudaMemsetAsync(p, 0, n * sizeof(T), stream));
  }
};

// Several host arrays to the device with ONE copy: packed (16-byte aligned)
// into a pinned staging block, copied into one device arena; add() returns
// each array's device address.  The staging block and the arena live as long
// as the Packed object (its owner frees it after syncing the stream).
struct PackedUpload {
  struct Part {
    const void* src;
    size_t bytes, off;
  };
  std::vector<Part> parts;
  size_t total = 0;
  size_t add(const void* src, size_t bytes) {
    parts.push_back({src, bytes, total});
    const size_t at = total;
    total += (bytes + 15) & ~(size_t)15;
    return at;
  }
};

}  // namespace sp

namespace sp {
// std::vector element allocator that leaves new elements uninitialised
// (resize of a 10^7-entry output must not memset what is overwritten next)
template <class T>
struct NoInitAlloc : std::allocator<T> {
  template <class U>
  struct rebind {
    using other = NoInitAlloc<U>;
  };
  NoInitAlloc() = default;
  template <class U>
  NoInitAlloc(const NoInitAlloc<U>&) noexcept {}
  template <class U>
  void construct(U* p) noexcept {
    ::new ((void*)p) U;
  }
  template <class U, class... A>
  void construct(U* p, A&&... a) {
    ::new ((void*)p) U(std::forward<A>(a)...);
  }
};
template <class T>
using PodVec = std::vector<T, NoInitAlloc<T>>;
}  // namespace sp

// The host copies a device graph keeps (sp_dgraph::h_*), recycled across
// uploads by the context: a fresh 20 MB of host vectors per upload is ~5k
// first-touch page faults (~1.2 ms at 10^5 nodes) on every e2e step.
struct HostGraphCopies {
  sp::PodVec<uint8_t> names, op, w_rank, w_train;
  sp::PodVec<int64_t> name_off, topo, in_off;
  sp::PodVec<int32_t> in_idx;
};

struct sp_ctx {
  int device = 0;
  int sm_count = 148;
  size_t smem_optin = 0;
  cudaStream_t stream = nullptr;
  cudaStream_t aux = nullptr;  // explain_all of a group while another search runs on `stream`
  cudaEvent_t ev[8] = {};

  std::string last_error;
  double fold_ms = 0, score_ms = 0, score_kernel_ms = 0;
  // device-only part of the last fold (events around the level loop) and its level count
  double fold_device_ms = 0;
  int32_t fold_levels = 0;
  int64_t own_launches = 0, cub_calls = 0;
  int skip = 1;  // exact prefix-failure skipping in sp_score / sp_search
  int host_layout = 1;  // small graphs: table layout on the host (SP_OPT_HOST_LAYOUT)
  int sim_rank = 0, sim_nranks = 1;  // SP_OPT_SIM_SHARD (measurement only)
  int memo = 0;  // with skip off: memoised brute force (re-route only dirty nodes); off: walk
  cudaEvent_t timer[2] = {};
  cudaEvent_t trace[4] = {};  // SP_SCORE_TRACE: reduce / explain / d2h boundaries
  // scratch reused across calls
  sp::DevBuf<uint8_t> cub_tmp;
  void* staging = nullptr;  // pinned host staging for graph uploads
  size_t staging_bytes = 0;
  // free pinned host blocks for score results (D2H enqueued at launch time)
  std::vector<std::pair<void*, size_t>> pinned_pool;
  // resident CTAs per SM by (kernel, smem): the runtime query costs ~10 us per launch
  std::vector<std::pair<std::pair<const void*, size_t>, int>> occupancy;
  std::vector<cudaEvent_t> event_pool;  // timing events of finished searches, reused
  std::vector<HostGraphCopies> host_copies;  // spare sp_dgraph host vectors (graph_upload / sp_graph_free)
  // multi-GPU (comm.cu).  Every device is a lane: this context's own
  // communicator handle (ncclComm_t), its rank among `nranks`, and how the
  // lanes exchange their per-block records (SP_TRANSPORT_*).  A context made
  // by sp_ctx_create(ngpu > 1, ...) is the primary lane and drives the others
  // (`peers`, devices[1..]); a process-per-GPU context has no peers and joins
  // a communicator with sp_ctx_comm_init.
  void* comm = nullptr;
  int32_t nranks = 1, rank = 0;
  int32_t transport = SP_TRANSPORT_NONE;
  std::vector<sp_ctx*> peers;
};

namespace sp {
// Pinned host block of at least `need` bytes from the context's pool (best
// fit; allocated when none fits).  Blocks go back with pinned_release.
inline uint8_t* pinned_acquire(sp_ctx* ctx, size_t need, size_t* got) {
  auto& pool = ctx->pinned_pool;
  size_t best = pool.size();
  for (size_t i = 0; i < pool.size(); i++)
    if (pool[i].second >= need && (best == pool.size() || pool[i].second < pool[best].second)) best = i;
  if (best < pool.size()) {
    uint8_t* p = (uint8_t*)pool[best].first;
    *got = pool[best].second;
    pool.erase(pool.begin() + (std::ptrdiff_t)best);
    return p;
  }
  const size_t n = need > ((size_t)64 << 10) ? need : ((size_t)64 << 10);
  void* p = nullptr;
  SP_CUDA(cudaHostAlloc(&p, n, cudaHostAllocDefault));
  *got = n;
  return (uint8_t*)p;
}
inline void pinned_release(sp_ctx* ctx, void* p, size_t n) {
  if (p) ctx->pinned_pool.push_back({p, n});
}
// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) only when `smem` exceeds
// what was already allowed for `kern`.  The attribute belongs to the function
// in the whole process (every context, every device of it), so the record is
// process-wide and the limit only ever grows: a context that needs less must
// not lower it under another context's launches.
inline std::mutex& smem_mutex() {
  static std::mutex m;
  return m;
}
inline std::vector<std::pair<std::pair<const void*, int>, int>>& smem_limits() {
  static std::vector<std::pair<std::pair<const void*, int>, int>> v;  // ((kernel, device), bytes)
  return v;
}
template <class K>
inline void allow_smem(sp_ctx* ctx, K* kern, size_t smem) {
  std::lock_guard<std::mutex> lock(smem_mutex());
  const std::pair<const void*, int> key{(const void*)kern, ctx->device};
  for (auto& e : smem_limits())
    if (e.first == key) {
      if ((size_t)e.second >= smem) return;
      SP_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      e.second = (int)smem;
      return;
    }
  SP_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  smem_limits().push_back({key, (int)smem});
}
// resident CTAs per SM of `kern` at `threads` x `smem` (cached per context)
template <class K>
inline int resident_ctas(sp_ctx* ctx, K* kern, int threads, size_t smem) {
  const std::pair<const void*, size_t> key{(const void*)kern, smem * 4096 + (size_t)threads};
  for (const auto& e : ctx->occupancy)
    if (e.first == key) return e.second;
  int per_sm = 0;
  SP_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, threads, smem));
  ctx->occupancy.push_back({key, per_sm});
  return per_sm;
}
}  // namespace sp

// Device-resident lowered graph (+ the host copies the library needs).
constexpr int64_t SP_HOST_LAYOUT_MAX = 8192;

struct sp_dgraph {
  sp_ctx* ctx = nullptr;
  int64_t n = 0, E = 0;
  int32_t max_depth = 1;
  // host copies the library needs (string order, slot order, op validity)
  sp::PodVec<uint8_t> h_names;  // filled by graph_upload's parallel copies (no zero fill)
  sp::PodVec<int64_t> h_name_off, h_topo;
  sp::PodVec<uint8_t> h_op, h_w_rank;
  // graphs of <= SP_HOST_LAYOUT_MAX nodes also keep the producer CSR and the
  // trainable flags: their table layout is computed on the host (no device
  // round trip between the fold and the fill)
  sp::PodVec<int64_t> h_in_off;
  sp::PodVec<int32_t> h_in_idx;
  sp::PodVec<uint8_t> h_w_train;
  // device copies: views into one arena filled by a single H2D copy
  sp::DevBuf<uint8_t> arena;
  template <class T>
  struct View {
    T* p = nullptr;
  };
  View<uint8_t> names, op, act_rank, w_rank, w_train;
  View<int64_t> name_off, topo, act_shape, act_bytes, w_shape, w_bytes, in_off;
  View<int32_t> in_idx;
  std::vector<sp_dgraph*> peers;  // the same graph on every peer lane of a multi-device context
  // the one-CTA fold's per-node name hashes (prefix / rel hash and prefix end
  // per depth, node depth): a function of the names and the seed only, kept
  // from the first search of the graph (ph | rh | pend | depth)
  sp::DevBuf<uint8_t> name_hash;
  uint64_t name_hash_seed = 0;
  int32_t name_hash_D = -1;
};


struct sp_fold {
  std::vector<int64_t> block_T, block_inst_off, block_member_off;
  sp::PodVec<int64_t> inst_prefix_node, inst_prefix_len;
  sp::PodVec<int32_t> members;
  sp_blocks view{};
};

// One block's table blob header (lives at the start of each blob in HBM and smem).
struct BlobHeader {
  uint64_t C;             // candidate count
  uint64_t radix3;        // bit q set: ENUMERATION position q has 3 options, else 2
  int32_t T, V, nt, npool;
  int32_t desc_off, prod_off, tab_off, dbl_off;  // byte offsets from blob start
  int32_t train_off, bytes, multi_dev, n_prod;    // multi_dev: device_count > 1; n_prod: internal edges
  double setup, c_ar, bw, eff_ar, keep_bwd;       // keep_bwd = 1.0 - overlap_fraction
  int64_t mu, chunk;
  uint64_t radix3_ref;    // bit s set: REFERENCE slot s (weight_nodes order) has 3 options
  int32_t skip_off;       // NodeSkip[T]
  int32_t stride_off;     // u64 reference stride per enumeration position, then int8 perm[V]
  int32_t dirty_off;      // u64 dirty[V+1]: nodes whose ancestor cone reaches position >= q (T <= 64)
  int32_t pad3;
  // lean walk (biased digits): FastNode[T], a zero block, (reach, state) offset
  // pairs of producers of fan-in >= 3 nodes, and 4-row routing tables
  int32_t fast_off, zero_off, fprod_off, tab4_off;
  // pack_gradients on the biased digit word (V <= 32): bias = the word of all-zero
  // digits; bit 2(V-1-q) of tmask_small / tmask_big set when enumeration
  // position q holds a trainable weight smaller than / at least mu
  uint64_t bias, tmask_small, tmask_big;
  int32_t tslot_off;  // double uterm[V], then int64 size[V]: each trainable weight's by enumeration position
  int32_t pad4;
};
static_assert(sizeof(BlobHeader) % 16 == 0, "blob header must stay 16-byte aligned");

// Per-node record of the lean scoring walk: every field is a ready-to-use
// shared-memory byte offset, so the walk does no unpacking beyond shifts.  The
// routing table of a node has 4 rows indexed by the node's BIASED digit field
// (row = digit + 4 - radix; unweighted nodes replicate their single row 4
// times), each row 3^k bytes keyed by the producer states in base 3.  A live
// value's state byte sits at 1/8 of its reach offset (reach at pool +
// (p*THREADS + t)*8, state at pool_states + p*THREADS + t), so the state
// offsets are not stored: two 16-byte loads per node instead of three.
struct __align__(16) FastNode {
  int32_t tab;           // smem offset of the node's 4-row routing table
  int32_t dbl;           // smem offset of own[4]; exitc[4] follows
  int32_t cb0, cb1;      // smem offsets of conv[0], conv[1] ([4][3] doubles; zero block if absent)
  int32_t r0, r1;        // reach byte offsets of producers 0/1 in the lane pool (k >= 3: fprod pair index)
  int32_t out_r;         // output reach offset (< 0: no internal consumer)
  int32_t kf;            // k << 16 | boundary << 13 | min(k,3) << 11 | one-hot kind << 8 | digit shift (0..62)
};
static_assert(sizeof(FastNode) == 32, "FastNode is two 16-byte smem loads");

struct __align__(16) NodeDesc {
  int16_t slot;      // weight slot (enumeration position) or -1
  uint8_t k;         // internal producers
  uint8_t nd;        // digit options (1 when unweighted)
  int16_t out_pool;  // pool slot receiving reach/state, -1 when no internal consumer
  uint16_t prod;     // index of first producer pool slot (int16 array)
  uint32_t tab;      // entry table byte offset within the entry section
  uint32_t dbl;      // double offset within the double section (own[4], exitc[4], conv[k][4][3])
};
static_assert(sizeof(NodeDesc) == 16, "NodeDesc is one 16-byte smem load");

// Exact prefix-failure skipping: if node i fails, every candidate that keeps
// the digits of the enumeration positions 0..m of its ancestor cone fails too,
// so the enumeration may jump to the next multiple of R = prod radix(q > m).
struct NodeSkip {
  uint64_t R;  // skip modulus (0 when the node has no weighted ancestor: skip to the end)
  int32_t m;   // highest enumeration position in the node's ancestor cone, -1 if none
  int32_t pad;
};
static_assert(sizeof(NodeSkip) == 16, "NodeSkip layout");

struct TrainDesc {
  int32_t slot;
  int32_t pad;
  int64_t size;
  double uterm;  // setup + AR(size) for an unfused gradient
};

struct sp_tables {
  sp_ctx* ctx = nullptr;
  int64_t n_blocks = 0;
  std::vector<BlobHeader> hdr;           // host copy of every block header
  std::vector<int64_t> blob_off;         // byte offset of each block blob
  std::vector<int64_t> edge_off;         // internal-edge offset of each block (explain output)
  std::vector<std::vector<int32_t>> slot_pos;  // weight slot -> template position
  std::vector<int64_t> tmpl_off;
  std::vector<int32_t> tmpl_nodes;
  int64_t max_blob = 0;
  int32_t max_pool = 0;
  int32_t max_T = 0;
  bool overflow = false;                 // some block has > 2^64 candidates
  sp::DevBuf<uint8_t> blobs;
  sp::DevBuf<int64_t> d_blob_off;
  sp::DevBuf<int32_t> d_tmpl_nodes;
  sp::DevBuf<int64_t> d_tmpl_off;
  sp_dgraph* dg = nullptr;
  void* priv = nullptr;  // sp::TablesPriv (device maps used by explain)
  std::vector<sp_tables*> peers;  // the same tables on every peer lane of a multi-device context
};

namespace sp {
void graph_upload(sp_ctx* ctx, const sp_graph* g, sp_dgraph* dg);
void fold_run(sp_ctx* ctx, sp_dgraph* dg, int32_t min_dup, sp_fold* out);
void tables_wait_built(sp_tables* t);
void tables_build(sp_ctx* ctx, sp_dgraph* dg, int64_t n_blocks, const int64_t* tmpl_off,
                  const int32_t* tmpl_nodes, const sp_mesh* mesh, int64_t mu, int64_t chunk,
                  sp_tables* out);
void score_all(sp_ctx* ctx, sp_tables* t, int32_t shard, int32_t n_shards, sp_score_out* out,
               void* xblocks = nullptr, int8_t* xnode = nullptr, int8_t* xedge = nullptr);
void score_launch(sp_ctx* ctx, sp_tables* t, int32_t shard, int32_t n_shards, bool explain, bool local = false);
void score_wait(sp_ctx* ctx, sp_tables* t, sp_score_out* out, void* xblocks, int8_t* xnode, int8_t* xedge);
void score_range(sp_ctx* ctx, sp_tables* t, int64_t block, uint64_t lo, uint64_t hi,
                 double* totals, sp_score_out* out);
void explain(sp_ctx* ctx, sp_tables* t, int64_t block, uint64_t index, sp_explain_out* out,
             sp_edge_conv* edges, int32_t max_edges, int32_t* n_edges);
void merge_key(sp_score_out* acc, const sp_score_out* o);
void tables_free_priv(sp_tables* t);
void explain_all(sp_ctx* ctx, sp_tables* t, const uint64_t* indices, void* blocks_out, int8_t* node_out,
                 int8_t* edge_out);
void route_search(sp_ctx* ctx, sp_dgraph* dg, int64_t nb, const int64_t* tmpl_off, const int32_t* tmpl_nodes,
                  const int16_t* ref_slot, const uint8_t* radix, const int64_t* edge_off, const sp_mesh* mesh,
                  int64_t mu, int64_t chunk, const uint64_t* indices, sp_score_out* scores, void* xblocks,
                  int8_t* xnode, int8_t* xedge);
// comm.cu: NCCL, loaded with dlopen on first use
int nccl_version();
void nccl_unique_id(uint8_t* out);
void nccl_init_rank(sp_ctx* ctx, int nranks, int rank, const uint8_t* id);
void nccl_init_all(const std::vector<sp_ctx*>& lanes);
void nccl_destroy(sp_ctx* ctx);
void nccl_group_start();
void nccl_group_end();
void nccl_allgather(sp_ctx* ctx, const void* send, void* recv, size_t bytes);
}  // namespace sp
