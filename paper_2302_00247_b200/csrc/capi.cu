// extern "C" boundary (include/shardsearch.h): exception -> status code,
// per-context last-error string, device timing accessors.
#include <cstdio>

#include "sp_internal.h"

namespace {

template <class F>
int guard(sp_ctx* ctx, F&& f) {
  try {
    // a non-sticky error some other CUDA user left in this thread's last-error
    // slot would otherwise surface at this call's first launch check
    cudaGetLastError();
    f();
    if (ctx) ctx->last_error.clear();
    return SP_OK;
  } catch (const sp::Error& e) {
    if (ctx) ctx->last_error = e.what();
    return e.code;
  } catch (const std::bad_alloc&) {
    if (ctx) ctx->last_error = "host allocation failed";
    return SP_ERR_CUDA;
  } catch (const std::exception& e) {
    if (ctx) ctx->last_error = e.what();
    return SP_ERR_CUDA;
  }
}

}  // namespace

extern "C" {

int sp_abi_version(void) { return SP_ABI_VERSION; }

static sp_ctx* ctx_create_one(int device) {
  sp_ctx* ctx = new sp_ctx();
  int rc = guard(ctx, [&] {
    SP_CUDA(cudaSetDevice(device));
    ctx->device = device;
    SP_CUDA(cudaDeviceGetAttribute(&ctx->sm_count, cudaDevAttrMultiProcessorCount, device));
    int optin = 0;
    SP_CUDA(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, device));
    ctx->smem_optin = (size_t)optin;
    SP_CUDA(cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking));
    SP_CUDA(cudaStreamCreateWithFlags(&ctx->aux, cudaStreamNonBlocking));
    // every scratch buffer is stream-ordered (cudaMallocAsync): keep freed
    // memory in the device pool instead of returning it at each sync, so the
    // per-call buffers of fold / tables / score are re-used, not re-mapped
    cudaMemPool_t pool;
    SP_CUDA(cudaDeviceGetDefaultMemPool(&pool, device));
    uint64_t keep = UINT64_MAX;
    SP_CUDA(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep));
    for (auto& e : ctx->ev) SP_CUDA(cudaEventCreate(&e));
    for (auto& e : ctx->timer) SP_CUDA(cudaEventCreate(&e));
    for (auto& e : ctx->trace) SP_CUDA(cudaEventCreate(&e));
  });
  if (rc != SP_OK) {
    std::fprintf(stderr, "sp_ctx_create: %s\n", ctx->last_error.c_str());
    delete ctx;
    return nullptr;
  }
  return ctx;
}

static void ctx_destroy_one(sp_ctx* ctx) {
  cudaSetDevice(ctx->device);
  ctx->cub_tmp.release();
  if (ctx->stream) cudaStreamSynchronize(ctx->stream);
  if (ctx->comm) sp::nccl_destroy(ctx);
  if (ctx->staging) cudaFreeHost(ctx->staging);
  for (auto& b : ctx->pinned_pool) cudaFreeHost(b.first);
  for (auto e : ctx->event_pool) cudaEventDestroy(e);
  for (auto& e : ctx->ev)
    if (e) cudaEventDestroy(e);
  for (auto& e : ctx->timer)
    if (e) cudaEventDestroy(e);
  if (ctx->aux) {
    sp::devcache_drop(ctx->aux);
    cudaStreamSynchronize(ctx->aux);
    cudaStreamDestroy(ctx->aux);
  }
  if (ctx->stream) {
    sp::devcache_drop(ctx->stream);
    cudaStreamSynchronize(ctx->stream);
    cudaStreamDestroy(ctx->stream);
  }
  delete ctx;
}

int sp_ctx_create(int ngpu, const int* devices, sp_ctx** out) {
  if (!out || ngpu < 1 || !devices) return SP_ERR_CONFIG;
  *out = nullptr;
  std::vector<sp_ctx*> lanes;
  for (int i = 0; i < ngpu; i++) {
    sp_ctx* c = ctx_create_one(devices[i]);
    if (!c) {
      for (sp_ctx* l : lanes) ctx_destroy_one(l);
      return SP_ERR_CUDA;
    }
    lanes.push_back(c);
  }
  sp_ctx* P = lanes[0];
  if (ngpu > 1) {
    bool distinct = true;
    for (int i = 0; i < ngpu; i++)
      for (int j = 0; j < i; j++) distinct = distinct && devices[i] != devices[j];
    const char* tr = getenv("SP_TRANSPORT");
    const bool p2p = !distinct || (tr && std::string(tr) == "p2p");
    int rc = guard(P, [&] {
      if (p2p) {
        for (int i = 0; i < ngpu; i++) {
          lanes[i]->nranks = ngpu;
          lanes[i]->rank = i;
          lanes[i]->transport = SP_TRANSPORT_P2P;
          // the records are copied onto the primary's device
          if (i && devices[i] != devices[0]) {
            int can = 0;
            SP_CUDA(cudaDeviceCanAccessPeer(&can, devices[0], devices[i]));
            if (can) {
              SP_CUDA(cudaSetDevice(devices[0]));
              cudaError_t e = cudaDeviceEnablePeerAccess(devices[i], 0);
              if (e == cudaErrorPeerAccessAlreadyEnabled) cudaGetLastError();
              else SP_CUDA(e);
            }
          }
        }
      } else {
        sp::nccl_init_all(lanes);
      }
    });
    if (rc != SP_OK) {
      std::fprintf(stderr, "sp_ctx_create: %s\n", P->last_error.c_str());
      for (sp_ctx* l : lanes) ctx_destroy_one(l);
      return rc;
    }
    P->peers.assign(lanes.begin() + 1, lanes.end());
    cudaSetDevice(devices[0]);
  }
  *out = P;
  return SP_OK;
}

void sp_ctx_destroy(sp_ctx* ctx) {
  if (!ctx) return;
  for (sp_ctx* p : ctx->peers) ctx_destroy_one(p);
  ctx->peers.clear();
  ctx_destroy_one(ctx);
}

int sp_comm_unique_id(uint8_t* id) {
  if (!id) return SP_ERR_CONFIG;
  return guard(nullptr, [&] { sp::nccl_unique_id(id); });
}

int sp_ctx_comm_init(sp_ctx* ctx, int32_t nranks, int32_t rank, const uint8_t* id) {
  if (!ctx || !id || nranks < 1 || rank < 0 || rank >= nranks) return SP_ERR_CONFIG;
  if (!ctx->peers.empty() || ctx->comm) {
    ctx->last_error = "context already has a communicator (multi-device or initialised)";
    return SP_ERR_CONFIG;
  }
  return guard(ctx, [&] { sp::nccl_init_rank(ctx, nranks, rank, id); });
}

int sp_ctx_comm_info(const sp_ctx* ctx, int32_t* nranks, int32_t* rank, int32_t* ndev, int32_t* transport,
                     int32_t* nccl_version) {
  if (!ctx) return SP_ERR_CONFIG;
  if (nranks) *nranks = ctx->nranks;
  if (rank) *rank = ctx->rank;
  if (ndev) *ndev = 1 + (int32_t)ctx->peers.size();
  if (transport) *transport = ctx->transport;
  if (nccl_version) {
    *nccl_version = 0;
    if (ctx->transport == SP_TRANSPORT_NCCL) {
      try {
        *nccl_version = sp::nccl_version();
      } catch (const std::exception&) {
      }
    }
  }
  return SP_OK;
}

const char* sp_last_error(const sp_ctx* ctx) { return ctx ? ctx->last_error.c_str() : "null context"; }

int sp_graph_upload(sp_ctx* ctx, const sp_graph* g, sp_dgraph** out) {
  if (!ctx || !g || !out) return SP_ERR_CONFIG;
  *out = nullptr;
  sp_dgraph* dg = new sp_dgraph();
  int rc = guard(ctx, [&] {
    SP_CUDA(cudaSetDevice(ctx->device));
    sp::graph_upload(ctx, g, dg);
    for (sp_ctx* p : ctx->peers) {  // the graph on every device of the context
      dg->peers.push_back(new sp_dgraph());
      SP_CUDA(cudaSetDevice(p->device));
      sp::graph_upload(p, g, dg->peers.back());
    }
    SP_CUDA(cudaSetDevice(ctx->device));
  });
  if (rc != SP_OK) {
    sp_graph_free(dg);
    return rc;
  }
  *out = dg;
  return SP_OK;
}

void sp_graph_free(sp_dgraph* dg) {
  if (!dg) return;
  for (sp_dgraph* p : dg->peers) sp_graph_free(p);
  dg->peers.clear();
  if (dg->ctx) {
    cudaSetDevice(dg->ctx->device);
    cudaStreamSynchronize(dg->ctx->stream);
    // keep the host vectors for the context's next upload (at most two sets)
    if (dg->ctx->host_copies.size() < 2) {
      HostGraphCopies hc;
      hc.names.swap(dg->h_names);
      hc.op.swap(dg->h_op);
      hc.w_rank.swap(dg->h_w_rank);
      hc.w_train.swap(dg->h_w_train);
      hc.name_off.swap(dg->h_name_off);
      hc.topo.swap(dg->h_topo);
      hc.in_off.swap(dg->h_in_off);
      hc.in_idx.swap(dg->h_in_idx);
      dg->ctx->host_copies.push_back(std::move(hc));
    }
  }
  delete dg;
}

int sp_fold_run(sp_ctx* ctx, sp_dgraph* dg, int32_t min_dup, sp_fold** out) {
  if (!ctx || !dg || !out) return SP_ERR_CONFIG;
  *out = nullptr;
  sp_fold* f = new sp_fold();
  int rc = guard(ctx, [&] {
    SP_CUDA(cudaSetDevice(ctx->device));
    SP_CUDA(cudaEventRecord(ctx->ev[4], ctx->stream));
    sp::Trace tr("fold_run");
    sp::fold_run(ctx, dg, min_dup, f);
    SP_CUDA(cudaEventRecord(ctx->ev[5], ctx->stream));
    SP_CUDA(cudaEventSynchronize(ctx->ev[5]));
    tr.mark("done");
    float ms = 0;
    SP_CUDA(cudaEventElapsedTime(&ms, ctx->ev[4], ctx->ev[5]));
    ctx->fold_ms = ms;
  });
  if (rc != SP_OK) {
    delete f;
    return rc;
  }
  *out = f;
  return SP_OK;
}

int sp_fold_view(const sp_fold* f, sp_blocks* view) {
  if (!f || !view) return SP_ERR_CONFIG;
  *view = f->view;
  return SP_OK;
}

void sp_fold_free(sp_fold* f) { delete f; }

int sp_tables_build(sp_ctx* ctx, sp_dgraph* dg, int64_t n_blocks, const int64_t* tmpl_off,
                    const int32_t* tmpl_nodes, const sp_mesh* mesh, int64_t mu, int64_t chunk_size,
                    sp_tables** out) {
  if (!ctx || !dg || !tmpl_off || !mesh || !out) return SP_ERR_CONFIG;
  *out = nullptr;
  sp_tables* t = new sp_tables();
  int rc = guard(ctx, [&] {
    SP_CUDA(cudaSetDevice(ctx->device));
    if (mesh->m < 1 || mesh->n < 1) throw sp::Error(SP_ERR_CONFIG, "mesh must be at least 1x1");
    sp::tables_build(ctx, dg, n_blocks, tmpl_off, tmpl_nodes, mesh, mu, chunk_size, t);
    if (dg->peers.size() != ctx->peers.size()) throw sp::Error(SP_ERR_CONFIG, "graph was not uploaded by this context");
    for (size_t i = 0; i < ctx->peers.size(); i++) {  // the tables on every device of the context
      t->peers.push_back(new sp_tables());
      SP_CUDA(cudaSetDevice(ctx->peers[i]->device));
      sp::tables_build(ctx->peers[i], dg->peers[i], n_blocks, tmpl_off, tmpl_nodes, mesh, mu, chunk_size,
                       t->peers.back());
    }
    SP_CUDA(cudaSetDevice(ctx->device));
  });
  if (rc != SP_OK) {
    sp_tables_free(t);
    return rc;
  }
  *out = t;
  return SP_OK;
}

void sp_tables_free(sp_tables* t) {
  if (!t) return;
  for (sp_tables* p : t->peers) sp_tables_free(p);
  t->peers.clear();
  sp::Trace tr("tables_free");
  if (t->ctx) {
    // the device buffers go back stream-ordered; only the build's own uploads
    // (pinned staging) must have run -- not whatever was queued behind them
    // (a cheap block group's tables are closed while the expensive group's
    // kernel still runs)
    cudaSetDevice(t->ctx->device);
    sp::tables_wait_built(t);
  }
  tr.mark("sync");
  sp::tables_free_priv(t);
  delete t;
  tr.mark("free");
}

struct sp_plan {
  sp_fold* fold = nullptr;
  std::vector<int64_t> toff, eoff;
  std::vector<int32_t> tnodes;
  std::vector<sp_score_out> scores;
  std::vector<sp_explain_block> detail;
  std::vector<int8_t> node, edge;
  // every array of the view packed into one block (16-byte aligned parts, in
  // the view's field order), so a caller maps the whole result with one buffer
  std::vector<uint8_t> arena;
  sp_plan_view view{};
  ~sp_plan() { delete fold; }
};

static void plan_pack(sp_plan* P) {
  const sp_blocks& B = P->fold->view;
  const int64_t nb = B.n_blocks;
  struct Part {
    const void* src;
    size_t bytes;
  };
  const Part parts[] = {
      {B.block_T, sizeof(int64_t) * (size_t)nb},
      {B.block_inst_off, sizeof(int64_t) * (size_t)(nb + 1)},
      {B.block_member_off, sizeof(int64_t) * (size_t)(nb + 1)},
      {B.inst_prefix_node, sizeof(int64_t) * (size_t)B.n_instances},
      {B.inst_prefix_len, sizeof(int64_t) * (size_t)B.n_instances},
      {B.members, sizeof(int32_t) * (size_t)B.n_members},
      {P->toff.data(), sizeof(int64_t) * P->toff.size()},
      {P->tnodes.data(), sizeof(int32_t) * P->tnodes.size()},
      {P->scores.data(), sizeof(sp_score_out) * P->scores.size()},
      {P->detail.data(), sizeof(sp_explain_block) * P->detail.size()},
      {P->node.data(), P->node.size()},
      {P->edge.data(), P->edge.size()},
      {P->eoff.data(), sizeof(int64_t) * P->eoff.size()},
  };
  constexpr int NP = sizeof(parts) / sizeof(parts[0]);
  size_t off[NP], total = 0;
  for (int i = 0; i < NP; i++) {
    off[i] = total;
    total += (parts[i].bytes + 15) & ~(size_t)15;
  }
  P->arena.resize(std::max<size_t>(total, 16));
  uint8_t* a = P->arena.data();
  for (int i = 0; i < NP; i++)
    if (parts[i].bytes) std::memcpy(a + off[i], parts[i].src, parts[i].bytes);
  sp_plan_view& v = P->view;
  v.blocks = B;
  v.blocks.block_T = (const int64_t*)(a + off[0]);
  v.blocks.block_inst_off = (const int64_t*)(a + off[1]);
  v.blocks.block_member_off = (const int64_t*)(a + off[2]);
  v.blocks.inst_prefix_node = (const int64_t*)(a + off[3]);
  v.blocks.inst_prefix_len = (const int64_t*)(a + off[4]);
  v.blocks.members = (const int32_t*)(a + off[5]);
  v.tmpl_off = (const int64_t*)(a + off[6]);
  v.tmpl_nodes = (const int32_t*)(a + off[7]);
  v.scores = (const sp_score_out*)(a + off[8]);
  v.detail = (const sp_explain_block*)(a + off[9]);
  v.node_detail = (const int8_t*)(a + off[10]);
  v.edge_detail = (const int8_t*)(a + off[11]);
  v.edge_off = (const int64_t*)(a + off[12]);
  v.n_entries = P->toff.empty() ? 0 : P->toff.back();
  v.n_edges = P->eoff.empty() ? 0 : P->eoff.back();
}

int sp_plan_run(sp_ctx* ctx, sp_dgraph* dg, int32_t min_dup, const sp_mesh* mesh, int64_t mu, int64_t chunk_size,
                sp_plan** out) {
  if (!ctx || !dg || !mesh || !out) return SP_ERR_CONFIG;
  *out = nullptr;
  if (!ctx->peers.empty() || ctx->comm) {
    ctx->last_error = "sp_plan_run: single-device contexts only";
    return SP_ERR_CONFIG;
  }
  sp_plan* P = new sp_plan();
  sp_tables* t = nullptr;
  int rc = guard(ctx, [&] {
    sp::Trace tr("plan");
    SP_CUDA(cudaSetDevice(ctx->device));
    if (mesh->m < 1 || mesh->n < 1) throw sp::Error(SP_ERR_CONFIG, "mesh must be at least 1x1");
    P->fold = new sp_fold();
    SP_CUDA(cudaEventRecord(ctx->ev[4], ctx->stream));
    sp::fold_run(ctx, dg, min_dup, P->fold);
    SP_CUDA(cudaEventRecord(ctx->ev[5], ctx->stream));
    tr.mark("fold");
    const sp_blocks& B = P->fold->view;
    const int64_t nb = B.n_blocks;
    P->toff.assign(nb + 1, 0);
    for (int64_t b = 0; b < nb; b++) {
      if (B.block_T[b] > SP_EXPLAIN_MAX_T) throw sp::Error(SP_ERR_UNSUPPORTED, "template with more than 256 nodes");
      P->toff[b + 1] = P->toff[b] + B.block_T[b];
    }
    P->tnodes.resize(P->toff[nb]);
    for (int64_t b = 0; b < nb; b++)
      std::memcpy(P->tnodes.data() + P->toff[b], B.members + B.block_member_off[b], sizeof(int32_t) * B.block_T[b]);
    t = new sp_tables();
    sp::tables_build(ctx, dg, nb, P->toff.data(), P->tnodes.empty() ? nullptr : P->tnodes.data(), mesh, mu,
                     chunk_size, t);
    tr.mark("tables");
    sp::score_launch(ctx, t, 0, 1, true);
    tr.mark("launch");
    P->scores.resize(std::max<int64_t>(nb, 1));
    P->detail.resize(std::max<int64_t>(nb, 1));
    P->node.resize(std::max<int64_t>(4 * P->toff[nb], 1));
    P->eoff = t->edge_off;
    P->edge.resize(std::max<int64_t>(2 * P->eoff[nb], 1));
    sp::score_wait(ctx, t, P->scores.data(), P->detail.data(), P->node.data(), P->edge.data());
    float ms = 0;
    SP_CUDA(cudaEventElapsedTime(&ms, ctx->ev[4], ctx->ev[5]));
    ctx->fold_ms = ms;
    tr.mark("search");
  });
  if (t) sp_tables_free(t);
  if (rc != SP_OK) {
    delete P;
    return rc;
  }
  plan_pack(P);
  *out = P;
  return SP_OK;
}

int sp_plan_view_get(const sp_plan* p, sp_plan_view* v) {
  if (!p || !v || !p->fold) return SP_ERR_CONFIG;
  *v = p->view;
  return SP_OK;
}

void sp_plan_free(sp_plan* p) { delete p; }

int sp_tables_candidates(const sp_tables* t, uint64_t* out) {
  if (!t || !out) return SP_ERR_CONFIG;
  for (int64_t b = 0; b < t->n_blocks; b++) out[b] = t->hdr[b].C;
  return t->overflow ? SP_ERR_UNSUPPORTED : SP_OK;
}

int sp_tables_bytes(const sp_tables* t, int64_t* bytes) {
  if (!t || !bytes) return SP_ERR_CONFIG;
  *bytes = t->blob_off.empty() ? 0 : t->blob_off.back();
  return SP_OK;
}

int sp_tables_slots(const sp_tables* t, int64_t block, int32_t* slot_pos, int32_t* n_slots) {
  if (!t || block < 0 || block >= t->n_blocks || !n_slots) return SP_ERR_CONFIG;
  const auto& v = t->slot_pos[block];
  if (slot_pos)
    for (size_t i = 0; i < v.size(); i++) slot_pos[i] = v[i];
  *n_slots = (int32_t)v.size();
  return SP_OK;
}

int sp_score(sp_ctx* ctx, sp_tables* t, int32_t shard, int32_t n_shards, sp_score_out* out) {
  if (!ctx || !t || !out) return SP_ERR_CONFIG;
  return guard(ctx, [&] {
    SP_CUDA(cudaSetDevice(ctx->device));
    sp::score_all(ctx, t, shard, n_shards, out);
  });
}

int sp_search(sp_ctx* ctx, sp_tables* t, sp_score_out* out, sp_explain_block* blocks, int8_t* node_detail,
              int8_t* edge_detail) {
  if (!ctx || !t || !out || !blocks || !node_detail || !edge_detail) return SP_ERR_CONFIG;
  return guard(ctx, [&] {
    SP_CUDA(cudaSetDevice(ctx->device));
    sp::score_all(ctx, t, 0, 1, out, blocks, node_detail, edge_detail);
  });
}

int sp_score_launch(sp_ctx* ctx, sp_tables* t, int32_t shard, int32_t n_shards, int32_t explain) {
  if (!ctx || !t) return SP_ERR_CONFIG;
  return guard(ctx, [&] {
    sp::Trace tr("score_launch");
    SP_CUDA(cudaSetDevice(ctx->device));
    sp::score_launch(ctx, t, shard, n_shards, (explain & 1) != 0, (explain & SP_SCORE_LOCAL) != 0);
    tr.mark("enqueued");
  });
}

int sp_score_wait(sp_ctx* ctx, sp_tables* t, sp_score_out* out, sp_explain_block* blocks, int8_t* node_detail,
                  int8_t* edge_detail) {
  if (!ctx || !t || !out) return SP_ERR_CONFIG;
  if (blocks && (!node_detail || !edge_detail)) return SP_ERR_CONFIG;
  return guard(ctx, [&] {
    sp::Trace tr("score_wait");
    SP_CUDA(cudaSetDevice(ctx->device));
    sp::score_wait(ctx, t, out, blocks, node_detail, edge_detail);
    tr.mark("done");
  });
}

int sp_score_range(sp_ctx* ctx, sp_tables* t, int64_t block, uint64_t lo, uint64_t hi, double* totals,
                   sp_score_out* out) {
  if (!ctx || !t || !out) return SP_ERR_CONFIG;
  return guard(ctx, [&] {
    SP_CUDA(cudaSetDevice(ctx->device));
    sp::score_range(ctx, t, block, lo, hi, totals, out);
  });
}

void sp_merge_keys(sp_score_out* acc, const sp_score_out* other) {
  if (acc && other) sp::merge_key(acc, other);
}

int sp_explain(sp_ctx* ctx, sp_tables* t, int64_t block, uint64_t index, sp_explain_out* out,
               sp_edge_conv* edges, int32_t max_edges, int32_t* n_edges) {
  if (!ctx || !t || !out || !n_edges) return SP_ERR_CONFIG;
  return guard(ctx, [&] {
    SP_CUDA(cudaSetDevice(ctx->device));
    sp::explain(ctx, t, block, index, out, edges, max_edges, n_edges);
  });
}

int sp_tables_sizes(const sp_tables* t, int64_t* n_entries, int64_t* n_edges) {
  if (!t) return SP_ERR_CONFIG;
  if (n_entries) *n_entries = t->tmpl_off.empty() ? 0 : t->tmpl_off.back();
  if (n_edges) *n_edges = t->edge_off.empty() ? 0 : t->edge_off.back();
  return SP_OK;
}

int sp_tables_edge_offsets(const sp_tables* t, int64_t* edge_off) {
  if (!t || !edge_off) return SP_ERR_CONFIG;
  for (size_t i = 0; i < t->edge_off.size(); i++) edge_off[i] = t->edge_off[i];
  return SP_OK;
}

int sp_explain_all(sp_ctx* ctx, sp_tables* t, const uint64_t* indices, sp_explain_block* blocks,
                   int8_t* node_detail, int8_t* edge_detail) {
  if (!ctx || !t || !indices || !blocks) return SP_ERR_CONFIG;
  static_assert(sizeof(sp_explain_block) == 104, "sp_explain_block layout");
  return guard(ctx, [&] {
    SP_CUDA(cudaSetDevice(ctx->device));
    sp::explain_all(ctx, t, indices, blocks, node_detail, edge_detail);
  });
}

int sp_route_search(sp_ctx* ctx, sp_dgraph* dg, int64_t n_blocks, const int64_t* tmpl_off, const int32_t* tmpl_nodes,
                    const int16_t* ref_slot, const uint8_t* radix, const int64_t* edge_off, const sp_mesh* mesh,
                    int64_t mu, int64_t chunk_size, const uint64_t* indices, sp_score_out* out,
                    sp_explain_block* blocks, int8_t* node_detail, int8_t* edge_detail) {
  if (!ctx || !dg || !tmpl_off || !mesh || n_blocks < 0 || !blocks || !node_detail || !edge_detail) return SP_ERR_CONFIG;
  if (!indices && !out) return SP_ERR_CONFIG;
  return guard(ctx, [&] {
    SP_CUDA(cudaSetDevice(ctx->device));
    if (mesh->m < 1 || mesh->n < 1) throw sp::Error(SP_ERR_CONFIG, "mesh must be at least 1x1");
    sp::route_search(ctx, dg, n_blocks, tmpl_off, tmpl_nodes, ref_slot, radix, edge_off, mesh, mu, chunk_size,
                     indices, out, blocks, node_detail, edge_detail);
  });
}

int sp_ctx_limits(const sp_ctx* ctx, int64_t* smem_per_block, int32_t* sm_count) {
  if (!ctx) return SP_ERR_CONFIG;
  if (smem_per_block) *smem_per_block = (int64_t)ctx->smem_optin;
  if (sm_count) *sm_count = ctx->sm_count;
  return SP_OK;
}

int sp_tables_block_info(const sp_tables* t, int64_t* blob_bytes, int32_t* pool_slots, int32_t* template_nodes) {
  if (!t) return SP_ERR_CONFIG;
  for (int64_t b = 0; b < t->n_blocks; b++) {
    if (blob_bytes) blob_bytes[b] = t->hdr[b].bytes;
    if (pool_slots) pool_slots[b] = t->hdr[b].npool;
    if (template_nodes) template_nodes[b] = t->hdr[b].T;
  }
  return SP_OK;
}

int sp_last_timings(const sp_ctx* ctx, double* fold_ms, double* score_ms, double* score_kernel_ms) {
  if (!ctx) return SP_ERR_CONFIG;
  if (fold_ms) *fold_ms = ctx->fold_ms;
  if (score_ms) *score_ms = ctx->score_ms;
  if (score_kernel_ms) *score_kernel_ms = ctx->score_kernel_ms;
  return SP_OK;
}

int sp_fold_stats(const sp_ctx* ctx, double* device_ms, int32_t* levels) {
  if (!ctx) return SP_ERR_CONFIG;
  if (device_ms) *device_ms = ctx->fold_device_ms;
  if (levels) *levels = ctx->fold_levels;
  return SP_OK;
}

int sp_set_option(sp_ctx* ctx, int32_t option, int64_t value) {
  if (!ctx) return SP_ERR_CONFIG;
  if (option == SP_OPT_PREFIX_SKIP || option == SP_OPT_MEMO) {
    for (size_t i = 0; i <= ctx->peers.size(); i++) {
      sp_ctx* c = i ? ctx->peers[i - 1] : ctx;
      (option == SP_OPT_PREFIX_SKIP ? c->skip : c->memo) = value ? 1 : 0;
    }
    return SP_OK;
  }
  if (option == SP_OPT_SIM_SHARD) {
    const int32_t n = (int32_t)(value >> 16), r = (int32_t)(value & 0xFFFF);
    if (value && (n < 1 || r >= n)) {
      ctx->last_error = "SP_OPT_SIM_SHARD: rank must be below the rank count";
      return SP_ERR_CONFIG;
    }
    ctx->sim_nranks = value ? n : 1;
    ctx->sim_rank = value ? r : 0;
    return SP_OK;
  }
  if (option == SP_OPT_HOST_LAYOUT) {
    for (size_t i = 0; i <= ctx->peers.size(); i++) (i ? ctx->peers[i - 1] : ctx)->host_layout = value ? 1 : 0;
    return SP_OK;
  }
  ctx->last_error = "unknown option";
  return SP_ERR_CONFIG;
}

int sp_timer_start(sp_ctx* ctx) {
  if (!ctx) return SP_ERR_CONFIG;
  return guard(ctx, [&] {
    SP_CUDA(cudaSetDevice(ctx->device));
    SP_CUDA(cudaEventRecord(ctx->timer[0], ctx->stream));
  });
}

int sp_timer_stop(sp_ctx* ctx, double* ms) {
  if (!ctx || !ms) return SP_ERR_CONFIG;
  return guard(ctx, [&] {
    SP_CUDA(cudaSetDevice(ctx->device));
    SP_CUDA(cudaEventRecord(ctx->timer[1], ctx->stream));
    SP_CUDA(cudaEventSynchronize(ctx->timer[1]));
    float f = 0;
    SP_CUDA(cudaEventElapsedTime(&f, ctx->timer[0], ctx->timer[1]));
    *ms = f;
  });
}

int sp_copy_bytes(int64_t* h2d, int64_t* d2h) {
  if (h2d) *h2d = sp::g_h2d_bytes.load();
  if (d2h) *d2h = sp::g_d2h_bytes.load();
  return SP_OK;
}

int sp_launch_counts(const sp_ctx* ctx, int64_t* own_kernels, int64_t* cub_calls) {
  if (!ctx) return SP_ERR_CONFIG;
  int64_t own = ctx->own_launches, cub = ctx->cub_calls;
  for (const sp_ctx* p : ctx->peers) {
    own += p->own_launches;
    cub += p->cub_calls;
  }
  if (own_kernels) *own_kernels = own;
  if (cub_calls) *cub_calls = cub;
  return SP_OK;
}

}  // extern "C"
