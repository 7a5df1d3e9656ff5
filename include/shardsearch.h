/*
 * shardsearch.h -- C ABI of the B200 search backend for TAP's plan search.
 *
 * The reference (shardplan, pure Python) has no FFI; its swap surface is the
 * Python seam  derive_plan -> prune_graph / search_subgraph -> _eval_range
 * (pkg/src/shardplan/search.py:289-379, pruning.py:123-201).  This header is
 * the flat, PyTorch-free boundary a ctypes/cffi shim binds in its place
 * (INTEGRATION.md shows the binding).  All inputs are caller-owned, C-contiguous,
 * little-endian arrays read only for the duration of a call; every handle
 * returned here is owned by the library and released with its *_free call.
 *
 * Error convention: functions return SP_OK (0) or an error code;
 * sp_last_error(ctx) returns the message of the last failure on that context.
 * Invalid candidates are data (valid bit / count), never errors -- mirroring
 * RoutingFailure (search.py:79-82, 198-199).
 */
#ifndef SHARDSEARCH_H
#define SHARDSEARCH_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SP_ABI_VERSION 2
#define SP_MAX_RANK 8

enum sp_status {
  SP_OK = 0,
  SP_ERR_CONFIG = 1,      /* -> shardplan.BadConfig (errors.py:29-30) */
  SP_ERR_UNSUPPORTED = 2, /* index space > u64, rank > SP_MAX_RANK, ... */
  SP_ERR_CUDA = 3,        /* CUDA / NCCL internal failure */
  SP_ERR_SPEC = 4,        /* -> shardplan.SpecMismatch (patterns_for on a non-shardable kind) */
  SP_ERR_PARSE = 5,       /* -> shardplan.ParseError (errors.py) : graph ingest */
  SP_ERR_CYCLE = 6,       /* -> shardplan.CycleError(src, dst)   : graph ingest */
  SP_ERR_DANGLING = 7,    /* -> shardplan.DanglingRef            : graph ingest */
  SP_ERR_EMPTY = 8,       /* -> shardplan.EmptyGraph             : graph ingest */
  SP_ERR_ONNX_PARSE = 9,  /* -> onnx_ingest.model.ModelParseError   : ONNX ingest */
  SP_ERR_ONNX_UNSUPPORTED = 10 /* -> onnx_ingest.convert.UnsupportedModel : ONNX ingest */
};

/* OpKind (ir.py:44-62) in declaration order. */
enum sp_op {
  SP_OP_MATMUL = 0,
  SP_OP_ELEMENTWISE = 1,
  SP_OP_LAYERNORM = 2,
  SP_OP_SOFTMAX = 3,
  SP_OP_EMBEDDING = 4,
  SP_OP_RESHAPE = 5,
  SP_OP_INPUT = 6,
  SP_OP_OUTPUT = 7,
  SP_OP_AUXILIARY = 8,
  SP_OP_COLLECTIVE = 9
};

/*
 * Grouped ModelGraph lowered to flat arrays: one row per
 * GraphNode (ir.py:164-202) in any fixed order; `topo_rank` carries the
 * position of the node in ModelGraph.topo_order (ir.py:250-274), which is the
 * only place the library needs the reference's lexicographic-heap order.
 */
typedef struct sp_graph {
  int64_t n_nodes;
  const uint8_t* name_bytes;  /* concatenated UTF-8 GraphNode scopes */
  const int64_t* name_off;    /* [n+1] */
  const int64_t* topo_rank;   /* [n] */
  const uint8_t* op;          /* [n] enum sp_op */
  const uint8_t* act_rank;    /* [n] 1..SP_MAX_RANK */
  const int64_t* act_shape;   /* [n*SP_MAX_RANK], unused dims 0 */
  const int64_t* act_bytes;   /* [n] TensorSpec.byte_size (ir.py:103-105) */
  const uint8_t* w_rank;      /* [n] 0 = no weight */
  const int64_t* w_shape;     /* [n*SP_MAX_RANK] */
  const int64_t* w_bytes;     /* [n] */
  const uint8_t* w_trainable; /* [n] */
  const int64_t* in_off;      /* [n+1] producer CSR */
  const int32_t* in_idx;      /* [E] producers in GraphNode.inputs order (deduplicated) */
} sp_graph;

/* ClusterSpec (costmodel.py:36-119) flattened. */
typedef struct sp_mesh {
  int64_t m, n;
  double intra_bw, inter_bw;
  double eff_allreduce, eff_allgather, eff_reducescatter, eff_alltoall;
  double overlap_fraction;
  double setup_latency_s;
} sp_mesh;

/*
 * Folding result (the list[Subgraph] of prune_graph, pruning.py:33-55, 123-201)
 * as a read-only view.  Blocks are in the reference's order (sorted by
 * template_prefix); instances of a block are sorted by prefix, instance 0 is
 * the template.  members[block_member_off[b] + i*block_T[b] + t] is the node
 * index of template position t in instance i of block b.  An instance prefix
 * is the first inst_prefix_len[j] bytes of node inst_prefix_node[j]'s scope.
 */
typedef struct sp_blocks {
  int64_t n_blocks;
  int64_t n_instances;
  int64_t n_members;
  const int64_t* block_T;          /* [n_blocks] */
  const int64_t* block_inst_off;   /* [n_blocks+1] */
  const int64_t* block_member_off; /* [n_blocks+1] */
  const int64_t* inst_prefix_node; /* [n_instances] */
  const int64_t* inst_prefix_len;  /* [n_instances] */
  const int32_t* members;          /* [n_members] */
} sp_blocks;

/* Per-block search result: SubgraphResult (search.py:236-242) + _plan_key. */
typedef struct sp_score_out {
  uint64_t candidates;  /* count_candidates (search.py:96-100) */
  uint64_t valid;       /* candidates whose pattern_routing succeeded */
  uint64_t best_index;  /* argmin of (total, num_split, index) */
  double best_total;    /* CostReport.total of the argmin (bit-exact) */
  int32_t best_num_split;
  int32_t has_best;     /* 0 when no candidate routes (reference asserts) */
} sp_score_out;

#define SP_EXPLAIN_MAX_T 256

/* Routing/cost detail of one candidate (RoutedPlan + CostReport fields). */
typedef struct sp_explain_out {
  int32_t valid;
  int32_t T;
  int32_t fail_pos;                       /* template position of RoutingFailure */
  int32_t pattern[SP_EXPLAIN_MAX_T];      /* index into patterns_for(op) */
  int32_t state_axis[SP_EXPLAIN_MAX_T];   /* final state: -1 replica, else split axis */
  int32_t exit_axis[SP_EXPLAIN_MAX_T];    /* -1 no exit AllGather, else gather axis */
  double forward_comm;
  double backward_comm;
  double total;
  int64_t bytes_allreduce, bytes_allgather, bytes_reducescatter, bytes_alltoall;
  int64_t calls_allreduce, calls_allgather, calls_reducescatter, calls_alltoall;
  int64_t collective_calls;
} sp_explain_out;

/* Conversion collective on an internal edge, reported by sp_explain_edges. */
typedef struct sp_edge_conv {
  int32_t consumer_pos; /* template position of the consumer */
  int32_t producer_pos; /* template position of the internal producer */
  int32_t kind;         /* 1 allreduce, 2 allgather, 3 reducescatter, 4 alltoall */
  int32_t axis;         /* collective axis, -1 when none */
} sp_edge_conv;

/* Per-block winner summary of sp_explain_all (plan_cost fields). */
typedef struct sp_explain_block {
  int32_t valid;
  int32_t fail_pos;
  double forward_comm, backward_comm, total;
  int64_t bytes[4]; /* allreduce, allgather, reducescatter, alltoall */
  int64_t calls[4];
  int64_t collective_calls;
} sp_explain_block;

typedef struct sp_ctx sp_ctx;
typedef struct sp_dgraph sp_dgraph;
typedef struct sp_fold sp_fold;
typedef struct sp_tables sp_tables;

int sp_abi_version(void);

/*
 * A context over `ngpu` devices of this process.  ngpu == 1: one
 * device -- the process-per-GPU form; join the other processes' devices with
 * sp_ctx_comm_init.  ngpu > 1: this process drives all `devices`; every entry
 * point below fans out over them (graph and tables replicated, the fold runs on
 * devices[0]) and a search deals each block's work items over the devices and
 * merges on devices[0] -- the reference's process-pool split and min-merge
 * (search.py:327-343) -- through ncclCommInitAll / one ncclAllGather (devices
 * listed twice share a GPU and exchange by peer copies instead; test use).
 */
int sp_ctx_create(int ngpu, const int* devices, sp_ctx** out);
void sp_ctx_destroy(sp_ctx* ctx);
const char* sp_last_error(const sp_ctx* ctx);

/*
 * Multi-process form (one process per GPU, e.g. under torchrun): rank 0 calls
 * sp_comm_unique_id and hands the SP_COMM_ID_BYTES-byte id to every rank by
 * any bootstrap (file, TCP store, MPI); each rank then calls sp_ctx_comm_init
 * on its single-device context (ncclCommInitRank; NCCL is loaded with dlopen
 * on first use, libnccl.so.2).  From then on sp_score_launch / sp_score /
 * sp_search score this rank's share (`shard`/`n_shards` are taken from the
 * communicator) and exchange the 40-byte per-block records with ONE
 * ncclAllGather over NVLink, merged on the device by (total, num_split, index)
 * with valid counts summed; every rank ends with the merged result, and the
 * winner detail (explain) is chained behind the merge on the device.
 */
#define SP_COMM_ID_BYTES 128
enum sp_transport { SP_TRANSPORT_NONE = 0, SP_TRANSPORT_NCCL = 1, SP_TRANSPORT_P2P = 2 };
int sp_comm_unique_id(uint8_t* id);
int sp_ctx_comm_init(sp_ctx* ctx, int32_t nranks, int32_t rank, const uint8_t* id);
/* nranks / rank of the context's communicator (1 / 0 without one), its local
 * device count and transport (enum sp_transport), the loaded NCCL version. */
int sp_ctx_comm_info(const sp_ctx* ctx, int32_t* nranks, int32_t* rank, int32_t* ndev, int32_t* transport,
                     int32_t* nccl_version);

/* Upload the lowered graph once; it stays resident in HBM. */
int sp_graph_upload(sp_ctx* ctx, const sp_graph* g, sp_dgraph** out);
void sp_graph_free(sp_dgraph* dg);

/* prune_graph(graph, min_duplicates) on the device (pruning.py:123-201). */
int sp_fold_run(sp_ctx* ctx, sp_dgraph* dg, int32_t min_dup, sp_fold** out);
int sp_fold_view(const sp_fold* f, sp_blocks* view);
void sp_fold_free(sp_fold* f);

/*
 * Per-block routing/cost tables for a set of templates (template node lists
 * in template order, as Subgraph.template).  mu/chunk are pack_gradients'
 * threshold and chunk size (rewrite.py:78-111).
 */
int sp_tables_build(sp_ctx* ctx, sp_dgraph* dg, int64_t n_blocks, const int64_t* tmpl_off,
                    const int32_t* tmpl_nodes, const sp_mesh* mesh, int64_t mu,
                    int64_t chunk_size, sp_tables** out);
void sp_tables_free(sp_tables* t);
/* count_candidates per block; returns SP_ERR_UNSUPPORTED if one exceeds u64. */
int sp_tables_candidates(const sp_tables* t, uint64_t* out);
/* Total bytes of the device routing tables (all blocks). */
int sp_tables_bytes(const sp_tables* t, int64_t* bytes);
/* Weight slot order of a block (weight_nodes, search.py:85-88): template positions. */
int sp_tables_slots(const sp_tables* t, int64_t block, int32_t* slot_pos, int32_t* n_slots);

/*
 * Batched scoring of every block (search_subgraph + _eval_range, search.py:289-345).
 * Shard `shard` of `n_shards` scores its contiguous slice of each block's index
 * range (search.py:331-336); results merge exactly with sp_merge_keys.
 */
int sp_score(sp_ctx* ctx, sp_tables* t, int32_t shard, int32_t n_shards, sp_score_out* out);
/*
 * Single-device search of every block in one call: sp_score followed by the
 * winner detail of sp_explain_all, chained on the device (one host sync).
 */
int sp_search(sp_ctx* ctx, sp_tables* t, sp_score_out* out, sp_explain_block* blocks,
              int8_t* node_detail, int8_t* edge_detail);
/*
 * Asynchronous form of sp_score / sp_search: sp_score_launch enqueues the
 * scoring of shard `shard` of `n_shards` (and, with `explain`, the winner
 * detail of sp_explain_all) on the context's stream and returns at once, so
 * the caller can assemble host-side results while the device searches;
 * sp_score_wait collects it (blocks/node_detail/edge_detail may be NULL, and
 * must be when `explain` was 0).  One search may be in flight per tables;
 * searches on different tables may be queued back to back: each copies its
 * results to pinned host memory behind its own kernels and sp_score_wait
 * waits on that search's event only, so an early search is collected while
 * later ones still run.
 * No reference counterpart: the reference's pool.map blocks (search.py:338).
 */
int sp_score_launch(sp_ctx* ctx, sp_tables* t, int32_t shard, int32_t n_shards, int32_t explain);
/* `explain` | SP_SCORE_LOCAL: score every candidate of `t` on this device and
 * exchange nothing, even when the context has a communicator, peer lanes or a
 * simulated shard -- for a search whose results only the root needs (the
 * cheap residual group of a multi-rank derive_plan: rank 0 scores it, the
 * other ranks never build it).  Every rank must agree which searches are
 * local: a non-local search is a collective. */
#define SP_SCORE_LOCAL 2
int sp_score_wait(sp_ctx* ctx, sp_tables* t, sp_score_out* out, sp_explain_block* blocks, int8_t* node_detail,
                  int8_t* edge_detail);
/* Score [lo, hi) of one block; optional per-candidate totals (NaN = invalid). */
int sp_score_range(sp_ctx* ctx, sp_tables* t, int64_t block, uint64_t lo, uint64_t hi,
                   double* totals, sp_score_out* out);
/* Lexicographic (total, num_split, index) merge of shard results, valid summed. */
void sp_merge_keys(sp_score_out* acc, const sp_score_out* other);

/* Full routing/cost detail of one candidate (for RoutedPlan/CostReport reconstruction). */
int sp_explain(sp_ctx* ctx, sp_tables* t, int64_t block, uint64_t index, sp_explain_out* out,
               sp_edge_conv* edges, int32_t max_edges, int32_t* n_edges);

/*
 * Routing detail of one candidate per block in a single launch (indices[b] ==
 * UINT64_MAX skips block b).  node_detail[4*e] = (pattern, state axis or -1,
 * exit AllGather axis or -1, 0) for template entry e (tmpl_off order);
 * edge_detail[2*k] = (collective kind 0..4, axis or -1) for every internal
 * edge, consumers in template order, producers in GraphNode.inputs order.
 */
int sp_tables_sizes(const sp_tables* t, int64_t* n_entries, int64_t* n_edges);
/* Internal-edge offset of every block in edge_detail ([n_blocks+1]). */
int sp_tables_edge_offsets(const sp_tables* t, int64_t* edge_off);
int sp_explain_all(sp_ctx* ctx, sp_tables* t, const uint64_t* indices, sp_explain_block* blocks,
                   int8_t* node_detail, int8_t* edge_detail);

/*
 * Route search: the blocks the table path cannot hold (a template of more than
 * SP_EXPLAIN_MAX_T nodes, a node with more than 6 internal producers, routing
 * tables larger than shared memory) scored without routing tables -- every
 * candidate routed node by node on the device (route_node: the reference's
 * per-node pattern choice, search.py:134-224) and costed as plan_cost
 * (costmodel.py:193-267) with reach/state in global scratch.  ref_slot[e] =
 * the weight slot (weight_nodes order, search.py:85-88) of template entry e or
 * -1, radix[e] its option count (2 or 3), edge_off = internal producer edges
 * per block (prefix sums).  Scores every block (out) and returns the winners'
 * detail in the layout of sp_explain_all, or -- with `indices` -- the detail of
 * the given candidates only (out may be NULL).  Up to 64 internal producers
 * per node and 2**64 candidates per block.
 */
int sp_route_search(sp_ctx* ctx, sp_dgraph* dg, int64_t n_blocks, const int64_t* tmpl_off, const int32_t* tmpl_nodes,
                    const int16_t* ref_slot, const uint8_t* radix, const int64_t* edge_off, const sp_mesh* mesh,
                    int64_t mu, int64_t chunk_size, const uint64_t* indices, sp_score_out* out,
                    sp_explain_block* blocks, int8_t* node_detail, int8_t* edge_detail);
/*
 * The device half of derive_plan in ONE call (search.py:348-379 up to the
 * report assembly): the fold (sp_fold_run), every block's template (instance
 * 0 of the fold's member matrix), the routing tables (sp_tables_build), the
 * search and the winners' detail (sp_search), with no host round trip in
 * between beyond the fold's and the table layout's own.  The result holds the
 * fold arrays, the template CSR and sp_search's outputs; sp_plan_view points
 * into it until sp_plan_free -- into ONE contiguous block, the arrays in the
 * view's field order, each 16-byte aligned (a caller may map it as a whole).  Single-device contexts only (SP_ERR_CONFIG on a
 * sharded one).  SP_ERR_UNSUPPORTED when a block is beyond the table path (a
 * template of more than SP_EXPLAIN_MAX_T nodes, more than 6 internal
 * producers, tables larger than shared memory, more than 2**64 candidates):
 * the caller then searches that graph block by block (sp_tables_build /
 * sp_route_search).  Replaces the sequence of calls, not a reference
 * interface: it exists to keep small searches free of per-call overhead.
 */
typedef struct sp_plan sp_plan;
typedef struct sp_plan_view {
  sp_blocks blocks;               /* the fold, as sp_fold_view */
  const int64_t* tmpl_off;        /* [n_blocks + 1] */
  const int32_t* tmpl_nodes;      /* [n_entries]: row of every template node */
  const sp_score_out* scores;     /* [n_blocks] */
  const sp_explain_block* detail; /* [n_blocks] winners (sp_explain_all layout) */
  const int8_t* node_detail;      /* [4 * n_entries] */
  const int8_t* edge_detail;      /* [2 * n_edges] */
  const int64_t* edge_off;        /* [n_blocks + 1] */
  int64_t n_entries, n_edges;
} sp_plan_view;
int sp_plan_run(sp_ctx* ctx, sp_dgraph* dg, int32_t min_dup, const sp_mesh* mesh, int64_t mu, int64_t chunk_size,
                sp_plan** out);
int sp_plan_view_get(const sp_plan* p, sp_plan_view* view);
void sp_plan_free(sp_plan* p);

/* Shared memory per CTA (opt-in) and SM count of the context's device. */
int sp_ctx_limits(const sp_ctx* ctx, int64_t* smem_per_block, int32_t* sm_count);
/* Per block of built tables: blob bytes, live-value pool slots, template nodes. */
int sp_tables_block_info(const sp_tables* t, int64_t* blob_bytes, int32_t* pool_slots, int32_t* template_nodes);

/*
 * Native graph ingest (host only, no context): the JSON graph document of
 * load_graph (ir.py:302-338, schema 1/2) -> ModelGraph validation and
 * lexicographic-heap toposort (ir.py:214-274) -> trim_and_group (ir.py:378-461)
 * -> the grouped graph as sp_graph arrays, rows in the grouped topological
 * order (what lowering.lower() produces from the Python objects).  Replaces
 * the reference's `load_graph` + `trim_and_group` in front of derive_plan
 * (SURVEY 8(f) rows 1-2).  Errors: SP_ERR_PARSE / CYCLE / DANGLING / EMPTY /
 * UNSUPPORTED; sp_ingest_error(0) is the message, (1)/(2) the CycleError
 * edge (src, dst), valid until the next sp_ingest_json on this thread.
 */
typedef struct sp_ingest sp_ingest;
int sp_ingest_json(const char* text, int64_t len, sp_ingest** out);
const char* sp_ingest_error(int32_t which);
int sp_ingest_view(const sp_ingest* g, sp_graph* view, int64_t* n_raw, int64_t* n_aux);
void sp_ingest_free(sp_ingest* g);
/*
 * ONNX ModelProto bytes -> the reference's onnx_ingest conversion
 * (wire.py:27-97, model.py:143-167, convert.py:84-274).  export_only != 0:
 * keep the schema-1 document (json.dumps text, sp_ingest_text(g, 0, 0)) and
 * the ConversionReport, as export_graph returns them; else continue into the
 * load_graph + trim_and_group pipeline of sp_ingest_json (sp_ingest_view).
 * has_batch/batch = the --batch option fixing a symbolic leading dimension.
 * counts[6] of sp_ingest_report: trainable_elements, skipped_elements,
 * initializer_elements, #warnings, #skipped, document bytes; texts:
 * kind 1 = warnings[i], kind 2 = skipped[i].
 */
int sp_ingest_onnx(const uint8_t* data, int64_t len, int32_t has_batch, int64_t batch, int32_t export_only,
                   sp_ingest** out);
int sp_ingest_report(const sp_ingest* g, int64_t* counts);
const char* sp_ingest_text(const sp_ingest* g, int32_t kind, int64_t i);

/* Device time (ms) of the last sp_score / sp_fold_run kernels (CUDA events). */
int sp_last_timings(const sp_ctx* ctx, double* fold_ms, double* score_ms, double* score_kernel_ms);

/*
 * Device-only part of the last sp_fold_run (CUDA events around the level loop,
 * excluding the host-side ordering of fold_finalize) and how many levels the
 * loop ran.  No reference counterpart: measurement hook for bench.py.
 */
int sp_fold_stats(const sp_ctx* ctx, double* device_ms, int32_t* levels);

/*
 * Options.  SP_OPT_PREFIX_SKIP (default 1): when a candidate fails routing at
 * node i, every candidate sharing the digits of i's ancestor cone fails too,
 * so the scorer jumps over them (exact; counts and argmin are unchanged).
 * 0 walks every candidate individually (brute force).
 */
#define SP_OPT_PREFIX_SKIP 1
/*
 * SP_OPT_MEMO (default 0, used when prefix skipping is off): every candidate is
 * still visited, but a node is re-routed only when a digit of its ancestor cone
 * changed since the lane's previous candidate (templates <= 64 nodes).  0 walks
 * every node of every candidate.
 */
#define SP_OPT_MEMO 2
/*
 * SP_OPT_HOST_LAYOUT (default 1): for graphs of <= 8192 nodes the table layout
 * (node maps, boundary flags, blob offsets) is computed on the host while the
 * tables are built, so building them needs no device round trip.  0 uses the
 * device layout for every graph (same tables).
 */
#define SP_OPT_HOST_LAYOUT 3
/*
 * SP_OPT_SIM_SHARD (measurement only, default 0): value (N << 16) | r makes
 * every single-device search score only rank r's share of an N-rank search,
 * with the winner detail chained on the device as after the multi-GPU merge:
 * one rank's step of the in-library multi-process search, simulated on one
 * GPU (the results are that share's, not the whole search's).  0: off.
 */
#define SP_OPT_SIM_SHARD 4
int sp_set_option(sp_ctx* ctx, int32_t option, int64_t value);

/* CUDA-event timer on the context's stream (brackets whole API calls for benchmarks). */
int sp_timer_start(sp_ctx* ctx);
int sp_timer_stop(sp_ctx* ctx, double* ms);
/* Kernel launches issued by this library since context creation: own kernels and CUB calls. */
int sp_launch_counts(const sp_ctx* ctx, int64_t* own_kernels, int64_t* cub_calls);
/* Host<->device bytes copied by the library in this process (all contexts). */
int sp_copy_bytes(int64_t* h2d, int64_t* d2h);

#ifdef __cplusplus
}
#endif

#endif /* SHARDSEARCH_H */
