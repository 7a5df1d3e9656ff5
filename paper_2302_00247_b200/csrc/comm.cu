// Multi-GPU exchange of the per-block search records, inside the library.
//
// The reference's data-parallel axis is the process pool's range split and
// exact min-merge (search.py:327-343).  Here every device (a lane) scores its
// share of every block's work items; the per-block records (sp_score_out, 40
// bytes) are exchanged with ONE ncclAllGather over NVLink/NVSwitch and merged
// on the device by k_merge_ranks (lexicographic (total, num_split, index) min,
// valid counts summed) -- a 64-bit allreduce-min cannot carry that key
// losslessly.  Two ways to form the communicator:
//   * one process per GPU: sp_comm_unique_id on rank 0, the 128-byte id handed
//     to the other ranks by any bootstrap, then sp_ctx_comm_init
//     (ncclCommInitRank);
//   * one process driving several GPUs: sp_ctx_create(ngpu, devices)
//     (ncclCommInitAll; collectives of the lanes inside one NCCL group call).
// NCCL is loaded with dlopen on first use (libnccl.so.2, the one torch has
// already loaded when present), so the library has no link-time NCCL
// dependency and a single-GPU user never loads it.
#include <dlfcn.h>
#include <nccl.h>

#include <cstdio>
#include <mutex>

#include "sp_internal.h"

namespace sp {
namespace {

struct NcclApi {
  void* so = nullptr;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommInitAll)(ncclComm_t*, int, const int*) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
  ncclResult_t (*GetVersion)(int*) = nullptr;
  std::string error;
};

NcclApi& api() {
  static NcclApi a;
  static std::once_flag once;
  std::call_once(once, [] {
    const char* env = getenv("SP_NCCL_LIB");
    const char* names[] = {env, "libnccl.so.2", "libnccl.so"};
    for (const char* n : names) {
      if (!n) continue;
      a.so = dlopen(n, RTLD_NOW | RTLD_GLOBAL);
      if (a.so) break;
    }
    if (!a.so) {
      a.error = std::string("cannot load NCCL (libnccl.so.2): ") + dlerror();
      return;
    }
#define SP_SYM(field, name)                                  \
  a.field = (decltype(a.field))dlsym(a.so, name);            \
  if (!a.field) {                                            \
    a.error = std::string("NCCL symbol missing: ") + name;   \
    return;                                                  \
  }
    SP_SYM(GetUniqueId, "ncclGetUniqueId");
    SP_SYM(CommInitRank, "ncclCommInitRank");
    SP_SYM(CommInitAll, "ncclCommInitAll");
    SP_SYM(CommDestroy, "ncclCommDestroy");
    SP_SYM(AllGather, "ncclAllGather");
    SP_SYM(GroupStart, "ncclGroupStart");
    SP_SYM(GroupEnd, "ncclGroupEnd");
    SP_SYM(GetErrorString, "ncclGetErrorString");
    SP_SYM(GetVersion, "ncclGetVersion");
#undef SP_SYM
  });
  if (!a.error.empty()) throw Error(SP_ERR_CUDA, a.error);
  return a;
}

void check(ncclResult_t r, const char* what) {
  if (r != ncclSuccess) throw Error(SP_ERR_CUDA, std::string(what) + ": " + api().GetErrorString(r));
}

}  // namespace

int nccl_version() {
  int v = 0;
  check(api().GetVersion(&v), "ncclGetVersion");
  return v;
}

void nccl_unique_id(uint8_t* out) {
  static_assert(sizeof(ncclUniqueId) == SP_COMM_ID_BYTES, "ncclUniqueId size");
  ncclUniqueId id;
  check(api().GetUniqueId(&id), "ncclGetUniqueId");
  std::memcpy(out, &id, sizeof(id));
}

void nccl_init_rank(sp_ctx* ctx, int nranks, int rank, const uint8_t* id) {
  ncclUniqueId uid;
  std::memcpy(&uid, id, sizeof(uid));
  ncclComm_t comm = nullptr;
  SP_CUDA(cudaSetDevice(ctx->device));
  check(api().CommInitRank(&comm, nranks, uid, rank), "ncclCommInitRank");
  ctx->comm = comm;
  ctx->nranks = nranks;
  ctx->rank = rank;
  ctx->transport = SP_TRANSPORT_NCCL;
}

void nccl_init_all(const std::vector<sp_ctx*>& lanes) {
  const int n = (int)lanes.size();
  std::vector<int> devs(n);
  std::vector<ncclComm_t> comms(n);
  for (int i = 0; i < n; i++) devs[i] = lanes[i]->device;
  check(api().CommInitAll(comms.data(), n, devs.data()), "ncclCommInitAll");
  for (int i = 0; i < n; i++) {
    lanes[i]->comm = comms[i];
    lanes[i]->nranks = n;
    lanes[i]->rank = i;
    lanes[i]->transport = SP_TRANSPORT_NCCL;
  }
}

void nccl_destroy(sp_ctx* ctx) {
  if (ctx->comm) {
    api().CommDestroy((ncclComm_t)ctx->comm);
    ctx->comm = nullptr;
  }
}

void nccl_group_start() { check(api().GroupStart(), "ncclGroupStart"); }
void nccl_group_end() { check(api().GroupEnd(), "ncclGroupEnd"); }

void nccl_allgather(sp_ctx* ctx, const void* send, void* recv, size_t bytes) {
  check(api().AllGather(send, recv, bytes, ncclUint8, (ncclComm_t)ctx->comm, ctx->stream), "ncclAllGather");
}

}  // namespace sp
