// (5) rl_comm: a library-owned NCCL communicator (NVLink 5 / NVSwitch), bootstrapped
// from a 128-byte unique id that the caller broadcasts (e.g. over the torch process group).
// Used for the token-parallel all-reduce of rl_batch_counts / rl_loss_stats (north_star:
// "an NCCL all-reduce of loss sums and token counts") and the vocab-parallel combine.
#include <nccl.h>

#include <cstring>

#include "common.cuh"

struct rl_comm {
  ncclComm_t nccl;
  int32_t nranks;
  int32_t rank;
};

namespace rl {
static rl_status nccl_fail(ncclResult_t r, const char* what) {
  return fail(RL_ERR_NCCL, "%s: %s", what, ncclGetErrorString(r));
}
ncclComm_t comm_nccl(rl_comm* c) { return c->nccl; }
int32_t comm_rank(const rl_comm* c) { return c->rank; }
int32_t comm_size(const rl_comm* c) { return c->nranks; }
}  // namespace rl

static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId is 128 bytes");

extern "C" rl_status rl_comm_unique_id(void* out_128_bytes_host) {
  if (!out_128_bytes_host) return rl::fail(RL_ERR_INVALID_ARGUMENT, "NULL out");
  ncclUniqueId id;
  ncclResult_t r = ncclGetUniqueId(&id);
  if (r != ncclSuccess) return rl::nccl_fail(r, "ncclGetUniqueId");
  memcpy(out_128_bytes_host, &id, sizeof(id));
  return RL_OK;
}

extern "C" rl_status rl_comm_init(rl_comm** out, const void* unique_id_host, int32_t nranks,
                                  int32_t rank) {
  if (!out || !unique_id_host) return rl::fail(RL_ERR_INVALID_ARGUMENT, "NULL out/unique_id");
  if (nranks < 1 || rank < 0 || rank >= nranks)
    return rl::fail(RL_ERR_INVALID_ARGUMENT, "bad nranks/rank %d/%d", nranks, rank);
  ncclUniqueId id;
  memcpy(&id, unique_id_host, sizeof(id));
  ncclComm_t c;
  ncclResult_t r = ncclCommInitRank(&c, nranks, id, rank);
  if (r != ncclSuccess) return rl::nccl_fail(r, "ncclCommInitRank");
  *out = new rl_comm{c, nranks, rank};
  return RL_OK;
}

extern "C" rl_status rl_comm_split(rl_comm* parent, int32_t color, int32_t key, rl_comm** out) {
  if (!parent || !out) return rl::fail(RL_ERR_INVALID_ARGUMENT, "NULL parent/out");
  ncclComm_t c = nullptr;
  ncclResult_t r = ncclCommSplit(parent->nccl, color, key, &c, nullptr);
  if (r != ncclSuccess) return rl::nccl_fail(r, "ncclCommSplit");
  if (!c) {  // color == NCCL_SPLIT_NOCOLOR
    *out = nullptr;
    return RL_OK;
  }
  int n = 0, me = 0;
  ncclCommCount(c, &n);
  ncclCommUserRank(c, &me);
  *out = new rl_comm{c, n, me};
  return RL_OK;
}

extern "C" rl_status rl_comm_destroy(rl_comm* c) {
  if (!c) return RL_OK;
  ncclResult_t r = ncclCommDestroy(c->nccl);
  delete c;
  if (r != ncclSuccess) return rl::nccl_fail(r, "ncclCommDestroy");
  return RL_OK;
}

extern "C" rl_status rl_comm_size(const rl_comm* c, int32_t* nranks, int32_t* rank) {
  if (!c) return rl::fail(RL_ERR_INVALID_ARGUMENT, "NULL comm");
  if (nranks) *nranks = c->nranks;
  if (rank) *rank = c->rank;
  return RL_OK;
}

extern "C" rl_status rl_comm_allreduce_f64(rl_comm* c, double* buf, size_t n, rl_stream stream) {
  if (!c || (!buf && n)) return rl::fail(RL_ERR_INVALID_ARGUMENT, "NULL comm/buf");
  if (n == 0) return RL_OK;
  ncclResult_t r = ncclAllReduce(buf, buf, n, ncclDouble, ncclSum, c->nccl, (cudaStream_t)stream);
  if (r != ncclSuccess) return rl::nccl_fail(r, "ncclAllReduce");
  return RL_OK;
}
