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
  // peer exchange (rl_comm_enable_peer_exchange): this rank's buffer and every rank's mapping
  void* xbuf = nullptr;
  void* peers[8] = {};
  int64_t max_tokens = 0;
  uint32_t epoch = 0;
};

namespace rl {
static rl_status nccl_fail(ncclResult_t r, const char* what) {
  return fail(RL_ERR_NCCL, "%s: %s", what, ncclGetErrorString(r));
}
ncclComm_t comm_nccl(rl_comm* c) { return c->nccl; }
int32_t comm_rank(const rl_comm* c) { return c->rank; }
int32_t comm_size(const rl_comm* c) { return c->nranks; }
// peer exchange layout (per rank buffer): two parity halves (the call epoch's low bit), each
// [P source ranks][max_tokens] records of two 8-byte words {epoch << 32 | float bits}
// (vp_ring_kernel, vocab_parallel.cu)
bool comm_peer_exchange(rl_comm* c, int64_t n_tokens, void** peers, int64_t* max_tokens, uint32_t* epoch) {
  if (!c->xbuf || n_tokens > c->max_tokens) return false;
  for (int r = 0; r < c->nranks; ++r) peers[r] = c->peers[r];
  *max_tokens = c->max_tokens;
  *epoch = ++c->epoch;
  return true;
}
static void release_peer_exchange(rl_comm* c) {
  for (int r = 0; r < c->nranks; ++r)
    if (c->peers[r] && c->peers[r] != c->xbuf) cudaIpcCloseMemHandle(c->peers[r]);
  if (c->xbuf) cudaFree(c->xbuf);
  c->xbuf = nullptr;
  for (auto& p : c->peers) p = nullptr;
}
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

extern "C" rl_status rl_comm_enable_peer_exchange(rl_comm* c, int64_t max_tokens) {
  using namespace rl;
  if (!c || max_tokens < 1) return fail(RL_ERR_INVALID_ARGUMENT, "NULL comm or max_tokens < 1");
  if (c->nranks > 8) return fail(RL_ERR_UNSUPPORTED, "peer exchange supports <= 8 ranks");
  release_peer_exchange(c);
  const size_t bytes = 2 * (size_t)c->nranks * max_tokens * 16;
  if (cudaMalloc(&c->xbuf, bytes) != cudaSuccess) return check_launch("cudaMalloc(peer exchange)");
  if (cudaMemset(c->xbuf, 0, bytes) != cudaSuccess) return check_launch("cudaMemset(peer exchange)");
  cudaIpcMemHandle_t mine;
  if (cudaIpcGetMemHandle(&mine, c->xbuf) != cudaSuccess) {
    release_peer_exchange(c);
    return check_launch("cudaIpcGetMemHandle");
  }
  char* dh = nullptr;
  const size_t hb = sizeof(cudaIpcMemHandle_t);
  if (cudaMalloc(&dh, hb * (c->nranks + 1)) != cudaSuccess) return check_launch("cudaMalloc(handles)");
  cudaMemcpy(dh + hb * c->nranks, &mine, hb, cudaMemcpyHostToDevice);
  ncclResult_t r = ncclAllGather(dh + hb * c->nranks, dh, hb, ncclChar, c->nccl, 0);
  if (r != ncclSuccess) {
    cudaFree(dh);
    release_peer_exchange(c);
    return nccl_fail(r, "ncclAllGather(ipc handles)");
  }
  cudaIpcMemHandle_t* all = new cudaIpcMemHandle_t[c->nranks];
  cudaDeviceSynchronize();
  cudaMemcpy(all, dh, hb * c->nranks, cudaMemcpyDeviceToHost);
  cudaFree(dh);
  rl_status st = RL_OK;
  for (int q = 0; q < c->nranks; ++q) {
    if (q == c->rank) {
      c->peers[q] = c->xbuf;
      continue;
    }
    void* p = nullptr;
    if (cudaIpcOpenMemHandle(&p, all[q], cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) {
      cudaGetLastError();
      st = fail(RL_ERR_UNSUPPORTED, "cudaIpcOpenMemHandle failed for rank %d (no P2P?)", q);
      break;
    }
    c->peers[q] = p;
  }
  delete[] all;
  // every rank must take the same path: enable only if every rank mapped every peer (a min
  // reduction of the per-rank success flag), else release on all ranks
  int32_t* okd = nullptr;
  int32_t ok = st == RL_OK ? 1 : 0;
  if (cudaMalloc(&okd, sizeof(int32_t)) != cudaSuccess) {
    release_peer_exchange(c);
    return check_launch("cudaMalloc(peer exchange flag)");
  }
  cudaMemcpy(okd, &ok, sizeof(int32_t), cudaMemcpyHostToDevice);
  r = ncclAllReduce(okd, okd, 1, ncclInt32, ncclMin, c->nccl, 0);
  cudaDeviceSynchronize();
  cudaMemcpy(&ok, okd, sizeof(int32_t), cudaMemcpyDeviceToHost);
  cudaFree(okd);
  if (r != ncclSuccess) {
    release_peer_exchange(c);
    return nccl_fail(r, "ncclAllReduce(peer exchange agreement)");
  }
  if (st == RL_OK && !ok) st = fail(RL_ERR_UNSUPPORTED, "another rank could not map its peers");
  if (st != RL_OK) {
    release_peer_exchange(c);
    return st;
  }
  c->max_tokens = max_tokens;
  c->epoch = 0;
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
  rl::release_peer_exchange(c);
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
