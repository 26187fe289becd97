// ipm_dist.cu — the multi-GPU clause (a9): contiguous shards, one NCCL collective, rank-ordered fold.
//
// Each rank reduces its shard with the single-GPU kernel into an ACCUMULATOR-typed partial (float32 `+`
// stays float64, so rounding happens once, globally), one ncclAllGather moves the P partials (8 bytes
// each) over NVLink/NVSwitch, and a one-warp kernel folds them in rank order, merges the variable's
// original value and rounds. AllGather + an ordered fold (rather than ncclAllReduce) is used for every op:
// NCCL has no & | ^ (nccl.h ncclRedOp_t: Sum, Prod, Max, Min, Avg), and an ordered fold gives every rank
// the same bits whatever NCCL's internal reduction order (ring / tree / NVLS). The message is 8 bytes per
// rank, so the collective is latency-bound either way.
#include <cuda_runtime.h>
#include <nccl.h>

#include <cstring>
#include <string>

#include "ipm.h"
#include "ipm_internal.h"

struct ipm_comm {
  ncclComm_t nccl;
  int rank, world, device;
};

using namespace ipm;

static ipm_status nccl_fail(ncclResult_t r, const char* where) {
  set_error(std::string(where) + ": " + ncclGetErrorString(r));
  return IPM_E_NCCL;
}

extern "C" {

size_t ipm_comm_id_bytes(void) { return sizeof(ncclUniqueId); }

ipm_status ipm_comm_unique_id(void* id_out) {
  if (!id_out) {
    set_error("NULL id buffer");
    return IPM_E_NULL;
  }
  ncclUniqueId id;
  ncclResult_t r = ncclGetUniqueId(&id);
  if (r != ncclSuccess) return nccl_fail(r, "ncclGetUniqueId");
  memcpy(id_out, &id, sizeof id);
  return IPM_OK;
}

ipm_status ipm_comm_init(ipm_comm** comm, int rank, int world, const void* id, int device) {
  if (!comm || !id) {
    set_error("NULL pointer");
    return IPM_E_NULL;
  }
  if (world < 1 || world > WS_MAX_RANKS || rank < 0 || rank >= world) {
    set_error("rank/world out of range (world <= 64)");
    return IPM_E_ARG;
  }
  cudaError_t e = cudaSetDevice(device);
  if (e != cudaSuccess) return cuda_fail(e, "cudaSetDevice");
  ncclUniqueId uid;
  memcpy(&uid, id, sizeof uid);
  ncclComm_t c;
  ncclResult_t r = ncclCommInitRank(&c, world, uid, rank);
  if (r != ncclSuccess) return nccl_fail(r, "ncclCommInitRank");
  *comm = new ipm_comm{c, rank, world, device};
  return IPM_OK;
}

ipm_status ipm_comm_destroy(ipm_comm* comm) {
  if (!comm) return IPM_OK;
  ncclResult_t r = ncclCommDestroy(comm->nccl);
  delete comm;
  if (r != ncclSuccess) return nccl_fail(r, "ncclCommDestroy");
  return IPM_OK;
}

ipm_status ipm_shard_range(int64_t n, int rank, int world, int64_t* lo, int64_t* hi) {
  if (!lo || !hi) {
    set_error("NULL pointer");
    return IPM_E_NULL;
  }
  if (n < 0) {
    set_error("negative element count");
    return IPM_E_SIZE;
  }
  if (world < 1 || rank < 0 || rank >= world) {
    set_error("rank/world out of range");
    return IPM_E_ARG;
  }
  // floor(r*n/P) with a 128-bit intermediate: shards differ by at most one element, later ranks larger
  *lo = (int64_t)(((__int128)n * rank) / world);
  *hi = (int64_t)(((__int128)n * (rank + 1)) / world);
  return IPM_OK;
}

ipm_status ipm_reduce_dist_async(ipm_comm* comm, ipm_op op, ipm_dtype dt, const void* dev_shard, int64_t n_shard,
                                 const void* init, void* dev_result, void* ws, void* stream) {
  ipm_status s;
  if (!comm) {
    set_error("NULL communicator");
    return IPM_E_NULL;
  }
  if ((s = validate(op, dt))) return s;
  if (n_shard < 0) {
    set_error("negative element count");
    return IPM_E_SIZE;
  }
  if ((n_shard > 0 && !dev_shard) || !dev_result) {
    set_error("NULL device pointer");
    return IPM_E_NULL;
  }
  if (!ws || ((uintptr_t)ws & 255u)) {
    set_error("workspace must be a non-NULL, 256-byte aligned device buffer");
    return IPM_E_WORKSPACE;
  }
  cudaStream_t st = (cudaStream_t)stream;
  uint64_t* local = (uint64_t*)((char*)ws + WS_LOCAL);
  uint64_t* slots = (uint64_t*)((char*)ws + WS_SLOTS);
  // local partial (an empty shard yields the identity: the kernel runs one CTA over nothing)
  if ((s = launch_flat(op, dt, dev_shard, n_shard, 0, 0, L_PARTIAL, local, ws, st))) return s;
  ncclResult_t r = ncclAllGather(local, slots, 1, ncclUint64, comm->nccl, st);
  if (r != ncclSuccess) return nccl_fail(r, "ncclAllGather");
  return launch_finalize(op, dt, slots, comm->world, scalar_bits(dt, init), init != nullptr, dev_result, st);
}

ipm_status ipm_reduce_dist(ipm_comm* comm, ipm_op op, ipm_dtype dt, const void* dev_shard, int64_t n_shard,
                           void* inout, void* ws, void* stream) {
  if (!inout) {
    set_error("NULL inout");
    return IPM_E_NULL;
  }
  void* res = (char*)ws + WS_RESULT;
  ipm_status s = ipm_reduce_dist_async(comm, op, dt, dev_shard, n_shard, inout, res, ws, stream);
  if (s) return s;
  cudaStream_t st = (cudaStream_t)stream;
  cudaError_t e = cudaMemcpyAsync(inout, res, esize(dt), cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) return cuda_fail(e, "ipm_reduce_dist");
  ncclResult_t ar;
  if (ncclCommGetAsyncError(comm->nccl, &ar) == ncclSuccess && ar != ncclSuccess)
    return nccl_fail(ar, "ncclCommGetAsyncError");
  return IPM_OK;
}

}  // extern "C"
