// ipm_dist.cu — the multi-GPU clause (a9): contiguous shards, one exchange of accumulator partials, a fold in
// rank order.
//
// Each rank reduces its shard into an ACCUMULATOR-typed partial (float32 `+` stays float64, so rounding
// happens once, globally). Two exchanges, same result bits:
//   fused (default when every peer's buffer is mapped): the reduction kernel itself, in the CTA that finishes
//     the shard, stores the partial into every peer's symmetric slot buffer over NVLink (CUDA IPC peer
//     mappings), waits for all ranks' slots, folds them in rank order and writes the result — ONE kernel per
//     rank, no collective launch, no second kernel (ipm_kernels.cuh dist_exchange);
//   NCCL: the kernel writes the partial, one ncclAllGather moves the P partials (8 bytes each), a one-warp
//     kernel folds them in rank order. AllGather + an ordered fold (rather than ncclAllReduce) because NCCL has
//     no & | ^ (nccl.h ncclRedOp_t: Sum, Prod, Max, Min, Avg) and so that every rank gets the same bits
//     whatever NCCL's internal reduction order.
// The message is 8 bytes per rank: both are latency-bound; the fused path removes two launches per call.
#include <cuda_runtime.h>
#include <nccl.h>

#include <cstring>
#include <string>

#include "ipm.h"
#include "ipm_internal.h"
#include "ipm_kernels.cuh"

struct ipm_comm {
  ncclComm_t nccl;
  int rank, world, device;
  int p2p;                      // every peer's symmetric buffer is mapped into this process
  uint64_t* sym;                // own symmetric slot buffer (cudaMalloc, IPC-exported)
  uint64_t** peers_dev;         // device array of world pointers (own buffer at [rank])
  void* opened[64];             // peer mappings to close
};

using namespace ipm;

static ipm_status nccl_fail(ncclResult_t r, const char* where) {
  set_error(std::string(where) + ": " + ncclGetErrorString(r));
  return IPM_E_NCCL;
}

// symmetric slot buffers: allocate and IPC-export one per rank, exchange the handles with one ncclAllGather,
// map every peer's buffer; all ranks then agree (ncclAllReduce min) on whether the fused path is usable.
constexpr size_t SYM_BYTES = 8 * 1024;  // >= SYM_WORDS * 8
static ipm_status setup_peer_memory(ipm_comm* m) {
  cudaError_t e;
  if ((e = cudaMalloc(&m->sym, SYM_BYTES)) != cudaSuccess) return cuda_fail(e, "cudaMalloc(sym)");
  if ((e = cudaMemset(m->sym, 0, SYM_BYTES)) != cudaSuccess) return cuda_fail(e, "cudaMemset(sym)");
  uint64_t* host_ptrs[64] = {nullptr};
  host_ptrs[m->rank] = m->sym;
  int ok = 1;
  if (m->world > 1) {
    cudaIpcMemHandle_t mine;
    if (cudaIpcGetMemHandle(&mine, m->sym) != cudaSuccess) ok = 0;
    char* dbuf = nullptr;
    const size_t hb = sizeof(cudaIpcMemHandle_t);
    if ((e = cudaMalloc(&dbuf, hb * m->world + sizeof(int))) != cudaSuccess) return cuda_fail(e, "cudaMalloc");
    cudaMemcpy(dbuf + hb * m->rank, &mine, hb, cudaMemcpyHostToDevice);
    ncclResult_t r = ncclAllGather(dbuf + hb * m->rank, dbuf, hb, ncclUint8, m->nccl, 0);
    if (r != ncclSuccess) {
      cudaFree(dbuf);
      return nccl_fail(r, "ncclAllGather(ipc handles)");
    }
    std::string all(hb * m->world, '\0');
    if ((e = cudaMemcpy(&all[0], dbuf, hb * m->world, cudaMemcpyDeviceToHost)) != cudaSuccess) {
      cudaFree(dbuf);
      return cuda_fail(e, "cudaMemcpy(handles)");
    }
    for (int q = 0; q < m->world && ok; ++q) {
      if (q == m->rank) continue;
      cudaIpcMemHandle_t h;
      memcpy(&h, &all[hb * q], hb);
      void* ptr = nullptr;
      if (cudaIpcOpenMemHandle(&ptr, h, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) {
        cudaGetLastError();
        ok = 0;
        break;
      }
      m->opened[q] = ptr;
      host_ptrs[q] = (uint64_t*)ptr;
    }
    // every rank must take the same path
    int* dok = (int*)(dbuf + hb * m->world);
    cudaMemcpy(dok, &ok, sizeof(int), cudaMemcpyHostToDevice);
    r = ncclAllReduce(dok, dok, 1, ncclInt32, ncclMin, m->nccl, 0);
    if (r == ncclSuccess) cudaMemcpy(&ok, dok, sizeof(int), cudaMemcpyDeviceToHost);
    else ok = 0;
    cudaFree(dbuf);
  }
  if ((e = cudaMalloc(&m->peers_dev, sizeof(uint64_t*) * m->world)) != cudaSuccess) return cuda_fail(e, "cudaMalloc");
  if ((e = cudaMemcpy(m->peers_dev, host_ptrs, sizeof(uint64_t*) * m->world, cudaMemcpyHostToDevice)) != cudaSuccess)
    return cuda_fail(e, "cudaMemcpy(peers)");
  m->p2p = ok;
  return IPM_OK;
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
  ipm_comm* m = new ipm_comm();
  m->nccl = c;
  m->rank = rank;
  m->world = world;
  m->device = device;
  ipm_status s = setup_peer_memory(m);
  if (s) {
    ipm_comm_destroy(m);
    return s;
  }
  *comm = m;
  return IPM_OK;
}

ipm_status ipm_comm_init_group(ipm_comm** comms, int world, int device) {
  if (!comms) {
    set_error("NULL pointer");
    return IPM_E_NULL;
  }
  if (world < 1 || world > WS_MAX_RANKS) {
    set_error("world out of range (1..64)");
    return IPM_E_ARG;
  }
  cudaError_t e = cudaSetDevice(device);
  if (e != cudaSuccess) return cuda_fail(e, "cudaSetDevice");
  uint64_t* ptrs[64] = {nullptr};
  for (int q = 0; q < world; ++q) {
    ipm_comm* m = new ipm_comm();
    m->nccl = nullptr;
    m->rank = q;
    m->world = world;
    m->device = device;
    m->p2p = 1;
    comms[q] = m;
    if ((e = cudaMalloc(&m->sym, SYM_BYTES)) != cudaSuccess || (e = cudaMemset(m->sym, 0, SYM_BYTES)) != cudaSuccess) {
      for (int k = 0; k <= q; ++k) ipm_comm_destroy(comms[k]);
      return cuda_fail(e, "cudaMalloc(sym)");
    }
    ptrs[q] = m->sym;
  }
  for (int q = 0; q < world; ++q) {
    ipm_comm* m = comms[q];
    if ((e = cudaMalloc(&m->peers_dev, sizeof(uint64_t*) * world)) != cudaSuccess ||
        (e = cudaMemcpy(m->peers_dev, ptrs, sizeof(uint64_t*) * world, cudaMemcpyHostToDevice)) != cudaSuccess) {
      for (int k = 0; k < world; ++k) ipm_comm_destroy(comms[k]);
      return cuda_fail(e, "peers");
    }
  }
  return IPM_OK;
}

size_t ipm_comm_ipc_handle_bytes(void) { return sizeof(cudaIpcMemHandle_t); }

ipm_status ipm_comm_create_ipc(ipm_comm** comm, int rank, int world, int device, void* handle_out) {
  if (!comm || !handle_out) {
    set_error("NULL pointer");
    return IPM_E_NULL;
  }
  if (world < 1 || world > WS_MAX_RANKS || rank < 0 || rank >= world) {
    set_error("rank/world out of range (world <= 64)");
    return IPM_E_ARG;
  }
  cudaError_t e = cudaSetDevice(device);
  if (e != cudaSuccess) return cuda_fail(e, "cudaSetDevice");
  ipm_comm* m = new ipm_comm();
  m->nccl = nullptr;
  m->rank = rank;
  m->world = world;
  m->device = device;
  m->p2p = 0;  // until ipm_comm_attach_ipc
  if ((e = cudaMalloc(&m->sym, SYM_BYTES)) != cudaSuccess || (e = cudaMemset(m->sym, 0, SYM_BYTES)) != cudaSuccess ||
      (e = cudaIpcGetMemHandle((cudaIpcMemHandle_t*)handle_out, m->sym)) != cudaSuccess) {
    ipm_comm_destroy(m);
    return cuda_fail(e, "symmetric slot buffer");
  }
  *comm = m;
  return IPM_OK;
}

ipm_status ipm_comm_attach_ipc(ipm_comm* comm, const void* handles) {
  if (!comm || !handles) {
    set_error("NULL pointer");
    return IPM_E_NULL;
  }
  if (comm->p2p || comm->nccl) {
    set_error("communicator is already connected");
    return IPM_E_ARG;
  }
  cudaError_t e = cudaSetDevice(comm->device);
  if (e != cudaSuccess) return cuda_fail(e, "cudaSetDevice");
  const size_t hb = sizeof(cudaIpcMemHandle_t);
  uint64_t* ptrs[64] = {nullptr};
  for (int q = 0; q < comm->world; ++q) {
    if (q == comm->rank) {
      ptrs[q] = comm->sym;
      continue;
    }
    cudaIpcMemHandle_t h;
    memcpy(&h, (const char*)handles + hb * q, hb);
    void* ptr = nullptr;
    if ((e = cudaIpcOpenMemHandle(&ptr, h, cudaIpcMemLazyEnablePeerAccess)) != cudaSuccess) {
      cudaGetLastError();
      for (int k = 0; k < q; ++k)
        if (comm->opened[k]) {
          cudaIpcCloseMemHandle(comm->opened[k]);
          comm->opened[k] = nullptr;
        }
      return cuda_fail(e, "cudaIpcOpenMemHandle(peer slot buffer)");
    }
    comm->opened[q] = ptr;
    ptrs[q] = (uint64_t*)ptr;
  }
  if ((e = cudaMalloc(&comm->peers_dev, sizeof(uint64_t*) * comm->world)) != cudaSuccess ||
      (e = cudaMemcpy(comm->peers_dev, ptrs, sizeof(uint64_t*) * comm->world, cudaMemcpyHostToDevice)) != cudaSuccess)
    return cuda_fail(e, "peers");
  comm->p2p = 1;
  return IPM_OK;
}

ipm_status ipm_comm_destroy(ipm_comm* comm) {
  if (!comm) return IPM_OK;
  cudaDeviceSynchronize();
  for (int q = 0; q < 64; ++q)
    if (comm->opened[q]) cudaIpcCloseMemHandle(comm->opened[q]);
  if (comm->peers_dev) cudaFree(comm->peers_dev);
  if (comm->sym) cudaFree(comm->sym);
  ncclResult_t r = comm->nccl ? ncclCommDestroy(comm->nccl) : ncclSuccess;
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
  if (!comm->p2p && !comm->nccl) {
    set_error("communicator not connected (ipm_comm_attach_ipc not called)");
    return IPM_E_ARG;
  }
  cudaStream_t st = (cudaStream_t)stream;
  if (comm->p2p && (dist_mode_option() == 0 || !comm->nccl)) {  // one kernel: reduction + exchange
    DistArgs d{comm->peers_dev, comm->rank, comm->world, dist_timeout_ns()};
    return launch_flat(op, dt, dev_shard, n_shard, scalar_bits(dt, init), init != nullptr, L_DIST, dev_result, ws,
                       st, &d);
  }
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
  void *mh, *md;
  ipm_status s = result_mailbox(&mh, &md);
  if (s) return s;
  if ((s = ipm_reduce_dist_async(comm, op, dt, dev_shard, n_shard, inout, md, ws, stream))) return s;
  cudaError_t e = cudaStreamSynchronize((cudaStream_t)stream);
  if (e != cudaSuccess) return cuda_fail(e, "ipm_reduce_dist");
  memcpy(inout, mh, esize(dt));
  ncclResult_t ar;
  if (comm->nccl && ncclCommGetAsyncError(comm->nccl, &ar) == ncclSuccess && ar != ncclSuccess)
    return nccl_fail(ar, "ncclCommGetAsyncError");
  int err = 0;
  if (comm->p2p && ipm_comm_error(comm, &err) == IPM_OK && err) {
    set_error("fused exchange: a peer did not arrive within the timeout (result undefined)");
    return IPM_E_NCCL;
  }
  return IPM_OK;
}

ipm_status ipm_reduce_host_dist(ipm_comm* comm, ipm_op op, ipm_dtype dt, const void* host_shard, int64_t n_shard,
                                void* inout, void* ws, void* stream) {
  ipm_status s;
  if (!comm || !inout || (n_shard > 0 && !host_shard)) {
    set_error("NULL pointer");
    return IPM_E_NULL;
  }
  if ((s = validate(op, dt))) return s;
  if (n_shard < 0) {
    set_error("negative element count");
    return IPM_E_SIZE;
  }
  if (!ws || ((uintptr_t)ws & 255u)) {
    set_error("workspace must be a non-NULL, 256-byte aligned device buffer");
    return IPM_E_WORKSPACE;
  }
  if (!comm->p2p && !comm->nccl) {
    set_error("communicator not connected (ipm_comm_attach_ipc not called)");
    return IPM_E_ARG;
  }
  cudaStream_t st = (cudaStream_t)stream;
  if ((s = stream_host_partial(op, dt, host_shard, n_shard, ws, st))) return s;
  const uint64_t* acc = (const uint64_t*)((char*)ws + WS_ACC);
  void *mh, *res;
  if ((s = result_mailbox(&mh, &res))) return s;
  const uint64_t ib = scalar_bits(dt, inout);
  if (comm->p2p && (dist_mode_option() == 0 || !comm->nccl)) {
    DistArgs d{comm->peers_dev, comm->rank, comm->world, dist_timeout_ns()};
    if ((s = launch_exchange(op, dt, acc, ib, 1, res, &d, st))) return s;
  } else {
    uint64_t* slots = (uint64_t*)((char*)ws + WS_SLOTS);
    ncclResult_t r = ncclAllGather(acc, slots, 1, ncclUint64, comm->nccl, st);
    if (r != ncclSuccess) return nccl_fail(r, "ncclAllGather");
    if ((s = launch_finalize(op, dt, slots, comm->world, ib, 1, res, st))) return s;
  }
  cudaError_t e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) return cuda_fail(e, "ipm_reduce_host_dist");
  memcpy(inout, mh, esize(dt));
  int err = 0;
  if (comm->p2p && ipm_comm_error(comm, &err) == IPM_OK && err) {
    set_error("fused exchange: a peer did not arrive within the timeout (result undefined)");
    return IPM_E_NCCL;
  }
  return IPM_OK;
}

int ipm_comm_uses_peer_memory(const ipm_comm* comm) {
  return comm && comm->p2p && (dist_mode_option() == 0 || !comm->nccl);
}

ipm_status ipm_comm_error(ipm_comm* comm, int* err) {
  if (!comm || !err) {
    set_error("NULL pointer");
    return IPM_E_NULL;
  }
  uint64_t v = 0;
  cudaError_t e = cudaMemcpy(&v, comm->sym + SYM_ERROR, 8, cudaMemcpyDeviceToHost);
  if (e != cudaSuccess) return cuda_fail(e, "cudaMemcpy(error word)");
  *err = v ? 1 : 0;
  if (v) cudaMemset(comm->sym + SYM_ERROR, 0, 8);
  return IPM_OK;
}

}  // extern "C"
