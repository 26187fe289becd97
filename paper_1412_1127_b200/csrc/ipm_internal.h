// ipm_internal.h — shared between the translation units of libipm (not part of the ABI).
#pragma once
#include <cuda_runtime.h>
#include <cstdint>
#include <string>
#include "ipm.h"

namespace ipm {

// workspace layout (bytes from the 256-aligned base); ipm_workspace_bytes() = WS_BYTES
constexpr size_t WS_TICKETS = 0;          // uint32 tickets[WS_MAX_ROWS]
constexpr int WS_MAX_ROWS = 1024;
constexpr size_t WS_RESULT = 4096;        // result slots (up to 4 elements of 8 bytes)
constexpr size_t WS_LOCAL = 4160;         // this rank's accumulator partial (multi-GPU)
constexpr size_t WS_ACC = 4224;           // running accumulator (host-streaming path)
constexpr size_t WS_COUNTER = 4288;       // dynamic tile counter of the flat kernel (left at zero)
constexpr size_t WS_PACKED = 4296;        // int32 + count-and-sum word of the static flat kernel (left at zero)
constexpr size_t WS_RAGGED_NW = 4320;     // int64: warp count of the ragged kernel that ran (auto)
constexpr size_t WS_SLOTS = 4352;         // gathered partials, one per rank
constexpr int WS_MAX_RANKS = 64;
constexpr size_t WS_PARTIALS = 8192;      // per-CTA partials
constexpr int WS_MAX_PARTIALS = 16384;
constexpr size_t WS_RAGGED = WS_PARTIALS + 8 * (size_t)WS_MAX_PARTIALS;  // ragged head/tail records
constexpr int WS_MAX_RAGGED_WARPS = 8192;
constexpr size_t WS_BYTES = WS_RAGGED + 4 * 8 * (size_t)WS_MAX_RAGGED_WARPS;

// error plumbing: thread-local detail string for ipm_last_error_message()
void set_error(const std::string& msg);
ipm_status cuda_fail(cudaError_t e, const char* where);

int sm_count();  // of the current device (cached)
// pinned, device-mapped 64-byte result buffer of the calling host thread on the current device
ipm_status result_mailbox(void** host, void** dev);

ipm_status validate(ipm_op op, ipm_dtype dt);
size_t esize(ipm_dtype dt);
uint64_t scalar_bits(ipm_dtype dt, const void* host_scalar);

// kernel launchers (ipm_api.cu); all asynchronous on `st`
enum { L_RESULT = 0, L_PARTIAL = 1, L_ACCUM_FIRST = 2, L_ACCUM = 3, L_DIST = 5 };
struct DistArgs {             // L_DIST: the fused multi-GPU exchange (ipm_kernels.cuh dist_exchange)
  uint64_t* const* peers;     // device array of world symmetric-buffer pointers
  int rank, world;
  long long timeout_ns;
};
ipm_status launch_flat(ipm_op op, ipm_dtype dt, const void* dev, int64_t n, uint64_t init, int has_init, int mode,
                       void* out, void* ws, cudaStream_t st, const DistArgs* dist = nullptr,
                       unsigned long long* done = nullptr, unsigned long long done_seq = 0);
ipm_status launch_exchange(ipm_op op, ipm_dtype dt, const uint64_t* acc, uint64_t init, int has_init, void* out,
                           const DistArgs* dist, cudaStream_t st);
// host-streaming copyin fused with the reduction: leaves the accumulator partial of host[0..n) at ws + WS_ACC
ipm_status stream_host_partial(ipm_op op, ipm_dtype dt, const void* host, int64_t n, void* ws, cudaStream_t st);
int dist_mode_option();       // IPM_OPT_DIST_MODE: 0 auto (peer memory when mapped), 1 NCCL
long long dist_timeout_ns();
ipm_status launch_finalize(ipm_op op, ipm_dtype dt, const uint64_t* slots, int P, uint64_t init, int has_init,
                           void* out, cudaStream_t st);

}  // namespace ipm
