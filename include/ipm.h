/* ipm.h — C ABI of libipm: B200-native execution of the OpenACC `reduction(op:var)` clause.
 *
 * The method (arxiv 1412.1127, IPMACC) lowers
 *
 *     #pragma acc loop reduction(op:var)        for (i = 0; i < n; ++i) var = var op a[i];
 *
 * to a kernel in which every thread folds its share of the iterations into a private copy of `var`
 * initialised to op's identity, the copies are combined along the threads of a thread block and then
 * across thread blocks, and the result is merged into the variable's original value
 * (PAPER.md:97 Step 4 "iii) performing variable reductions"; PAPER.md:106 Step 7 "extra code ... that
 * merges results across different thread blocks ... according to [Harris 2006]"; PAPER.md:205 the two-level
 * scheme; SPEC.md:317 the per-thread private copy and the fold "into the original host variable").
 * OpenACC's levels map to gang/worker/vector. Here: vector = a warp (warp-level reduce
 * instructions), worker = a CTA (shared-memory combine), gang = the grid (a last-CTA finish on the GPU
 * instead of the paper's host loop — see DESIGN.md "What differs from the paper").
 *
 * Data clauses (`copyin`, `create`, `present`, `copyout`, `delete`) follow PAPER.md:26/63 ("the [start:n]
 * pair indicates that n elements should be copied from the start element") and PAPER.md:99-100 (Step 5,
 * "host-accelerator pointer exchange, data copy in/out ... and memory allocation"); the present-table
 * semantics and error codes follow SPEC.md:296-304 and :391 (E_SIZE, E_PRESENT).
 *
 * Conventions for every entry point:
 *   - `stream` is a cudaStream_t passed as void* (NULL = the legacy default stream).
 *   - Device pointers are CUDA device (or managed) addresses; host pointers are ordinary (pageable or
 *     pinned) host addresses. Nothing is retained after a call returns unless stated.
 *   - Every call returns an ipm_status; no exception or exit() crosses the ABI. IPM_E_CUDA / IPM_E_NCCL
 *     carry the library's error string in ipm_last_error_message() (thread-local).
 *   - The library never allocates on the reduce path; the caller owns inputs, outputs and workspaces.
 *   - Element types: IPM_I32 = int32_t, IPM_I64 = int64_t, IPM_F32 = float, IPM_F64 = double.
 *   - "init" is the variable's value before the loop (a host scalar of the element type); NULL means the
 *     op's identity. The result is init ⊕ a[0] ⊕ ... ⊕ a[n-1] (reading R1).
 *
 * Semantics of the ops: integer + and * wrap modulo 2^w; max/min compare signed;
 * & | ^ act on the two's-complement bits and are illegal on floats (IPM_E_REDOP); && and || use C
 * truthiness (x != 0; for floats -0.0 is false and NaN is true) and yield 0/1 in the element type;
 * float max/min are IEEE 754-2019 maximum/minimum (-0 < +0; any NaN gives the canonical quiet NaN);
 * float + and * accumulate float32 inputs in float64 and round once at the end.
 */
#ifndef IPM_H
#define IPM_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum { IPM_ADD = 0, IPM_MUL, IPM_MAX, IPM_MIN, IPM_BAND, IPM_BOR, IPM_BXOR, IPM_LAND, IPM_LOR } ipm_op;
typedef enum { IPM_I32 = 0, IPM_I64, IPM_F32, IPM_F64 } ipm_dtype;

typedef enum {
  IPM_OK = 0,
  IPM_E_REDOP,     /* op illegal for the element type (& | ^ on floats), or an unknown op */
  IPM_E_DTYPE,     /* unknown element type */
  IPM_E_NULL,      /* a required pointer is NULL (e.g. dev == NULL with n > 0) */
  IPM_E_SIZE,      /* negative or overflowing count, row_stride < cols, bytes == 0 for a data clause */
  IPM_E_PRESENT,   /* `present`/`copyout`/`delete` on host memory with no live device copy */
  IPM_E_ALIGN,     /* a device pointer not aligned to its element size */
  IPM_E_WORKSPACE, /* workspace NULL or not aligned to 256 bytes */
  IPM_E_CUDA,      /* a CUDA runtime error; detail in ipm_last_error_message() */
  IPM_E_NCCL,      /* an NCCL error; detail in ipm_last_error_message() */
  IPM_E_ARG        /* any other invalid argument (rank/world out of range, ...) */
} ipm_status;

const char* ipm_status_str(ipm_status s);
const char* ipm_last_error_message(void);
/* 1 if reduction(op) is legal on dtype (30 of the 36 pairs), else 0 */
int ipm_op_legal(ipm_op op, ipm_dtype dt);
/* element size in bytes, 0 for an unknown dtype */
size_t ipm_dtype_size(ipm_dtype dt);
/* library version as 10000*major + 100*minor + patch */
int ipm_version(void);

/* ------------------------------------------------------------------ device-memory allocator hook
 * Device memory for the data clauses comes from this allocator (default: cudaMallocAsync/cudaFreeAsync on
 * the call's stream). The Python binding installs PyTorch's caching allocator here. `ctx` is passed back
 * untouched. Passing NULL restores the default. The structure is copied. */
typedef struct {
  void* (*alloc)(size_t bytes, void* stream, void* ctx);
  void (*free)(void* p, void* stream, void* ctx);
  void* ctx;
} ipm_allocator;
ipm_status ipm_set_allocator(const ipm_allocator* a);

/* ------------------------------------------------------------------ data environment (present table)
 * The table maps a host byte range [host, host+bytes) to a device buffer with a reference count, like an
 * OpenACC runtime's present table. Lookups accept any sub-range of a live entry.
 *   ipm_copyin : if the range is present, ++ref and return its device address; otherwise allocate `bytes`,
 *                copy host -> device on `stream` (the call returns after the copy completed) and ref = 1.
 *   ipm_create : like copyin but without the transfer (acc `create`).
 *   ipm_present: *dev = device address corresponding to `host` (which may point inside an entry whose range
 *                covers [host, host+bytes)); IPM_E_PRESENT if none. No transfer, no ref change.
 *   ipm_update_device / ipm_update_host: copy the sub-range host <-> device (acc `update`); IPM_E_PRESENT
 *                if absent. Synchronous with respect to the host.
 *   ipm_copyout: copy device -> host for the entry starting at `host` (`bytes` of it), then --ref and free
 *                at 0. ipm_delete: --ref, free at 0, no transfer.
 *   ipm_present_count: number of live entries (for leak tests). */
ipm_status ipm_copyin(const void* host, size_t bytes, void** dev, void* stream);
ipm_status ipm_create(const void* host, size_t bytes, void** dev, void* stream);
ipm_status ipm_present(const void* host, size_t bytes, void** dev);
ipm_status ipm_update_device(const void* host, size_t bytes, void* stream);
ipm_status ipm_update_host(void* host, size_t bytes, void* stream);
ipm_status ipm_copyout(void* host, size_t bytes, void* stream);
ipm_status ipm_delete(const void* host, void* stream);
int ipm_present_count(void);

/* ------------------------------------------------------------------ reductions
 * Workspace: a device buffer of ipm_workspace_bytes() bytes, 256-byte aligned, ZEROED once before first
 * use (ipm_workspace_init does that). It holds the per-CTA partials, the cross-CTA ticket, the result slot
 * and the cross-rank gather slots. Every reduce leaves the ticket at zero again, so one workspace can be
 * reused by back-to-back calls on the same stream (and inside a CUDA graph); concurrent streams need
 * separate workspaces. */
size_t ipm_workspace_bytes(void);
ipm_status ipm_workspace_init(void* ws, void* stream);

/* Flat clause over a[0..n): *inout = *inout ⊕ a[0] ⊕ ... ⊕ a[n-1].
 * dev: device array of n elements of dt, aligned to the element size. inout: host scalar of dt (in: the
 * variable's original value, out: the result). Blocks until the result is on the host (the end of an acc
 * compute region is a synchronisation point). n == 0 is not an error: no kernel is
 * launched and *inout becomes init ⊕ identity (= init, normalised to 0/1 for && ||). */
ipm_status ipm_reduce(ipm_op op, ipm_dtype dt, const void* dev, int64_t n, void* inout, void* workspace,
                      void* stream);

/* Same fold, asynchronous: init (host scalar, NULL = identity) is read during the call; the result (one
 * element of dt) is written to device memory dev_result by the kernel, in stream order. No host
 * synchronisation; capturable in a CUDA graph. One kernel launch (none when n == 0: a 1-thread finalize
 * kernel writes init ⊕ identity). */
ipm_status ipm_reduce_async(ipm_op op, ipm_dtype dt, const void* dev, int64_t n, const void* init,
                            void* dev_result, void* workspace, void* stream);

/* Nested gang-outer / vector-inner clause (BASELINE.json north_star "segmented per-row reduction"):
 *   for r in [0, rows): dev_out[r] = init ⊕ fold_{j<cols} dev[r*row_stride + j]
 * dev: device array, row-major, row_stride >= cols elements between row starts (any alignment to the
 * element size). init: host scalar (NULL = identity). dev_out: rows elements of dt, device. Asynchronous
 * (stream order). workspace may be NULL unless rows < 2 x the SM count and cols >= 2048 x (32 / element size)
 * elements, in which case each row is split across several CTAs and a workspace (as above) is required
 * (IPM_E_WORKSPACE otherwise). Passing a workspace always is safe. */
ipm_status ipm_reduce_segmented(ipm_op op, ipm_dtype dt, const void* dev, int64_t rows, int64_t cols,
                                int64_t row_stride, const void* init, void* dev_out, void* workspace,
                                void* stream);

/* The two levels of the paper's scheme as separate calls ("reducing along threads of thread
 * block on GPU and reducing along thread block on CPU"; the CUDA SRAD variant it compares against merges on the
 * GPU with "multiple serial kernel launches"). Used by tools/ablation_twolevel.py to measure that design
 * point against the one-launch path; ipm_reduce does both levels in one kernel.
 *   ipm_reduce_partials: one partial per thread block of the flat kernel, written to dev_partials as 8-byte
 *     slots holding the op's accumulator (for + and * on float32/float64 a double; for integer + * & | ^ and
 *     the logical ops the unsigned word, zero-extended; for integer max/min the signed word, sign-extended);
 *     *count = number of blocks (<= max_partials, else IPM_E_SIZE; ipm_flat_geometry gives it in advance).
 *   ipm_finalize_partials: one-warp kernel: *dev_result = init ⊕ slot[0] ⊕ ... ⊕ slot[count-1] (index order). */
ipm_status ipm_reduce_partials(ipm_op op, ipm_dtype dt, const void* dev, int64_t n, void* dev_partials,
                               int max_partials, int* count, void* stream);
ipm_status ipm_finalize_partials(ipm_op op, ipm_dtype dt, const void* dev_partials, int count, const void* init,
                                 void* dev_result, void* stream);

/* One scalar over a strided 2-D region: a gang loop over rows collapsed with the
 * vector loop over columns (SPEC.md:148 nest depth <= 2),
 *   *inout = *inout ⊕ fold_{r<rows, j<cols} dev[r*row_stride + j]
 * Rows need not be contiguous (row_stride >= cols) nor aligned beyond the element size. One kernel launch
 * (the flat kernel when row_stride == cols). rows or cols == 0 -> init ⊕ identity. */
ipm_status ipm_reduce_2d(ipm_op op, ipm_dtype dt, const void* dev, int64_t rows, int64_t cols, int64_t row_stride,
                         void* inout, void* workspace, void* stream);
ipm_status ipm_reduce_2d_async(ipm_op op, ipm_dtype dt, const void* dev, int64_t rows, int64_t cols,
                               int64_t row_stride, const void* init, void* dev_result, void* workspace,
                               void* stream);

/* Several reduction variables over ONE pass: a loop that carries more than one
 * reduction variable (">=1 scalar variable"; SPEC.md:253 a reduction list per kernel) and folds an
 * expression of the element — SRAD's reduction region accumulates the image's sum and sum of squares
 * (PAPER.md:205). Signatures (vars in this order; + wraps for integers, float32 expressions and sums in float64):
 *   IPM_FUSED_SUM_SUMSQ  v0 += x[i];      v1 += x[i]*x[i]
 *   IPM_FUSED_DOT        v0 += x[i]*y[i]                         (y: a second array, same n)
 *   IPM_FUSED_MINMAX     v0 = min(v0, x[i]); v1 = max(v1, x[i])   (float: IEEE 754-2019 minimum/maximum)
 *   IPM_FUSED_STATS      v0 += x; v1 += x*x; v2 = min; v3 = max
 * x, y: device arrays of n elements of dt; init / inout: host arrays of ipm_fused_nvars(f) elements (init
 * NULL = identities); dev_result: device array of nvars elements. One kernel launch. */
typedef enum { IPM_FUSED_SUM_SUMSQ = 0, IPM_FUSED_DOT, IPM_FUSED_MINMAX, IPM_FUSED_STATS } ipm_fused;
int ipm_fused_nvars(ipm_fused f);
ipm_status ipm_reduce_fused(ipm_fused f, ipm_dtype dt, const void* x, const void* y, int64_t n, void* inout,
                            void* workspace, void* stream);
ipm_status ipm_reduce_fused_async(ipm_fused f, ipm_dtype dt, const void* x, const void* y, int64_t n,
                                  const void* init, void* dev_result, void* workspace, void* stream);

/* Ragged nested clause: an outer gang loop over rows whose inner vector loop has
 * data-dependent bounds — BFS's adjacency loops — given in CSR form:
 *   for r in [0, rows): dev_out[r] = init ⊕ fold_{j = off[r] .. off[r+1]-1} dev[j]
 * dev_offsets: device array of rows+1 int64 element indices, non-decreasing (off[0] need not be 0; results are
 * undefined otherwise). dev: the element array (indices off[0] .. off[rows]-1 are read). dev_out: rows
 * elements. Work is balanced by elements, not rows: rows of any length, including a few huge ones, spread over
 * all SMs; rows split between warps are finished by a second one-warp-per-split kernel, folding the pieces in
 * order (deterministic). Two kernel launches; workspace required. rows < 2^31 - 1 (else IPM_E_SIZE). */
ipm_status ipm_reduce_ragged(ipm_op op, ipm_dtype dt, const void* dev, const int64_t* dev_offsets, int64_t rows,
                             const void* init, void* dev_out, void* workspace, void* stream);

/* The same clause and the same parity bar as ipm_reduce_ragged (bit-exact for integer, bitwise, logical, max and
 * min; float + * within the stated tolerance — rows are split into lane and chunk pieces at other positions, so the
 * float64 association order, and in rare cases the last bit of a float32 row sum, can differ from the default
 * kernel's; deterministic from run to run), computed in two passes over caller-owned scratch: a row-parallel pass marks where every row starts in a bitmap over the elements, counts the row starts
 * per chunk of 512 elements (256 for 8-byte types) and writes every EMPTY row (init ⊕ identity); an
 * element-parallel pass then folds the elements, reading each lane's row-start flags from the bitmap and naming
 * rows by rank within their chunk instead of walking the row offsets per chunk.
 * nvalues: the element array's length, >= off[rows] (the bound the scratch is sized from).
 * scratch: 256-byte aligned device buffer of at least ipm_ragged_scratch_bytes(dt, nvalues, rows) bytes, caller-owned;
 *   its contents on entry do not matter (the library zeroes it in stream order); not used after the call's
 *   kernels complete. Too small -> IPM_E_WORKSPACE; misaligned -> IPM_E_ALIGN.
 * Four launches on `stream` (memset, mark, fold, fix-up); workspace as for ipm_reduce_ragged. */
size_t ipm_ragged_scratch_bytes(ipm_dtype dt, int64_t nvalues, int64_t rows);
ipm_status ipm_reduce_ragged_marked(ipm_op op, ipm_dtype dt, const void* dev, int64_t nvalues,
                                    const int64_t* dev_offsets, int64_t rows, const void* init, void* dev_out,
                                    void* workspace, void* scratch, size_t scratch_bytes, void* stream);

/* End-to-end clause over a HOST array: the data clause `copyin(a[0:n])` fused with the reduction. The host
 * array is streamed to the device in chunks through two library-owned staging buffers (allocated once
 * through the allocator hook and kept until ipm_release_staging), each chunk's H2D copy overlapping the
 * reduction of the previous chunk; partial results stay on the device; one 8-byte D2H at the end.
 * Pinned host memory is fastest; pageable memory works. Blocks until *inout holds the result.
 * Thread safety: concurrent calls from several host threads on different streams (each with its own workspace)
 * are safe — they share the staging buffers, and a call's copies into a buffer wait for the previous caller's
 * last kernel that read it (so concurrent host-path calls partly serialise on the two buffers). */
ipm_status ipm_reduce_host(ipm_op op, ipm_dtype dt, const void* host, int64_t n, void* inout, void* workspace,
                           void* stream);
ipm_status ipm_release_staging(void);

/* Kernel timing (tracing): while enabled, the library records a CUDA event pair on the launch stream around
 * each reduction kernel it launches (not the one-warp finalize), up to max_records launches (later launches
 * are not recorded). ipm_profile_read waits for the recorded events and returns the per-launch durations in
 * milliseconds, in launch order, plus the number of recorded launches; it also returns the kernel kind of each
 * record in `kinds` when non-NULL: 0 flat (incl. per-block partials and the fused multi-GPU exchange),
 * 1 segmented, 2 several variables (fused), 3 strided 2-D, 4 ragged (one record covers the ragged kernel and
 * its fix-up). Disable frees the events. Not thread-safe with concurrent launches from other threads. */
ipm_status ipm_profile_enable(int max_records);
ipm_status ipm_profile_read(float* ms, int* kinds, int max, int* count);
ipm_status ipm_profile_disable(void);

/* Tuning options (process-wide; the defaults are the measured best):
 *   IPM_OPT_FLAT_CTAS_PER_SM  CTAs per SM of the flat kernel's persistent grid, 1..8 (-1 = default 4)
 *   IPM_OPT_SEG_KERNEL        segmented rows: 0 auto (= 1), 1 one warp per row with direct 256-bit loads,
 *                             2 one warp per row fed by TMA bulk copies into a per-warp shared-memory ring
 *                             (rows of >= 64 bytes). (One CTA per row was measured slower: profiles/
 *                             r01_seg_kernels.txt.)
 *   IPM_OPT_DETERMINISTIC     1 (default): the flat clause uses the guided schedule — ~90% of the tiles
 *                             dealt statically, the rest in fixed chunks claimed dynamically, one partial per
 *                             element range, folded in a fixed order — so repeated runs give identical bits
 *                             for every op; 0: purely dynamic tiles (float + and * may then differ in the last
 *                             bits between runs); 2: static grid-stride tiles (deterministic, no balancing).
 * IPM_E_ARG for an unknown key or an out-of-range value. */
typedef enum {
  IPM_OPT_FLAT_CTAS_PER_SM = 0,
  IPM_OPT_SEG_KERNEL = 1,
  IPM_OPT_DETERMINISTIC = 2,
  IPM_OPT_DIST_MODE = 3,        /* 0 (default): fused peer-memory exchange when every peer is mapped; 1: NCCL */
  IPM_OPT_DIST_TIMEOUT_MS = 4,  /* fused exchange: give up waiting for a peer after this long (default 30000) */
  IPM_OPT_RAGGED_KERNEL = 5     /* ragged rows: 0 auto (1 below 256 elements per row on average over the whole
                                   input, 128 for 8-byte types, else 4; both launched, the device picks, no host
                                   sync),
                                   1 one warp per element range (k_ragged_vec),
                                   2 one CTA per element range in tiles (k_ragged_tile),
                                   3 one warp per element range, rows finished in row order (k_ragged_rank),
                                   4 one warp per element range, lane per row over shared-memory windows
                                     (k_ragged_lpr). Measured on one B200: 1 the fastest on
                                     rows of tens of elements, 3 on short power-law rows, 4 on rows of >= 256.
                                   The two-pass form is a separate entry point, ipm_reduce_ragged_marked (the
                                   fastest on short power-law rows; this option does not apply to it). */
} ipm_option;
ipm_status ipm_set_option(ipm_option key, int64_t value);

/* Launch geometry the library uses for a flat reduce of n elements (for tests and the roofline report). */
ipm_status ipm_flat_geometry(ipm_dtype dt, int64_t n, int* grid, int* block);
/* Which flat kernel ipm_reduce / ipm_reduce_async would launch for n elements of dt under the current options
 * (the same decision function the launch uses): 0 static grid-stride tiles (inputs <= 64 MiB, or
 * IPM_OPT_DETERMINISTIC = 2), 1 the guided deterministic schedule (k_flat_guided, the default above 64 MiB),
 * 2 purely dynamic tiles (IPM_OPT_DETERMINISTIC = 0), -1 no reduction kernel (n == 0). For tests that must
 * know which schedule they exercised. */
ipm_status ipm_flat_schedule(ipm_dtype dt, int64_t n, int* schedule);
/* The identity of op on dt as one element of dt ("per-thread private v initialized to op's
 * identity"): 0 for + | ^ ||; 1 (1.0) for * &&; the type's minimum (-inf) for max, maximum (+inf) for min; all
 * bits set for &. init = identity makes init ⊕ fold == fold, so a caller of the synchronous calls (whose `inout`
 * always carries an original value) passes this when the variable has none. IPM_E_REDOP for an illegal pair. */
ipm_status ipm_identity(ipm_op op, ipm_dtype dt, void* out);

/* ------------------------------------------------------------------ multi-GPU (one process per GPU)
 * The iteration space is sharded contiguously: rank r owns [r*n/P, (r+1)*n/P) (floor division, 128-bit
 * intermediate) — ipm_shard_range computes it (pure host function). Each rank reduces its shard on its GPU
 * into an accumulator-typed partial (no host sync); the P partials are exchanged and every rank folds them in
 * rank order, merges init and rounds — so every rank gets the same bits. Exchange:
 * fused (default when every peer's 8 KiB symmetric slot buffer is mapped through CUDA IPC): the reduction
 * kernel's last CTA stores the partial into every peer's buffer over NVLink and folds the P slots — one kernel
 * per rank per call; otherwise ONE ncclAllGather of the partials + a one-warp fold kernel.
 * Bootstrap with NCCL: rank 0 calls ipm_comm_unique_id, the id (ipm_comm_id_bytes() bytes) is broadcast out
 * of band (the Python binding uses the torch.distributed store), then every rank calls ipm_comm_init (which
 * also exchanges the slot-buffer IPC handles with ncclAllGather and agrees on the fused path). */
typedef struct ipm_comm ipm_comm;
size_t ipm_comm_id_bytes(void);
ipm_status ipm_comm_unique_id(void* id_out);
ipm_status ipm_comm_init(ipm_comm** comm, int rank, int world, const void* id, int device);
ipm_status ipm_comm_destroy(ipm_comm* comm);
/* `world` ranks in ONE process on ONE device (comms[0..world-1]), exchanging through each other's slot buffers
 * with the fused path only (no NCCL). Each rank's calls go on its own stream with its own workspace; the ranks'
 * kernels then run concurrently on the device. Used to exercise the multi-rank exchange on a single GPU. */
ipm_status ipm_comm_init_group(ipm_comm** comms, int world, int device);
/* Bootstrap WITHOUT NCCL (fused exchange only): every rank calls ipm_comm_create_ipc, which allocates its
 * symmetric slot buffer and writes its CUDA IPC handle (ipm_comm_ipc_handle_bytes() bytes) to handle_out; the
 * caller moves the handles between the ranks out of band (any transport) and every rank calls
 * ipm_comm_attach_ipc with all `world` handles in rank order (its own included, ignored). The ranks are
 * processes on the GPUs of one node (peer mappings over NVLink) or on the same GPU. attach returns IPM_E_CUDA
 * if a peer buffer cannot be mapped; the ranks must then all give up (there is no fallback without NCCL). Until
 * attach succeeds, reduce calls on the communicator return IPM_E_ARG. */
size_t ipm_comm_ipc_handle_bytes(void);
ipm_status ipm_comm_create_ipc(ipm_comm** comm, int rank, int world, int device, void* handle_out);
ipm_status ipm_comm_attach_ipc(ipm_comm* comm, const void* handles);
ipm_status ipm_shard_range(int64_t n, int rank, int world, int64_t* lo, int64_t* hi);
/* dev_shard: this rank's n_shard elements (device); inout: host scalar, the same init on every rank (in),
 * the global result (out). Blocks until *inout is written. */
ipm_status ipm_reduce_dist(ipm_comm* comm, ipm_op op, ipm_dtype dt, const void* dev_shard, int64_t n_shard,
                           void* inout, void* workspace, void* stream);
/* End-to-end multi-GPU clause over HOST shards: each rank's host_shard (n_shard elements, pinned fastest) is
 * streamed to its device through the staging ring of ipm_reduce_host and folded into an accumulator partial on
 * the device, then the partials are exchanged exactly as in ipm_reduce_dist. inout: host scalar, the same init on
 * every rank (in) and the global result (out). Blocks until *inout is written. */
ipm_status ipm_reduce_host_dist(ipm_comm* comm, ipm_op op, ipm_dtype dt, const void* host_shard, int64_t n_shard,
                                void* inout, void* workspace, void* stream);
/* 1 if ipm_reduce_dist on this communicator takes the fused path: every peer's symmetric slot buffer is mapped
 * (CUDA IPC over NVLink) and IPM_OPT_DIST_MODE is 0 — the reduction kernel then exchanges the rank partials
 * itself (one kernel per rank per call). 0: ncclAllGather + a one-warp fold kernel. */
int ipm_comm_uses_peer_memory(const ipm_comm* comm);
/* Fused path only: *err = 1 if a call since the last check gave up waiting for a peer (IPM_OPT_DIST_TIMEOUT_MS);
 * the flag is cleared. ipm_reduce_dist checks it itself and returns IPM_E_NCCL. */
ipm_status ipm_comm_error(ipm_comm* comm, int* err);
/* Asynchronous form: result written to dev_result (device, one element) in stream order. */
ipm_status ipm_reduce_dist_async(ipm_comm* comm, ipm_op op, ipm_dtype dt, const void* dev_shard,
                                 int64_t n_shard, const void* init, void* dev_result, void* workspace,
                                 void* stream);

#ifdef __cplusplus
}
#endif
#endif /* IPM_H */
