/*
 * grkan_b200.h -- C ABI of the B200-native GR-KAN group-rational activation.
 *
 * The drop-in boundary for the FlashKAT hot path: plain pointers, sizes and a
 * CUDA stream handle; no torch or CUDA types in the signatures.  Every call is
 * stream-ordered, allocation-free, sync-free (except grkan_read_status) and
 * reentrant; the library keeps no mutable globals besides a once-initialised
 * device-attribute cache.
 *
 * Reference interfaces replaced (all in /root/reference):
 *   grkan_fwd          forward_tensor(x, params, layout, validate)
 *                        pkg/src/grkan/rational.py:325-345
 *                      (element math rational_values, rational.py:218-224)
 *   grkan_bwd          backward_blocked(x, upstream, params, plan, ...) -> GradBundle
 *                        pkg/src/grkan/backward.py:275-372
 *                      (gradient_terms rational.py:227-278, block_partial_totals
 *                       backward.py:122-139, combine_partials backward.py:142-179,
 *                       _check_accumulators backward.py:182-184)
 *   grkan_bwd_workspace_bytes
 *                      ExecutionPlan.blocked geometry, backward.py:51-98
 *   grkan_bwd_atomic   backward_naive as the model of the paper's Alg. 1
 *                        pkg/src/grkan/backward.py:187-246 (comparator only)
 *   grkan_status       GrkanError taxonomy, pkg/src/grkan/errors.py:4-37
 *
 * Tensor layout: x, dy, y, dx are dense row-major [rows, d] (rows = B*L),
 * element type given by `dtype`.  The feature dim is split into n_groups equal
 * contiguous groups of width d / n_groups (GroupLayout, rational.py:31-55).
 * Coefficients: a = [n_groups, m1] (a_0..a_m), b = [n_groups, n] (b_1..b_n),
 * both float32 for GRKAN_F32 / GRKAN_BF16 tensors and float64 for GRKAN_F64
 * (the reference casts its fp64 parameters to the tensor dtype at use,
 * rational.py:220-221).  da/db come back in that same coefficient dtype.
 */
#ifndef GRKAN_B200_H_
#define GRKAN_B200_H_

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define GRKAN_API __attribute__((visibility("default")))
#else
#define GRKAN_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

/* Status codes: the reference's error classes (errors.py:4-37) plus CUDA. */
typedef enum grkan_status {
  GRKAN_OK = 0,
  GRKAN_ERR_LAYOUT = 1,            /* LayoutMismatchError   (rational.py:41-45, 313-322) */
  GRKAN_ERR_GRID = 2,              /* GridGeometryError     (backward.py:86-98, 298-299) */
  GRKAN_ERR_NONFINITE_INPUT = 3,   /* NonFiniteInputError   (rational.py:174-179)        */
  GRKAN_ERR_ACCUM_OVERFLOW = 4,    /* AccumulationOverflowError (backward.py:182-184)    */
  GRKAN_ERR_UNSUPPORTED = 5,       /* dtype / degree this build does not provide         */
  GRKAN_ERR_CUDA = 6,              /* a CUDA runtime call failed                         */
  GRKAN_ERR_INVALID = 7,           /* null pointer, short workspace, bad flag            */
  GRKAN_ERR_PEER_TIMEOUT = 8       /* grkan_bwd_p2p: a peer rank never arrived            */
} grkan_status;

/* Element types; 0/1 match the GRKB dump dtype codes (cli.py:54). */
typedef enum grkan_dtype { GRKAN_F32 = 0, GRKAN_F64 = 1, GRKAN_BF16 = 2 } grkan_dtype;

/* Flags. */
#define GRKAN_FLAG_FAST 0u         /* FMA + approximate reciprocal; max-scaled <= 1e-5 */
#define GRKAN_FLAG_EXACT 1u        /* reference op order, IEEE-rounded ops: bitwise y/dx */
#define GRKAN_FLAG_CHECK_FINITE 2u /* checked mode: flag NaN/Inf inputs (validate=True) */
#define GRKAN_FLAG_DETERMINISTIC 4u /* grkan_bwd: partials per global row block (see below) */

/* Highest supported degrees (m1 = m + 1 numerator coefficients, n denominator). */
#define GRKAN_MAX_M1 12
#define GRKAN_MAX_N 12

GRKAN_API const char* grkan_version(void);
GRKAN_API const char* grkan_status_string(int status);
/* Message for the last non-OK status returned on this host thread. */
GRKAN_API const char* grkan_last_error(void);

/* Device status words written by the kernels (checked mode / overflow). */
typedef struct grkan_device_status {
  int32_t nonfinite_input; /* 1 if any x / dy element was NaN or Inf (CHECK_FINITE) */
  int32_t accum_overflow;  /* 1 if any da / db entry is non-finite                  */
  int32_t peer_timeout;    /* 1 if grkan_bwd_p2p's wait for the peers expired        */
  int32_t reserved;
} grkan_device_status;

/* Forward: y = P(x) / (1 + |A(x)|) per group.  `status` may be NULL unless
 * GRKAN_FLAG_CHECK_FINITE is set; it is zeroed and then written in-stream. */
GRKAN_API int grkan_fwd(const void* x, void* y, const void* a, const void* b, int64_t rows, int32_t d,
              int32_t n_groups, int32_t m1, int32_t n, int32_t dtype, uint32_t flags,
              grkan_device_status* status, void* stream);

/* Workspace for grkan_bwd: status words + one partial per (row tile, group). */
GRKAN_API size_t grkan_bwd_workspace_bytes(int64_t rows, int32_t d, int32_t n_groups, int32_t m1,
                                 int32_t n, int32_t dtype);

/* Backward: dx (like x) and da [n_groups, m1], db [n_groups, n].
 * Two kernels, no atomics: per-CTA partials, then a fixed-order reduction
 * (bitwise reproducible run to run).  The device status (overflow, and
 * non-finite inputs under CHECK_FINITE) lands at the start of `ws`. */
GRKAN_API int grkan_bwd(const void* x, const void* dy, const void* a, const void* b, void* dx, void* da,
              void* db, void* ws, size_t ws_bytes, int64_t rows, int32_t d, int32_t n_groups,
              int32_t m1, int32_t n, int32_t dtype, uint32_t flags, void* stream);

/* Fused forward + backward step: y (forward_tensor) and dx, da, db
 * (backward_blocked) of the same x and upstream dy in ONE pass -- x is read once
 * and y comes from the backward's own P(x) and 1/Q(x) (rational.py:218-278 share
 * them).  Same results as grkan_fwd + grkan_bwd (EXACT: y, dx bitwise; da/db the
 * per-CTA fold).  For plans without the fused kernel (non-(5,4) degrees,
 * unaligned tensors, DETERMINISTIC) it runs the two passes back to back.  `ws`
 * as for grkan_bwd (the forward's CHECK_FINITE status shares it). */
GRKAN_API int grkan_fwd_bwd(const void* x, const void* dy, const void* a, const void* b, void* y, void* dx,
                            void* da, void* db, void* ws, size_t ws_bytes, int64_t rows, int32_t d,
                            int32_t n_groups, int32_t m1, int32_t n, int32_t dtype, uint32_t flags,
                            void* stream);

/* The paper's Alg. 1 (per-element global atomicAdd into da/db).  Comparator
 * for the speed and rounding claims only; not used by the product path.
 * `status` receives the overflow flag (may be NULL). */
GRKAN_API int grkan_bwd_atomic(const void* x, const void* dy, const void* a, const void* b, void* dx,
                     void* da, void* db, int64_t rows, int32_t d, int32_t n_groups, int32_t m1,
                     int32_t n, int32_t dtype, uint32_t flags, grkan_device_status* status,
                     void* stream);

/* Deterministic (row-sharding-invariant) coefficient gradients.
 *
 * The multi-GPU analogue of backward_blocked's worker-count invariance
 * (backward.py:275-372 with combine_partials' ordered fold, 142-179;
 * pkg/tests/test_acceptance.py:232-252): rows are cut into global blocks of
 * grkan_det_block_rows() rows; each block's m1 + n partial sums are computed in
 * a fixed order that depends only on the block's data, stored slot-major
 * part[(block * n_groups + g) * (m1 + n) + k], and folded by
 * grkan_reduce_partials in global block order.  A run sharded over any number
 * of ranks at block-aligned row boundaries, with the per-rank partial arrays
 * concatenated in rank order (an all-gather), gives bitwise the da / db of
 * grkan_bwd(..., GRKAN_FLAG_DETERMINISTIC) on the whole tensor (for one
 * kernel family: 16-byte-aligned tensors on every rank).  dx is unaffected. */
GRKAN_API int64_t grkan_det_block_rows(int32_t d, int32_t n_groups, int32_t dtype);
GRKAN_API size_t grkan_det_partials_bytes(int64_t rows, int32_t d, int32_t n_groups, int32_t m1, int32_t n,
                                          int32_t dtype);
/* dx plus this shard's per-block partials (no reduction).  `status` may be
 * NULL unless GRKAN_FLAG_CHECK_FINITE is set. */
GRKAN_API int grkan_bwd_partials(const void* x, const void* dy, const void* a, const void* b, void* dx,
                                 void* part, size_t part_bytes, int64_t rows, int32_t d, int32_t n_groups,
                                 int32_t m1, int32_t n, int32_t dtype, uint32_t flags,
                                 grkan_device_status* status, void* stream);
/* Fixed-order fp64 fold of n_blocks slot-major partials into da / db; the
 * overflow flag lands in `status` (required). */
GRKAN_API int grkan_reduce_partials(const void* part, int64_t n_blocks, int32_t n_groups, int32_t m1,
                                    int32_t n, void* da, void* db, int32_t dtype, grkan_device_status* status,
                                    void* stream);

/* Fused GR-KAN layer backward through its linear map (the
 * reference's layer_backward, pkg/src/grkan/layer.py:318-379, step by step):
 *   dF = dY . W  on the tcgen05 tensor cores (bf16 x bf16 -> fp32 in TMEM),
 *   dX = R'(X, dF) and the per-tile da / db partials in the epilogue,
 * then the fixed-order fold (as grkan_bwd) -- dF never touches HBM.
 * dY [M, K], W [K, N] (torch Linear weight [out, in]), X / dX [M, N]: bf16,
 * row-major, 16-byte aligned; a [n_groups, 6], b [n_groups, 4], da, db: fp32
 * (degrees (5, 4)); FAST policy.  Needs K % 64 == 0 and a group width
 * N / n_groups that is a multiple of 32.  Status words at the start of `ws`. */
GRKAN_API size_t grkan_linear_bwd_workspace_bytes(int64_t M, int32_t N, int32_t K, int32_t n_groups);
GRKAN_API int grkan_linear_bwd(const void* dy, const void* w, const void* x, const void* a, const void* b,
                               void* dx, void* da, void* db, void* ws, size_t ws_bytes, int64_t M, int32_t N,
                               int32_t K, int32_t n_groups, uint32_t flags, void* stream);


/* K3 fused with the cross-GPU da||db sum over peer memory:
 * grkan_bwd_p2p runs K2, then ONE kernel that folds this rank's partials,
 * stores the fp64 column values into every rank's exchange buffer through
 * CUDA-IPC-mapped pointers (NVLink), bumps every rank's arrival counter and,
 * once all ranks arrived, folds the world values in rank order -- no NCCL
 * launch, bitwise-identical da/db on every rank.  `peer_bufs` is a DEVICE
 * array of `world` pointers: rank r's exchange buffer mapped into this
 * process (own buffer at index `rank`); each buffer comes from
 * grkan_p2p_alloc(grkan_p2p_buffer_bytes(...)) (zeroed); `epoch` counts calls
 * from 1 and must advance identically on every rank. */
#define GRKAN_IPC_HANDLE_BYTES 64
GRKAN_API size_t grkan_p2p_buffer_bytes(int32_t world, int32_t n_groups, int32_t m1, int32_t n);
GRKAN_API int grkan_p2p_alloc(size_t bytes, void** out);
GRKAN_API int grkan_p2p_free(void* ptr);
GRKAN_API int grkan_ipc_get_handle(const void* dev_ptr, void* handle_out);
GRKAN_API int grkan_ipc_open_handle(const void* handle, void** dev_ptr_out);
GRKAN_API int grkan_ipc_close_handle(void* dev_ptr);
GRKAN_API int grkan_bwd_p2p(const void* x, const void* dy, const void* a, const void* b, void* dx, void* da,
                            void* db, void* ws, size_t ws_bytes, int64_t rows, int32_t d, int32_t n_groups,
                            int32_t m1, int32_t n, int32_t dtype, uint32_t flags, void* const* peer_bufs,
                            int32_t rank, int32_t world, uint64_t epoch, void* stream);

/* Per-element gradient terms (the reference's gradient_terms,
 * pkg/src/grkan/rational.py:227-278): dx plus the m1 + n per-element
 * contributions, unreduced, into terms[(k) * rows * d + i] (coefficient dtype).
 * Introspection / parity only (10x the output of grkan_bwd); EXACT gives the
 * reference's terms bit for bit. */
GRKAN_API int grkan_bwd_terms(const void* x, const void* dy, const void* a, const void* b, void* dx, void* terms,
                              int64_t rows, int32_t d, int32_t n_groups, int32_t m1, int32_t n, int32_t dtype,
                              uint32_t flags, void* stream);

/* Synchronise `stream` and copy the device status to the host; maps it to a
 * status code (NONFINITE_INPUT first, then PEER_TIMEOUT, then ACCUM_OVERFLOW,
 * else OK). */
GRKAN_API int grkan_read_status(const grkan_device_status* status, void* stream,
                      grkan_device_status* host_out);

/* Backward launch geometry for 16-byte-aligned tensors on a 148-SM B200 (for
 * tests / the access model): out[0]=vector width, out[1]=threads per CTA,
 * out[2]=rows per tile (direct kernels) or per pipeline stage (staged),
 * out[3]=partials per group, out[4]=CTAs, out[5]=1 if TMA-staged. */
GRKAN_API int grkan_plan(int64_t rows, int32_t d, int32_t n_groups, int32_t m1, int32_t n, int32_t dtype,
                         int64_t* out6);

/* The reference's combine_partials fold itself (pkg/src/grkan/backward.py:142-179):
 * d_a[g] += pa from zeros, entry by entry in the given fold order (the caller sorts by
 * block_id for deterministic_ordered, keeps the submission order for
 * unordered_scatter), in the partials' dtype (GRKAN_F32 / GRKAN_F64) with separately
 * rounded adds -- bitwise the reference's result, absorption included
 * (pkg/tests/test_backward.py:193-209).  part[i * (num_w + den_w) + k] holds entry i's
 * numerator then denominator partials; group_of[i] = block_id % n_groups.  All
 * pointers are device pointers; stream-ordered. */
GRKAN_API int grkan_combine_partials(const void* part, const int32_t* group_of, int64_t n_entries,
                                     int32_t n_groups, int32_t num_w, int32_t den_w, void* da, void* db,
                                     int32_t dtype, void* stream);

/* Access instrumentation: the reference's counter= / coverage= arguments of
 * backward_blocked / backward_naive (pkg/src/grkan/backward.py:187-195, 275-285,
 * 326-351) and instrumented_backward (pkg/src/grkan/access.py:129-161).  Runs the
 * SAME kernels as grkan_bwd (naive = 0) or grkan_bwd_atomic (naive = 1), in their
 * counting instantiations: every element a thread processes adds 1 to
 * coverage[row * d + col] (device int32 [rows * d]), and every kernel adds the
 * element-sized global accesses it performs to counts[0..2] = {reads, writes, rmw}
 * (device uint64[3]; an atomic add is 1 read + 1 write + 1 rmw, as the reference
 * models it).  Both accumulate: zero them first.  Unchecked, per-CTA partials; the
 * device status (overflow) lands at the start of `ws` as for grkan_bwd. */
GRKAN_API int grkan_bwd_instrumented(const void* x, const void* dy, const void* a, const void* b, void* dx,
                                     void* da, void* db, void* ws, size_t ws_bytes, int32_t* coverage,
                                     unsigned long long* counts, int64_t rows, int32_t d, int32_t n_groups,
                                     int32_t m1, int32_t n, int32_t dtype, uint32_t flags, int32_t naive,
                                     void* stream);
/* CTAs one launch uses on this device (kernel 0 = grkan_fwd, 1 = grkan_bwd's K2,
 * 2 = grkan_bwd_atomic) for 16-byte-aligned tensors; -1 on a layout error.  The
 * access model's closed forms need it (one coefficient row load per CTA). */
GRKAN_API int64_t grkan_launch_ctas(int64_t rows, int32_t d, int32_t n_groups, int32_t m1, int32_t n,
                                    int32_t dtype, int32_t kernel);

/* ---- Host-array calls (the reference's own calling convention) -------------------
 *
 * The reference's forward_tensor / backward_blocked take and return host (NumPy)
 * arrays (pkg/src/grkan/rational.py:325-345, pkg/src/grkan/backward.py:275-372).
 * These calls accept plain pageable host pointers, stream the rows through
 * pinned staging slots with host copies, PCIe transfers and kernels overlapped,
 * and return when the outputs are in host memory (synchronous).  A context owns
 * the staging memory, three streams and a pool of host copy threads; one
 * context per host thread (calls on one context are not concurrent-safe).
 *   grkan_host_fwd  forward_tensor    (status: LAYOUT / GRID / NONFINITE_INPUT)
 *   grkan_host_bwd  backward_blocked  (status: ... / ACCUM_OVERFLOW); da / db are the
 *                   deterministic-family fold (bitwise independent of chunk_bytes:
 *                   equal to grkan_bwd(..., GRKAN_FLAG_DETERMINISTIC) on the whole tensor).
 * Coefficients a / b and da / db are host arrays in the coefficient dtype.  Page-locked
 * x / dy / y / dx buffers are transferred in place (no staging copy). */
typedef struct grkan_host_ctx grkan_host_ctx;
/* chunk_bytes: staging per tensor per slot (0 = 32 MiB); threads: host copy threads
 * (0 = min(16, hardware threads)). */
GRKAN_API int grkan_host_create(int32_t device, size_t chunk_bytes, int32_t threads, grkan_host_ctx** out);
GRKAN_API int grkan_host_destroy(grkan_host_ctx* ctx);
GRKAN_API int grkan_host_threads(const grkan_host_ctx* ctx);
GRKAN_API const char* grkan_host_last_error(void);
GRKAN_API int grkan_host_fwd(grkan_host_ctx* ctx, const void* x, void* y, const void* a, const void* b,
                             int64_t rows, int32_t d, int32_t n_groups, int32_t m1, int32_t n, int32_t dtype,
                             uint32_t flags);
GRKAN_API int grkan_host_bwd(grkan_host_ctx* ctx, const void* x, const void* dy, const void* a, const void* b,
                             void* dx, void* da, void* db, int64_t rows, int32_t d, int32_t n_groups, int32_t m1,
                             int32_t n, int32_t dtype, uint32_t flags);

#ifdef __cplusplus
}
#endif

#endif /* GRKAN_B200_H_ */
