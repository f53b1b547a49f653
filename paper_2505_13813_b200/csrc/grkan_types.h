// grkan_types.h -- plain types shared by the host launch code and the kernels.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace grkan {

struct Geom {
  int64_t rows;     // B*L
  int64_t n_tiles;  // ceil(rows / R)
  int32_t d;        // feature dim (row stride, elements)
  int32_t ng;       // groups
  int32_t dg;       // group width
  int32_t V;        // 16-byte vectors per row segment = dg / W
  int32_t R;        // rows per tile (direct kernels)
  int32_t dr, dc;   // kBlock = dr * V + dc: flat-index step in (row, vector) units
  // staged kernels: persistent, statically balanced partition
  int32_t RS;       // rows per pipeline stage
  int32_t pg;       // CTAs per group (= partials per group = n_tiles)
  int64_t nsu;      // stage units per group = ceil(rows / RS)
  float one;        // 1.0f, opaque to ptxas (see grkan_math.cuh xmad2)
  int32_t flush;    // staged backward: stages between per-lane accumulator flushes
  int32_t RU;       // staged: rows per partition unit (RS; RB in deterministic mode)
  int32_t det;      // deterministic (global row-block) partials: slot-major
                    // part[(block * ng + g) * kc + k], one partial per RB-row block
  int32_t spb;      // staged deterministic: stages per block (RB / RS)
  // staged bf16 FAST backward: per-CTA table of the x-only factors over the x
  // exponent window [lut_e0, lut_e0 + lut_ne) (biased fp32/bf16 exponents)
  int32_t lut_e0;
  int32_t lut_ne;   // 0: no table
  uint32_t lut_c;   // (0x4000 - (lut_e0 << 7)) * 0x10001: the slot offset of both halves of a bf16 pair
  // staged kernels: rows per TMA box (tensor-map copies of RS-row stages,
  // RS / tma_rows boxes per tensor); 0: one bulk copy per row segment.  The map
  // views [rows, d] as [rows, d / tma_ci, tma_ci] (box inner extent <= 256).
  int32_t tma_rows;
  int32_t tma_ci;
  // staged backward at two or more CTAs per SM: the first wave of CTAs (bid <
  // wave, one per SM) gets w1/64 of a later CTA's share of the group's stage
  // units (the warp schedulers favour the older CTA: without it, the second CTA
  // of every SM finished ~10 us after the first at KAT-S fp32).  w1 = 64: even.
  int32_t w1;
  int32_t wave;
  // staged backward without CHECK_FINITE: CTA 0 zeroes the status block at its
  // start instead of a cudaMemsetAsync before the launch (no other K2 CTA
  // writes it, K3 writes it only after griddepcontrol.wait, i.e. after K2)
  int32_t zst;
  // instrumented launches only (grkan_bwd_instrumented; null otherwise): per-element
  // visit counts [rows * d] and element-access tallies {reads, writes, rmw}
  int32_t* cov;
  unsigned long long* cnt;
};

struct DevStatus {
  int32_t nonfinite_input;
  int32_t accum_overflow;
  int32_t peer_timeout;  // grkan_bwd_p2p: a peer never arrived (bounded wait expired)
  int32_t reserved;
};

constexpr int kBlock = 256;    // threads per CTA for K1 / K2 / K4
constexpr int kMinBlocks = 3;  // register cap 85 / thread -> 24 warps per SM

// Vectors per tensor each thread loads before computing (must match Engine::U).
inline int unroll_for_width(int W) { return W >= 2 ? 2 : 4; }

struct Plan {
  int W = 1;          // elements per 16-byte vector (1 = scalar path)
  int threads = kBlock;
  int cw = 0;         // staged backward: consumer warps per CTA (GRKAN_CONSUMER_WARPS or GRKAN_WIDE_WARPS)
  int64_t ctas = 0;
  Geom geo{};
  bool staged = false;  // TMA-bulk-staged persistent kernels (grkan_staged.cuh)
  int stages = 0;       // shared-memory ring depth
  size_t smem = 0;      // dynamic shared memory per CTA
};

// Staged-kernel geometry (compile-time; overridable with -D for tuning builds,
// see tools/build_variant.py).  Shared by the host planner and the kernels.
#ifndef GRKAN_CONSUMER_WARPS
#define GRKAN_CONSUMER_WARPS 8     // consumer warps per staged CTA (+1 producer warp)
#endif
#ifndef GRKAN_STAGE_VECS
#define GRKAN_STAGE_VECS 768       // 16-byte vectors per tensor per pipeline stage
#endif
#ifndef GRKAN_BWD_CTAS
#define GRKAN_BWD_CTAS 2           // staged backward CTAs per SM (register cap)
#endif
#ifndef GRKAN_BWD_STAGES
#define GRKAN_BWD_STAGES 4         // staged backward ring depth
#endif
#ifndef GRKAN_WIDE_WARPS
#define GRKAN_WIDE_WARPS 16        // wide backward geometry: consumer warps of its one CTA per SM
#endif
#ifndef GRKAN_SIGN_GUARD
#define GRKAN_SIGN_GUARD 1        // FAST: FMA-evaluated A(x) with the sign guard (0: reference-rounded A)
#endif
#ifndef GRKAN_BF16_GUARD
#define GRKAN_BF16_GUARD 0        // sign guard for bf16 I/O too
#endif
#ifndef GRKAN_GUARD_NP
#define GRKAN_GUARD_NP 2          // FAST sign guard: element pairs per guard branch
#endif
#ifndef GRKAN_FWD_CONSUMER_WARPS
#define GRKAN_FWD_CONSUMER_WARPS 2 // consumer warps per staged forward CTA
#endif
#ifndef GRKAN_FWD_STAGE_VECS
#define GRKAN_FWD_STAGE_VECS 192   // 16-byte vectors per forward pipeline stage
#endif
#ifndef GRKAN_FWD_STAGES
#define GRKAN_FWD_STAGES 4         // staged forward ring depth
#endif
#ifndef GRKAN_FULL_STAGE
#define GRKAN_FULL_STAGE 1        // staged backward: branch-free path for full stages
#endif
#ifndef GRKAN_DET_ROWS
#define GRKAN_DET_ROWS 128        // deterministic mode: minimum rows per global block
#endif
#ifndef GRKAN_PROBE_NOMEM
#define GRKAN_PROBE_NOMEM 0       // diagnostic only: staged backward computes on unfilled shared memory
#endif
#ifndef GRKAN_LUT_PAIRED
#define GRKAN_LUT_PAIRED 1        // bf16 table as (1/Q, factor) float2 pairs: one 8-byte load per element (0: two arrays)
#endif
#ifndef GRKAN_SKEW64
#define GRKAN_SKEW64 64           // staged backward, >= 2 CTAs per SM: first-wave share in 1/64 units
#endif
#ifndef GRKAN_PROBE_TIMES
#define GRKAN_PROBE_TIMES 0       // diagnostic only: %globaltimer stamps of the staged backward's CTAs
#endif
#ifndef GRKAN_FWD_CTAS
#define GRKAN_FWD_CTAS 8
#endif
#ifndef GRKAN_LUT
#define GRKAN_LUT 1               // bf16 FAST backward: per-CTA table of the x-only factors
#endif
#ifndef GRKAN_TMA2D_MAX_ROW_BYTES
#define GRKAN_TMA2D_MAX_ROW_BYTES 512  // staged backward: tensor-map stage copies for row segments up to this size
#endif
#ifndef GRKAN_TMA_BF16_BWD
#define GRKAN_TMA_BF16_BWD 1      // bf16 backward (issue-bound): tensor-map stage copies at any row length
#endif
#ifndef GRKAN_TMA2D_MAX_ROW_BYTES_FWD
#define GRKAN_TMA2D_MAX_ROW_BYTES_FWD 128  // staged forward: the same, smaller stages
#endif
#ifndef GRKAN_WAIT_HINT_NS
#define GRKAN_WAIT_HINT_NS 1000000  // staged ring waits: mbarrier.try_wait suspend-time hint (0: none)
#endif
#ifndef GRKAN_LUT_STAGES
#define GRKAN_LUT_STAGES 3        // ring depth when the table shares shared memory
#endif
#ifndef GRKAN_LUT_TOP
#define GRKAN_LUT_TOP 129         // highest tabulated biased exponent: |x| < 2^3
#endif
constexpr int kLutSignStride = 2048;  // table slots: [t] for x >= 0, [2048 + t] for x < 0
constexpr int kConsumerWarpsHost = GRKAN_CONSUMER_WARPS;
constexpr int kStagedThreadsHost = 32 * (GRKAN_CONSUMER_WARPS + 1);
constexpr int kStageVecsHost = GRKAN_STAGE_VECS;
constexpr int kBwdCtasPerSmHost = GRKAN_BWD_CTAS;
constexpr int kFwdCtasPerSmHost = GRKAN_FWD_CTAS;
constexpr int kFwdThreadsHost = 32 * (GRKAN_FWD_CONSUMER_WARPS + 1);
constexpr int kFwdStageVecsHost = GRKAN_FWD_STAGE_VECS;
static_assert(GRKAN_STAGE_VECS % (32 * GRKAN_CONSUMER_WARPS) == 0, "stage must split evenly over consumers");
static_assert(GRKAN_FWD_STAGE_VECS % (32 * GRKAN_FWD_CONSUMER_WARPS) == 0, "stage must split evenly over consumers");
// per-lane fp32 register chains <= 12 vectors per flush (4 stages at 3 vectors per thread)
constexpr int kFlushStages = (12 * 32 * GRKAN_CONSUMER_WARPS / GRKAN_STAGE_VECS) > 0
                                 ? (12 * 32 * GRKAN_CONSUMER_WARPS / GRKAN_STAGE_VECS) : 1;

struct LaunchArgs {
  const Plan* plan;
  const void* x;
  const void* dy;   // backward only
  void* out;        // y (forward) or dx (backward)
  const void* a;
  const void* b;
  void* part;       // backward partials (SoA)
  void* da;
  void* db;
  DevStatus* st;
  int m1, n;
  bool exact, vec, check;
  bool partials_only;  // backward: K2 only (deterministic multi-GPU path)
  bool instr;          // backward: the instrumented instantiations (coverage + access counts)
  void* y2;            // backward: also write the forward value here (fused step; staged plans only)
  CUtensorMap tmx, tmu;  // staged plans with geo.tma_rows > 0: x and dy as tiled maps
  cudaStream_t stream;
};

// One entry per I/O dtype; each lives in its own translation unit.
cudaError_t launch_fwd_f32(const LaunchArgs&);
cudaError_t launch_fwd_bf16(const LaunchArgs&);
cudaError_t launch_fwd_f64(const LaunchArgs&);
cudaError_t launch_bwd_f32(const LaunchArgs&);
cudaError_t launch_bwd_bf16(const LaunchArgs&);
cudaError_t launch_bwd_f64(const LaunchArgs&);
cudaError_t launch_atomic_f32(const LaunchArgs&);
cudaError_t launch_atomic_bf16(const LaunchArgs&);
cudaError_t launch_atomic_f64(const LaunchArgs&);
cudaError_t launch_reduce_f32(const void* part, int64_t n_tiles, int64_t slot_stride, int ng, int m1, int n,
                              void* da, void* db, DevStatus* st, cudaStream_t s);
cudaError_t launch_reduce_f64(const void* part, int64_t n_tiles, int64_t slot_stride, int ng, int m1, int n,
                              void* da, void* db, DevStatus* st, cudaStream_t s);

// Record `msg` as this thread's grkan_last_error() message and return `code`
// (library-internal; defined in grkan_capi.cu).
int set_error(int code, const char* msg);

}  // namespace grkan
