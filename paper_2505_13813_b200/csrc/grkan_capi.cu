// grkan_capi.cu -- the C ABI (include/grkan_b200.h): validation, launch planning
// and dispatch onto the per-dtype launchers (grkan_inst_*.cu -> grkan_kernels.cuh).
//
// Host-side argument checks mirror the reference's synchronous errors:
//   layout   GroupLayout.__post_init__ / check_compatible (rational.py:38-45, 313-322)
//   geometry backward_blocked shape / plan checks (backward.py:298-300)
// Device-side conditions (non-finite inputs in checked mode, non-finite da/db)
// land in a status block that grkan_read_status() maps to the same codes.
#include <atomic>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <numeric>
#include <cstdlib>

#include "../../include/grkan_b200.h"
#include "grkan_tmap.h"
#include "grkan_types.h"

#define GRKAN_VERSION_STRING "grkan_b200 0.1.0 (sm_100a)"

namespace {

using grkan::DevStatus;
using grkan::Geom;

thread_local char g_err[512] = "";

int fail(int code, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
  return code;
}

int cuda_fail(cudaError_t e, const char* where) {
  return fail(GRKAN_ERR_CUDA, "%s: %s", where, cudaGetErrorString(e));
}

// Once-initialised per-device SM count (the only library-global state).
int sm_count() {
  static std::atomic<int> cache[128];
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 128) return 148;
  int v = cache[dev].load(std::memory_order_relaxed);
  if (v == 0) {
    if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || v <= 0)
      v = 148;
    cache[dev].store(v, std::memory_order_relaxed);
  }
  return v;
}

size_t elem_size(int dtype) {
  switch (dtype) {
    case GRKAN_F32: return 4;
    case GRKAN_F64: return 8;
    case GRKAN_BF16: return 2;
    default: return 0;
  }
}
size_t acc_size(int dtype) { return dtype == GRKAN_F64 ? 8 : 4; }

using grkan::Plan;

constexpr int kEltsPerThread = 64;  // target elements per thread per CTA

// Tile geometry: one CTA per (row tile, group); R rows chosen so each of the
// kBlock threads handles ~kEltsPerThread elements and, when cheap, so the
// tile's vector count is a whole number of unrolled steps (no ragged steps).
// GRKAN_STAGED=0 in the environment selects the register-direct kernels even
// where the TMA-staged ones apply (A/B measurements; results are identical
// for y/dx and within fp32 reassociation for da/db).
// Forward: fp32 defaults to the register-direct kernel (measured 99.7% of
// copy bandwidth at KAT-B vs 87% staged); 2-byte I/O carries twice the math
// per byte and runs faster staged (84% vs 72%).  GRKAN_STAGED_FWD=0/1 forces;
// GRKAN_STAGED=0 selects the register-direct backward.
bool staged_enabled(int nt, size_t es) {
  const char* v = getenv(nt == 1 ? "GRKAN_STAGED_FWD" : "GRKAN_STAGED");
  if (v && (v[0] == '0' || v[0] == '1')) return v[0] == '1';
  return nt == 2 || es == 2;
}

constexpr int kStagesPerTensorPair = GRKAN_BWD_STAGES;  // backward ring depth (2 tensors)
constexpr int kStagesSingle = GRKAN_FWD_STAGES;  // forward ring depth (1 tensor)
constexpr size_t kSmemPerSm = 228 * 1024;

// Deterministic mode's global row block RB: a whole number of staged
// pipeline stages (RS = stage vectors / V rows) of >= 128 rows.  Depends only
// on (d, n_groups, element size), so every rank of a sharded run agrees on it.
int64_t det_rows(int32_t d, int32_t ng, size_t es) {
  const int dg = d / ng;
  const int W = static_cast<int>(16 / es);
  const int V = dg % W == 0 ? dg / W : 0;
  const int RS = (V >= 1 && V <= grkan::kStageVecsHost) ? grkan::kStageVecsHost / V : 1;
  return static_cast<int64_t>(RS) * ((GRKAN_DET_ROWS + RS - 1) / RS);
}

// bf16 FAST backward: the x-factor table (grkan_staged.cuh LUT); results agree
// with the table-free kernel within the FAST tolerance.  The choice depends on
// the layout only, never on the row count: the table path rounds each term
// differently, and dx must not depend on deterministic mode or on how rows
// are sharded.  GRKAN_LUT=0 in the environment disables it (A/B).
bool lut_enabled() {
  const char* v = getenv("GRKAN_LUT");
  if (v && (v[0] == '0' || v[0] == '1')) return v[0] == '1';
  return GRKAN_LUT != 0;
}

// Short row segments: the staged producers copy whole stages as tensor-map
// boxes instead of one bulk copy per row (GRKAN_TMA2D=0: per-row copies,
// =2: boxes at every row length; A/B).
int tma2d_mode() {
  const char* v = getenv("GRKAN_TMA2D");
  if (v && (v[0] == '0' || v[0] == '2')) return v[0] - '0';
  return 1;
}

// The wide backward geometry (one CTA of GRKAN_WIDE_WARPS consumer warps per
// SM, stages twice as large): measured on one B200 at 1965 MHz, KAT-B fp32
// 308 -> 296 us, bf16 216 -> 208 us, KAT-S bf16 68 -> 66 us, but KAT-S fp32
// 89 -> 119 us (768-byte rows: its single producer cannot issue the per-row
// copies fast enough; with tensor-map boxes 92 us).  So: 2-byte I/O, and
// 4-byte I/O with row segments of at least 1536 bytes.  GRKAN_WIDE=0/1 forces
// (A/B).  Never for deterministic partials (the geometry must not depend on
// the shard) or the fused / instrumented instantiations (wide_ok = false).
bool wide_geometry(size_t es, int dg, bool wide_ok) {
  if (!wide_ok || es > 4) return false;
  const char* v = getenv("GRKAN_WIDE");
  if (v && (v[0] == '0' || v[0] == '1')) return v[0] == '1';
  return es == 2 || static_cast<size_t>(dg) * es >= 1536;
}

// Staged backward at >= 2 CTAs per SM: the first wave's share of stage units,
// in 1/64 of a later CTA's (Geom::w1).  GRKAN_SKEW=<n> overrides (A/B).
int first_wave_weight() {
  const char* v = getenv("GRKAN_SKEW");
  if (v && *v) {
    const int w = atoi(v);
    if (w >= 16 && w <= 256) return w;
  }
  return GRKAN_SKEW64;
}

// The status block of a staged backward without CHECK_FINITE is zeroed by the
// kernel's CTA 0 (Geom::zst): one stream operation less per call.
// GRKAN_ZST=0 in the environment keeps the memset (A/B).
bool zero_status_in_kernel(const Plan& p, uint32_t flags) {
  if (!p.staged || (flags & GRKAN_FLAG_CHECK_FINITE) != 0) return false;
  const char* v = getenv("GRKAN_ZST");
  return !(v && v[0] == '0');
}

// nt = tensors streamed in (1 forward, 2 backward).  det: one partial per
// global RB-row block (slot-major), independent of the launch geometry.
// lut: the caller runs the bf16 FAST backward (grkan_bwd / grkan_bwd_partials).
// wide_ok: the caller launches the plain backward (grkan_bwd), which has the
// wide-geometry instantiations.
Plan make_plan(int64_t rows, int32_t d, int32_t ng, int32_t m1, int32_t n, size_t es, bool vec, int nt,
               int sms, bool det = false, bool lut = false, bool wide_ok = false) {
  Plan p;
  const int dg = d / ng;
  const int64_t RB = det ? det_rows(d, ng, es) : 0;
  p.geo.det = det ? 1 : 0;
  p.geo.one = 1.0f;
  p.geo.w1 = 64;  // even partition unless the staged backward below skews it
  p.geo.wave = sms;
  p.W = vec ? static_cast<int>(16 / es) : 1;
  const bool wide = nt == 2 && !det && vec && wide_geometry(es, dg, wide_ok);
  const int cw = wide ? GRKAN_WIDE_WARPS : grkan::kConsumerWarpsHost;
  const int ctas_per_sm = wide ? 1 : grkan::kBwdCtasPerSmHost;
  const int stage_vecs = nt == 2 ? grkan::kStageVecsHost / grkan::kConsumerWarpsHost * cw : grkan::kFwdStageVecsHost;
  // staged kernels: compile-time degrees (5, 4) (the paper) and (3, 2)
  const bool staged_deg = (m1 == 6 && n == 4) || (m1 == 4 && n == 2);
  if (vec && staged_deg && dg / p.W <= stage_vecs && staged_enabled(nt, es)) {
    // TMA-staged persistent kernels (grkan_staged.cuh)
    const int V = dg / p.W;
    const int RS = stage_vecs / V;
    const int64_t RU = det ? RB : RS;  // rows per partition unit
    const int64_t nsu = rows > 0 ? (rows + RU - 1) / RU : 0;
    p.staged = true;
    p.stages = nt == 2 ? kStagesPerTensorPair : kStagesSingle;
    p.smem = static_cast<size_t>(p.stages) * nt * RS * dg * es;
    if (nt == 2)  // + per-lane accumulator totals [10][256] in the accumulation type
      p.smem += static_cast<size_t>(m1 + n) * 32 * cw * (es == 8 ? 8 : 4);
    // (measured faster at KAT-B and KAT-S; the ~1-2 us table build matters only
    // for tensors that take a few microseconds anyway)
    if (nt == 2 && es == 2 && lut && m1 == 6 && n == 4 && lut_enabled()) {
      // the table (two float arrays over a 16-exponent window) takes a ring
      // stage's place and the accumulator totals go one slot per lane pair, so
      // kBwdCtasPerSm CTAs stay resident
      const size_t ring = static_cast<size_t>(GRKAN_LUT_STAGES) * nt * RS * dg * es;
      const size_t acc = static_cast<size_t>(m1 + n) * 16 * cw * 4;
      const size_t sm = ring + acc + 2 * 2 * grkan::kLutSignStride * sizeof(float);
      if (kSmemPerSm / (sm + 2048) >= static_cast<size_t>(ctas_per_sm)) {
        p.stages = GRKAN_LUT_STAGES;
        p.smem = sm;
        p.geo.lut_ne = 16;
        p.geo.lut_e0 = GRKAN_LUT_TOP - 15;  // <= 128: the slot arithmetic needs base <= 0x4000
        p.geo.lut_c = (0x4000u - (static_cast<uint32_t>(p.geo.lut_e0) << 7)) * 0x10001u;
      }
    }
    // Tensor-map stage copies (measured: the backward gains from boxes up to
    // 384-byte rows and, fp32, loses at 768; the bf16 backward is issue-bound and
    // gains at any length; the forward's small stages only below ~100-byte rows).
    // Box inner extent: the largest 16-byte-multiple divisor of dg that is <= 256.
    {
      int ci = 0;
      for (int c = dg < 256 ? dg : 256; c >= 1; --c)
        if (dg % c == 0 && (static_cast<size_t>(c) * es) % 16 == 0) {
          ci = c;
          break;
        }
      const size_t row_bytes = static_cast<size_t>(dg) * es;
      const int mode = tma2d_mode();
      const bool want = mode == 2 || (nt == 2 ? (row_bytes <= GRKAN_TMA2D_MAX_ROW_BYTES || (es == 2 && GRKAN_TMA_BF16_BWD))
                                              : row_bytes <= GRKAN_TMA2D_MAX_ROW_BYTES_FWD);
      if (mode != 0 && want && ci > 0 && (static_cast<size_t>(RS) * dg * es) % 128 == 0 &&
          rows < (int64_t{1} << 31)) {
        const int nbox = (RS + 255) / 256;  // box dimensions are <= 256
        if (RS % nbox == 0) {
          p.geo.tma_rows = RS / nbox;
          p.geo.tma_ci = ci;
        }
      }
    }
    const int occ_regs = nt == 2 ? ctas_per_sm : grkan::kFwdCtasPerSmHost;
    int occ = static_cast<int>(kSmemPerSm / (p.smem + 2048));
    occ = occ < 1 ? 1 : (occ > occ_regs ? occ_regs : occ);
    const int64_t slots = static_cast<int64_t>(sms) * occ;
    int64_t pg = slots / ng;
    if (pg > nsu) pg = nsu;
    if (pg < 1) pg = 1;
    p.threads = nt == 2 ? 32 * (cw + 1) : grkan::kFwdThreadsHost;
    p.cw = nt == 2 ? cw : 0;
    p.geo.rows = rows;
    p.geo.d = d;
    p.geo.ng = ng;
    p.geo.dg = dg;
    p.geo.V = V;
    p.geo.R = 0;
    p.geo.RS = RS;
    p.geo.nsu = nsu;
    p.geo.pg = static_cast<int32_t>(pg);
    p.geo.flush = grkan::kFlushStages;
    p.geo.RU = static_cast<int32_t>(RU);
    p.geo.spb = static_cast<int32_t>(RU / RS);
    // partials per (group, coefficient) for K3 (backward: one per consumer
    // warp; deterministic: one per RB-row block)
    p.geo.n_tiles = det ? nsu : (nt == 2 ? pg * cw : pg);
    if (nt == 2 && !det && occ >= 2 && pg * ng > sms && nsu >= 4 * pg) p.geo.w1 = first_wave_weight();
    p.ctas = rows > 0 ? pg * ng : 0;
    return p;
  }
  const int U = nt == 1 ? 4 : grkan::unroll_for_width(p.W);  // = Engine::UF / Engine::U
  const int V = dg / p.W;
  const int64_t step = static_cast<int64_t>(grkan::kBlock) * U;
  const int64_t target_vecs = static_cast<int64_t>(grkan::kBlock) * kEltsPerThread / p.W;
  int64_t R = (target_vecs + V - 1) / V;
  if (R < 1) R = 1;
  for (int64_t r = R; r <= 2 * R; ++r) {
    if ((r * V) % step == 0) {
      R = r;
      break;
    }
  }
  if (rows > 0 && R > rows) R = rows;
  int64_t n_tiles = rows > 0 ? (rows + R - 1) / R : 0;
  // small tensors: shrink tiles until there are a few CTAs per SM
  while (!det && R > 1 && n_tiles * ng < 4LL * sms) {
    R = (R + 1) / 2;
    n_tiles = (rows + R - 1) / R;
  }
  if (det) {  // fixed global row blocks, whatever the shard size
    R = RB;
    n_tiles = rows > 0 ? (rows + R - 1) / R : 0;
  }
  p.threads = grkan::kBlock;
  p.geo.rows = rows;
  p.geo.n_tiles = n_tiles;
  p.geo.d = d;
  p.geo.ng = ng;
  p.geo.dg = dg;
  p.geo.V = V;
  p.geo.R = static_cast<int32_t>(R);
  p.geo.dr = grkan::kBlock / V;
  p.geo.dc = grkan::kBlock % V;
  p.ctas = n_tiles * ng;
  return p;
}

// The tiled maps of x and dy for a plan with geo.tma_rows > 0: [rows, d] viewed
// as [rows, d / ci, ci], boxes of tma_rows rows x one group's dg / ci chunks; on
// any encode failure the plan falls back to per-row copies.
void attach_maps(Plan& p, grkan::LaunchArgs& L, const void* x, const void* u, int32_t dtype) {
  if (p.geo.tma_rows <= 0) return;
  auto fn = grkan::encode_fn();
  const size_t es = elem_size(dtype);
  const CUtensorMapDataType ty = dtype == GRKAN_F32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32
                                 : dtype == GRKAN_BF16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16
                                                       : CU_TENSOR_MAP_DATA_TYPE_FLOAT64;
  const int ci = p.geo.tma_ci;
  const cuuint64_t dims[3] = {static_cast<cuuint64_t>(ci), static_cast<cuuint64_t>(p.geo.d / ci),
                              static_cast<cuuint64_t>(p.geo.rows)};
  const cuuint64_t strides[2] = {static_cast<cuuint64_t>(ci) * es, static_cast<cuuint64_t>(p.geo.d) * es};
  const cuuint32_t box[3] = {static_cast<cuuint32_t>(ci), static_cast<cuuint32_t>(p.geo.dg / ci),
                             static_cast<cuuint32_t>(p.geo.tma_rows)};
  const cuuint32_t estr[3] = {1, 1, 1};
  auto enc = [&](CUtensorMap* m, const void* base) {
    return fn && base &&
           fn(m, ty, 3, const_cast<void*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
              CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
  };
  if (!enc(&L.tmx, x) || (u && !enc(&L.tmu, u))) p.geo.tma_rows = 0;
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

bool vec_ok(int32_t d, int32_t ng, size_t es, std::initializer_list<const void*> ptrs) {
  const size_t dg = static_cast<size_t>(d / ng);
  if ((dg * es) % 16 != 0 || (static_cast<size_t>(d) * es) % 16 != 0) return false;
  for (const void* p : ptrs)
    if (p && !aligned16(p)) return false;
  return true;
}

int check_layout(int64_t rows, int32_t d, int32_t ng, int32_t m1, int32_t n, int32_t dtype,
                 uint32_t flags) {
  if (elem_size(dtype) == 0) return fail(GRKAN_ERR_UNSUPPORTED, "unsupported dtype code %d", dtype);
  if (d < 1 || ng < 1)
    return fail(GRKAN_ERR_LAYOUT, "layout mismatch: dimensions must be positive (d=%d, groups=%d)", d, ng);
  if (d % ng != 0)
    return fail(GRKAN_ERR_LAYOUT, "layout mismatch: feature_dim %d not divisible by num_groups %d", d, ng);
  if (rows < 0) return fail(GRKAN_ERR_GRID, "grid geometry invalid: negative row count");
  if (m1 < 1 || n < 0)
    return fail(GRKAN_ERR_INVALID, "need at least one numerator coefficient and n >= 0 (m1=%d, n=%d)", m1, n);
  if (m1 > GRKAN_MAX_M1 || n > GRKAN_MAX_N)
    return fail(GRKAN_ERR_UNSUPPORTED, "degrees (m1=%d, n=%d) exceed this build (max %d, %d)", m1, n,
                GRKAN_MAX_M1, GRKAN_MAX_N);
  if (flags & ~(GRKAN_FLAG_EXACT | GRKAN_FLAG_CHECK_FINITE | GRKAN_FLAG_DETERMINISTIC))
    return fail(GRKAN_ERR_INVALID, "unknown flag bits 0x%x", flags);
  return GRKAN_OK;
}

using grkan::LaunchArgs;

cudaError_t launch_reduce(int dtype, const void* part, int64_t n_tiles, int64_t slot_stride, int ng, int m1,
                          int n, void* da, void* db, DevStatus* st, cudaStream_t s) {
  if (dtype == GRKAN_F64) return grkan::launch_reduce_f64(part, n_tiles, slot_stride, ng, m1, n, da, db, st, s);
  return grkan::launch_reduce_f32(part, n_tiles, slot_stride, ng, m1, n, da, db, st, s);
}

cudaError_t launch(const char* which, int dtype, const LaunchArgs& L) {
  const bool f = which[0] == 'f', b = which[0] == 'b';
  switch (dtype) {
    case GRKAN_F32: return f ? grkan::launch_fwd_f32(L) : b ? grkan::launch_bwd_f32(L) : grkan::launch_atomic_f32(L);
    case GRKAN_BF16: return f ? grkan::launch_fwd_bf16(L) : b ? grkan::launch_bwd_bf16(L) : grkan::launch_atomic_bf16(L);
    case GRKAN_F64: return f ? grkan::launch_fwd_f64(L) : b ? grkan::launch_bwd_f64(L) : grkan::launch_atomic_f64(L);
    default: return cudaErrorInvalidValue;
  }
}

bool plan_fits(const Plan& p) {
  return p.ctas <= 0x7fffffffLL && static_cast<int64_t>(p.geo.R) * p.geo.V <= 0x7fffffffLL &&
         (!p.staged || p.smem <= 227 * 1024);
}

size_t ws_bytes_for(const Plan& p, int32_t m1, int32_t n, int32_t dtype) {
  const size_t part = static_cast<size_t>(p.geo.ng) * (m1 + n) * p.geo.n_tiles * acc_size(dtype);
  return 256 + ((part + 255) / 256) * 256;
}

}  // namespace

namespace grkan {
cudaError_t launch_reduce_p2p(int dtype, const void* part, int64_t n_tiles, int ng, int m1, int n, void* const* bufs,
                              int rank, int world, unsigned long long epoch, void* da, void* db, DevStatus* st,
                              cudaStream_t stream);  // grkan_p2p.cu
// Error reporting for the other C-ABI translation units (grkan_fused.cu).
int set_error(int code, const char* msg) { return fail(code, "%s", msg); }
}  // namespace grkan

extern "C" {

const char* grkan_version(void) { return GRKAN_VERSION_STRING; }

const char* grkan_last_error(void) { return g_err; }

const char* grkan_status_string(int status) {
  switch (status) {
    case GRKAN_OK: return "ok";
    case GRKAN_ERR_LAYOUT: return "layout mismatch";
    case GRKAN_ERR_GRID: return "grid geometry invalid";
    case GRKAN_ERR_NONFINITE_INPUT: return "non-finite input";
    case GRKAN_ERR_ACCUM_OVERFLOW: return "accumulation overflow";
    case GRKAN_ERR_UNSUPPORTED: return "unsupported";
    case GRKAN_ERR_CUDA: return "cuda error";
    case GRKAN_ERR_INVALID: return "invalid argument";
    case GRKAN_ERR_PEER_TIMEOUT: return "peer exchange timed out";
    default: return "unknown status";
  }
}

int grkan_plan(int64_t rows, int32_t d, int32_t n_groups, int32_t m1, int32_t n, int32_t dtype,
               int64_t* out6) {
  int rc = check_layout(rows, d, n_groups, m1, n, dtype, 0);
  if (rc) return rc;
  if (!out6) return fail(GRKAN_ERR_INVALID, "null output");
  const size_t es = elem_size(dtype);
  const Plan p = make_plan(rows, d, n_groups, m1, n, es, vec_ok(d, n_groups, es, {}), 2, 148);
  out6[0] = p.W;
  out6[1] = p.threads;
  out6[2] = p.staged ? p.geo.RS : p.geo.R;
  out6[3] = p.geo.n_tiles;
  out6[4] = p.ctas;
  out6[5] = p.staged ? 1 : 0;
  return GRKAN_OK;
}

int64_t grkan_launch_ctas(int64_t rows, int32_t d, int32_t n_groups, int32_t m1, int32_t n, int32_t dtype,
                          int32_t kernel) {
  if (check_layout(rows, d, n_groups, m1, n, dtype, 0) != GRKAN_OK || kernel < 0 || kernel > 2) return -1;
  const size_t es = elem_size(dtype);
  const bool vec = vec_ok(d, n_groups, es, {});
  const Plan p = kernel == 2 ? make_plan(rows, d, n_groups, 0, n, es, vec, 2, sm_count())
                             : make_plan(rows, d, n_groups, m1, n, es, vec, kernel == 0 ? 1 : 2, sm_count());
  return p.ctas;
}

size_t grkan_bwd_workspace_bytes(int64_t rows, int32_t d, int32_t n_groups, int32_t m1, int32_t n,
                                 int32_t dtype) {
  if (check_layout(rows, d, n_groups, m1, n, dtype, 0) != GRKAN_OK) return 0;
  const size_t es = elem_size(dtype);
  // the vector / scalar choice depends on pointer alignment: size for both
  // The vector / scalar choice depends on pointer alignment and the small-tensor
  // tile shrink on the SM count: size for both widths at the maximum shrink
  // (an SM count no device reaches), which bounds every plan grkan_bwd can pick.
  const int kAnySms = 1 << 20;
  const bool can_vec = vec_ok(d, n_groups, es, {});
  size_t a = 0;
  if (can_vec)  // both staged geometries (make_plan picks the wide one per shape)
    for (int wide = 0; wide < 2; ++wide) {
      const size_t w =
          ws_bytes_for(make_plan(rows, d, n_groups, m1, n, es, true, 2, kAnySms, false, true, wide == 1), m1, n, dtype);
      a = w > a ? w : a;
    }
  const size_t b = ws_bytes_for(make_plan(rows, d, n_groups, m1, n, es, false, 2, kAnySms), m1, n, dtype);
  // GRKAN_FLAG_DETERMINISTIC: one partial per global row block
  const size_t c = ws_bytes_for(make_plan(rows, d, n_groups, m1, n, es, false, 2, kAnySms, true), m1, n, dtype);
  const size_t ab = a > b ? a : b;
  return ab > c ? ab : c;
}

int grkan_fwd(const void* x, void* y, const void* a, const void* b, int64_t rows, int32_t d,
              int32_t n_groups, int32_t m1, int32_t n, int32_t dtype, uint32_t flags,
              grkan_device_status* status, void* stream) {
  int rc = check_layout(rows, d, n_groups, m1, n, dtype, flags);
  if (rc) return rc;
  const bool check = (flags & GRKAN_FLAG_CHECK_FINITE) != 0;
  if (check && !status) return fail(GRKAN_ERR_INVALID, "CHECK_FINITE needs a status block");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (check) {
    cudaError_t e = cudaMemsetAsync(status, 0, sizeof(grkan_device_status), s);
    if (e != cudaSuccess) return cuda_fail(e, "cudaMemsetAsync(status)");
  }
  if (rows == 0) return GRKAN_OK;
  if (!x || !y || !a || (n > 0 && !b)) return fail(GRKAN_ERR_INVALID, "null tensor pointer");
  const size_t es = elem_size(dtype);
  const bool vec = vec_ok(d, n_groups, es, {x, y});
  Plan p = make_plan(rows, d, n_groups, m1, n, es, vec, 1, sm_count());
  if (!plan_fits(p)) return fail(GRKAN_ERR_GRID, "grid geometry invalid: %lld CTAs", (long long)p.ctas);
  LaunchArgs L{};
  L.plan = &p;
  L.x = x;
  L.out = y;
  L.a = a;
  L.b = b;
  L.st = reinterpret_cast<DevStatus*>(status);
  L.m1 = m1;
  L.n = n;
  L.exact = (flags & GRKAN_FLAG_EXACT) != 0;
  L.vec = vec;
  L.check = check;
  L.stream = s;
  attach_maps(p, L, x, nullptr, dtype);
  cudaError_t e = launch("fwd", dtype, L);
  if (e != cudaSuccess) return cuda_fail(e, "k_fwd launch");
  return GRKAN_OK;
}

int grkan_bwd(const void* x, const void* dy, const void* a, const void* b, void* dx, void* da,
              void* db, void* ws, size_t ws_bytes, int64_t rows, int32_t d, int32_t n_groups,
              int32_t m1, int32_t n, int32_t dtype, uint32_t flags, void* stream) {
  int rc = check_layout(rows, d, n_groups, m1, n, dtype, flags);
  if (rc) return rc;
  if (!ws || !da || (n > 0 && !db)) return fail(GRKAN_ERR_INVALID, "null workspace / gradient pointer");
  if (!aligned16(ws)) return fail(GRKAN_ERR_INVALID, "workspace must be 16-byte aligned");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  DevStatus* st = reinterpret_cast<DevStatus*>(ws);
  cudaError_t e;
  const size_t as = acc_size(dtype);
  if (rows == 0) {  // nothing to fold: the gradients are exact zeros
    e = cudaMemsetAsync(ws, 0, sizeof(DevStatus), s);
    if (e != cudaSuccess) return cuda_fail(e, "cudaMemsetAsync(status)");
    e = cudaMemsetAsync(da, 0, static_cast<size_t>(n_groups) * m1 * as, s);
    if (e == cudaSuccess && n > 0) e = cudaMemsetAsync(db, 0, static_cast<size_t>(n_groups) * n * as, s);
    return e == cudaSuccess ? GRKAN_OK : cuda_fail(e, "cudaMemsetAsync(da/db)");
  }
  if (!x || !dy || !dx || !a || (n > 0 && !b)) return fail(GRKAN_ERR_INVALID, "null tensor pointer");
  const size_t es = elem_size(dtype);
  const bool vec = vec_ok(d, n_groups, es, {x, dy, dx});
  const bool det = (flags & GRKAN_FLAG_DETERMINISTIC) != 0;
  Plan p = make_plan(rows, d, n_groups, m1, n, es, vec, 2, sm_count(), det,
                           (flags & GRKAN_FLAG_EXACT) == 0, true);
  if (!plan_fits(p)) return fail(GRKAN_ERR_GRID, "grid geometry invalid: %lld CTAs", (long long)p.ctas);
  const size_t need = ws_bytes_for(p, m1, n, dtype);
  if (ws_bytes < need)
    return fail(GRKAN_ERR_INVALID, "workspace too small: %zu < %zu bytes", ws_bytes, need);
  p.geo.zst = zero_status_in_kernel(p, flags);
  if (!p.geo.zst) {
    e = cudaMemsetAsync(ws, 0, sizeof(DevStatus), s);
    if (e != cudaSuccess) return cuda_fail(e, "cudaMemsetAsync(status)");
  }
  LaunchArgs L{};
  L.plan = &p;
  L.x = x;
  L.dy = dy;
  L.out = dx;
  L.a = a;
  L.b = b;
  L.part = static_cast<char*>(ws) + 256;
  L.da = da;
  L.db = db;
  L.st = st;
  L.m1 = m1;
  L.n = n;
  L.exact = (flags & GRKAN_FLAG_EXACT) != 0;
  L.vec = vec;
  L.check = (flags & GRKAN_FLAG_CHECK_FINITE) != 0;
  L.stream = s;
  attach_maps(p, L, x, dy, dtype);
  e = launch("bwd", dtype, L);
  if (e != cudaSuccess) return cuda_fail(e, "k_bwd launch");
  return GRKAN_OK;
}

int grkan_fwd_bwd(const void* x, const void* dy, const void* a, const void* b, void* y, void* dx, void* da,
                  void* db, void* ws, size_t ws_bytes, int64_t rows, int32_t d, int32_t n_groups, int32_t m1,
                  int32_t n, int32_t dtype, uint32_t flags, void* stream) {
  int rc = check_layout(rows, d, n_groups, m1, n, dtype, flags);
  if (rc) return rc;
  const size_t es = elem_size(dtype);
  const bool det = (flags & GRKAN_FLAG_DETERMINISTIC) != 0;
  const bool vec = vec_ok(d, n_groups, es, {x, dy, dx, y});
  Plan p = make_plan(rows, d, n_groups, m1, n, es, vec, 2, sm_count(), det, false, true);
  if (rows == 0 || !p.staged || det) {
    // no fused instantiation for this plan: the two passes back to back (same results)
    // (grkan_bwd's CHECK_FINITE covers x, so the forward runs unchecked)
    rc = grkan_fwd(x, y, a, b, rows, d, n_groups, m1, n, dtype,
                   flags & ~(GRKAN_FLAG_DETERMINISTIC | GRKAN_FLAG_CHECK_FINITE), nullptr, stream);
    if (rc) return rc;
    return grkan_bwd(x, dy, a, b, dx, da, db, ws, ws_bytes, rows, d, n_groups, m1, n, dtype, flags, stream);
  }
  if (!ws || !da || (n > 0 && !db)) return fail(GRKAN_ERR_INVALID, "null workspace / gradient pointer");
  if (!aligned16(ws)) return fail(GRKAN_ERR_INVALID, "workspace must be 16-byte aligned");
  if (!x || !dy || !dx || !y || !a || (n > 0 && !b)) return fail(GRKAN_ERR_INVALID, "null tensor pointer");
  if (!plan_fits(p)) return fail(GRKAN_ERR_GRID, "grid geometry invalid: %lld CTAs", (long long)p.ctas);
  const size_t need = ws_bytes_for(p, m1, n, dtype);
  if (ws_bytes < need) return fail(GRKAN_ERR_INVALID, "workspace too small: %zu < %zu bytes", ws_bytes, need);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  p.geo.zst = zero_status_in_kernel(p, flags);
  if (!p.geo.zst) {
    cudaError_t e = cudaMemsetAsync(ws, 0, sizeof(DevStatus), s);
    if (e != cudaSuccess) return cuda_fail(e, "cudaMemsetAsync(status)");
  }
  cudaError_t e;
  LaunchArgs L{};
  L.plan = &p;
  L.x = x;
  L.dy = dy;
  L.out = dx;
  L.y2 = y;
  L.a = a;
  L.b = b;
  L.part = static_cast<char*>(ws) + 256;
  L.da = da;
  L.db = db;
  L.st = reinterpret_cast<DevStatus*>(ws);
  L.m1 = m1;
  L.n = n;
  L.exact = (flags & GRKAN_FLAG_EXACT) != 0;
  L.vec = vec;
  L.check = (flags & GRKAN_FLAG_CHECK_FINITE) != 0;
  L.stream = s;
  attach_maps(p, L, x, dy, dtype);
  e = launch("bwd", dtype, L);
  if (e != cudaSuccess) return cuda_fail(e, "k_bwd (fused step) launch");
  return GRKAN_OK;
}

int grkan_bwd_p2p(const void* x, const void* dy, const void* a, const void* b, void* dx, void* da, void* db,
                  void* ws, size_t ws_bytes, int64_t rows, int32_t d, int32_t n_groups, int32_t m1, int32_t n,
                  int32_t dtype, uint32_t flags, void* const* peer_bufs, int32_t rank, int32_t world,
                  uint64_t epoch, void* stream) {
  int rc = check_layout(rows, d, n_groups, m1, n, dtype, flags);
  if (rc) return rc;
  if (flags & GRKAN_FLAG_DETERMINISTIC)
    return fail(GRKAN_ERR_INVALID, "the peer-memory exchange folds per-CTA partials; no DETERMINISTIC flag");
  if (!ws || !da || (n > 0 && !db) || !peer_bufs) return fail(GRKAN_ERR_INVALID, "null workspace / gradient / peer pointer");
  if (world < 1 || rank < 0 || rank >= world || epoch == 0)
    return fail(GRKAN_ERR_INVALID, "bad rank %d / world %d / epoch (must start at 1)", rank, world);
  if (!aligned16(ws)) return fail(GRKAN_ERR_INVALID, "workspace must be 16-byte aligned");
  if (!x || !dy || !dx || !a || (n > 0 && !b)) {
    if (rows > 0) return fail(GRKAN_ERR_INVALID, "null tensor pointer");
  }
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  DevStatus* st = reinterpret_cast<DevStatus*>(ws);
  cudaError_t e = cudaMemsetAsync(ws, 0, sizeof(DevStatus), s);
  if (e != cudaSuccess) return cuda_fail(e, "cudaMemsetAsync(status)");
  const size_t es = elem_size(dtype);
  const bool vec = rows > 0 && vec_ok(d, n_groups, es, {x, dy, dx});
  Plan p = make_plan(rows, d, n_groups, m1, n, es, vec, 2, sm_count());
  if (!plan_fits(p)) return fail(GRKAN_ERR_GRID, "grid geometry invalid: %lld CTAs", (long long)p.ctas);
  const size_t need = ws_bytes_for(p, m1, n, dtype);
  if (ws_bytes < need) return fail(GRKAN_ERR_INVALID, "workspace too small: %zu < %zu bytes", ws_bytes, need);
  if (rows > 0) {
    LaunchArgs L{};
    L.plan = &p;
    L.x = x;
    L.dy = dy;
    L.out = dx;
    L.a = a;
    L.b = b;
    L.part = static_cast<char*>(ws) + 256;
    L.st = st;
    L.m1 = m1;
    L.n = n;
    L.exact = (flags & GRKAN_FLAG_EXACT) != 0;
    L.vec = vec;
    L.check = (flags & GRKAN_FLAG_CHECK_FINITE) != 0;
    L.partials_only = true;
    L.stream = s;
    attach_maps(p, L, x, dy, dtype);
    e = launch("bwd", dtype, L);
    if (e != cudaSuccess) return cuda_fail(e, "k_bwd (partials) launch");
  }
  // an empty shard still takes part in the exchange: no partials, a zero fold
  const int64_t n_tiles = rows > 0 ? p.geo.n_tiles : 0;
  e = grkan::launch_reduce_p2p(dtype, static_cast<char*>(ws) + 256, n_tiles, n_groups, m1, n, peer_bufs, rank, world,
                               epoch, da, db, st, s);
  if (e != cudaSuccess) return cuda_fail(e, "k_bwd_reduce_p2p launch");
  return GRKAN_OK;
}

int64_t grkan_det_block_rows(int32_t d, int32_t n_groups, int32_t dtype) {
  if (elem_size(dtype) == 0 || d < 1 || n_groups < 1 || d % n_groups) return 0;
  return det_rows(d, n_groups, elem_size(dtype));
}

size_t grkan_det_partials_bytes(int64_t rows, int32_t d, int32_t n_groups, int32_t m1, int32_t n,
                                int32_t dtype) {
  if (check_layout(rows, d, n_groups, m1, n, dtype, 0) != GRKAN_OK) return 0;
  const int64_t rb = det_rows(d, n_groups, elem_size(dtype));
  const int64_t blocks = (rows + rb - 1) / rb;
  return static_cast<size_t>(blocks) * n_groups * (m1 + n) * acc_size(dtype);
}

int grkan_bwd_partials(const void* x, const void* dy, const void* a, const void* b, void* dx, void* part,
                       size_t part_bytes, int64_t rows, int32_t d, int32_t n_groups, int32_t m1, int32_t n,
                       int32_t dtype, uint32_t flags, grkan_device_status* status, void* stream) {
  int rc = check_layout(rows, d, n_groups, m1, n, dtype, flags);
  if (rc) return rc;
  const bool check = (flags & GRKAN_FLAG_CHECK_FINITE) != 0;
  if (check && !status) return fail(GRKAN_ERR_INVALID, "CHECK_FINITE needs a status block");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (check) {
    cudaError_t e = cudaMemsetAsync(status, 0, sizeof(grkan_device_status), s);
    if (e != cudaSuccess) return cuda_fail(e, "cudaMemsetAsync(status)");
  }
  if (rows == 0) return GRKAN_OK;
  const size_t need = grkan_det_partials_bytes(rows, d, n_groups, m1, n, dtype);
  if (!part || part_bytes < need)
    return fail(GRKAN_ERR_INVALID, "partials buffer too small: %zu < %zu bytes", part ? part_bytes : 0, need);
  if (!x || !dy || !dx || !a || (n > 0 && !b)) return fail(GRKAN_ERR_INVALID, "null tensor pointer");
  const size_t es = elem_size(dtype);
  const bool vec = vec_ok(d, n_groups, es, {x, dy, dx});
  Plan p = make_plan(rows, d, n_groups, m1, n, es, vec, 2, sm_count(), true,
                           (flags & GRKAN_FLAG_EXACT) == 0);
  if (!plan_fits(p)) return fail(GRKAN_ERR_GRID, "grid geometry invalid: %lld CTAs", (long long)p.ctas);
  LaunchArgs L{};
  L.plan = &p;
  L.x = x;
  L.dy = dy;
  L.out = dx;
  L.a = a;
  L.b = b;
  L.part = part;
  L.st = reinterpret_cast<DevStatus*>(status);
  L.m1 = m1;
  L.n = n;
  L.exact = (flags & GRKAN_FLAG_EXACT) != 0;
  L.vec = vec;
  L.check = check;
  L.partials_only = true;
  L.stream = s;
  attach_maps(p, L, x, dy, dtype);
  cudaError_t e = launch("bwd", dtype, L);
  if (e != cudaSuccess) return cuda_fail(e, "k_bwd (partials) launch");
  return GRKAN_OK;
}

int grkan_reduce_partials(const void* part, int64_t n_blocks, int32_t n_groups, int32_t m1, int32_t n,
                          void* da, void* db, int32_t dtype, grkan_device_status* status, void* stream) {
  int rc = check_layout(0, n_groups, n_groups, m1, n, dtype, 0);
  if (rc) return rc;
  if (n_blocks < 0) return fail(GRKAN_ERR_GRID, "grid geometry invalid: negative block count");
  if (!da || (n > 0 && !db) || !status) return fail(GRKAN_ERR_INVALID, "null gradient / status pointer");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  cudaError_t e = cudaMemsetAsync(status, 0, sizeof(grkan_device_status), s);
  if (e != cudaSuccess) return cuda_fail(e, "cudaMemsetAsync(status)");
  if (n_blocks == 0) {
    const size_t as = acc_size(dtype);
    e = cudaMemsetAsync(da, 0, static_cast<size_t>(n_groups) * m1 * as, s);
    if (e == cudaSuccess && n > 0) e = cudaMemsetAsync(db, 0, static_cast<size_t>(n_groups) * n * as, s);
    return e == cudaSuccess ? GRKAN_OK : cuda_fail(e, "cudaMemsetAsync(da/db)");
  }
  if (!part) return fail(GRKAN_ERR_INVALID, "null partials pointer");
  e = launch_reduce(dtype, part, n_blocks, static_cast<int64_t>(n_groups) * (m1 + n), n_groups, m1, n, da, db,
                    reinterpret_cast<DevStatus*>(status), s);
  if (e != cudaSuccess) return cuda_fail(e, "k_bwd_reduce launch");
  return GRKAN_OK;
}

int grkan_bwd_instrumented(const void* x, const void* dy, const void* a, const void* b, void* dx, void* da,
                           void* db, void* ws, size_t ws_bytes, int32_t* coverage, unsigned long long* counts,
                           int64_t rows, int32_t d, int32_t n_groups, int32_t m1, int32_t n, int32_t dtype,
                           uint32_t flags, int32_t naive, void* stream) {
  if (flags & (GRKAN_FLAG_CHECK_FINITE | GRKAN_FLAG_DETERMINISTIC))
    return fail(GRKAN_ERR_INVALID, "instrumented backward: CHECK_FINITE / DETERMINISTIC not supported");
  int rc = check_layout(rows, d, n_groups, m1, n, dtype, flags);
  if (rc) return rc;
  if (!coverage || !counts) return fail(GRKAN_ERR_INVALID, "instrumented backward needs coverage and counts");
  if (!ws || !da || (n > 0 && !db)) return fail(GRKAN_ERR_INVALID, "null workspace / gradient pointer");
  if (!aligned16(ws)) return fail(GRKAN_ERR_INVALID, "workspace must be 16-byte aligned");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  DevStatus* st = reinterpret_cast<DevStatus*>(ws);
  cudaError_t e = cudaMemsetAsync(ws, 0, sizeof(DevStatus), s);
  const size_t as = acc_size(dtype);
  if (e == cudaSuccess && (naive || rows == 0)) {
    e = cudaMemsetAsync(da, 0, static_cast<size_t>(n_groups) * m1 * as, s);
    if (e == cudaSuccess && n > 0) e = cudaMemsetAsync(db, 0, static_cast<size_t>(n_groups) * n * as, s);
  }
  if (e != cudaSuccess) return cuda_fail(e, "cudaMemsetAsync");
  if (rows == 0) return GRKAN_OK;
  if (!x || !dy || !dx || !a || (n > 0 && !b)) return fail(GRKAN_ERR_INVALID, "null tensor pointer");
  const size_t es = elem_size(dtype);
  const bool vec = vec_ok(d, n_groups, es, {x, dy, dx});
  // the same plan grkan_bwd / grkan_bwd_atomic pick for these tensors
  Plan p = naive ? make_plan(rows, d, n_groups, /*m1=*/0, n, es, vec, 2, sm_count())
                 : make_plan(rows, d, n_groups, m1, n, es, vec, 2, sm_count());
  if (!plan_fits(p)) return fail(GRKAN_ERR_GRID, "grid geometry invalid: %lld CTAs", (long long)p.ctas);
  if (!naive && ws_bytes < ws_bytes_for(p, m1, n, dtype))
    return fail(GRKAN_ERR_INVALID, "workspace too small: %zu < %zu bytes", ws_bytes, ws_bytes_for(p, m1, n, dtype));
  p.geo.cov = coverage;
  p.geo.cnt = counts;
  LaunchArgs L{};
  L.plan = &p;
  L.x = x;
  L.dy = dy;
  L.out = dx;
  L.a = a;
  L.b = b;
  L.part = static_cast<char*>(ws) + 256;
  L.da = da;
  L.db = db;
  L.st = st;
  L.m1 = m1;
  L.n = n;
  L.exact = (flags & GRKAN_FLAG_EXACT) != 0;
  L.vec = vec;
  L.check = false;
  L.instr = true;
  L.stream = s;
  if (!naive) attach_maps(p, L, x, dy, dtype);
  e = launch(naive ? "atomic" : "bwd", dtype, L);
  if (e != cudaSuccess) return cuda_fail(e, "instrumented backward launch");
  return GRKAN_OK;
}

int grkan_bwd_atomic(const void* x, const void* dy, const void* a, const void* b, void* dx,
                     void* da, void* db, int64_t rows, int32_t d, int32_t n_groups, int32_t m1,
                     int32_t n, int32_t dtype, uint32_t flags, grkan_device_status* status,
                     void* stream) {
  int rc = check_layout(rows, d, n_groups, m1, n, dtype, flags & GRKAN_FLAG_EXACT);
  if (rc) return rc;
  if (!da || (n > 0 && !db)) return fail(GRKAN_ERR_INVALID, "null gradient pointer");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const size_t as = acc_size(dtype);
  cudaError_t e = cudaMemsetAsync(da, 0, static_cast<size_t>(n_groups) * m1 * as, s);
  if (e == cudaSuccess && n > 0) e = cudaMemsetAsync(db, 0, static_cast<size_t>(n_groups) * n * as, s);
  if (e == cudaSuccess && status) e = cudaMemsetAsync(status, 0, sizeof(grkan_device_status), s);
  if (e != cudaSuccess) return cuda_fail(e, "cudaMemsetAsync");
  if (rows == 0) return GRKAN_OK;
  if (!x || !dy || !dx || !a || (n > 0 && !b)) return fail(GRKAN_ERR_INVALID, "null tensor pointer");
  const size_t es = elem_size(dtype);
  const bool vec = vec_ok(d, n_groups, es, {x, dy, dx});
  const Plan p = make_plan(rows, d, n_groups, /*m1=*/0, n, es, vec, 2, sm_count());  // never staged
  if (!plan_fits(p)) return fail(GRKAN_ERR_GRID, "grid geometry invalid: %lld CTAs", (long long)p.ctas);
  LaunchArgs L{};
  L.plan = &p;
  L.x = x;
  L.dy = dy;
  L.out = dx;
  L.a = a;
  L.b = b;
  L.da = da;
  L.db = db;
  L.st = reinterpret_cast<DevStatus*>(status);
  L.m1 = m1;
  L.n = n;
  L.exact = (flags & GRKAN_FLAG_EXACT) != 0;
  L.vec = vec;
  L.check = false;
  L.stream = s;
  e = launch("atomic", dtype, L);
  if (e != cudaSuccess) return cuda_fail(e, "k_bwd_atomic launch");
  return GRKAN_OK;
}

int grkan_read_status(const grkan_device_status* status, void* stream,
                      grkan_device_status* host_out) {
  if (!status || !host_out) return fail(GRKAN_ERR_INVALID, "null status pointer");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  cudaError_t e = cudaMemcpyAsync(host_out, status, sizeof(grkan_device_status), cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) return cuda_fail(e, "grkan_read_status");
  if (host_out->nonfinite_input) return fail(GRKAN_ERR_NONFINITE_INPUT, "non-finite input");
  if (host_out->peer_timeout)
    return fail(GRKAN_ERR_PEER_TIMEOUT, "peer exchange timed out: a rank never arrived (grkan_bwd_p2p)");
  if (host_out->accum_overflow) return fail(GRKAN_ERR_ACCUM_OVERFLOW, "accumulation overflow");
  return GRKAN_OK;
}

}  // extern "C"
