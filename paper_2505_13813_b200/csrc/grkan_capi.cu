// grkan_capi.cu -- the C ABI (include/grkan_b200.h): validation, launch planning
// and dispatch onto the sm_100a kernels in grkan_kernels.cuh.
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

#include "../../include/grkan_b200.h"
#include "grkan_kernels.cuh"

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

struct Plan {
  int W = 1;
  int threads = 0;
  int64_t ctas = 0;
  Geom geo{};
};

constexpr int kEltsPerThread = 64;  // target elements per thread per CTA
constexpr int kTargetThreads = 256;

Plan make_plan(int64_t rows, int32_t d, int32_t ng, size_t es, bool vec, int sms) {
  Plan p;
  const int dg = d / ng;
  p.W = vec ? static_cast<int>(16 / es) : 1;
  const int U = p.W >= 8 ? 2 : 4;  // must match grkan::Unroll
  const int V = dg / p.W;
  int CT, RPB;
  if (V <= 384) {
    CT = V;
    const int step = 32 / std::gcd(V, 32);  // makes CT * RPB a multiple of 32
    long k = lround(static_cast<double>(kTargetThreads) / (static_cast<double>(V) * step));
    if (k < 1) k = 1;
    RPB = static_cast<int>(step * k);
    if (CT * RPB > grkan::kMaxThreads) {
      CT = 256;
      RPB = 1;
    }
  } else {
    CT = 256;
    RPB = 1;
  }
  const int col_iters = (V + CT - 1) / CT;
  auto rows_per_thread = [&](int ept) {
    int ptr = (ept + p.W * col_iters - 1) / (p.W * col_iters);
    ptr = ((ptr + U - 1) / U) * U;
    return ptr < U ? U : ptr;
  };
  int ptr = rows_per_thread(kEltsPerThread);
  int64_t R = static_cast<int64_t>(RPB) * ptr;
  int64_t n_tiles = (rows + R - 1) / R;
  // small tensors: shrink tiles until there are a few CTAs per SM
  while (ptr > U && n_tiles * ng < 4LL * sms) {
    ptr = ((ptr / 2 + U - 1) / U) * U;
    R = static_cast<int64_t>(RPB) * ptr;
    n_tiles = (rows + R - 1) / R;
  }
  p.threads = CT * RPB;
  p.geo.rows = rows;
  p.geo.n_tiles = n_tiles;
  p.geo.d = d;
  p.geo.ng = ng;
  p.geo.dg = dg;
  p.geo.V = V;
  p.geo.CT = CT;
  p.geo.RPB = RPB;
  p.geo.R = static_cast<int32_t>(R);
  p.ctas = n_tiles * ng;
  return p;
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
  if (flags & ~(GRKAN_FLAG_EXACT | GRKAN_FLAG_CHECK_FINITE))
    return fail(GRKAN_ERR_INVALID, "unknown flag bits 0x%x", flags);
  return GRKAN_OK;
}

// ---------------------------------------------------------------------------
// Compile-time dispatch: dtype x {fast, exact} x {(6,4) fixed, generic <=12/12}
// x {128-bit vector, scalar}.
// ---------------------------------------------------------------------------
template <typename T>
struct TT {
  using type = T;
};
template <bool B>
struct BT {
  static constexpr bool value = B;
};
template <int I>
struct IT {
  static constexpr int value = I;
};

template <typename F>
cudaError_t dispatch(int dtype, bool exact, bool fixed, bool vec, F&& f) {
  auto with_t = [&](auto tt) -> cudaError_t {
    using T = typename decltype(tt)::type;
    constexpr int WV = static_cast<int>(16 / sizeof(T));
    auto with_e = [&](auto et) -> cudaError_t {
      auto with_f = [&](auto ft) -> cudaError_t {
        return vec ? f(tt, et, ft, IT<WV>{}) : f(tt, et, ft, IT<1>{});
      };
      return fixed ? with_f(BT<true>{}) : with_f(BT<false>{});
    };
    return exact ? with_e(BT<true>{}) : with_e(BT<false>{});
  };
  switch (dtype) {
    case GRKAN_F32: return with_t(TT<float>{});
    case GRKAN_BF16: return with_t(TT<__nv_bfloat16>{});
    case GRKAN_F64: return with_t(TT<double>{});
    default: return cudaErrorInvalidValue;
  }
}

constexpr int kFixM1 = 6, kFixN = 4;  // the paper's degrees (5, 4)
constexpr int kGenM1 = GRKAN_MAX_M1, kGenN = GRKAN_MAX_N;

size_t ws_bytes_for(const Plan& p, int32_t m1, int32_t n, int32_t dtype) {
  const size_t part = static_cast<size_t>(p.geo.ng) * (m1 + n) * p.geo.n_tiles * acc_size(dtype);
  return 256 + ((part + 255) / 256) * 256;
}

}  // namespace

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
    default: return "unknown status";
  }
}

int grkan_plan(int64_t rows, int32_t d, int32_t n_groups, int32_t m1, int32_t n, int32_t dtype,
               int64_t* out5) {
  int rc = check_layout(rows, d, n_groups, m1, n, dtype, 0);
  if (rc) return rc;
  if (!out5) return fail(GRKAN_ERR_INVALID, "null output");
  const size_t es = elem_size(dtype);
  const Plan p = make_plan(rows, d, n_groups, es, vec_ok(d, n_groups, es, {}), 148);
  out5[0] = p.W;
  out5[1] = p.threads;
  out5[2] = p.geo.R;
  out5[3] = p.geo.n_tiles;
  out5[4] = p.ctas;
  return GRKAN_OK;
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
  const size_t a = can_vec ? ws_bytes_for(make_plan(rows, d, n_groups, es, true, kAnySms), m1, n, dtype) : 0;
  const size_t b = ws_bytes_for(make_plan(rows, d, n_groups, es, false, kAnySms), m1, n, dtype);
  return a > b ? a : b;
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
  const Plan p = make_plan(rows, d, n_groups, es, vec, sm_count());
  if (p.ctas > 0x7fffffffLL) return fail(GRKAN_ERR_GRID, "grid geometry invalid: %lld CTAs", (long long)p.ctas);
  const bool fixed = (m1 == kFixM1 && n == kFixN);
  DevStatus* st = reinterpret_cast<DevStatus*>(status);
  cudaError_t e = dispatch(dtype, flags & GRKAN_FLAG_EXACT, fixed, vec, [&](auto tt, auto et, auto ft, auto wt) {
    using T = typename decltype(tt)::type;
    constexpr bool E = decltype(et)::value;
    constexpr bool FX = decltype(ft)::value;
    constexpr int W = decltype(wt)::value;
    using A = typename grkan::VecIO<T, W>::A;
    constexpr int MM1 = FX ? kFixM1 : kGenM1;
    constexpr int MN = FX ? kFixN : kGenN;
    grkan::k_fwd<T, E, MM1, MN, FX, W><<<static_cast<unsigned>(p.ctas), p.threads, 0, s>>>(
        static_cast<const T*>(x), static_cast<T*>(y), static_cast<const A*>(a),
        static_cast<const A*>(b), p.geo, m1, n, check ? 1 : 0, st);
    return cudaGetLastError();
  });
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
  cudaError_t e = cudaMemsetAsync(ws, 0, sizeof(DevStatus), s);
  if (e != cudaSuccess) return cuda_fail(e, "cudaMemsetAsync(status)");
  const size_t as = acc_size(dtype);
  if (rows == 0) {  // nothing to fold: the gradients are exact zeros
    e = cudaMemsetAsync(da, 0, static_cast<size_t>(n_groups) * m1 * as, s);
    if (e == cudaSuccess && n > 0) e = cudaMemsetAsync(db, 0, static_cast<size_t>(n_groups) * n * as, s);
    return e == cudaSuccess ? GRKAN_OK : cuda_fail(e, "cudaMemsetAsync(da/db)");
  }
  if (!x || !dy || !dx || !a || (n > 0 && !b)) return fail(GRKAN_ERR_INVALID, "null tensor pointer");
  const size_t es = elem_size(dtype);
  const bool vec = vec_ok(d, n_groups, es, {x, dy, dx});
  const Plan p = make_plan(rows, d, n_groups, es, vec, sm_count());
  if (p.ctas > 0x7fffffffLL) return fail(GRKAN_ERR_GRID, "grid geometry invalid: %lld CTAs", (long long)p.ctas);
  const size_t need = ws_bytes_for(p, m1, n, dtype);
  if (ws_bytes < need)
    return fail(GRKAN_ERR_INVALID, "workspace too small: %zu < %zu bytes", ws_bytes, need);
  void* part = static_cast<char*>(ws) + 256;
  const bool fixed = (m1 == kFixM1 && n == kFixN);
  const bool check = (flags & GRKAN_FLAG_CHECK_FINITE) != 0;
  e = dispatch(dtype, flags & GRKAN_FLAG_EXACT, fixed, vec, [&](auto tt, auto et, auto ft, auto wt) {
    using T = typename decltype(tt)::type;
    constexpr bool E = decltype(et)::value;
    constexpr bool FX = decltype(ft)::value;
    constexpr int W = decltype(wt)::value;
    using A = typename grkan::VecIO<T, W>::A;
    constexpr int MM1 = FX ? kFixM1 : kGenM1;
    constexpr int MN = FX ? kFixN : kGenN;
    grkan::k_bwd_main<T, E, MM1, MN, FX, W><<<static_cast<unsigned>(p.ctas), p.threads, 0, s>>>(
        static_cast<const T*>(x), static_cast<const T*>(dy), static_cast<T*>(dx),
        static_cast<const A*>(a), static_cast<const A*>(b), static_cast<A*>(part), p.geo, m1, n,
        check ? 1 : 0, st);
    cudaError_t le = cudaGetLastError();
    if (le != cudaSuccess) return le;
    // K3 with programmatic dependent launch: its launch overlaps K2's tail,
    // its griddepcontrol.wait orders it after K2's memory.
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(static_cast<unsigned>(n_groups * (m1 + n)));
    cfg.blockDim = dim3(256);
    cfg.dynamicSmemBytes = 0;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, grkan::k_bwd_reduce<A>, static_cast<const A*>(part),
                              p.geo.n_tiles, m1, n, static_cast<A*>(da), static_cast<A*>(db), st);
  });
  if (e != cudaSuccess) return cuda_fail(e, "k_bwd launch");
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
  const Plan p = make_plan(rows, d, n_groups, es, vec, sm_count());
  const bool fixed = (m1 == kFixM1 && n == kFixN);
  DevStatus* st = reinterpret_cast<DevStatus*>(status);
  e = dispatch(dtype, flags & GRKAN_FLAG_EXACT, fixed, vec, [&](auto tt, auto et, auto ft, auto wt) {
    using T = typename decltype(tt)::type;
    constexpr bool E = decltype(et)::value;
    constexpr bool FX = decltype(ft)::value;
    constexpr int W = decltype(wt)::value;
    using A = typename grkan::VecIO<T, W>::A;
    constexpr int MM1 = FX ? kFixM1 : kGenM1;
    constexpr int MN = FX ? kFixN : kGenN;
    grkan::k_bwd_atomic<T, E, MM1, MN, FX, W><<<static_cast<unsigned>(p.ctas), p.threads, 0, s>>>(
        static_cast<const T*>(x), static_cast<const T*>(dy), static_cast<T*>(dx),
        static_cast<const A*>(a), static_cast<const A*>(b), static_cast<A*>(da), static_cast<A*>(db),
        p.geo, m1, n);
    cudaError_t le = cudaGetLastError();
    if (le != cudaSuccess || !st) return le;
    grkan::k_check_finite<A><<<1, 256, 0, s>>>(static_cast<const A*>(da), (int64_t)n_groups * m1, st);
    if (n > 0) grkan::k_check_finite<A><<<1, 256, 0, s>>>(static_cast<const A*>(db), (int64_t)n_groups * n, st);
    return cudaGetLastError();
  });
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
  if (host_out->accum_overflow) return fail(GRKAN_ERR_ACCUM_OVERFLOW, "accumulation overflow");
  return GRKAN_OK;
}

}  // extern "C"
