// grkan_launch.cuh -- compile-time dispatch from LaunchArgs onto the kernel
// instantiations: {fast, exact} x {(5,4) fixed, generic <= 12/12} x
// {128-bit vector, scalar} x {checked, unchecked}.  Included once per dtype TU.
#pragma once

#include <atomic>

#include "grkan_kernels.cuh"
#include "grkan_staged.cuh"
#include "grkan_types.h"

namespace grkan {

constexpr int kFixM1 = 6, kFixN = 4;   // the paper's degrees (5, 4)
constexpr int kGenM1 = 12, kGenN = 12; // GRKAN_MAX_M1 / GRKAN_MAX_N

template <typename T>
constexpr int vec_width() { return static_cast<int>(16 / sizeof(T)); }

// Degree shapes of the register-direct kernels: 0 = the paper's (5, 4) and
// -1 = (3, 2) (the reference's small test degrees, run_bench --num-coeffs 4
// --den-coeffs 2) at compile time; C = 4, 8, 12 = run-time degrees up to
// capacity C for both polynomials (the generic Horner evaluates all C steps
// with uniform selects, so a small capacity is several times cheaper than the
// 12/12 maximum).
template <int S>
struct Deg {
  static constexpr bool FX = S <= 0;
  static constexpr int M1 = S == 0 ? kFixM1 : (S < 0 ? 4 : S);
  static constexpr int N = S == 0 ? kFixN : (S < 0 ? 2 : S);
};

inline int deg_shape(const LaunchArgs& L) {
  if (L.m1 == kFixM1 && L.n == kFixN) return 0;
  if (L.m1 == 4 && L.n == 2) return -1;
  const int c = L.m1 > L.n ? L.m1 : L.n;
  return c <= 4 ? 4 : (c <= 8 ? 8 : kGenM1);
}

template <typename F>
cudaError_t with_shape(int s, F&& f) {
  switch (s) {
    case 0: return f(std::integral_constant<int, 0>{});
    case -1: return f(std::integral_constant<int, -1>{});
    case 4: return f(std::integral_constant<int, 4>{});
    case 8: return f(std::integral_constant<int, 8>{});
    default: return f(std::integral_constant<int, kGenM1>{});
  }
}

// Calls f(bool_constant<EXACT>, int_constant<degree shape>, int_constant<W>, bool_constant<CHECK>).
template <typename T, typename F>
cudaError_t dispatch(const LaunchArgs& L, F&& f) {
  auto w = [&](auto e, auto sh, auto ck) -> cudaError_t {
    if (L.vec) return f(e, sh, std::integral_constant<int, vec_width<T>()>{}, ck);
    return f(e, sh, std::integral_constant<int, 1>{}, ck);
  };
  auto c = [&](auto e, auto sh) -> cudaError_t {
    return L.check ? w(e, sh, std::true_type{}) : w(e, sh, std::false_type{});
  };
  auto x = [&](auto e) -> cudaError_t {
    return with_shape(deg_shape(L), [&](auto sh) { return c(e, sh); });
  };
  return L.exact ? x(std::true_type{}) : x(std::false_type{});
}

// Opt a kernel into its dynamic shared memory size (static + dynamic > 48 KB
// needs the attribute).  The attribute is per device: one cache per kernel
// instantiation and device.
template <auto Kernel>
cudaError_t allow_smem(size_t bytes) {
  static std::atomic<size_t> granted_per_dev[64];
  int dev = 0;
  cudaGetDevice(&dev);
  std::atomic<size_t>& granted = granted_per_dev[dev & 63];
  if (bytes <= granted.load(std::memory_order_relaxed)) return cudaSuccess;
  cudaError_t e = cudaFuncSetAttribute(Kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(bytes));
  if (e == cudaSuccess) {
    size_t cur = granted.load(std::memory_order_relaxed);
    while (cur < bytes && !granted.compare_exchange_weak(cur, bytes, std::memory_order_relaxed)) {
    }
  }
  return e;
}

// Staged kernels: f(bool_constant<EXACT>, bool_constant<CHECK>, int_constant<M1>,
// int_constant<N>) for the two compile-time degree pairs make_plan stages:
// the paper's (5, 4) and (3, 2).
template <typename T, typename F>
cudaError_t dispatch_staged(const LaunchArgs& L, F&& f) {
  auto d = [&](auto e, auto ck) -> cudaError_t {
    if (L.m1 == 4 && L.n == 2) return f(e, ck, std::integral_constant<int, 4>{}, std::integral_constant<int, 2>{});
    return f(e, ck, std::integral_constant<int, kFixM1>{}, std::integral_constant<int, kFixN>{});
  };
  auto c = [&](auto e) -> cudaError_t {
    return L.check ? d(e, std::true_type{}) : d(e, std::false_type{});
  };
  return L.exact ? c(std::true_type{}) : c(std::false_type{});
}

template <typename T>
cudaError_t launch_fwd_t(const LaunchArgs& L) {
  using A = typename VecIO<T, 1>::A;
  const Plan& p = *L.plan;
  if (p.staged) {
    return dispatch_staged<T>(L, [&](auto e, auto ck, auto m1, auto n) -> cudaError_t {
      constexpr auto kern = k_fwd_staged<T, decltype(e)::value, decltype(ck)::value, decltype(m1)::value,
                                         decltype(n)::value>;
      cudaError_t ae = allow_smem<kern>(p.smem);
      if (ae != cudaSuccess) return ae;
      kern<<<static_cast<unsigned>(p.ctas), kFwdThreads, p.smem, L.stream>>>(
          static_cast<const T*>(L.x), static_cast<T*>(L.out), static_cast<const A*>(L.a),
          static_cast<const A*>(L.b), p.geo, p.stages, L.st, L.tmx);
      return cudaGetLastError();
    });
  }
  return dispatch<T>(L, [&](auto e, auto sh, auto wc, auto ck) -> cudaError_t {
    using DG = Deg<decltype(sh)::value>;
    k_fwd<T, decltype(e)::value, DG::M1, DG::N, DG::FX, decltype(wc)::value,
          decltype(ck)::value><<<static_cast<unsigned>(p.ctas), kBlock, 0, L.stream>>>(
        static_cast<const T*>(L.x), static_cast<T*>(L.out), static_cast<const A*>(L.a),
        static_cast<const A*>(L.b), p.geo, L.m1, L.n, L.st);
    return cudaGetLastError();
  });
}

template <typename A>
cudaError_t launch_reduce_t(const A* part, int64_t n_tiles, int64_t slot_stride, int ng, int m1, int n, A* da,
                            A* db, DevStatus* st, cudaStream_t stream, unsigned long long* cnt = nullptr);

template <typename T>
cudaError_t launch_bwd_t(const LaunchArgs& L) {
  using A = typename VecIO<T, 1>::A;
  const Plan& p = *L.plan;
  cudaError_t e0;
  if (L.instr) {
    // the instrumented instantiations: same kernels, counting (unchecked, per-CTA partials)
    auto ex = [&](auto e) -> cudaError_t {
      if (p.staged && L.m1 == 4) {
        constexpr auto kern = k_bwd_staged<T, decltype(e)::value, false, false, true, false, false, 4, 2>;
        cudaError_t ae = allow_smem<kern>(p.smem);
        if (ae != cudaSuccess) return ae;
        kern<<<static_cast<unsigned>(p.ctas), kStagedThreads, p.smem, L.stream>>>(
            static_cast<const T*>(L.x), static_cast<const T*>(L.dy), static_cast<T*>(L.out), nullptr,
            static_cast<const A*>(L.a), static_cast<const A*>(L.b), static_cast<A*>(L.part), p.geo, p.stages,
            L.st, L.tmx, L.tmu);
        return cudaGetLastError();
      }
      if (p.staged) {
        constexpr auto kern = k_bwd_staged<T, decltype(e)::value, false, false, true>;
        cudaError_t ae = allow_smem<kern>(p.smem);
        if (ae != cudaSuccess) return ae;
        kern<<<static_cast<unsigned>(p.ctas), kStagedThreads, p.smem, L.stream>>>(
            static_cast<const T*>(L.x), static_cast<const T*>(L.dy), static_cast<T*>(L.out), nullptr,
            static_cast<const A*>(L.a), static_cast<const A*>(L.b), static_cast<A*>(L.part), p.geo, p.stages,
            L.st, L.tmx, L.tmu);
        return cudaGetLastError();
      }
      auto fw = [&](auto sh, auto wc) -> cudaError_t {
        using DG = Deg<decltype(sh)::value>;
        k_bwd_main<T, decltype(e)::value, DG::M1, DG::N, DG::FX, decltype(wc)::value,
                   false, true><<<static_cast<unsigned>(p.ctas), kBlock, 0, L.stream>>>(
            static_cast<const T*>(L.x), static_cast<const T*>(L.dy), static_cast<T*>(L.out),
            static_cast<const A*>(L.a), static_cast<const A*>(L.b), static_cast<A*>(L.part), p.geo, L.m1, L.n,
            L.st);
        return cudaGetLastError();
      };
      auto w = [&](auto sh) -> cudaError_t {
        if (L.vec) return fw(sh, std::integral_constant<int, vec_width<T>()>{});
        return fw(sh, std::integral_constant<int, 1>{});
      };
      return with_shape(deg_shape(L), w);
    };
    e0 = L.exact ? ex(std::true_type{}) : ex(std::false_type{});
    if (e0 != cudaSuccess) return e0;
    return launch_reduce_t<A>(static_cast<const A*>(L.part), p.geo.n_tiles, 1, p.geo.ng, L.m1, L.n,
                              static_cast<A*>(L.da), static_cast<A*>(L.db), L.st, L.stream, p.geo.cnt);
  }
  if (p.staged) {
    e0 = dispatch_staged<T>(L, [&](auto e, auto ck, auto m1, auto n) -> cudaError_t {
      auto go = [&](auto det, auto fwd, auto lut, auto cw) -> cudaError_t {
        constexpr auto kern = k_bwd_staged<T, decltype(e)::value, decltype(ck)::value, decltype(det)::value, false,
                                           decltype(fwd)::value, decltype(lut)::value, decltype(m1)::value,
                                           decltype(n)::value, decltype(cw)::value>;
        cudaError_t ae = allow_smem<kern>(p.smem);
        if (ae != cudaSuccess) return ae;
        kern<<<static_cast<unsigned>(p.ctas), staged_threads<decltype(cw)::value>(), p.smem, L.stream>>>(
            static_cast<const T*>(L.x), static_cast<const T*>(L.dy), static_cast<T*>(L.out), static_cast<T*>(L.y2),
            static_cast<const A*>(L.a), static_cast<const A*>(L.b), static_cast<A*>(L.part), p.geo,
            p.stages, L.st, L.tmx, L.tmu);
        return cudaGetLastError();
      };
      const std::false_type no;
      const std::integral_constant<int, kConsumerWarps> cw0;
      if (L.y2) {  // fused step: per-CTA partials only, the geometry grkan_bwd would pick
        if constexpr (sizeof(T) <= 4)
          if (p.cw == kWideWarps) return go(no, std::true_type{}, no, std::integral_constant<int, kWideWarps>{});
        return go(no, std::true_type{}, no, cw0);
      }
      constexpr bool kPaper = decltype(m1)::value == kFixM1 && decltype(n)::value == kFixN;
      constexpr bool kLutType = std::is_same<T, __nv_bfloat16>::value && !decltype(e)::value && kPaper;
      if constexpr (sizeof(T) <= 4) {
        if (p.cw == kWideWarps && !p.geo.det) {  // the wide geometry (make_plan, grkan_bwd only)
          const std::integral_constant<int, kWideWarps> cww;
          if constexpr (kLutType)
            if (p.geo.lut_ne > 0) return go(no, no, std::true_type{}, cww);
          return go(no, no, no, cww);
        }
      }
      if constexpr (kLutType) {
        if (p.geo.lut_ne > 0)  // the x-factor table (make_plan decides; sizes its shared memory)
          return p.geo.det ? go(std::true_type{}, no, std::true_type{}, cw0) : go(no, no, std::true_type{}, cw0);
      }
      return p.geo.det ? go(std::true_type{}, no, no, cw0) : go(no, no, no, cw0);
    });
  } else e0 = dispatch<T>(L, [&](auto e, auto sh, auto wc, auto ck) -> cudaError_t {
    using DG = Deg<decltype(sh)::value>;
    k_bwd_main<T, decltype(e)::value, DG::M1, DG::N, DG::FX,
               decltype(wc)::value, decltype(ck)::value>
        <<<static_cast<unsigned>(p.ctas), kBlock, 0, L.stream>>>(
            static_cast<const T*>(L.x), static_cast<const T*>(L.dy), static_cast<T*>(L.out),
            static_cast<const A*>(L.a), static_cast<const A*>(L.b), static_cast<A*>(L.part), p.geo,
            L.m1, L.n, L.st);
    return cudaGetLastError();
  });
  if (e0 != cudaSuccess || L.partials_only) return e0;
  return launch_reduce_t<A>(static_cast<const A*>(L.part), p.geo.n_tiles, p.geo.det ? (int64_t)p.geo.ng * (L.m1 + L.n) : 1,
                            p.geo.ng, L.m1, L.n, static_cast<A*>(L.da), static_cast<A*>(L.db), L.st, L.stream);
}

// K3 alone: fixed-order fold of n_tiles partials per (group, coefficient)
// (column-major, slot_stride 1; or slot-major, slot_stride ng * kc).
template <typename A>
cudaError_t launch_reduce_t(const A* part, int64_t n_tiles, int64_t slot_stride, int ng, int m1, int n, A* da,
                            A* db, DevStatus* st, cudaStream_t stream, unsigned long long* cnt) {
  // K3 with programmatic dependent launch: its launch overlaps K2's tail and
  // its griddepcontrol.wait orders it after all of K2's memory operations.
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(static_cast<unsigned>(ng * (m1 + n)));
  cfg.blockDim = dim3(256);
  cfg.dynamicSmemBytes = 0;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, k_bwd_reduce<A>, part, n_tiles, m1, n, da, db, st, slot_stride, cnt);
}

template <typename T>
cudaError_t launch_atomic_t(const LaunchArgs& L) {
  using A = typename VecIO<T, 1>::A;
  const Plan& p = *L.plan;
  LaunchArgs L2 = L;
  L2.check = false;
  cudaError_t e0 = dispatch<T>(L2, [&](auto e, auto sh, auto wc, auto) -> cudaError_t {
    using DG = Deg<decltype(sh)::value>;
    auto go = [&](auto ins) -> cudaError_t {
      k_bwd_atomic<T, decltype(e)::value, DG::M1, DG::N, DG::FX, decltype(wc)::value,
                   decltype(ins)::value><<<static_cast<unsigned>(p.ctas), kBlock, 0, L.stream>>>(
          static_cast<const T*>(L.x), static_cast<const T*>(L.dy), static_cast<T*>(L.out),
          static_cast<const A*>(L.a), static_cast<const A*>(L.b), static_cast<A*>(L.da),
          static_cast<A*>(L.db), p.geo, L.m1, L.n);
      return cudaGetLastError();
    };
    return L.instr ? go(std::true_type{}) : go(std::false_type{});
  });
  if (e0 != cudaSuccess || !L.st) return e0;
  k_check_finite<A><<<1, 256, 0, L.stream>>>(static_cast<const A*>(L.da), (int64_t)p.geo.ng * L.m1, L.st);
  if (L.n > 0) k_check_finite<A><<<1, 256, 0, L.stream>>>(static_cast<const A*>(L.db), (int64_t)p.geo.ng * L.n, L.st);
  return cudaGetLastError();
}

}  // namespace grkan

#define GRKAN_DEFINE_LAUNCHERS(T, SUF)                                                       \
  namespace grkan {                                                                          \
  cudaError_t launch_fwd_##SUF(const LaunchArgs& L) { return launch_fwd_t<T>(L); }           \
  cudaError_t launch_bwd_##SUF(const LaunchArgs& L) { return launch_bwd_t<T>(L); }           \
  cudaError_t launch_atomic_##SUF(const LaunchArgs& L) { return launch_atomic_t<T>(L); }     \
  cudaError_t launch_reduce_##SUF(const void* part, int64_t n_tiles, int64_t slot_stride, int ng, int m1, \
                                  int n, void* da, void* db, DevStatus* st, cudaStream_t s) {   \
    using A = typename VecIO<T, 1>::A;                                                       \
    return launch_reduce_t<A>(static_cast<const A*>(part), n_tiles, slot_stride, ng, m1, n,   \
                              static_cast<A*>(da), static_cast<A*>(db), st, s);             \
  }                                                                                          \
  }
