// grkan_fused.cu -- fused GR-KAN layer backward through its linear map
// (SURVEY.md section 8f #3), tcgen05 tensor cores + TMA + TMEM on sm_100a.
//
// A GR-KAN layer is F = R(X) (the group-rational unit) followed by a linear
// map Y = F W^T (W = torch Linear weight [out = K, in = N]); the reference's
// layer_forward / layer_backward (pkg/src/grkan/layer.py:318-379) do the two
// steps separately, so dF = dY W makes a round trip through memory before the
// rational backward reads it.  Here one kernel computes
//
//     dF = dY [M, K] . W [K, N]          bf16 x bf16 -> fp32, accumulated in TMEM
//     dX = R'(X, dF),  da / db partials  in the epilogue, straight from TMEM
//
// so dF never exists in HBM.  Per CTA: one 128 x BN output tile (BN divides
// the group width, so the tile's coefficients are CTA-uniform) and the whole
// K loop.  Warp roles (192 threads):
//   warp 0      TMA producer: dY tile [128 x 64] (K-major, 128B swizzle) and
//               W tile [64 x BN] (N-major, 128B/64B swizzle atoms) per stage
//   warp 1      TMEM allocator + MMA issuer (one elected lane issues
//               tcgen05.mma.cta_group::1.kind::f16, M=128, N=BN, K=16 x 4 per stage;
//               tcgen05.commit frees the stage / signals the epilogue)
//   warps 2-5   epilogue: tcgen05.ld 32 columns at a time (thread = tile row =
//               TMEM lane), X from global (32-byte sectors), RationalX2 grad on
//               element pairs (the unfused backward's math, FAST policy), dX to
//               global, ten fp32 accumulators -> one partial per tile per
//               coefficient (fixed butterfly + fixed warp order, no atomics)
// then the unfused path's K3 folds the partials in fixed order.  Two CTAs per
// SM (3-stage ring, 96 KB smem, 2 x BN TMEM columns) overlap one CTA's
// epilogue with the other's MMA.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstring>

#include "../../include/grkan_b200.h"
#include "grkan_staged.cuh"
#include "grkan_types.h"

namespace grkan {

int set_error(int code, const char* msg);  // grkan_capi.cu

namespace fused {

constexpr int kBM = 128;          // tile rows (UMMA M, TMEM lanes)
constexpr int kBK = 64;           // K per stage (one 128-byte swizzle row of bf16)
constexpr int kStages = 3;
constexpr int kThreads = 192;     // producer, MMA, 4 epilogue warps
constexpr int kKC = 10;           // coefficient terms (degrees (5, 4))

__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int c0, int c1, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}

// UMMA shared-memory matrix descriptor (sm_100 format: version 1, base offset 0).
__device__ __forceinline__ uint64_t smem_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo, uint32_t layout) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((saddr >> 4) & 0x3FFFu);
  d |= static_cast<uint64_t>((lbo >> 4) & 0x3FFFu) << 16;
  d |= static_cast<uint64_t>((sbo >> 4) & 0x3FFFu) << 32;
  d |= static_cast<uint64_t>(1) << 46;
  d |= static_cast<uint64_t>(layout & 7u) << 61;
  return d;
}

// Instruction descriptor: D f32, A/B bf16, A K-major, B MN-major, M = 128, N = BN.
template <int BN>
__device__ __forceinline__ uint32_t instr_desc() {
  return (1u << 4) | (1u << 7) | (1u << 10) | (0u << 15) | (1u << 16) | (static_cast<uint32_t>(BN >> 3) << 17) |
         (static_cast<uint32_t>(kBM >> 4) << 24);
}

__device__ __forceinline__ void umma_bf16(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                          uint32_t accumulate) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}

__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}

// 32 lanes x 32 columns of fp32 from TMEM: thread t gets its lane's 32 columns.
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float (&v)[32]) {
  uint32_t r[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
      "%15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
        "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}

struct FusedGeom {
  int64_t M;
  int32_t N, K, ng, dg;
  int32_t n_tiles_n;   // N / BN
  int32_t tiles_pg;    // partials per group = m_tiles * (dg / BN)
  float one;
};

// B tile (W rows k0..k0+63, columns n0..n0+BN-1) is loaded as BN / ATOM boxes
// of ATOM columns x 64 rows; ATOM = 64 (128B swizzle) or 32 (64B swizzle).
template <int BN, int ATOM>
__global__ void __launch_bounds__(kThreads, 2)
    k_linear_bwd_fused(const __grid_constant__ CUtensorMap map_dy, const __grid_constant__ CUtensorMap map_w,
                       const __nv_bfloat16* __restrict__ x, __nv_bfloat16* __restrict__ dx,
                       const float* __restrict__ ca, const float* __restrict__ cb, float* __restrict__ part,
                       FusedGeom geo) {
  constexpr int A_BYTES = kBM * kBK * 2;            // 16 KB
  constexpr int B_BYTES = kBK * BN * 2;             // BN * 128 B
  constexpr int STAGE = A_BYTES + B_BYTES;
  constexpr int ATOM_BYTES = ATOM * 2 * kBK;        // one swizzle-atom column block
  constexpr uint32_t B_LAYOUT = ATOM == 64 ? 2u : 4u;      // SWIZZLE_128B / SWIZZLE_64B
  constexpr uint32_t B_SBO = ATOM * 2 * 8;                 // 8 K-rows of one atom
  constexpr int TMEM_COLS = BN <= 32 ? 32 : BN <= 64 ? 64 : BN <= 128 ? 128 : 256;

  extern __shared__ __align__(1024) unsigned char smem_raw[];
  // 1024-byte alignment for the swizzle atoms
  unsigned char* smem = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t full[kStages], empty[kStages], tmem_full;
  __shared__ uint32_t tmem_base;
  __shared__ float red[4][kKC];

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n_tile = blockIdx.x % geo.n_tiles_n;
  const int64_t m_tile = blockIdx.x / geo.n_tiles_n;
  const int n0 = n_tile * BN;
  const int64_t m0 = m_tile * kBM;
  const int kblocks = geo.K / kBK;

  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(&tmem_full, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {  // TMEM allocation (whole warp), base address to smem
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base)),
                 "n"(TMEM_COLS)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem_d = tmem_base;

  if (warp == 0) {
    if (lane == 0) {  // ---- TMA producer
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_dy)) : "memory");
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_w)) : "memory");
      int slot = 0;
      uint32_t phase = 0;
      for (int kb = 0; kb < kblocks; ++kb) {
        if (kb >= kStages) mbar_wait(&empty[slot], phase ^ 1);
        unsigned char* sa = smem + slot * STAGE;
        unsigned char* sb = sa + A_BYTES;
        mbar_arrive_expect_tx(&full[slot], STAGE);
        tma_load_2d(sa, &map_dy, kb * kBK, static_cast<int>(m0), &full[slot]);
#pragma unroll
        for (int a = 0; a < BN / ATOM; ++a) tma_load_2d(sb + a * ATOM_BYTES, &map_w, n0 + a * ATOM, kb * kBK, &full[slot]);
        if (++slot == kStages) {
          slot = 0;
          phase ^= 1;
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // ---- MMA issuer
      const uint32_t idesc = instr_desc<BN>();
      int slot = 0;
      uint32_t phase = 0;
      for (int kb = 0; kb < kblocks; ++kb) {
        mbar_wait(&full[slot], phase);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t sa = smem_u32(smem + slot * STAGE);
        const uint32_t sb = sa + A_BYTES;
#pragma unroll
        for (int k = 0; k < kBK / 16; ++k) {
          // A: K-major SW128, +32 B per 16-element K step inside the swizzle row
          const uint64_t ad = smem_desc(sa + k * 32, 16, 1024, 2);
          // B: MN-major, K step = two 8-row groups
          const uint64_t bd = smem_desc(sb + k * 2 * B_SBO, ATOM_BYTES, B_SBO, B_LAYOUT);
          umma_bf16(tmem_d, ad, bd, idesc, (kb | k) != 0);
        }
        umma_commit(&empty[slot]);  // frees the stage when these MMAs complete
        if (kb == kblocks - 1) umma_commit(&tmem_full);
        if (++slot == kStages) {
          slot = 0;
          phase ^= 1;
        }
      }
    }
  } else {
    // ---- epilogue: warps 2..5; TMEM lanes 32 * (warp % 4) ..
    const int q = warp & 3;
    const int row = q * 32 + lane;
    const int64_t grow = m0 + row;
    const bool live = grow < geo.M;
    const int g = n0 / geo.dg;
    RationalX2<false> rp;
    rp.load(ca, cb, g, geo.one);
    float2 acc2[kKC];
#pragma unroll
    for (int k = 0; k < kKC; ++k) acc2[k] = make_float2(0.f, 0.f);
    mbar_wait(&tmem_full, 0);
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t taddr = tmem_d + (static_cast<uint32_t>(q * 32) << 16);
    const __nv_bfloat16* xrow = x + grow * geo.N + n0;
    __nv_bfloat16* dxrow = dx + grow * geo.N + n0;
#pragma unroll 1
    for (int c = 0; c < BN; c += 32) {
      float u[32];
      tmem_ld32(taddr + c, u);  // warp-collective: every lane participates
      if (live) {
        uint4 xr[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) xr[i] = __ldcs(reinterpret_cast<const uint4*>(xrow + c) + i);
        uint4 o4[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          float xv[8], o[8];
          Raw16<__nv_bfloat16>::unpack(xr[i], xv);
          float uv[8];
#pragma unroll
          for (int e = 0; e < 8; ++e) uv[e] = u[i * 8 + e];
          rp.template grad_n<4, false>(xv, uv, o, acc2);
          o4[i] = Raw16<__nv_bfloat16>::pack(o);
        }
#pragma unroll
        for (int i = 0; i < 4; ++i) __stcs(reinterpret_cast<uint4*>(dxrow + c) + i, o4[i]);
      }
    }
    // one partial per tile per coefficient: fixed butterfly, fixed warp order
#pragma unroll
    for (int k = 0; k < kKC; ++k) {
      float v = acc2[k].x + acc2[k].y;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
      if (lane == 0) red[q][k] = v;
    }
    asm volatile("bar.sync 1, 128;" ::: "memory");
    if (warp == 2 && lane < kKC) {
      const float v = ((red[0][lane] + red[1][lane]) + red[2][lane]) + red[3][lane];
      const int64_t t = m_tile * (geo.dg / BN) + (n0 % geo.dg) / BN;
      part[(static_cast<int64_t>(g) * kKC + lane) * geo.tiles_pg + t] = v;
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  if (warp == 1)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_d), "n"(TMEM_COLS) : "memory");
}

// ---- host -------------------------------------------------------------------

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

bool make_map(CUtensorMap* m, const void* base, uint64_t inner, uint64_t outer, uint32_t box_in, uint32_t box_out,
              CUtensorMapSwizzle sw) {
  auto fn = encode_fn();
  if (!fn) return false;
  const cuuint64_t dims[2] = {inner, outer};
  const cuuint64_t strides[1] = {inner * 2};
  const cuuint32_t box[2] = {box_in, box_out};
  const cuuint32_t estr[2] = {1, 1};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, estr,
            CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// Widest BN in {256, 192, 128, 64} dividing the group width, else a multiple
// of 32 (64B-swizzle B atoms): {224, 160, 96, 32}.
int pick_bn(int dg, int* atom) {
  const int c128[] = {256, 192, 128, 64};
  for (int bn : c128)
    if (dg % bn == 0) {
      *atom = 64;
      return bn;
    }
  const int c64[] = {224, 160, 96, 32};
  for (int bn : c64)
    if (dg % bn == 0) {
      *atom = 32;
      return bn;
    }
  return 0;
}

template <int BN, int ATOM>
cudaError_t launch_t(const CUtensorMap& mdy, const CUtensorMap& mw, const void* x, void* dx, const float* a,
                     const float* b, float* part, const FusedGeom& geo, int64_t ctas, cudaStream_t s) {
  constexpr size_t smem = static_cast<size_t>(kStages) * (kBM * kBK * 2 + kBK * BN * 2) + 1024;
  auto kern = k_linear_bwd_fused<BN, ATOM>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
  if (e != cudaSuccess) return e;
  kern<<<static_cast<unsigned>(ctas), kThreads, smem, s>>>(mdy, mw, static_cast<const __nv_bfloat16*>(x),
                                                            static_cast<__nv_bfloat16*>(dx), a, b, part, geo);
  return cudaGetLastError();
}

}  // namespace fused
}  // namespace grkan

extern "C" {

size_t grkan_linear_bwd_workspace_bytes(int64_t M, int32_t N, int32_t K, int32_t n_groups) {
  if (M < 0 || N < 1 || K < 1 || n_groups < 1 || N % n_groups) return 0;
  int atom = 0;
  const int bn = grkan::fused::pick_bn(N / n_groups, &atom);
  if (!bn) return 0;
  const int64_t tiles_pg = ((M + grkan::fused::kBM - 1) / grkan::fused::kBM) * ((N / n_groups) / bn);
  const size_t part = static_cast<size_t>(n_groups) * grkan::fused::kKC * tiles_pg * sizeof(float);
  return 256 + ((part + 255) / 256) * 256;
}

int grkan_linear_bwd(const void* dy, const void* w, const void* x, const void* a, const void* b, void* dx,
                     void* da, void* db, void* ws, size_t ws_bytes, int64_t M, int32_t N, int32_t K,
                     int32_t n_groups, uint32_t flags, void* stream) {
  using namespace grkan::fused;
  char msg[256];
  if (N < 1 || n_groups < 1 || N % n_groups) {
    snprintf(msg, sizeof msg, "layout mismatch: feature_dim %d not divisible by num_groups %d", N, n_groups);
    return grkan::set_error(GRKAN_ERR_LAYOUT, msg);
  }
  if (M < 0 || K < 1) return grkan::set_error(GRKAN_ERR_GRID, "grid geometry invalid: M >= 0 and K >= 1 required");
  if (flags & ~GRKAN_FLAG_FAST)
    return grkan::set_error(GRKAN_ERR_UNSUPPORTED, "fused linear backward: FAST policy only");
  const int dg = N / n_groups;
  int atom = 0;
  const int bn = pick_bn(dg, &atom);
  if (!bn || K % kBK) {
    snprintf(msg, sizeof msg, "fused linear backward needs group width %% 32 == 0 and K %% 64 == 0 (dg=%d, K=%d)", dg, K);
    return grkan::set_error(GRKAN_ERR_UNSUPPORTED, msg);
  }
  if (!ws || !da || !db || !dx || !dy || !w || !x || !a || !b)
    return grkan::set_error(GRKAN_ERR_INVALID, "null pointer");
  const size_t need = grkan_linear_bwd_workspace_bytes(M, N, K, n_groups);
  if (ws_bytes < need) return grkan::set_error(GRKAN_ERR_INVALID, "workspace too small");
  for (const void* p : {dy, w, x, (const void*)dx})
    if (reinterpret_cast<uintptr_t>(p) & 15) return grkan::set_error(GRKAN_ERR_INVALID, "tensors must be 16-byte aligned");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  grkan::DevStatus* st = static_cast<grkan::DevStatus*>(ws);
  cudaError_t e = cudaMemsetAsync(ws, 0, sizeof(grkan::DevStatus), s);
  if (e != cudaSuccess) return grkan::set_error(GRKAN_ERR_CUDA, cudaGetErrorString(e));
  if (M == 0) {
    e = cudaMemsetAsync(da, 0, static_cast<size_t>(n_groups) * 6 * 4, s);
    if (e == cudaSuccess) e = cudaMemsetAsync(db, 0, static_cast<size_t>(n_groups) * 4 * 4, s);
    return e == cudaSuccess ? GRKAN_OK : grkan::set_error(GRKAN_ERR_CUDA, cudaGetErrorString(e));
  }
  CUtensorMap mdy, mw;
  if (!make_map(&mdy, dy, static_cast<uint64_t>(K), static_cast<uint64_t>(M), kBK, kBM, CU_TENSOR_MAP_SWIZZLE_128B) ||
      !make_map(&mw, w, static_cast<uint64_t>(N), static_cast<uint64_t>(K), atom, kBK,
                atom == 64 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B))
    return grkan::set_error(GRKAN_ERR_CUDA, "cuTensorMapEncodeTiled failed");
  FusedGeom geo;
  geo.M = M;
  geo.N = N;
  geo.K = K;
  geo.ng = n_groups;
  geo.dg = dg;
  geo.n_tiles_n = N / bn;
  const int64_t m_tiles = (M + kBM - 1) / kBM;
  geo.tiles_pg = static_cast<int32_t>(m_tiles * (dg / bn));
  geo.one = 1.0f;
  const int64_t ctas = m_tiles * geo.n_tiles_n;
  float* part = reinterpret_cast<float*>(static_cast<char*>(ws) + 256);
  const float* fa = static_cast<const float*>(a);
  const float* fb = static_cast<const float*>(b);
  switch (bn) {
    case 256: e = launch_t<256, 64>(mdy, mw, x, dx, fa, fb, part, geo, ctas, s); break;
    case 192: e = launch_t<192, 64>(mdy, mw, x, dx, fa, fb, part, geo, ctas, s); break;
    case 128: e = launch_t<128, 64>(mdy, mw, x, dx, fa, fb, part, geo, ctas, s); break;
    case 64: e = launch_t<64, 64>(mdy, mw, x, dx, fa, fb, part, geo, ctas, s); break;
    case 224: e = launch_t<224, 32>(mdy, mw, x, dx, fa, fb, part, geo, ctas, s); break;
    case 160: e = launch_t<160, 32>(mdy, mw, x, dx, fa, fb, part, geo, ctas, s); break;
    case 96: e = launch_t<96, 32>(mdy, mw, x, dx, fa, fb, part, geo, ctas, s); break;
    default: e = launch_t<32, 32>(mdy, mw, x, dx, fa, fb, part, geo, ctas, s); break;
  }
  if (e != cudaSuccess) return grkan::set_error(GRKAN_ERR_CUDA, cudaGetErrorString(e));
  e = grkan::launch_reduce_f32(part, geo.tiles_pg, 1, n_groups, 6, 4, da, db, st, s);
  if (e != cudaSuccess) return grkan::set_error(GRKAN_ERR_CUDA, cudaGetErrorString(e));
  return GRKAN_OK;
}

}  // extern "C"
