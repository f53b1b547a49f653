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
// so dF never exists in HBM.  Tiles are 128 x BN (BN divides the group width,
// so a tile's coefficients are uniform) with the whole K loop; a persistent
// CTA per SM walks its tiles with two TMEM accumulator buffers.  Warp roles:
//   warp 0      TMA producer: dY tile [128 x 64] (K-major, 128B swizzle) and
//               W tile [64 x BN] (N-major, 128B/64B swizzle atoms) per stage
//   warp 1      TMEM allocator + MMA issuer (one elected lane issues
//               tcgen05.mma.cta_group::1.kind::f16, M=128, N=BN, K=16 x 4 per stage;
//               tcgen05.commit frees the stage / signals the epilogue)
//   warps 2..  4 * ES epilogue warps: tcgen05.ld 32 columns at a time (thread =
//               tile row = TMEM lane; ES warps per lane quadrant split the
//               columns), X from global (32-byte sectors, prefetched one chunk
//               ahead), RationalX2 grad on element pairs (the unfused
//               backward's math, FAST policy), dX to global, ten fp32
//               accumulators -> one partial per (tile, warp) per coefficient
//               (fixed butterfly, no atomics)
// then the unfused path's K3 folds the partials in fixed order.  The epilogue
// releases a TMEM buffer as soon as its last tcgen05.ld lands, so the next
// tile's MMA overlaps the rational math.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <type_traits>

#include "../../include/grkan_b200.h"
#include "grkan_staged.cuh"
#include "grkan_tmap.h"
#include "grkan_types.h"

namespace grkan {

int set_error(int code, const char* msg);  // grkan_capi.cu

namespace fused {

constexpr int kBM = 128;          // tile rows (UMMA M, TMEM lanes)
constexpr int kBK = 64;           // K per stage (one 128-byte swizzle row of bf16)
#ifndef GRKAN_FUSED_SMEM_KB
#define GRKAN_FUSED_SMEM_KB 200
#endif
constexpr int kSmemBudget = GRKAN_FUSED_SMEM_KB * 1024;  // operand ring + X tiles (the rest: alignment, barriers)
constexpr int kKC = 10;           // coefficient terms (degrees (5, 4))
constexpr int kMaxGroups = 64;    // coefficient table in shared memory
#ifndef GRKAN_FUSED_PROBE_NOEPI
#define GRKAN_FUSED_PROBE_NOEPI 0  // diagnostic only: 1 = backward epilogue skips the rational math and dX; 2 = math only skipped
#endif
#ifndef GRKAN_FUSED_PROBE_NOMMA
#define GRKAN_FUSED_PROBE_NOMMA 0  // diagnostic only: one MMA per tile (wrong results), times the epilogue side
#endif
#ifndef GRKAN_FUSED_SK_BN
#define GRKAN_FUSED_SK_BN 192     // short-K (X staged) tile width ...
#endif
#ifndef GRKAN_FUSED_SK_CH
#define GRKAN_FUSED_SK_CH 16      // ... and TMEM columns per epilogue load
#endif
#ifndef GRKAN_FUSED_SK_ES
#define GRKAN_FUSED_SK_ES 3       // ... and epilogue warps per TMEM lane quadrant
#endif

__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int c0, int c1, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}

// TMA prefetch of a tensor box into L2 (no shared memory, no barrier).
__device__ __forceinline__ void tma_prefetch_2d(const CUtensorMap* map, int c0, int c1) {
  asm volatile("cp.async.bulk.prefetch.tensor.2d.L2.global.tile [%0, {%1, %2}];" ::"l"(reinterpret_cast<uint64_t>(map)),
               "r"(c0), "r"(c1)
               : "memory");
}

#ifndef GRKAN_FUSED_NACC
#define GRKAN_FUSED_NACC 2  // backward: TMEM accumulator buffers (more than 2 only where NACC * BN <= 512)
#endif
#ifndef GRKAN_FUSED_XALL
#define GRKAN_FUSED_XALL 1  // backward epilogue: load all of a warp's X columns before the accumulator wait
#endif
#ifndef GRKAN_FUSED_XPF
#define GRKAN_FUSED_XPF 0  // long-K backward: TMA-prefetch each tile's X block into L2 when its MMA starts
#endif

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

// 32 lanes x 16 columns.
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float (&v)[16]) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
      "%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}

// 32 lanes x 8 columns.
__device__ __forceinline__ void tmem_ld8(uint32_t taddr, float (&v)[8]) {
  uint32_t r[8];
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
               : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 8; ++i) v[i] = __uint_as_float(r[i]);
}

template <int CH>
__device__ __forceinline__ void tmem_ld(uint32_t taddr, float (&v)[CH]) {
  if constexpr (CH == 32) tmem_ld32(taddr, v);
  else if constexpr (CH == 16) tmem_ld16(taddr, v);
  else tmem_ld8(taddr, v);
}

// ---- CTA-pair (cta_group::2) helpers --------------------------------------
__device__ __forceinline__ uint32_t cluster_ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// Both CTAs of the pair load into their own shared memory; the transaction
// bytes land on the leader's (CTA 0's) barrier: clear the peer bit.
__device__ __forceinline__ void tma_load_2d_pair(void* dst, const CUtensorMap* map, int c0, int c1, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar) & 0xFEFFFFFFu)
      : "memory");
}
__device__ __forceinline__ void umma_bf16_pair(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                               uint32_t accumulate) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
// commit to the barrier at this offset in BOTH CTAs of the pair
__device__ __forceinline__ void umma_commit_pair(uint64_t* bar) {
  asm volatile(
      "{\n"
      ".reg .b16 m;\n"
      "mov.b16 m, 3;\n"
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], m;\n"
      "}\n" ::"r"(smem_u32(bar))
      : "memory");
}
// arrive on the leader CTA's copy of a barrier
__device__ __forceinline__ void mbar_arrive_leader(uint64_t* bar) {
  uint32_t remote;
  asm volatile("mapa.shared::cluster.u32 %0, %1, 0;" : "=r"(remote) : "r"(smem_u32(bar)));
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(remote) : "memory");
}

struct FusedGeom {
  int64_t M;
  int32_t N, K, ng, dg;
  int32_t n_tiles_n;   // N / BN
  int32_t ppg;         // partials per group = m_tiles * (dg / CW) * 4 (one per warp sub-tile)
  float one;
};

// Persistent, warp-specialised: grid = min(tiles, SMs), CTA c takes tiles
// c, c + grid, ...; two TMEM accumulator buffers so the MMA of tile i + 1 runs
// while the epilogue drains tile i.  B tile (W rows k0..k0+63, columns
// n0..n0+BN-1) is loaded as BN / ATOM boxes of ATOM columns x 64 rows; ATOM =
// 64 (128B swizzle) or 32 (64B swizzle).  ES epilogue warps per TMEM lane
// quadrant split the tile's columns (4 * ES epilogue warps in all).
// XS: the producer also TMA-streams each tile's X block [128 x BN] (64-column
// 128B-swizzled boxes) into a double-buffered smem tile, so the epilogue reads
// X with conflict-free LDS.128 instead of waiting on global loads.
// PAIR: CTA pairs (cluster of 2) run tcgen05.mma.cta_group::2 on 256-row
// tiles -- each CTA loads its 128 rows of dY and HALF of the W tile, the
// leader issues the MMA over both shared memories, each CTA's TMEM receives
// its 128 rows, and each CTA's epilogue drains its own.  Halves the W traffic
// into each SM's shared memory (the long-K shape's limiter).
template <int BN, int ATOM, int ES, int CH, bool XS, int kStages, bool PAIR = false>
__global__ void __launch_bounds__(64 + 128 * ES, 1)
    k_linear_bwd_fused(const __grid_constant__ CUtensorMap map_dy, const __grid_constant__ CUtensorMap map_w,
                       const __grid_constant__ CUtensorMap map_x, const __nv_bfloat16* __restrict__ x, __nv_bfloat16* __restrict__ dx,
                       const float* __restrict__ ca, const float* __restrict__ cb, float* __restrict__ part,
                       FusedGeom geo) {
  static_assert(!(PAIR && XS), "CTA pairs serve the long-K (unstaged X) shapes");
  constexpr int A_BYTES = kBM * kBK * 2;            // 16 KB
  constexpr int B_BYTES = kBK * BN * 2 / (PAIR ? 2 : 1);  // BN * 128 B (half of it per CTA of a pair)
  constexpr int STAGE = A_BYTES + B_BYTES;
  constexpr int ATOM_BYTES = ATOM * 2 * kBK;        // one swizzle-atom column block
  constexpr int B_BOXES = (PAIR ? BN / 2 : BN) / ATOM;
  static_assert(!PAIR || (BN / 2) % ATOM == 0, "each CTA of a pair loads whole B atoms");
  constexpr uint32_t B_LAYOUT = ATOM == 64 ? 2u : 4u;      // SWIZZLE_128B / SWIZZLE_64B
  constexpr uint32_t B_SBO = ATOM * 2 * 8;                 // 8 K-rows of one atom
  // TMEM accumulator buffers: NACC tiles in flight between the MMA and the epilogue
  constexpr int NACC = (GRKAN_FUSED_NACC > 2 && GRKAN_FUSED_NACC * BN <= 512) ? GRKAN_FUSED_NACC : 2;
  constexpr int TMEM_COLS = NACC * BN <= 64 ? 64 : NACC * BN <= 128 ? 128 : NACC * BN <= 256 ? 256 : 512;
  constexpr int NE = 4 * ES;                        // epilogue warps
  constexpr int CW = BN / ES;                       // columns per epilogue warp
  static_assert(CW % CH == 0, "epilogue columns come in CH-column TMEM loads");
  constexpr int NV = CH / 8;                        // 16-byte X / dX vectors per chunk
  constexpr int XBOX = kBM * 64 * 2;                // one 64-column X box (16 KB)
  constexpr int XBYTES = XS ? BN * kBM * 2 : 0;     // one X tile buffer
  static_assert(!XS || BN % 64 == 0, "X staging uses 64-column boxes");

  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t full[kStages], empty[kStages], tfull[NACC], tempty[NACC], xfull[2], xempty[2];
  __shared__ uint32_t tmem_base;
  __shared__ float scoef[kMaxGroups * kKC];  // every group's a (6) || b (4)
  unsigned char* const xs = smem + kStages * STAGE;  // X tile buffers (XS)

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // PAIR: units are 256-row pair tiles walked by clusters; else 128-row tiles by CTAs
  const uint32_t crank = PAIR ? cluster_ctarank() : 0;
  const bool leader = crank == 0;
  const int64_t unit0 = PAIR ? (blockIdx.x >> 1) : blockIdx.x;
  const int64_t ustep = PAIR ? (gridDim.x >> 1) : gridDim.x;
  const int64_t n_tiles = ((geo.M + (PAIR ? 2 : 1) * kBM - 1) / ((PAIR ? 2 : 1) * kBM)) * geo.n_tiles_n;
  const int kblocks = geo.K / kBK;

  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int s = 0; s < NACC; ++s) {
      mbar_init(&tfull[s], 1);
      mbar_init(&tempty[s], PAIR ? 2 * NE : NE);  // PAIR: both CTAs' epilogues drain into the leader's
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&xfull[s], 1);
      mbar_init(&xempty[s], NE);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {  // TMEM allocation (whole warp), base address to smem
    if constexpr (PAIR) {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base)),
                   "n"(TMEM_COLS)
                   : "memory");
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
    } else {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base)),
                   "n"(TMEM_COLS)
                   : "memory");
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
  }
  for (int t = threadIdx.x; t < geo.ng * kKC; t += blockDim.x) {
    const int g = t / kKC, k = t - g * kKC;
    scoef[t] = k < 6 ? ca[g * 6 + k] : cb[g * 4 + (k - 6)];
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  if constexpr (PAIR) cluster_sync_all(); else __syncthreads();  // barriers visible to the peer
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem_d = tmem_base;

  if (warp == 0) {
    if (lane == 0) {  // ---- TMA producer
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_dy)) : "memory");
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_w)) : "memory");
      int slot = 0;
      uint32_t phase = 0;
      int64_t it = 0;
      int i = 0;
      for (int64_t tile = unit0; tile < n_tiles; tile += ustep, ++i) {
        const int n0 = static_cast<int>(tile % geo.n_tiles_n) * BN;
        const int m0 = static_cast<int>((tile / geo.n_tiles_n) * (PAIR ? 2 : 1) * kBM + crank * kBM);
        if constexpr (!XS && GRKAN_FUSED_XPF) {  // the epilogue's X reads then hit L2
#pragma unroll
          for (int a = 0; a < (BN + 63) / 64; ++a) tma_prefetch_2d(&map_x, n0 + a * 64, m0);
        }
        if constexpr (XS) {  // the tile's X block, into buffer i & 1
          const int xb = i & 1;
          mbar_wait(&xempty[xb], ((i >> 1) & 1) ^ 1);
          mbar_arrive_expect_tx(&xfull[xb], XBYTES);
#pragma unroll
          for (int a = 0; a < BN / 64; ++a) tma_load_2d(xs + xb * XBYTES + a * XBOX, &map_x, n0 + a * 64, m0, &xfull[xb]);
        }
        for (int kb = 0; kb < kblocks; ++kb, ++it) {
          if (it >= kStages) mbar_wait(&empty[slot], phase ^ 1);
          unsigned char* sa = smem + slot * STAGE;
          unsigned char* sb = sa + A_BYTES;
          if constexpr (PAIR) {
            if (leader) mbar_arrive_expect_tx(&full[slot], 2 * STAGE);  // both CTAs' bytes
            tma_load_2d_pair(sa, &map_dy, kb * kBK, m0, &full[slot]);
#pragma unroll
            for (int a = 0; a < B_BOXES; ++a)
              tma_load_2d_pair(sb + a * ATOM_BYTES, &map_w, n0 + crank * (BN / 2) + a * ATOM, kb * kBK, &full[slot]);
          } else {
            mbar_arrive_expect_tx(&full[slot], STAGE);
            tma_load_2d(sa, &map_dy, kb * kBK, m0, &full[slot]);
#pragma unroll
            for (int a = 0; a < B_BOXES; ++a) tma_load_2d(sb + a * ATOM_BYTES, &map_w, n0 + a * ATOM, kb * kBK, &full[slot]);
          }
          if (++slot == kStages) {
            slot = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0 && leader) {  // ---- MMA issuer (the pair's leader issues for both CTAs)
      const uint32_t idesc = PAIR ? (instr_desc<BN>() & ~(31u << 24)) | (static_cast<uint32_t>(2 * kBM >> 4) << 24)
                                  : instr_desc<BN>();
      int slot = 0;
      uint32_t phase = 0;
      int i = 0;
      for (int64_t tile = unit0; tile < n_tiles; tile += ustep, ++i) {
        const int acc = i % NACC;
        mbar_wait(&tempty[acc], ((i / NACC) & 1) ^ 1);  // epilogue has drained this buffer
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t dcol = tmem_d + static_cast<uint32_t>(acc * BN);
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
            if (GRKAN_FUSED_PROBE_NOMMA && (kb | k) != 0) continue;  // probe: epilogue-only timing
            if constexpr (PAIR)
              umma_bf16_pair(dcol, ad, bd, idesc, (kb | k) != 0);
            else
              umma_bf16(dcol, ad, bd, idesc, (kb | k) != 0);
          }
          if constexpr (PAIR)
            umma_commit_pair(&empty[slot]);  // frees the stage in both CTAs
          else
            umma_commit(&empty[slot]);  // frees the stage when these MMAs complete
          if (++slot == kStages) {
            slot = 0;
            phase ^= 1;
          }
        }
        if constexpr (PAIR)
          umma_commit_pair(&tfull[acc]);
        else
          umma_commit(&tfull[acc]);  // accumulator ready for the epilogue
      }
    }
  } else {
    // ---- epilogue warps: lanes 32 * (warp % 4) .. of TMEM, columns cs*CW ..
    const int e = warp - 2;
    const int q = warp & 3;
    const int cs = e >> 2;
    const int row = q * 32 + lane;
    int i = 0;
    int g_loaded = -1;
    RationalX2<false> rp;  // the warp's column block lies in one group (CW | dg)
    for (int64_t tile = unit0; tile < n_tiles; tile += ustep, ++i) {
      const int acc = i % NACC;  // TMEM accumulator buffer
      const int xb = i & 1;      // X staging buffer (XS)
      const int n0 = static_cast<int>(tile % geo.n_tiles_n) * BN;
      const int64_t m_tile = (tile / geo.n_tiles_n) * (PAIR ? 2 : 1) + crank;  // 128-row tile index
      const int64_t grow = m_tile * kBM + row;
      const bool live = grow < geo.M;
      const int c0 = n0 + cs * CW;
      const int g = c0 / geo.dg;
      if (g != g_loaded) {
        rp.load_row(scoef + g * kKC, geo.one);
        g_loaded = g;
      }
      const __nv_bfloat16* xrow = x + grow * geo.N + c0;
      __nv_bfloat16* dxrow = dx + grow * geo.N + c0;
      // X is independent of the MMA: fetch the first chunk (or, XALL, every
      // chunk of this warp's columns) before waiting for the accumulator
      constexpr bool XALL = GRKAN_FUSED_XALL && !XS;
      constexpr int XB = XALL ? CW / CH : 2;  // X register buffers
      uint4 xr[XB][NV];
      if (!XS && live) {
#pragma unroll
        for (int cc = 0; cc < (XALL ? CW / CH : 1); ++cc)
#pragma unroll
          for (int v = 0; v < NV; ++v) xr[cc][v] = __ldcs(reinterpret_cast<const uint4*>(xrow + cc * CH) + v);
      }
      const unsigned char* xtile = xs + xb * XBYTES;
      if constexpr (XS) mbar_wait(&xfull[xb], (i >> 1) & 1);
      // accumulators: float2 (packed FFMA2) when the register budget allows
      // (ES <= 3: <= 14 warps, 128 registers), else one float per coefficient
      using AccT = std::conditional_t<(ES <= 3 || CH <= 8), float2, float>;
      AccT sacc[kKC];
#pragma unroll
      for (int k = 0; k < kKC; ++k) sacc[k] = AccT{};
      mbar_wait(&tfull[acc], (i / NACC) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const uint32_t taddr = tmem_d + (static_cast<uint32_t>(q * 32) << 16) + static_cast<uint32_t>(acc * BN + cs * CW);
#pragma unroll
      for (int c = 0; c < CW / CH; ++c) {
        if (!XS && !XALL && live && c + 1 < CW / CH) {
#pragma unroll
          for (int v = 0; v < NV; ++v) xr[(c + 1) % XB][v] = __ldcs(reinterpret_cast<const uint4*>(xrow + (c + 1) * CH) + v);
        }
        if constexpr (XS) {  // 128B-swizzled box: 16-byte chunk j of row r sits at (j ^ (r & 7))
#pragma unroll
          for (int v = 0; v < NV; ++v) {
            const int col = cs * CW + c * CH + v * 8;
            const int j = (col & 63) >> 3;
            xr[c % XB][v] = *reinterpret_cast<const uint4*>(xtile + (col >> 6) * XBOX + row * 128 + ((j ^ (row & 7)) << 4));
          }
          if (c + 1 == CW / CH) {  // done with this X buffer
            __syncwarp();
            if (lane == 0) mbar_arrive(&xempty[xb]);
          }
        }
        float u[CH];
        tmem_ld<CH>(taddr + c * CH, u);  // warp-collective: every lane participates
        if (c + 1 == CW / CH) {          // this warp is done with the accumulator buffer
          asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
          __syncwarp();
          if (lane == 0) {
            if constexpr (PAIR)
              mbar_arrive_leader(&tempty[acc]);
            else
              mbar_arrive(&tempty[acc]);
          }
        }
        if (live && GRKAN_FUSED_PROBE_NOEPI == 2) {  // probe: dX traffic without the math
#pragma unroll
          for (int v = 0; v < NV; ++v) {
            float o[8];
#pragma unroll
            for (int k = 0; k < 8; ++k) o[k] = u[v * 8 + k];
            __stcs(reinterpret_cast<uint4*>(dxrow + c * CH) + v, Raw16<__nv_bfloat16>::pack(o));
          }
        }
        if (live && !GRKAN_FUSED_PROBE_NOEPI) {
          uint4 o4[NV];
#pragma unroll
          for (int v = 0; v < NV; ++v) {
            float xv[8], o[8], uv[8];
            Raw16<__nv_bfloat16>::unpack(xr[c % XB][v], xv);
#pragma unroll
            for (int k = 0; k < 8; ++k) uv[k] = u[v * 8 + k];
            rp.template grad_n<4, false, AccT>(xv, uv, o, sacc);
            o4[v] = Raw16<__nv_bfloat16>::pack(o);
          }
#pragma unroll
          for (int v = 0; v < NV; ++v) __stcs(reinterpret_cast<uint4*>(dxrow + c * CH) + v, o4[v]);
        }
      }
      // one partial per (128-row x CW-column warp block) per coefficient: fixed butterfly
      const int64_t t = (m_tile * (geo.dg / CW) + (c0 % geo.dg) / CW) * 4 + q;
#pragma unroll
      for (int k = 0; k < kKC; ++k) {
        float v;
        if constexpr (ES <= 3 || CH <= 8) v = sacc[k].x + sacc[k].y; else v = sacc[k];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if (lane == 0) part[(static_cast<int64_t>(g) * kKC + k) * geo.ppg + t] = v;
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  if constexpr (PAIR) cluster_sync_all(); else __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  if (warp == 1) {
    if constexpr (PAIR)
      asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_d), "n"(TMEM_COLS) : "memory");
    else
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_d), "n"(TMEM_COLS) : "memory");
  }
}

// ---- host -------------------------------------------------------------------

using grkan::encode_fn;

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

// Tile shapes, best first: (BN, B swizzle atom, epilogue warps per lane
// quadrant ES).  A shape fits when BN divides N and each epilogue warp's
// column block CW = BN / ES lies inside one group (CW divides the group width).
// ES = 4 (16 epilogue warps, 576 threads) uses 16-column TMEM loads to fit
// the 112-register budget; ES <= 2 loads 32 columns at a time.
// xs: X staged through shared memory (chosen when the epilogue dominates,
// i.e. small K: it costs ring stages the MMA needs at large K).
struct TileShape {
  int bn, atom, es, ch;
  bool xs;
};
#ifndef GRKAN_FUSED_LK_BN  // tuning knobs: the long-K shape tried first
#define GRKAN_FUSED_LK_BN 256
#define GRKAN_FUSED_LK_ATOM 64
#define GRKAN_FUSED_LK_ES 4
#define GRKAN_FUSED_LK_CH 16
#endif
constexpr TileShape kShapesLongK[] = {{GRKAN_FUSED_LK_BN, GRKAN_FUSED_LK_ATOM, GRKAN_FUSED_LK_ES, GRKAN_FUSED_LK_CH, false}, {192, 64, 4, 16, false}, {256, 64, 2, 32, false},
                                      {192, 64, 2, 32, false}, {128, 64, 4, 16, false}, {128, 64, 2, 32, false},
                                      {96, 32, 1, 32, false},  {64, 64, 2, 32, false},  {64, 64, 1, 32, false},
                                      {32, 32, 1, 32, false}};
constexpr TileShape kShapesShortK[] = {{GRKAN_FUSED_SK_BN, 64, GRKAN_FUSED_SK_ES, GRKAN_FUSED_SK_CH, true},
                                       {128, 64, 4, 16, true},
                                       {64, 64, 2, 32, true}, {96, 32, 1, 32, false},
                                       {32, 32, 1, 32, false}};

bool pick_shape(int N, int dg, int K, TileShape* out) {
  const bool short_k = K <= 1024;
  const TileShape* list = short_k ? kShapesShortK : kShapesLongK;
  const int n = short_k ? 5 : 10;
  for (int i = 0; i < n; ++i) {
    const TileShape& t = list[i];
    const int cw = t.bn / t.es;
    if (N % t.bn == 0 && cw % t.ch == 0 && cw % 8 == 0 && dg % cw == 0) {
      *out = t;
      return true;
    }
  }
  return false;
}

int sms_of_device() {
  int dev = 0, v = 148;
  if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
  return v > 0 ? v : 148;
}

template <int BN, int ATOM, int ES, int CH, bool XS>
cudaError_t launch_t(const CUtensorMap& mdy, const CUtensorMap& mw, const CUtensorMap& mx, const void* x, void* dx,
                     const float* a, const float* b, float* part, const FusedGeom& geo, int64_t tiles,
                     cudaStream_t s) {
  constexpr int kStageBytes = kBM * kBK * 2 + kBK * BN * 2;
  constexpr int kXBytes = XS ? 2 * BN * kBM * 2 : 0;
  constexpr int kRing = kSmemBudget - kXBytes;
  constexpr int kSt = kRing / kStageBytes > 8 ? 8 : kRing / kStageBytes;
  static_assert(kSt >= 2, "operand ring needs two stages");
  constexpr size_t smem = static_cast<size_t>(kSt) * kStageBytes + kXBytes + 1024;
  auto kern = k_linear_bwd_fused<BN, ATOM, ES, CH, XS, kSt>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
  if (e != cudaSuccess) return e;
  const int64_t grid = tiles < sms_of_device() ? tiles : sms_of_device();
  kern<<<static_cast<unsigned>(grid), 64 + 128 * ES, smem, s>>>(mdy, mw, mx, static_cast<const __nv_bfloat16*>(x),
                                                                 static_cast<__nv_bfloat16*>(dx), a, b, part, geo);
  return cudaGetLastError();
}

// CTA-pair launch (cluster of 2, cta_group::2 MMA on 256-row tiles).
template <int BN, int ATOM, int ES, int CH>
cudaError_t launch_pair_t(const CUtensorMap& mdy, const CUtensorMap& mw, const CUtensorMap& mx, const void* x,
                          void* dx, const float* a, const float* b, float* part, const FusedGeom& geo,
                          cudaStream_t s) {
  constexpr int kStageBytes = kBM * kBK * 2 + kBK * BN;  // A + half of B
  constexpr int kSt = kSmemBudget / kStageBytes > 8 ? 8 : kSmemBudget / kStageBytes;
  constexpr size_t smem = static_cast<size_t>(kSt) * kStageBytes + 1024;
  auto kern = k_linear_bwd_fused<BN, ATOM, ES, CH, false, kSt, true>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
  if (e != cudaSuccess) return e;
  const int64_t pair_tiles = ((geo.M + 2 * kBM - 1) / (2 * kBM)) * geo.n_tiles_n;
  const int64_t pairs = pair_tiles < sms_of_device() / 2 ? pair_tiles : sms_of_device() / 2;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(static_cast<unsigned>(2 * pairs));
  cfg.blockDim = dim3(64 + 128 * ES);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, mdy, mw, mx, static_cast<const __nv_bfloat16*>(x),
                            static_cast<__nv_bfloat16*>(dx), a, b, part, geo);
}

bool pair_enabled() {
  const char* v = getenv("GRKAN_FUSED_PAIR");
  return v && v[0] == '1';
}

}  // namespace fused
}  // namespace grkan

extern "C" {

size_t grkan_linear_bwd_workspace_bytes(int64_t M, int32_t N, int32_t K, int32_t n_groups) {
  if (M < 0 || N < 1 || K < 1 || n_groups < 1 || N % n_groups) return 0;
  grkan::fused::TileShape t;
  if (!grkan::fused::pick_shape(N, N / n_groups, K, &t)) return 0;
  // 128-row tiles, rounded up to an even count: CTA pairs cover 256 rows and the
  // second CTA of a ragged last pair writes (zero) partials for its tile too
  const int64_t m_tiles = 2 * ((M + 2 * grkan::fused::kBM - 1) / (2 * grkan::fused::kBM));
  const int64_t ppg = m_tiles * ((N / n_groups) / (t.bn / t.es)) * 4;
  const size_t part = static_cast<size_t>(n_groups) * grkan::fused::kKC * ppg * sizeof(float);
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
  TileShape ts;
  if (!pick_shape(N, dg, K, &ts) || K % kBK || n_groups > kMaxGroups) {
    snprintf(msg, sizeof msg,
             "fused linear backward needs group width %% 32 == 0, K %% 64 == 0, groups <= %d (dg=%d, K=%d, groups=%d)",
             kMaxGroups, dg, K, n_groups);
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
  CUtensorMap mdy, mw, mx;
  if (!make_map(&mdy, dy, static_cast<uint64_t>(K), static_cast<uint64_t>(M), kBK, kBM, CU_TENSOR_MAP_SWIZZLE_128B) ||
      !make_map(&mw, w, static_cast<uint64_t>(N), static_cast<uint64_t>(K), ts.atom, kBK,
                ts.atom == 64 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B) ||
      !make_map(&mx, x, static_cast<uint64_t>(N), static_cast<uint64_t>(M), 64, kBM, CU_TENSOR_MAP_SWIZZLE_128B))
    return grkan::set_error(GRKAN_ERR_CUDA, "cuTensorMapEncodeTiled failed");
  FusedGeom geo;
  geo.M = M;
  geo.N = N;
  geo.K = K;
  geo.ng = n_groups;
  geo.dg = dg;
  geo.n_tiles_n = N / ts.bn;
  const int64_t m_tiles = (M + kBM - 1) / kBM;
  // CTA pairs write partials for an even number of 128-row tiles (the second
  // CTA of a ragged last pair contributes zeros); the workspace covers both
  const bool pair = !ts.xs && ts.bn == 192 && ts.es == 4 && ts.ch == 16 && pair_enabled();
  const int64_t m_slots = pair ? 2 * ((M + 2 * kBM - 1) / (2 * kBM)) : m_tiles;
  geo.ppg = static_cast<int32_t>(m_slots * (dg / (ts.bn / ts.es)) * 4);
  geo.one = 1.0f;
  const int64_t tiles = m_tiles * geo.n_tiles_n;
  float* part = reinterpret_cast<float*>(static_cast<char*>(ws) + 256);
  const float* fa = static_cast<const float*>(a);
  const float* fb = static_cast<const float*>(b);
#define GRKAN_FUSED_CASE(BN_, AT_, ES_, CH_, XS_)                                             \
  if (ts.bn == BN_ && ts.atom == AT_ && ts.es == ES_ && ts.ch == CH_ && ts.xs == XS_)           \
    e = launch_t<BN_, AT_, ES_, CH_, XS_>(mdy, mw, mx, x, dx, fa, fb, part, geo, tiles, s);    \
  else
  if (pair) {
    // each CTA of the pair loads 96 of the 192 W columns: 64B-swizzle, 32-column atoms
    CUtensorMap mw32;
    if (!make_map(&mw32, w, static_cast<uint64_t>(N), static_cast<uint64_t>(K), 32, kBK, CU_TENSOR_MAP_SWIZZLE_64B))
      return grkan::set_error(GRKAN_ERR_CUDA, "cuTensorMapEncodeTiled failed");
    e = launch_pair_t<192, 32, 4, 16>(mdy, mw32, mx, x, dx, fa, fb, part, geo, s);
  } else
  GRKAN_FUSED_CASE(256, 64, 4, 16, false)
  GRKAN_FUSED_CASE(192, 64, 4, 16, false)
  GRKAN_FUSED_CASE(256, 64, 2, 32, false)
  GRKAN_FUSED_CASE(192, 64, 2, 32, false)
  GRKAN_FUSED_CASE(128, 64, 4, 16, false)
  GRKAN_FUSED_CASE(128, 64, 2, 32, false)
  GRKAN_FUSED_CASE(96, 32, 1, 32, false)
  GRKAN_FUSED_CASE(64, 64, 2, 32, false)
  GRKAN_FUSED_CASE(64, 64, 1, 32, false)
  GRKAN_FUSED_CASE(128, 64, 4, 16, true)
#if GRKAN_FUSED_SK_BN != 128 || GRKAN_FUSED_SK_ES != 4 || GRKAN_FUSED_SK_CH != 16
  GRKAN_FUSED_CASE(GRKAN_FUSED_SK_BN, 64, GRKAN_FUSED_SK_ES, GRKAN_FUSED_SK_CH, true)
#endif
  GRKAN_FUSED_CASE(64, 64, 2, 32, true)
  e = launch_t<32, 32, 1, 32, false>(mdy, mw, mx, x, dx, fa, fb, part, geo, tiles, s);
#undef GRKAN_FUSED_CASE
  if (e != cudaSuccess) return grkan::set_error(GRKAN_ERR_CUDA, cudaGetErrorString(e));
  e = grkan::launch_reduce_f32(part, geo.ppg, 1, n_groups, 6, 4, da, db, st, s);
  if (e != cudaSuccess) return grkan::set_error(GRKAN_ERR_CUDA, cudaGetErrorString(e));
  return GRKAN_OK;
}

}  // extern "C"
