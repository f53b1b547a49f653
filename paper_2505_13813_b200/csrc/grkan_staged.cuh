// grkan_staged.cuh -- TMA-bulk-staged K1 / K2 for the paper's degrees (5, 4).
//
// The register-direct kernels (grkan_kernels.cuh) keep their loads in
// registers, so bytes in flight per SM are bounded by register pressure and
// the backward stalls on L1TEX (ncu: ~55% of DRAM peak, 62% of stall cycles
// on long scoreboard).  Here a producer warp streams the CTA's rows into a
// shared-memory ring with cp.async.bulk (the sm_90+/sm_100a TMA bulk-copy
// engine: one instruction per contiguous row segment, completion counted in
// bytes on an mbarrier), and eight consumer warps compute out of shared memory.
// Bytes in flight per SM = stages x stage bytes x resident CTAs (~150 KB),
// independent of registers.
//
// Stage = RS rows of the group's columns, RS = floor(768 / V) so a stage is at
// most 768 16-byte vectors per tensor: exactly 3 per consumer thread when V
// divides 768 (KAT-S/B, fp32 and bf16).  Each consumer thread owns the same 3
// (row, vector) slots in every stage, so its smem and global offsets are fixed
// per thread.  dx / y leave straight from registers with 128-bit streaming
// stores (coalesced: consecutive threads write consecutive 16-byte vectors).
#pragma once

#include "grkan_kernels.cuh"

namespace grkan {

constexpr int kConsumerWarps = GRKAN_CONSUMER_WARPS;
constexpr int kStagedThreads = 32 * (kConsumerWarps + 1);  // + 1 producer warp
constexpr int kStageVecs = GRKAN_STAGE_VECS;               // per tensor per stage
constexpr int kVPT = kStageVecs / (32 * kConsumerWarps);   // 3 vectors per consumer thread
// The wide backward geometry: one CTA per SM with kWideWarps consumer warps
// and kVPT * 32 * kWideWarps-vector stages (make_plan chooses it per shape).
constexpr int kWideWarps = GRKAN_WIDE_WARPS;
template <int CW>
__host__ __device__ constexpr int staged_threads() { return 32 * (CW + 1); }
template <int CW>
__host__ __device__ constexpr int stage_vecs() { return kVPT * 32 * CW; }
constexpr int kMaxStages = 8;
// Backward CTAs per SM (register cap = 64K / (288 * MINB)).  Measured at
// KAT-B: 2 CTAs, 4-stage ring, unrolled vectors is best for both fp32 and
// bf16 (bf16 with 3 CTAs at 72 registers, 2-stage ring, serial vectors:
// 311 us vs 279 us -- the bf16 backward is FMA-pipe bound, not warp bound).
// kFullStage: branch-free body for full stages -- measured 260 -> 255 us for
// bf16 I/O but 308 -> 320 us for fp32 (KAT-B), so bf16 only.
template <typename T, int CW = kConsumerWarps>
struct BwdCfg {
  static constexpr int kMinBlocks = CW == kConsumerWarps ? GRKAN_BWD_CTAS : 1;
  static constexpr bool kSerialVectors = false;
  static constexpr bool kFullStage = GRKAN_FULL_STAGE && std::is_same<T, __nv_bfloat16>::value;
};
constexpr int kFwdCtasPerSm = GRKAN_FWD_CTAS;
// Forward geometry (separately tunable: one tensor in, little math per byte).
constexpr int kFwdConsumerWarps = GRKAN_FWD_CONSUMER_WARPS;
constexpr int kFwdThreads = 32 * (kFwdConsumerWarps + 1);
constexpr int kFwdVPT = GRKAN_FWD_STAGE_VECS / (32 * kFwdConsumerWarps);

// ---- PTX helpers: shared addresses, mbarriers, bulk copies ------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
// With a suspend-time hint the waiting warp is parked until the phase flips (or
// the hint expires) instead of re-issuing try_wait: a spinning producer or an
// early consumer otherwise takes issue slots from the consumer warps that share
// its scheduler (ncu: ~7% of the bf16 backward's instructions were retry loops).
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
#if GRKAN_WAIT_HINT_NS > 0
  asm volatile(
      "{\n"
      "  .reg .pred p;\n"
      "WAIT_%=:\n"
      "  mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n"
      "  @!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity), "n"(GRKAN_WAIT_HINT_NS)
      : "memory");
#else
  asm volatile(
      "{\n"
      "  .reg .pred p;\n"
      "WAIT_%=:\n"
      "  mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "  @!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
#endif
}
// global -> shared bulk copy (TMA engine), completion counted on `bar`;
// L2 evict-first: every byte is read exactly once.
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar,
                                         uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}
// 3-D tiled tensor copy (TMA): box at (c0, c1 = column chunk, c2 = row) of a
// [rows, d / ci, ci] map.
__device__ __forceinline__ void tma3d_g2s(void* dst, const CUtensorMap* map, int c0, int c1, int c2, uint64_t* bar,
                                          uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1, {%2, %3, %4}], [%5], %6;" ::"r"(
          smem_u32(dst)),
      "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}
__device__ __forceinline__ uint64_t evict_first_policy() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}

// ---- raw 16-byte vector <-> W math values ------------------------------------
template <typename T>
struct Raw16;

template <>
struct Raw16<float> {
  static constexpr int W = 4;
  static __device__ __forceinline__ void unpack(const uint4& r, float (&v)[4]) {
    v[0] = __uint_as_float(r.x); v[1] = __uint_as_float(r.y);
    v[2] = __uint_as_float(r.z); v[3] = __uint_as_float(r.w);
  }
  static __device__ __forceinline__ uint4 pack(const float (&v)[4]) {
    return make_uint4(__float_as_uint(v[0]), __float_as_uint(v[1]), __float_as_uint(v[2]),
                      __float_as_uint(v[3]));
  }
};

template <>
struct Raw16<__nv_bfloat16> {
  static constexpr int W = 8;
  static __device__ __forceinline__ void unpack(const uint4& r, float (&v)[8]) {
    const uint32_t w[4] = {r.x, r.y, r.z, r.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      v[2 * i] = __uint_as_float(__byte_perm(w[i], 0u, 0x1044));  // w << 16 on the ALU pipe (PRMT)
      v[2 * i + 1] = __uint_as_float(w[i] & 0xffff0000u);
    }
  }
  static __device__ __forceinline__ uint4 pack(const float (&v)[8]) {
    uint32_t w[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const __nv_bfloat162 h = __floats2bfloat162_rn(v[2 * i], v[2 * i + 1]);
      w[i] = *reinterpret_cast<const uint32_t*>(&h);
    }
    return make_uint4(w[0], w[1], w[2], w[3]);
  }
};

template <>
struct Raw16<double> {
  static constexpr int W = 2;
  static __device__ __forceinline__ void unpack(const uint4& r, double (&v)[2]) {
    v[0] = __hiloint2double(static_cast<int>(r.y), static_cast<int>(r.x));
    v[1] = __hiloint2double(static_cast<int>(r.w), static_cast<int>(r.z));
  }
  static __device__ __forceinline__ uint4 pack(const double (&v)[2]) {
    return make_uint4(static_cast<uint32_t>(__double2loint(v[0])), static_cast<uint32_t>(__double2hiint(v[0])),
                      static_cast<uint32_t>(__double2loint(v[1])), static_cast<uint32_t>(__double2hiint(v[1])));
  }
};

// Accumulator flush: every geo.flush stages each lane folds its register
// accumulators into a private fp32 slot in shared memory ([k][thread], bank-
// conflict free) and restarts them, so per-lane fp32 chains stay short
// (<= 6 * flush terms) at ~40 instructions per flush.  SH = 1: one slot per
// lane pair (the pair's totals meet by one shuffle first) -- half the shared
// memory, for the bf16 table kernel.
template <int SH, int CW = kConsumerWarps>
__device__ __forceinline__ int acc_slot(int k) {
  return k * ((32 * CW) >> SH) + (static_cast<int>(threadIdx.x) >> SH);
}

template <typename A, int KC, bool PK, int SH = 0, int CW = kConsumerWarps>
__device__ __forceinline__ void lane_flush(A (&acc)[KC], float2 (&acc2)[KC], A* __restrict__ sacc) {
#pragma unroll
  for (int k = 0; k < KC; ++k) {
    A v;
    if constexpr (PK) {
      v = acc2[k].x + acc2[k].y;
      acc2[k] = make_float2(0.f, 0.f);
    } else {
      v = acc[k];
      acc[k] = A(0);
    }
    if constexpr (SH == 1) {
      v += __shfl_xor_sync(0xffffffffu, v, 1);
      if ((threadIdx.x & 1) == 0) sacc[acc_slot<SH, CW>(k)] += v;
    } else {
      sacc[acc_slot<SH, CW>(k)] += v;
    }
  }
}

// This warp's lanes' slot values for coefficient k (SH = 1: 16 slots, lanes >= 16 add 0).
template <typename A, int SH, int CW = kConsumerWarps>
__device__ __forceinline__ A warp_slot_value(const A* __restrict__ sacc, int k) {
  const int lane = threadIdx.x & 31;
  if constexpr (SH == 1)
    return lane < 16 ? sacc[k * (16 * CW) + (threadIdx.x >> 5) * 16 + lane] : A(0);
  else
    return sacc[acc_slot<0, CW>(k)];
}

// End of CTA: each consumer warp folds its lanes' shared-memory totals with a
// fixed butterfly into partial slot (CTA j, warp w):
// part[((g * KC + k) * pg + j) * CW + w]  ->  n_tiles = pg * CW per (group, coefficient).
template <typename A, int KC, int SH = 0, int CW = kConsumerWarps>
__device__ __forceinline__ void warp_store(const A* __restrict__ sacc, A* __restrict__ part, int g, int64_t j,
                                           int warp, const Geom& geo) {
  const int lane = threadIdx.x & 31;
  const int64_t n_tiles = (int64_t)geo.pg * CW;
#pragma unroll
  for (int k = 0; k < KC; ++k) {
    A v = warp_slot_value<A, SH, CW>(sacc, k);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (lane == 0) part[((int64_t)g * KC + k) * n_tiles + j * CW + warp] = v;
  }
}

// Persistent, statically balanced partition: CTA (g, j) of pg per group owns
// stage units [j*nsu/pg, (j+1)*nsu/pg) of group g -- every CTA gets the same
// number of RS-row stages to within one, so there is no tail wave.  Linear
// id = j * ng + g: resident CTAs of all groups stream the same row band.
__device__ __forceinline__ void staged_range(const Geom& geo, int& g, int64_t& j, int64_t& row0, int& nr) {
  const int64_t bid = blockIdx.x;
  g = static_cast<int>(bid % geo.ng);
  j = bid / geo.ng;
  int64_t s0, s1;
  if (geo.w1 == 64) {
    s0 = (j * geo.nsu) / geo.pg;
    s1 = ((j + 1) * geo.nsu) / geo.pg;
  } else {  // weighted: CTAs j < J of this group are in the first wave (bid < wave)
    const int64_t J = geo.wave > g ? (geo.wave - g + geo.ng - 1) / geo.ng : 0;
    auto cum = [&](int64_t jj) {
      const int64_t f = jj < J ? jj : J;
      return f * geo.w1 + (jj - f) * 64;
    };
    const int64_t tot = cum(geo.pg);
    s0 = cum(j) * geo.nsu / tot;
    s1 = cum(j + 1) * geo.nsu / tot;
  }
  row0 = s0 * geo.RU;
  const int64_t r1 = s1 * geo.RU < geo.rows ? s1 * geo.RU : geo.rows;
  nr = static_cast<int>(r1 - row0);
}

// Deterministic mode: the CTA's lanes have just flushed one RB-row block into
// sacc.  Fixed butterfly per warp -> red[buf][warp], consumer-warp barrier,
// warp 0 folds the warps in order -> part[(blk * ng + g) * KC + k]; sacc is
// re-zeroed for the next block.  The partial depends only on the block's
// data (the thread -> element map is fixed per stage), never on which CTA
// processed it: bitwise identical for any row sharding aligned to RB.
template <typename A, int KC, int SH = 0>
__device__ __forceinline__ void block_store(A* __restrict__ sacc, A (&red)[2][kConsumerWarps][KC], int buf,
                                            A* __restrict__ part, int g, int64_t blk, int warp,
                                            const Geom& geo) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int k = 0; k < KC; ++k) {
    A v = warp_slot_value<A, SH>(sacc, k);
    __syncwarp();
    if (SH == 0 || lane < 16) sacc[SH == 1 ? k * (16 * kConsumerWarps) + warp * 16 + lane : acc_slot<0>(k)] = A(0);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (lane == 0) red[buf][warp][k] = v;
  }
  asm volatile("bar.sync 1, %0;" ::"r"(32 * kConsumerWarps) : "memory");
  if (warp == 0) {
#pragma unroll
    for (int k = 0; k < KC; ++k) {
      A v = lane < kConsumerWarps ? red[buf][lane][k] : A(0);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
      if (lane == 0) part[(blk * geo.ng + g) * KC + k] = v;
    }
  }
}

// ---------------------------------------------------------------------------
// Producer: lane 0 of the last warp fills the ring, one bulk copy per row
// segment per tensor -- or, with geo.tma_rows > 0 (short row segments, where
// per-row copies cost more than they move), RS / tma_rows tensor-map boxes
// per tensor (full boxes: rows past the tensor end arrive zero-filled, rows past
// the CTA's run are read and ignored).  `nt` tensors (1 forward, 2 backward).
// ---------------------------------------------------------------------------
template <typename T, int NT>
__device__ __forceinline__ void produce(const T* const (&src)[NT], T* const (&ring)[NT], const Geom& geo,
                                        int64_t row0, int nr, int stages, uint64_t* full,
                                        uint64_t* empty, int g, const CUtensorMap* const (&maps)[NT]) {
  const uint64_t policy = evict_first_policy();
  const int RS = geo.RS;
  const int nst = (nr + RS - 1) / RS;
  const uint32_t seg = static_cast<uint32_t>(geo.dg * sizeof(T));
  const int tr = geo.tma_rows;
  int slot = 0;
  uint32_t phase = 0;  // parity of the current pass over the ring
  for (int s = 0; s < nst; ++s) {
    if (s >= stages) mbar_wait(&empty[slot], phase ^ 1);  // released by the previous pass
    if (tr > 0) {
      mbar_arrive_expect_tx(&full[slot], static_cast<uint32_t>(RS) * seg * NT);
      for (int r = 0; r < RS; r += tr) {
#pragma unroll
        for (int t = 0; t < NT; ++t)
          tma3d_g2s(ring[t] + ((size_t)slot * RS + r) * geo.dg, maps[t], 0, g * (geo.dg / geo.tma_ci),
                    static_cast<int>(row0 + (int64_t)s * RS + r), &full[slot], policy);
      }
    } else {
      const int rows_here = min(RS, nr - s * RS);
      mbar_arrive_expect_tx(&full[slot], static_cast<uint32_t>(rows_here) * seg * NT);
      for (int r = 0; r < rows_here; ++r) {
        const int64_t goff = (row0 + s * RS + r) * geo.d + (int64_t)g * geo.dg;
#pragma unroll
        for (int t = 0; t < NT; ++t)
          bulk_g2s(ring[t] + ((size_t)slot * RS + r) * geo.dg, src[t] + goff, seg, &full[slot], policy);
      }
    }
    if (++slot == stages) {
      slot = 0;
      phase ^= 1;
    }
  }
}

// ---------------------------------------------------------------------------
// K2 staged: backward main pass, degrees (5, 4).
// FWD: the fused forward + backward step -- the forward value y = P/Q of every
// element falls out of the backward's own P and 1/Q (pq), so y is written beside
// dx from the same shared-memory x (x read once for both passes).
// ---------------------------------------------------------------------------
// LUT (bf16 I/O, FAST): the x-only factors {1/Q, -sign(A) P/Q^2} of every x in
// a 16-exponent window come from a per-CTA shared-memory table built at start
// (RationalX2::lut_entry); elements outside the window evaluate the same
// function inline, so results do not depend on the window.  Table: kLutSlots
// float2 entries {1/Q, -sign(A)P/Q^2} (GRKAN_LUT_PAIRED; 0: two float arrays),
// slot = t | sign << 11 with t = bf16 magnitude bits - window base
// (0 <= t < 2048).  One 8-byte load per element instead of two 4-byte ones
// (random banks: ~6.1 vs 2 x 3.5 wavefronts per warp in a half-warp bank
// model; measured 0.4% faster at KAT-B and KAT-S).
constexpr int kLutSlots = 2 * kLutSignStride;

// The two bf16 values of one 32-bit word at once: d = w + C puts each half at
// sign * 0x8000 + 0x4000 + (magnitude - base), so a half is inside the window
// iff its bits 11-14 read 1000b, and its slot is its low 11 bits plus its sign
// moved to bit 11 (carries between the halves only occur for |x| >= 2^115 or
// non-finite x, which are outside the window and make the check fail).
// Returns the packed slots (lo | hi << 16); `bad` collects window misses.
__device__ __forceinline__ uint32_t lut_slots2(uint32_t w, uint32_t c, uint32_t& bad) {
  const uint32_t d = w + c;
  bad |= (d ^ 0x40004000u) & 0x78007800u;
  return (d & 0x07ff07ffu) | ((d & 0x80008000u) >> 4);
}

template <typename T, bool EXACT, bool CHECK, bool DET, bool INSTR = false, bool FWD = false, bool LUT = false,
          int M1 = 6, int N = 4, int CW = kConsumerWarps>
__global__ void __launch_bounds__(staged_threads<CW>(), BwdCfg<T, CW>::kMinBlocks)
    k_bwd_staged(const T* __restrict__ x, const T* __restrict__ dy, T* __restrict__ dx, T* __restrict__ y,
                 const typename VecIO<T, 1>::A* __restrict__ ca,
                 const typename VecIO<T, 1>::A* __restrict__ cb,
                 typename VecIO<T, 1>::A* __restrict__ part, Geom geo, int stages,
                 DevStatus* __restrict__ st, const __grid_constant__ CUtensorMap tmx,
                 const __grid_constant__ CUtensorMap tmu) {
  using A = typename VecIO<T, 1>::A;
  using RW = Raw16<T>;
  constexpr int W = RW::W;
  constexpr bool PK = std::is_same<A, float>::value;
  constexpr int KC = M1 + N;
  static_assert(!LUT || (std::is_same<T, __nv_bfloat16>::value && !EXACT && !INSTR && !FWD && M1 == 6 && N == 4),
                "the x-factor table is the bf16 FAST backward at the paper's degrees only");
  static_assert(CW == kConsumerWarps || !DET, "deterministic partials use the default geometry on every rank");
  extern __shared__ __align__(128) unsigned char smem_raw[];
  __shared__ uint64_t full[kMaxStages], empty[kMaxStages];
  __shared__ A red[DET ? 2 : 1][DET ? CW : 1][DET ? KC : 1];
  pdl_launch_dependents();

  int g;
  int64_t tile, row0;
  int nr;
  if (threadIdx.x == 0) GRKAN_STAMP(0);
  if (geo.zst && blockIdx.x == 0 && threadIdx.x == 0) *reinterpret_cast<int4*>(st) = make_int4(0, 0, 0, 0);
  staged_range(geo, g, tile, row0, nr);
  if (DET) tile = row0 / geo.RU;  // first RB-row block of this CTA
  const size_t ring_elems = (size_t)stages * geo.RS * geo.dg;
  T* const sx = reinterpret_cast<T*>(smem_raw);
  T* const su = sx + ring_elems;
  // per-consumer-lane accumulator totals, [KC][256], after the two rings
  A* const sacc = reinterpret_cast<A*>(su + ring_elems);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], CW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (threadIdx.x < 32 * CW) {
#pragma unroll
    for (int k = 0; k < KC; ++k)
      if (!LUT || (threadIdx.x & 1) == 0) sacc[acc_slot<LUT ? 1 : 0, CW>(k)] = 0;
  }
  __syncthreads();

  A acc[KC];
#pragma unroll
  for (int k = 0; k < KC; ++k) acc[k] = A(0);
  Checker<A> chk;
  Tally tl;

  if (warp == CW) {
    if (lane == 0) {
      const T* const src[2] = {x, dy};
      T* const ring[2] = {sx, su};
      const CUtensorMap* const maps[2] = {&tmx, &tmu};
      if (!GRKAN_PROBE_NOMEM) produce<T, 2>(src, ring, geo, row0, nr, stages, full, empty, g, maps);
    }
  } else {
    RationalX2<EXACT, M1, N> rp;
    Rational<A, EXACT, M1, N, true> rs;
    float2 acc2[KC];
    if constexpr (PK) {
      rp.load(reinterpret_cast<const float*>(ca), reinterpret_cast<const float*>(cb), g, geo.one);
#pragma unroll
      for (int k = 0; k < KC; ++k) acc2[k] = make_float2(0.f, 0.f);
    } else {
      rs.load(ca, cb, g, M1, N);
    }
    // the x-factor table after the accumulator totals: built once by the
    // consumer warps (the producer is already streaming the first stages)
    float* const tiq = reinterpret_cast<float*>(sacc + KC * ((32 * CW) >> (LUT ? 1 : 0)));
    const uint32_t lut_base = static_cast<uint32_t>(geo.lut_e0) << 7;
    const uint32_t lut_c = geo.lut_c;  // a kernel parameter: one IADD3 per pair, not an IMAD
    if constexpr (LUT) {
      for (int i = threadIdx.x; i < kLutSlots; i += 32 * CW) {
        const uint32_t t = i & (kLutSignStride - 1), neg = static_cast<uint32_t>(i) >> 11;
        const float2 e = rp.lut_entry(__uint_as_float(((lut_base + t) | (neg << 15)) << 16));
        if constexpr (GRKAN_LUT_PAIRED) {
          reinterpret_cast<float2*>(tiq)[i] = e;
        } else {
          tiq[i] = e.x;
          tiq[kLutSlots + i] = e.y;
        }
      }
      asm volatile("bar.sync 1, %0;" ::"r"(32 * CW) : "memory");
    }
    // this thread's fixed (row, vector) slots in every stage
    int sr[kVPT], so[kVPT];
    T* gp[kVPT];  // running global pointers: advance by RS rows per stage
    const int svecs = geo.RS * geo.V;
#pragma unroll
    for (int j = 0; j < kVPT; ++j) {
      const int k = threadIdx.x + j * 32 * CW;
      const int r = k / geo.V, c = (k - (k / geo.V) * geo.V) * W;
      sr[j] = k < svecs ? r : 0x7fffffff;  // never valid outside the stage
      so[j] = r * geo.dg + c;
      gp[j] = dx + (row0 + r) * geo.d + (int64_t)g * geo.dg + c;
    }
    const int64_t gstep = (int64_t)geo.RS * geo.d;
    const bool full_slots = svecs == stage_vecs<CW>();  // every thread slot maps into the stage
    const int slot_elems = geo.RS * geo.dg;
    const int nst = (nr + geo.RS - 1) / geo.RS;
    int slot = 0, since_flush = 0;
    uint32_t phase = 0;
    for (int s = 0; s < nst; ++s) {
      if (!GRKAN_PROBE_NOMEM) mbar_wait(&full[slot], phase);
      if (GRKAN_PROBE_TIMES && s == 0 && threadIdx.x == 0) GRKAN_STAMP(1);
      const int rows_here = min(geo.RS, nr - s * geo.RS);
      const T* xs = sx + slot * slot_elems;
      const T* us = su + slot * slot_elems;
      auto vec = [&](int j) {
        A vx[W], vu[W], o[W], yo[W];
        const uint4 rx = *reinterpret_cast<const uint4*>(xs + so[j]);
        RW::unpack(rx, vx);
        RW::unpack(*reinterpret_cast<const uint4*>(us + so[j]), vu);
        if constexpr (LUT) {
          const uint32_t wx[4] = {rx.x, rx.y, rx.z, rx.w};
          uint32_t sl[4], bad = 0;
#pragma unroll
          for (int i = 0; i < 4; ++i) sl[i] = lut_slots2(wx[i], lut_c, bad);
          float iq[W], wf[W];
          if (__builtin_expect(bad == 0, 1)) {
#pragma unroll
            for (int i = 0; i < 4; ++i) {
              const uint32_t s0 = sl[i] & 0xffffu, s1 = sl[i] >> 16;
              if constexpr (GRKAN_LUT_PAIRED) {  // one 8-byte load per element
                const float2 e0 = reinterpret_cast<const float2*>(tiq)[s0];
                const float2 e1 = reinterpret_cast<const float2*>(tiq)[s1];
                iq[2 * i] = e0.x;
                wf[2 * i] = e0.y;
                iq[2 * i + 1] = e1.x;
                wf[2 * i + 1] = e1.y;
              } else {
                iq[2 * i] = tiq[s0];
                iq[2 * i + 1] = tiq[s1];
                wf[2 * i] = tiq[kLutSlots + s0];
                wf[2 * i + 1] = tiq[kLutSlots + s1];
              }
            }
          } else {  // an x outside the window: that element evaluates the table function itself
#pragma unroll
            for (int e = 0; e < W; ++e) {
              const uint32_t h = (e & 1) ? (wx[e >> 1] >> 16) : (wx[e >> 1] & 0xffffu);
              const uint32_t t = (h & 0x7fffu) - lut_base;
              float2 en;
              if (t < static_cast<uint32_t>(kLutSignStride)) {
                const uint32_t sidx = t | ((h >> 4) & 0x800u);
                en = GRKAN_LUT_PAIRED ? reinterpret_cast<const float2*>(tiq)[sidx]
                                      : make_float2(tiq[sidx], tiq[kLutSlots + sidx]);
              } else {
                en = rp.lut_entry(vx[e]);
              }
              iq[e] = en.x;
              wf[e] = en.y;
            }
          }
#pragma unroll
          for (int p = 0; p < W / 2; ++p) {
            const float2 r = rp.grad_lut(make_float2(vx[2 * p], vx[2 * p + 1]), make_float2(vu[2 * p], vu[2 * p + 1]),
                                         make_float2(iq[2 * p], iq[2 * p + 1]), make_float2(wf[2 * p], wf[2 * p + 1]),
                                         acc2);
            o[2 * p] = r.x;
            o[2 * p + 1] = r.y;
          }
        } else if constexpr (PK) {
          if constexpr (FWD)
            rp.template grad_n<W / 2, kGuard<T>, float2, true>(vx, vu, o, acc2, &yo);
          else
            rp.template grad_n<W / 2, kGuard<T>>(vx, vu, o, acc2);
        } else {
#pragma unroll
          for (int e = 0; e < W; ++e) {
            o[e] = rs.grad(vx[e], vu[e], acc);
            if constexpr (FWD) yo[e] = rs.value(vx[e]);
          }
        }
        if constexpr (FWD) __stcs(reinterpret_cast<uint4*>(y + (gp[j] - dx)), RW::pack(yo));
        if constexpr (CHECK) {
#pragma unroll
          for (int e = 0; e < W; ++e) {
            chk.add(vx[e]);
            chk.add(vu[e]);
          }
        }
        __stcs(reinterpret_cast<uint4*>(gp[j]), RW::pack(o));
        if constexpr (INSTR) {
          visit<W>(geo, gp[j] - dx);
          tl.r += 2 * W;  // x, dy (staged through shared memory by the bulk copies)
          tl.w += W;      // dx
        }
      };
      if (BwdCfg<T, CW>::kFullStage && full_slots && rows_here == geo.RS) {
        // every slot of a full stage is valid: one branch-free block the
        // scheduler can interleave across the thread's kVPT vectors
#pragma unroll
        for (int j = 0; j < kVPT; ++j) vec(j);
      } else {
#pragma unroll(BwdCfg<T, CW>::kSerialVectors ? 1 : kVPT)
        for (int j = 0; j < kVPT; ++j)
          if (sr[j] < rows_here) vec(j);
      }
#pragma unroll
      for (int j = 0; j < kVPT; ++j) gp[j] += gstep;
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[slot]);  // this warp is done with the slot
      // Short per-lane fp32 chains keep the da/db rounding error near the fp32
      // term-evaluation floor (see lane_flush).
      const bool block_end = DET && ((s + 1) % geo.spb == 0 || s + 1 == nst);
      if (++since_flush == geo.flush || s + 1 == nst || block_end) {
        lane_flush<A, KC, PK, LUT ? 1 : 0, CW>(acc, acc2, sacc);
        since_flush = 0;
      }
      if constexpr (DET) {
        if (block_end) {
          __syncwarp();
          block_store<A, KC, LUT ? 1 : 0>(sacc, red, (s / geo.spb) & 1, part, g, tile + s / geo.spb, warp, geo);
        }
      }
      if (++slot == stages) {
        slot = 0;
        phase ^= 1;
      }
    }
    if constexpr (!DET) {
      __syncwarp();
      warp_store<A, KC, LUT ? 1 : 0, CW>(sacc, part, g, tile, warp, geo);
    }
#if GRKAN_PROBE_TIMES
    if (lane == 0) {
      if (warp == 0) {  // slot 2: the SM this CTA ran on (<< 32) | its row count
        unsigned smid;
        asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
        g_probe_t[4 * (blockIdx.x % kProbeCtas) + 2] = (static_cast<unsigned long long>(smid) << 32) | nr;
      }
      GRKAN_STAMP_MAX(3);
    }
#endif
    if constexpr (INSTR) {
      if (lane == 0) {
        if (warp == 0) tl.r += KC;  // the CTA's coefficient row (registers afterwards)
        tl.w += KC;                 // this warp's one partial per coefficient
      }
      tl.flush(geo);
    }
  }
  if (CHECK && chk.bad()) st->nonfinite_input = 1;
}

// ---------------------------------------------------------------------------
// K1 staged: forward, degrees (5, 4).
// ---------------------------------------------------------------------------
template <typename T, bool EXACT, bool CHECK, int M1 = 6, int N = 4>
__global__ void __launch_bounds__(kFwdThreads, kFwdCtasPerSm)
    k_fwd_staged(const T* __restrict__ x, T* __restrict__ y, const typename VecIO<T, 1>::A* __restrict__ ca,
                 const typename VecIO<T, 1>::A* __restrict__ cb, Geom geo, int stages,
                 DevStatus* __restrict__ st, const __grid_constant__ CUtensorMap tmx) {
  using A = typename VecIO<T, 1>::A;
  using RW = Raw16<T>;
  constexpr int W = RW::W;
  constexpr bool PK = std::is_same<A, float>::value;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  __shared__ uint64_t full[kMaxStages], empty[kMaxStages];

  int g;
  int64_t tile, row0;
  int nr;
  staged_range(geo, g, tile, row0, nr);
  T* const sx = reinterpret_cast<T*>(smem_raw);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kFwdConsumerWarps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (warp == kFwdConsumerWarps) {
    if (lane == 0) {
      const T* const src[1] = {x};
      T* const ring[1] = {sx};
      const CUtensorMap* const maps[1] = {&tmx};
      produce<T, 1>(src, ring, geo, row0, nr, stages, full, empty, g, maps);
    }
    return;
  }
  RationalX2<EXACT, M1, N> rp;
  Rational<A, EXACT, M1, N, true> rs;
  if constexpr (PK)
    rp.load(reinterpret_cast<const float*>(ca), reinterpret_cast<const float*>(cb), g, geo.one);
  else
    rs.load(ca, cb, g, M1, N);
  int sr[kFwdVPT], soff[kFwdVPT];
  int64_t goff[kFwdVPT];
  const int svecs = geo.RS * geo.V;
#pragma unroll
  for (int j = 0; j < kFwdVPT; ++j) {
    const int k = threadIdx.x + j * 32 * kFwdConsumerWarps;
    const int r = k / geo.V, c = k - (k / geo.V) * geo.V;
    sr[j] = k < svecs ? r : 0x7fffffff;
    soff[j] = r * geo.dg + c * W;
    goff[j] = (int64_t)r * geo.d + (int64_t)g * geo.dg + c * W;
  }
  Checker<A> chk;
  const int nst = (nr + geo.RS - 1) / geo.RS;
  int slot = 0;
  uint32_t phase = 0;
  for (int s = 0; s < nst; ++s) {
    mbar_wait(&full[slot], phase);
    const int rows_here = min(geo.RS, nr - s * geo.RS);
    const T* xs = sx + (size_t)slot * geo.RS * geo.dg;
    T* ys = y + (row0 + (int64_t)s * geo.RS) * geo.d;
    uint4 rx[kFwdVPT];
#pragma unroll
    for (int j = 0; j < kFwdVPT; ++j)
      if (sr[j] < rows_here) rx[j] = *reinterpret_cast<const uint4*>(xs + soff[j]);
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[slot]);
#pragma unroll
    for (int j = 0; j < kFwdVPT; ++j) {
      if (sr[j] < rows_here) {
        A v[W], o[W];
        RW::unpack(rx[j], v);
        if constexpr (PK) {
#pragma unroll
          for (int e = 0; e < W; e += 2) {
            const float2 r2 = rp.value(make_float2(v[e], v[e + 1]));
            o[e] = r2.x;
            o[e + 1] = r2.y;
          }
        } else {
#pragma unroll
          for (int e = 0; e < W; ++e) o[e] = rs.value(v[e]);
        }
        if constexpr (CHECK) {
#pragma unroll
          for (int e = 0; e < W; ++e) chk.add(v[e]);
        }
        __stcs(reinterpret_cast<uint4*>(ys + goff[j]), RW::pack(o));
      }
    }
    if (++slot == stages) {
      slot = 0;
      phase ^= 1;
    }
  }
  if (CHECK && chk.bad()) st->nonfinite_input = 1;
}

}  // namespace grkan
