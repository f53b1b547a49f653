// grkan_p2p.cu -- K3 fused with the cross-GPU da||db exchange over peer memory.
//
// The data-parallel backward's one collective is the sum over ranks of the
// per-group coefficient gradients (m1 + n values per group, 320 B at the
// paper's shape).  Instead of K3 followed by an NCCL all-reduce, one kernel
// ("optional B200-native fusion"):
//   1. each CTA folds one (group, coefficient) column of this rank's K2
//      partials in fixed order (fp64), as K3 does;
//   2. thread 0 stores the fp64 value into slot [parity][rank][col] of EVERY
//      rank's exchange buffer (plain stores through CUDA-IPC-mapped peer
//      pointers: NVLink / NVSwitch on a B200 node), __threadfence_system(),
//      then bumps every rank's arrival counter with a system-scope atomic;
//   3. it waits (ld.acquire.sys, bounded: a peer that never arrives sets
//      DevStatus.peer_timeout after kPeerTimeoutNs instead of hanging) until
//      its own counter reaches epoch * world * CTAs, and folds the world slots
//      in rank order.  A fixed grid of <= 128 CTAs loops over the columns, so
//      any group count works without whole-grid co-residency.
// Every rank therefore computes the same fp64 sum in the same order: da/db are
// bitwise identical on all ranks, and no NCCL launch sits on the step.  The
// slot parity (epoch & 1) keeps a fast rank's next step from overwriting
// values a slow rank has not read yet: reaching step e + 2 requires every
// rank to have arrived in step e + 1, i.e. to have finished reading step e.
// Exchange buffer per rank: [u32 arrival counter, pad to 256 B][2][world][cols] fp64.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>
#include <cstring>

#include "../../include/grkan_b200.h"
#include "grkan_kernels.cuh"
#include "grkan_types.h"

namespace grkan {


namespace {

constexpr size_t kHeader = 256;

// Bounded wait for the peers' arrivals: a rank that failed before launching
// (validation error, exception) must not hang every other GPU forever.
// Default 20 s; GRKAN_P2P_TIMEOUT_MS overrides it (tests).
constexpr unsigned long long kPeerTimeoutNs = 20ull * 1000 * 1000 * 1000;
// Fixed CTA count (independent of the GPU): every rank expects the same number
// of arrivals, and 128 CTAs of 256 threads are co-resident on any B200 once
// K2 has drained, so the in-kernel wait cannot deadlock on residency.
constexpr int kP2pCtas = 128;

__device__ __forceinline__ unsigned long long globaltimer_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

template <typename A>
__global__ void __launch_bounds__(256)
    k_bwd_reduce_p2p(const A* __restrict__ part, int64_t n_tiles, int m1, int n, int ncol,
                     void* const* __restrict__ bufs, int rank, int world, unsigned long long epoch,
                     unsigned long long timeout_ns, A* __restrict__ da, A* __restrict__ db,
                     DevStatus* __restrict__ st) {
  pdl_wait();  // K2's partials are complete and visible after this
  const int kc = m1 + n;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int par = static_cast<int>(epoch & 1ull);
  __shared__ double red[8];
  // 1. this CTA's columns: fixed-order fp64 fold, stored into every rank's slot
  for (int col = blockIdx.x; col < ncol; col += gridDim.x) {
    const A* src = part + (int64_t)col * n_tiles;
    double s = 0.0;
    for (int64_t t = threadIdx.x; t < n_tiles; t += blockDim.x) s += static_cast<double>(src[t]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) red[warp] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
      double mine = 0.0;
      for (int w = 0; w < (int)((blockDim.x + 31) >> 5); ++w) mine += red[w];
      const size_t slot = (static_cast<size_t>(par) * world + rank) * ncol + col;
      for (int p = 0; p < world; ++p)
        reinterpret_cast<double*>(static_cast<char*>(bufs[p]) + kHeader)[slot] = mine;
    }
    __syncthreads();  // red[] is reused by the next column
  }
  if (threadIdx.x != 0) return;
  __threadfence_system();  // the slot values before the arrivals that announce them
  for (int p = 0; p < world; ++p) atomicAdd_system(static_cast<unsigned int*>(bufs[p]), 1u);
  // 2. wait for epoch * world * gridDim.x arrivals (bounded)
  const unsigned int target = static_cast<unsigned int>(epoch * static_cast<unsigned long long>(world) * gridDim.x);
  const unsigned int* my_flag = static_cast<const unsigned int*>(bufs[rank]);
  const unsigned long long t0 = globaltimer_ns();
  bool timed_out = false;
  unsigned int v;
  for (;;) {
    asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(my_flag) : "memory");
    if (static_cast<int>(v - target) >= 0) break;
    if (globaltimer_ns() - t0 > timeout_ns) {
      timed_out = true;
      break;
    }
    __nanosleep(200);
  }
  if (timed_out) st->peer_timeout = 1;
  // 3. fold the world values of this CTA's columns in rank order
  const double* slots =
      reinterpret_cast<const double*>(static_cast<const char*>(bufs[rank]) + kHeader) + static_cast<size_t>(par) * world * ncol;
  for (int col = blockIdx.x; col < ncol; col += gridDim.x) {
    double tot = 0.0;
    for (int r = 0; r < world; ++r) tot += __ldcv(slots + static_cast<size_t>(r) * ncol + col);
    const A out = static_cast<A>(tot);
    const int g = col / kc, k = col % kc;
    if (k < m1)
      da[(int64_t)g * m1 + k] = out;
    else
      db[(int64_t)g * n + (k - m1)] = out;
    if (nonfinite(out)) st->accum_overflow = 1;
  }
}

}  // namespace

cudaError_t launch_reduce_p2p(int dtype, const void* part, int64_t n_tiles, int ng, int m1, int n, void* const* bufs,
                              int rank, int world, unsigned long long epoch, void* da, void* db, DevStatus* st,
                              cudaStream_t stream) {
  cudaLaunchConfig_t cfg = {};
  const int ncol = ng * (m1 + n);
  unsigned long long timeout_ns = kPeerTimeoutNs;
  if (const char* env = std::getenv("GRKAN_P2P_TIMEOUT_MS")) timeout_ns = std::strtoull(env, nullptr, 10) * 1000000ull;
  cfg.gridDim = dim3(static_cast<unsigned>(ncol < kP2pCtas ? ncol : kP2pCtas));
  cfg.blockDim = dim3(256);
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  if (dtype == GRKAN_F64)
    return cudaLaunchKernelEx(&cfg, k_bwd_reduce_p2p<double>, static_cast<const double*>(part), n_tiles, m1, n, ncol, bufs,
                              rank, world, epoch, timeout_ns, static_cast<double*>(da), static_cast<double*>(db), st);
  return cudaLaunchKernelEx(&cfg, k_bwd_reduce_p2p<float>, static_cast<const float*>(part), n_tiles, m1, n, ncol, bufs,
                            rank, world, epoch, timeout_ns, static_cast<float*>(da), static_cast<float*>(db), st);
}

}  // namespace grkan

extern "C" {

size_t grkan_p2p_buffer_bytes(int32_t world, int32_t n_groups, int32_t m1, int32_t n) {
  if (world < 1 || n_groups < 1 || m1 < 1 || n < 0) return 0;
  return grkan::kHeader + 2ull * world * n_groups * (m1 + n) * sizeof(double);
}

int grkan_p2p_alloc(size_t bytes, void** out) {
  if (!out || bytes == 0) return grkan::set_error(GRKAN_ERR_INVALID, "p2p buffer: null output or zero size");
  cudaError_t e = cudaMalloc(out, bytes);  // its own allocation: an IPC handle maps exactly this range
  if (e == cudaSuccess) e = cudaMemset(*out, 0, bytes);
  if (e == cudaSuccess) e = cudaDeviceSynchronize();
  return e == cudaSuccess ? GRKAN_OK : grkan::set_error(GRKAN_ERR_CUDA, cudaGetErrorString(e));
}

int grkan_p2p_free(void* ptr) {
  cudaError_t e = cudaFree(ptr);
  return e == cudaSuccess ? GRKAN_OK : grkan::set_error(GRKAN_ERR_CUDA, cudaGetErrorString(e));
}

int grkan_ipc_get_handle(const void* dev_ptr, void* handle_out) {
  if (!dev_ptr || !handle_out) return grkan::set_error(GRKAN_ERR_INVALID, "ipc: null pointer");
  cudaIpcMemHandle_t h;
  cudaError_t e = cudaIpcGetMemHandle(&h, const_cast<void*>(dev_ptr));
  if (e != cudaSuccess) return grkan::set_error(GRKAN_ERR_CUDA, cudaGetErrorString(e));
  static_assert(sizeof(h) == GRKAN_IPC_HANDLE_BYTES, "IPC handle size");
  std::memcpy(handle_out, &h, sizeof(h));
  return GRKAN_OK;
}

int grkan_ipc_open_handle(const void* handle, void** dev_ptr_out) {
  if (!handle || !dev_ptr_out) return grkan::set_error(GRKAN_ERR_INVALID, "ipc: null pointer");
  cudaIpcMemHandle_t h;
  std::memcpy(&h, handle, sizeof(h));
  cudaError_t e = cudaIpcOpenMemHandle(dev_ptr_out, h, cudaIpcMemLazyEnablePeerAccess);
  return e == cudaSuccess ? GRKAN_OK : grkan::set_error(GRKAN_ERR_CUDA, cudaGetErrorString(e));
}

int grkan_ipc_close_handle(void* dev_ptr) {
  cudaError_t e = cudaIpcCloseMemHandle(dev_ptr);
  return e == cudaSuccess ? GRKAN_OK : grkan::set_error(GRKAN_ERR_CUDA, cudaGetErrorString(e));
}

}  // extern "C"
