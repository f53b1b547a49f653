// Microbenchmark: achievable HBM bandwidth for the read:write mixes of the
// GR-KAN path on B200, with the kernels' own access style (16-byte vectors,
// evict-first, grid-stride over 148 x k CTAs), at KAT-B tensor sizes
// (620 MB per fp32 tensor, each far above the 126 MB L2: no flush needed).
//
//   copy  1 read : 1 write   (K1 forward:  x -> y)
//   add   2 reads: 1 write   (K2 backward: x, dy -> dx)
//   read  1 read : 0 writes  (checksum)
//   write 0 reads: 1 write   (fill)
//   memcpy                   cudaMemcpyAsync D2D (the MEASURED_PEAKS style copy)
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o hbm_mix hbm_mix.cu && ./hbm_mix
// Prints one JSON line per mode: algorithmic bytes / time (best of reps and mean).
#include <cuda_runtime.h>

#include <cstdio>
#include <vector>
#include <algorithm>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("%s\n", cudaGetErrorString(e_)); return 1; } } while (0)

// streaming (evict-first) 16-byte accesses, as the kernels use (LDG/STG .EF)
__device__ __forceinline__ uint4 ld_ef(const uint4* p) { return __ldcs(p); }
__device__ __forceinline__ void st_ef(uint4* p, uint4 v) { __stcs(p, v); }

template <int MODE, int U>  // 0 copy, 1 add, 2 read, 3 write
__global__ void __launch_bounds__(256) k(const uint4* __restrict__ a, const uint4* __restrict__ b,
                                        uint4* __restrict__ c, size_t n, unsigned* sink) {
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  unsigned acc = 0;
  size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (; i + (U - 1) * stride < n; i += U * stride) {
    uint4 va[U], vb[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (MODE != 3) va[u] = ld_ef(a + i + u * stride);
      if (MODE == 1) vb[u] = ld_ef(b + i + u * stride);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      uint4 v = MODE == 3 ? make_uint4((unsigned)i, 1, 2, 3) : va[u];
      if (MODE == 1) { v.x += vb[u].x; v.y += vb[u].y; v.z += vb[u].z; v.w += vb[u].w; }
      if (MODE == 2) acc ^= v.x ^ v.y ^ v.z ^ v.w;
      else st_ef(c + i + u * stride, v);
    }
  }
  for (; i < n; i += stride) {
    uint4 v = MODE == 3 ? make_uint4((unsigned)i, 1, 2, 3) : ld_ef(a + i);
    if (MODE == 1) { const uint4 w = ld_ef(b + i); v.x += w.x; v.y += w.y; v.z += w.z; v.w += w.w; }
    if (MODE == 2) acc ^= v.x ^ v.y ^ v.z ^ v.w;
    else st_ef(c + i, v);
  }
  if (MODE == 2 && acc == 0x12345678u) *sink = acc;
}

// add over group column segments, the K2 partition: CTA b owns group b % 8
// (a 1536 B segment of every 12 KB row) over a contiguous run of rows.
template <int U>
__global__ void __launch_bounds__(256) k_seg(const uint4* __restrict__ a, const uint4* __restrict__ b,
                                            uint4* __restrict__ c, size_t rows, int vrow, int vseg, int ng) {
  const int g = blockIdx.x % ng;
  const size_t per = gridDim.x / ng;
  const size_t ci = blockIdx.x / ng;
  const size_t r0 = rows * ci / per, r1 = rows * (ci + 1) / per;
  const size_t nv = (r1 - r0) * vseg;
  for (size_t k0 = threadIdx.x; k0 < nv; k0 += (size_t)U * blockDim.x) {
    uint4 va[U], vb[U];
    size_t off[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const size_t k = k0 + (size_t)u * blockDim.x;
      const size_t r = r0 + k / vseg;
      off[u] = k < nv ? r * vrow + (size_t)g * vseg + k % vseg : (size_t)-1;
      if (off[u] != (size_t)-1) { va[u] = ld_ef(a + off[u]); vb[u] = ld_ef(b + off[u]); }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (off[u] == (size_t)-1) continue;
      uint4 v = va[u];
      v.x += vb[u].x; v.y += vb[u].y; v.z += vb[u].z; v.w += vb[u].w;
      st_ef(c + off[u], v);
    }
  }
}

int main() {
  const size_t bytes = 256ull * 197 * 3072 * 4;  // one KAT-B fp32 tensor
  const size_t n = bytes / 16;
  uint4 *a, *b, *c;
  unsigned* sink;
  CK(cudaMalloc(&a, bytes));
  CK(cudaMalloc(&b, bytes));
  CK(cudaMalloc(&c, bytes));
  CK(cudaMalloc(&sink, 4));
  CK(cudaMemset(a, 1, bytes));
  CK(cudaMemset(b, 2, bytes));
  CK(cudaMemset(c, 0, bytes));
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  const char* names[] = {"copy", "add", "read", "write", "memcpy"};
  const double traffic[] = {2.0 * bytes, 3.0 * bytes, 1.0 * bytes, 1.0 * bytes, 2.0 * bytes};
  const int reps = 30;
  for (int mode = 0; mode < 5; ++mode) {
    for (int ctas_per_sm : {4, 8, 16}) {
      if (mode == 4 && ctas_per_sm != 4) continue;
      const int grid = sms * ctas_per_sm;
      auto launch = [&]() {
        switch (mode) {
          case 0: k<0, 4><<<grid, 256>>>(a, b, c, n, sink); break;
          case 1: k<1, 4><<<grid, 256>>>(a, b, c, n, sink); break;
          case 2: k<2, 4><<<grid, 256>>>(a, b, c, n, sink); break;
          case 3: k<3, 4><<<grid, 256>>>(a, b, c, n, sink); break;
          default: cudaMemcpyAsync(c, a, bytes, cudaMemcpyDeviceToDevice); break;
        }
      };
      for (int w = 0; w < 5; ++w) launch();
      CK(cudaDeviceSynchronize());
      std::vector<float> ms(reps);
      for (int r = 0; r < reps; ++r) {
        CK(cudaEventRecord(e0));
        launch();
        CK(cudaEventRecord(e1));
        CK(cudaEventSynchronize(e1));
        CK(cudaEventElapsedTime(&ms[r], e0, e1));
      }
      CK(cudaGetLastError());
      const float best = *std::min_element(ms.begin(), ms.end());
      double mean = 0;
      for (float m : ms) mean += m;
      mean /= reps;
      printf("{\"mode\": \"%s\", \"ctas_per_sm\": %d, \"bytes\": %.0f, \"best_gbs\": %.1f, \"mean_gbs\": %.1f, "
             "\"best_us\": %.1f}\n",
             names[mode], mode == 4 ? 0 : ctas_per_sm, traffic[mode], traffic[mode] / best / 1e6,
             traffic[mode] / mean / 1e6, best * 1e3);
    }
  }
  // K2-like partition: 8 groups x (k x 148 / 8) CTAs, 96-vector segments of 768-vector rows
  for (int ctas_per_sm : {2, 4, 8}) {
    const int per = sms * ctas_per_sm / 8;
    const int grid = per * 8;
    const size_t rows = n / 768;
    auto launch = [&]() { k_seg<4><<<grid, 256>>>(a, b, c, rows, 768, 96, 8); };
    for (int w = 0; w < 5; ++w) launch();
    CK(cudaDeviceSynchronize());
    std::vector<float> ms(reps);
    for (int r = 0; r < reps; ++r) {
      CK(cudaEventRecord(e0));
      launch();
      CK(cudaEventRecord(e1));
      CK(cudaEventSynchronize(e1));
      CK(cudaEventElapsedTime(&ms[r], e0, e1));
    }
    CK(cudaGetLastError());
    const float best = *std::min_element(ms.begin(), ms.end());
    double mean = 0;
    for (float m : ms) mean += m;
    mean /= reps;
    printf("{\"mode\": \"add_group_segments\", \"ctas_per_sm\": %d, \"bytes\": %.0f, \"best_gbs\": %.1f, "
           "\"mean_gbs\": %.1f, \"best_us\": %.1f}\n",
           ctas_per_sm, 3.0 * bytes, 3.0 * bytes / best / 1e6, 3.0 * bytes / mean / 1e6, best * 1e3);
  }
  return 0;
}
