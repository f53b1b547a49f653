// Microbenchmark: FP32 lane-FMA throughput per SM per clock, scalar FFMA vs packed FFMA2.
#include <cstdio>
#include <cuda_runtime.h>
template <int MODE>
__global__ void k(float* out, float s, int iters) {
  float a[16];
  for (int i = 0; i < 16; ++i) a[i] = threadIdx.x * 0.001f + i;
  float2 b[8];
  for (int i = 0; i < 8; ++i) b[i] = make_float2(a[2*i], a[2*i+1]);
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    if (MODE == 0) {
#pragma unroll
      for (int i = 0; i < 16; ++i) a[i] = fmaf(a[i], s, 0.5f);
    } else if (MODE == 1) {
#pragma unroll
      for (int i = 0; i < 8; ++i) b[i] = __ffma2_rn(b[i], make_float2(s, s), make_float2(0.5f, 0.5f));
    } else {
#pragma unroll
      for (int i = 0; i < 8; ++i) a[i] = fmaf(a[i], s, 0.5f);
#pragma unroll
      for (int i = 0; i < 4; ++i) b[i] = __ffma2_rn(b[i], make_float2(s, s), make_float2(0.5f, 0.5f));
    }
  }
  long long t1 = clock64();
  float acc = 0;
  for (int i = 0; i < 16; ++i) acc += a[i];
  for (int i = 0; i < 8; ++i) acc += b[i].x + b[i].y;
  if (acc == 12345.f) out[0] = acc;
  if (threadIdx.x == 0 && blockIdx.x == 0) out[1] = (float)(t1 - t0);
}
int main() {
  float* d; cudaMalloc(&d, 8);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int iters = 20000, threads = 512, blocks = sms * 4;
  const char* names[3] = {"FFMA x16 chains", "FFMA2 x8 chains", "mix 8 FFMA + 4 FFMA2"};
  double lanes_per_iter[3] = {16, 16, 16};
  for (int mode = 0; mode < 3; ++mode) {
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(e0);
      if (mode == 0) k<0><<<blocks, threads>>>(d, 0.999f, iters);
      if (mode == 1) k<1><<<blocks, threads>>>(d, 0.999f, iters);
      if (mode == 2) k<2><<<blocks, threads>>>(d, 0.999f, iters);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
    }
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    float cyc; cudaMemcpy(&cyc, d + 1, 4, cudaMemcpyDeviceToHost);
    double lane_fma = (double)blocks * threads * iters * lanes_per_iter[mode];
    double per_sm_per_ns = lane_fma / sms / (ms * 1e6);
    printf("%-24s %.3f ms  %.1f lane-FMA/ns/SM  (~%.1f per clk at 1.965 GHz)\n", names[mode], ms, per_sm_per_ns,
           per_sm_per_ns / 1.965);
  }
  return 0;
}
