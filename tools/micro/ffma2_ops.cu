// Microbenchmark: packed FP32 (FFMA2 / FMUL2) throughput by operand form and by
// occupancy x chain count -- what bounds the FMA-dense bf16 backward at 4 warps per
// scheduler?  Prints lane-ops per clock per SM (128 = the FMA pipe's peak).
//   build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/micro/ffma2_ops tools/micro/ffma2_ops.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ float2 f2(float a, float b) { return make_float2(a, b); }

// MODE 0: acc = acc * pairB + pairC           (three F32x2 register operands)
// MODE 1: acc = acc * scalarReg + pairC       (.F32 broadcast from a vector register)
// MODE 2: acc = acc * kernelParam + pairC     (.F32 broadcast from a uniform register)
// MODE 3: acc = acc * pairB                   (FMUL2, two F32x2 operands)
// MODE 4: acc = pairB * acc + acc2            (both multiplicands pairs, addend another chain)
// MODE 5: acc_i = shared * pairB_i + acc_i     (the coefficient-term accumulation: one pair
//                                              operand common to consecutive FFMA2s -> .reuse)
template <int MODE, int CH>
__global__ void k(float* out, const float* __restrict__ init, float s, float t, int iters) {
  // operands loaded at run time, so the loop holds real register operands (no
  // rematerialised constants)
  float2 acc[CH], b[CH], c[CH];
#pragma unroll
  for (int i = 0; i < CH; ++i) {
    acc[i] = f2(init[(threadIdx.x + 3 * i) & 63], init[(threadIdx.x + 3 * i + 1) & 63]);
    b[i] = f2(init[64 + ((threadIdx.x + i) & 63)], init[64 + ((threadIdx.x + i + 7) & 63)]);
    c[i] = f2(init[128 + ((threadIdx.x + 5 * i) & 63)], init[128 + ((threadIdx.x + i + 9) & 63)]);
  }
  const float sr = s * (threadIdx.x & 1 ? 1.0f : 0.9999f);  // a per-thread (vector) register
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < CH; ++i) {
      if (MODE == 0) acc[i] = __ffma2_rn(acc[i], b[i], c[i]);
      if (MODE == 1) acc[i] = __ffma2_rn(acc[i], f2(sr, sr), c[i]);
      if (MODE == 2) acc[i] = __ffma2_rn(acc[i], f2(t, t), c[i]);
      if (MODE == 3) acc[i] = __fmul2_rn(acc[i], b[i]);
      if (MODE == 4) acc[i] = __ffma2_rn(b[i], acc[i], acc[(i + 1) % CH]);
      if (MODE == 5) acc[i] = __ffma2_rn(c[0], b[i], acc[i]);
    }
  }
  float r = 0;
#pragma unroll
  for (int i = 0; i < CH; ++i) r += acc[i].x + acc[i].y;
  if (r == 12345.f) out[0] = r;
}

template <int MODE, int CH>
void run(const char* name, float* dbuf, int sms, int warps_per_sm) {
  const int iters = 20000, threads = 32 * warps_per_sm, blocks = sms;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float ms = 0;
  for (int rep = 0; rep < 3; ++rep) {
    cudaEventRecord(e0);
    k<MODE, CH><<<blocks, threads>>>(dbuf, dbuf + 8, 0.999f, 0.9995f, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
  }
  int clk_khz;
  cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
  const double clks = ms * 1e-3 * clk_khz * 1e3;
  const double ops = (double)threads * iters * CH * 2;  // lane-ops per SM
  printf("%-34s warps/SM %2d chains %d  %7.3f ms  %6.1f lane-ops/clk/SM\n", name, warps_per_sm, CH, ms, ops / clks);
}

int main() {
  float* d;
  cudaMalloc(&d, 256 * sizeof(float));
  float h[256];
  for (int i = 0; i < 256; ++i) h[i] = i < 8 ? 0.f : (i < 72 ? 0.5f + i * 1e-3f : (i < 136 ? 0.9999f - (i % 64) * 1e-6f : 1e-4f * (i % 64)));
  cudaMemcpy(d, h, sizeof h, cudaMemcpyHostToDevice);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int w : {16, 32}) {
    run<0, 8>("FFMA2 pair*pair+pair", d, sms, w);
    run<1, 8>("FFMA2 pair*vreg.F32+pair", d, sms, w);
    run<2, 8>("FFMA2 pair*ureg.F32+pair", d, sms, w);
    run<3, 8>("FMUL2 pair*pair", d, sms, w);
    run<4, 8>("FFMA2 pair*pair+pair(other chain)", d, sms, w);
    run<5, 8>("FFMA2 shared*pair+acc (reuse)", d, sms, w);
  }
  for (int w : {16, 32}) {
    run<0, 1>("FFMA2 pair*pair+pair", d, sms, w);
    run<0, 2>("FFMA2 pair*pair+pair", d, sms, w);
    run<0, 4>("FFMA2 pair*pair+pair", d, sms, w);
    run<2, 1>("FFMA2 pair*ureg.F32+pair", d, sms, w);
    run<2, 2>("FFMA2 pair*ureg.F32+pair", d, sms, w);
    run<2, 4>("FFMA2 pair*ureg.F32+pair", d, sms, w);
  }
  return 0;
}
