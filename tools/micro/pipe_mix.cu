// Microbenchmark: does FP64 (DFMA) work overlap with packed FP32 (FFMA2) work
// on B200?  And what do the bf16 backward's side ops (IMAD, F2F.F64.F32,
// F2FP.BF16 pack) cost against the FMA pipe?
// Each mode runs independent chains; prints lane-ops per clock per SM.
#include <cstdio>
#include <cuda_runtime.h>

template <int NF2, int ND, int NI, int NCV>
__global__ void k(float* out, float s, int iters) {
  float2 f[NF2 > 0 ? NF2 : 1];
  double d[ND > 0 ? ND : 1];
  int ii[NI > 0 ? NI : 1];
  float c[NCV > 0 ? NCV : 1];
  double cd[NCV > 0 ? NCV : 1];
  for (int i = 0; i < (NF2 > 0 ? NF2 : 1); ++i) f[i] = make_float2(threadIdx.x * 1e-3f + i, i * 0.5f);
  for (int i = 0; i < (ND > 0 ? ND : 1); ++i) d[i] = threadIdx.x * 1e-3 + i;
  for (int i = 0; i < (NI > 0 ? NI : 1); ++i) ii[i] = threadIdx.x + i;
  for (int i = 0; i < (NCV > 0 ? NCV : 1); ++i) { c[i] = threadIdx.x * 1e-3f + i; cd[i] = 0; }
  const double sd = s;
  const int si = (int)(s * 3.0f) | 1;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NF2; ++i) f[i] = __ffma2_rn(f[i], make_float2(s, s), make_float2(0.5f, 0.5f));
#pragma unroll
    for (int i = 0; i < ND; ++i) d[i] = fma(d[i], sd, 0.25);
#pragma unroll
    for (int i = 0; i < NI; ++i) ii[i] = ii[i] * si + 7;
#pragma unroll
    for (int i = 0; i < NCV; ++i) { cd[i] = fma((double)c[i], sd, cd[i]); c[i] = c[i] * 0.999f; }
  }
  float acc = 0;
  for (int i = 0; i < NF2; ++i) acc += f[i].x + f[i].y;
  for (int i = 0; i < ND; ++i) acc += (float)d[i];
  for (int i = 0; i < NI; ++i) acc += (float)ii[i];
  for (int i = 0; i < NCV; ++i) acc += (float)cd[i] + c[i];
  if (acc == 12345.f) out[0] = acc;
}

template <int NF2, int ND, int NI, int NCV>
void run(const char* name, float* dbuf, int sms) {
  const int iters = 4000, threads = 512, blocks = sms * 4;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float ms = 0;
  for (int rep = 0; rep < 3; ++rep) {
    cudaEventRecord(e0);
    k<NF2, ND, NI, NCV><<<blocks, threads>>>(dbuf, 0.999f, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
  }
  int clk_khz;
  cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
  const double clks = ms * 1e-3 * clk_khz * 1e3;
  const double per = (double)blocks * threads * iters / sms / clks;  // thread-iterations per clk per SM
  printf("%-40s %.3f ms  FFMA2 lane-ops %.1f  DFMA %.1f  IMAD %.1f  cvt+dfma %.1f  (per clk per SM)\n", name, ms,
         per * NF2 * 2, per * ND, per * NI, per * NCV);
}

int main() {
  float* d;
  cudaMalloc(&d, 8);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  run<8, 0, 0, 0>("FFMA2 x8", d, sms);
  run<0, 8, 0, 0>("DFMA x8", d, sms);
  run<8, 4, 0, 0>("FFMA2 x8 + DFMA x4", d, sms);
  run<8, 8, 0, 0>("FFMA2 x8 + DFMA x8", d, sms);
  run<0, 0, 8, 0>("IMAD x8", d, sms);
  run<8, 0, 4, 0>("FFMA2 x8 + IMAD x4", d, sms);
  run<0, 0, 0, 8>("F2F.F64.F32 + DFMA + FMUL x8", d, sms);
  run<8, 0, 0, 4>("FFMA2 x8 + (cvt+DFMA+FMUL) x4", d, sms);
  return 0;
}
