/* capi_demo.c -- the drop-in boundary from plain C (no Python, no torch).
 *
 * Calls include/grkan_b200.h exactly as a C/C++ (or cgo / JNI / ctypes)
 * binding of the reference's forward_tensor / backward_blocked would
 * (pkg/src/grkan/rational.py:325-345, pkg/src/grkan/backward.py:275-372):
 * device buffers from cudaMalloc, a CUDA stream, status codes.
 * Checks EXACT forward against the C restatement of the reference
 * (oracle/, test infrastructure) bit for bit, runs the FAST backward,
 * reads the device status and exercises a host-side error.
 *
 *   build: see tests/test_gpu_capi_c.py
 */
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "grkan_b200.h"

/* oracle/_build/liboracle.so: the reference's forward in C (checker only) */
void orc_fwd_f(const float* x, float* y, const double* num, const double* den, int64_t rows, int d, int ng,
               int m1, int n);

static uint64_t rng = 0x9E3779B97F4A7C15ull;
static float randn(void) { /* Box-Muller on a 64-bit LCG */
  rng = rng * 6364136223846793005ull + 1442695040888963407ull;
  double u1 = ((rng >> 11) + 1.0) / 9007199254740993.0;
  rng = rng * 6364136223846793005ull + 1442695040888963407ull;
  double u2 = (rng >> 11) / 9007199254740992.0;
  return (float)(sqrt(-2.0 * log(u1)) * cos(6.283185307179586 * u2));
}

#define CK(x)                                                               \
  do {                                                                      \
    cudaError_t e_ = (x);                                                   \
    if (e_ != cudaSuccess) {                                                \
      fprintf(stderr, "%s: %s\n", #x, cudaGetErrorString(e_));              \
      return 1;                                                             \
    }                                                                       \
  } while (0)

int main(void) {
  const int64_t rows = 3 * 197;
  const int d = 768, ng = 8, m1 = 6, n = 4;
  const size_t E = (size_t)rows * d;
  float* x = malloc(E * 4);
  float* u = malloc(E * 4);
  float* y = malloc(E * 4);
  float* y_ref = malloc(E * 4);
  float a[8 * 6], b[8 * 4];
  double a64[8 * 6], b64[8 * 4];
  for (size_t i = 0; i < E; ++i) x[i] = randn(), u[i] = randn();
  for (int i = 0; i < ng * m1; ++i) a[i] = randn(), a64[i] = a[i];
  for (int i = 0; i < ng * n; ++i) b[i] = randn(), b64[i] = b[i];

  void *dx_, *du, *dy, *ddx, *da_, *db_, *dA, *dB, *ws;
  cudaStream_t s;
  CK(cudaStreamCreate(&s));
  CK(cudaMalloc(&dx_, E * 4));
  CK(cudaMalloc(&du, E * 4));
  CK(cudaMalloc(&dy, E * 4));
  CK(cudaMalloc(&ddx, E * 4));
  CK(cudaMalloc(&dA, sizeof a));
  CK(cudaMalloc(&dB, sizeof b));
  CK(cudaMalloc(&da_, sizeof a));
  CK(cudaMalloc(&db_, sizeof b));
  size_t ws_bytes = grkan_bwd_workspace_bytes(rows, d, ng, m1, n, GRKAN_F32);
  CK(cudaMalloc(&ws, ws_bytes));
  CK(cudaMemcpy(dx_, x, E * 4, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(du, u, E * 4, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dA, a, sizeof a, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dB, b, sizeof b, cudaMemcpyHostToDevice));

  /* forward_tensor: EXACT reproduces the reference's rounding */
  int rc = grkan_fwd(dx_, dy, dA, dB, rows, d, ng, m1, n, GRKAN_F32, GRKAN_FLAG_EXACT, NULL, s);
  if (rc != GRKAN_OK) return fprintf(stderr, "grkan_fwd: %s\n", grkan_last_error()), 1;
  CK(cudaMemcpyAsync(y, dy, E * 4, cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  orc_fwd_f(x, y_ref, a64, b64, rows, d, ng, m1, n);
  if (memcmp(y, y_ref, E * 4) != 0) return fprintf(stderr, "EXACT forward differs from the reference\n"), 1;

  /* backward_blocked: FAST policy, then the device status (AccumulationOverflowError analogue) */
  rc = grkan_bwd(dx_, du, dA, dB, ddx, da_, db_, ws, ws_bytes, rows, d, ng, m1, n, GRKAN_F32, GRKAN_FLAG_FAST, s);
  if (rc != GRKAN_OK) return fprintf(stderr, "grkan_bwd: %s\n", grkan_last_error()), 1;
  grkan_device_status st;
  rc = grkan_read_status((const grkan_device_status*)ws, s, &st);
  if (rc != GRKAN_OK) return fprintf(stderr, "status: %s\n", grkan_last_error()), 1;
  float da[8 * 6];
  CK(cudaMemcpy(da, da_, sizeof da, cudaMemcpyDeviceToHost));
  for (int i = 0; i < ng * m1; ++i)
    if (!isfinite(da[i])) return fprintf(stderr, "non-finite da\n"), 1;

  /* LayoutMismatchError analogue: d not divisible by the group count */
  rc = grkan_fwd(dx_, dy, dA, dB, rows, 770, ng, m1, n, GRKAN_F32, 0, NULL, s);
  if (rc != GRKAN_ERR_LAYOUT) return fprintf(stderr, "expected a layout error, got %d\n", rc), 1;
  printf("capi demo ok: %s; EXACT y bitwise == reference (%zu elements); da[0][0]=%.6g; \"%s\"\n",
         grkan_version(), E, da[0], grkan_last_error());
  return 0;
}
