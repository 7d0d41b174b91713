// FP64 tensor-core (DMMA) and DFMA peak microbenchmark for B200 (sm_100a).
// Measures the roofline denominator for the BCSS sttsm path: the FP64 DMMA
// issue-rate ceiling with operands in registers, at several warps/SM.
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  fprintf(stderr, "CUDA %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); exit(1);} } while (0)

template <int NACC>
__global__ void dmma_loop(double* out, int iters) {
  double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
  double c[NACC][2];
#pragma unroll
  for (int i = 0; i < NACC; ++i) { c[i][0] = 0.0; c[i][1] = 0.0; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NACC; ++i) {
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < NACC; ++i) s += c[i][0] + c[i][1];
  if (s == 12345.0) out[threadIdx.x] = s;
}

template <int NACC>
__global__ void dfma_loop(double* out, int iters) {
  double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
  double c[NACC];
#pragma unroll
  for (int i = 0; i < NACC; ++i) c[i] = i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NACC; ++i) c[i] = fma(a, c[i], b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < NACC; ++i) s += c[i];
  if (s == 12345.0) out[threadIdx.x] = s;
}

int main() {
  int dev = 0; cudaDeviceProp prop; CK(cudaGetDeviceProperties(&prop, dev));
  int sms = prop.multiProcessorCount;
  double* out; CK(cudaMalloc(&out, 4096 * sizeof(double)));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  printf("{\"gpu\": \"%s\", \"sms\": %d}\n", prop.name, sms);
  const int iters = 20000;
  for (int warps : {1, 2, 4, 8, 16}) {
    for (int ctas_per_sm : {1, 2}) {
      dim3 grid(sms * ctas_per_sm), block(32 * warps);
      dmma_loop<16><<<grid, block>>>(out, 100); CK(cudaDeviceSynchronize());
      float best = 1e30f;
      for (int r = 0; r < 5; ++r) {
        cudaEventRecord(e0); dmma_loop<16><<<grid, block>>>(out, iters); cudaEventRecord(e1);
        CK(cudaEventSynchronize(e1)); float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
      }
      double flops = 2.0 * 256 * 16 * (double)iters * grid.x * warps;
      printf("{\"kind\": \"dmma_m8n8k4\", \"warps_per_cta\": %d, \"ctas_per_sm\": %d, \"tflops\": %.3f}\n",
             warps, ctas_per_sm, flops / best / 1e9);
    }
  }
  for (int warps : {4, 8, 16, 32}) {
    dim3 grid(sms * 2), block(32 * warps);
    dfma_loop<8><<<grid, block>>>(out, 100); CK(cudaDeviceSynchronize());
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
      cudaEventRecord(e0); dfma_loop<8><<<grid, block>>>(out, iters); cudaEventRecord(e1);
      CK(cudaEventSynchronize(e1)); float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
    }
    double flops = 2.0 * 8 * (double)iters * grid.x * block.x;
    printf("{\"kind\": \"dfma\", \"warps_per_cta\": %d, \"ctas_per_sm\": 2, \"tflops\": %.3f}\n", warps, flops / best / 1e9);
  }
  return 0;
}
