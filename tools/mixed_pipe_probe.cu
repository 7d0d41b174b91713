// Do DMMA (tensor pipe) and DFMA (fp64 pipe) run concurrently on B200?
// Half the warps of each CTA run a DMMA loop, the other half a DFMA loop.
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
}

__global__ void mixed(double* out, int iters_mma, int iters_fma, int mma_warps) {
  const int warp = threadIdx.x >> 5;
  double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
  double s = 0;
  if (warp < mma_warps) {
    double c[16][2];
#pragma unroll
    for (int i = 0; i < 16; ++i) c[i][0] = c[i][1] = 0;
    for (int it = 0; it < iters_mma; ++it)
#pragma unroll
      for (int i = 0; i < 16; ++i) dmma(c[i][0], c[i][1], a, b);
#pragma unroll
    for (int i = 0; i < 16; ++i) s += c[i][0] + c[i][1];
  } else {
    double c[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) c[i] = i;
    for (int it = 0; it < iters_fma; ++it)
#pragma unroll
      for (int i = 0; i < 8; ++i) c[i] = fma(a, c[i], b);
#pragma unroll
    for (int i = 0; i < 8; ++i) s += c[i];
  }
  if (s == 1234.5) out[threadIdx.x] = s;
}

int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* out; cudaMalloc(&out, 4096 * 8);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  struct Cfg { int warps, mma_warps, im, ifm; };
  Cfg cfgs[] = {{8, 8, 4000, 0}, {8, 0, 0, 32000}, {16, 8, 4000, 32000}, {16, 8, 4000, 16000},
                {16, 8, 4000, 64000}, {12, 8, 4000, 32000}, {16, 4, 4000, 32000}};
  for (auto c : cfgs) {
    mixed<<<sms, 32 * c.warps>>>(out, 10, 10, c.mma_warps);
    float best = 1e30f;
    for (int r = 0; r < 3; ++r) {
      cudaEventRecord(e0);
      mixed<<<sms, 32 * c.warps>>>(out, c.im, c.ifm, c.mma_warps);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
    }
    double fl_mma = 2.0 * 256 * 16 * (double)c.im * c.mma_warps * sms;
    double fl_fma = 2.0 * 8 * (double)c.ifm * 32 * (c.warps - c.mma_warps) * sms;
    printf("{\"warps\": %d, \"mma_warps\": %d, \"ms\": %.3f, \"mma_tflops\": %.2f, \"fma_tflops\": %.2f, \"total\": %.2f}\n",
           c.warps, c.mma_warps, best, fl_mma / best / 1e9, fl_fma / best / 1e9, (fl_mma + fl_fma) / best / 1e9);
  }
  return 0;
}
