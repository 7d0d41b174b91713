// Dev probe: can a green context reserve SMs for an upload kernel while the
// rest of the GPU runs the compute?  Splits the SMs into a small group and the
// remainder, launches with the runtime API (<<<>>>) into streams of both green
// contexts on memory from the primary context, and records which SMs ran what.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/green_probe tools/green_probe.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <set>
#include <vector>

#define CU(x)                                                             \
  do {                                                                    \
    CUresult r = (x);                                                     \
    if (r != CUDA_SUCCESS) {                                              \
      const char* s = nullptr;                                            \
      cuGetErrorString(r, &s);                                            \
      printf("{\"error\": \"%s: %s\"}\n", #x, s ? s : "?");               \
      return 1;                                                           \
    }                                                                     \
  } while (0)
#define CK(x)                                                              \
  do {                                                                     \
    cudaError_t e = (x);                                                   \
    if (e != cudaSuccess) {                                                \
      printf("{\"error\": \"%s: %s\"}\n", #x, cudaGetErrorString(e));      \
      return 1;                                                            \
    }                                                                      \
  } while (0)

__global__ void spin(long long cycles, int* smid, double* buf) {
  const long long t0 = clock64();
  while (clock64() - t0 < cycles) {
  }
  if (threadIdx.x == 0) {
    unsigned s;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(s));
    smid[blockIdx.x] = (int)s;
    buf[blockIdx.x] += 1.0;  // touches primary-context memory
  }
}

int main() {
  CK(cudaSetDevice(0));
  CK(cudaFree(0));
  CUdevice dev;
  CU(cuDeviceGet(&dev, 0));
  CUdevResource all;
  CU(cuDeviceGetDevResource(dev, &all, CU_DEV_RESOURCE_TYPE_SM));
  CUdevResource grp[1], rem;
  unsigned nb = 1;
  CU(cuDevSmResourceSplitByCount(grp, &nb, &all, &rem, 0, 8));
  printf("{\"sms\": %u, \"group_sms\": %u, \"remainder_sms\": %u}\n", all.sm.smCount, grp[0].sm.smCount,
         rem.sm.smCount);
  CUdevResourceDesc dA, dB;
  CU(cuDevResourceGenerateDesc(&dA, grp, 1));
  CU(cuDevResourceGenerateDesc(&dB, &rem, 1));
  CUgreenCtx gA, gB;
  CU(cuGreenCtxCreate(&gA, dA, dev, CU_GREEN_CTX_DEFAULT_STREAM));
  CU(cuGreenCtxCreate(&gB, dB, dev, CU_GREEN_CTX_DEFAULT_STREAM));
  CUstream sA, sB;
  CU(cuGreenCtxStreamCreate(&sA, gA, CU_STREAM_NON_BLOCKING, 0));
  CU(cuGreenCtxStreamCreate(&sB, gB, CU_STREAM_NON_BLOCKING, 0));
  int *smA, *smB;
  double* buf;
  CK(cudaMalloc(&smA, 4096 * sizeof(int)));
  CK(cudaMalloc(&smB, 4096 * sizeof(int)));
  CK(cudaMalloc(&buf, 4096 * sizeof(double)));
  CK(cudaMemset(buf, 0, 4096 * sizeof(double)));
  const long long ms = 1965000;  // cycles per ms at 1965 MHz
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  // A: 8 CTAs of 100 ms; B: 4 rounds of a 148-CTA grid, 10 ms each
  CK(cudaEventRecord(e0, (cudaStream_t)sB));
  spin<<<8, 128, 0, (cudaStream_t)sA>>>(100 * ms, smA, buf);
  CK(cudaGetLastError());
  for (int r = 0; r < 4; ++r) spin<<<148, 128, 0, (cudaStream_t)sB>>>(10 * ms, smB, buf + 8);
  CK(cudaGetLastError());
  CK(cudaEventRecord(e1, (cudaStream_t)sB));
  CK(cudaDeviceSynchronize());
  float el = 0;
  CK(cudaEventElapsedTime(&el, e0, e1));
  std::vector<int> a(8), b(148);
  std::vector<double> hb(156);
  CK(cudaMemcpy(a.data(), smA, 8 * sizeof(int), cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(b.data(), smB, 148 * sizeof(int), cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(hb.data(), buf, 156 * sizeof(double), cudaMemcpyDeviceToHost));
  std::set<int> sa(a.begin(), a.end()), sbs(b.begin(), b.end());
  int overlap = 0;
  for (int s : sbs) overlap += sa.count(s);
  printf("{\"A_sms_used\": %zu, \"B_sms_used\": %zu, \"overlap\": %d, \"B_4x10ms_elapsed_ms\": %.2f, "
         "\"buf_A\": %.0f, \"buf_B\": %.0f}\n",
         sa.size(), sbs.size(), overlap, el, hb[0], hb[8]);
  // B's 148-CTA grid on ~140 SMs takes 2 waves per round if the partition holds
  return 0;
}
