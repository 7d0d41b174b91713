// Microbenchmark: DMMA fed from shared memory fragments (the level kernel's
// inner loop without global loads), to find the smem-fed DMMA ceiling.
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
}

template <int FM, int FN, int WM, int WN, int SYNC_EVERY>
__global__ void kern(double* out, int iters) {
  constexpr int BK = 32, WTM = FM * 8, WTN = FN * 8, BM = WM * WTM, BN = WN * WTN;
  constexpr int LDA = BK + 4, LDB = BN + 4;
  extern __shared__ double sm[];
  double* As = sm;
  double* Bs = sm + BM * LDA;
  for (int i = threadIdx.x; i < BM * LDA + BK * LDB; i += blockDim.x) sm[i] = 1e-3 * (i % 97);
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, wm = warp / WN, wn = warp % WN;
  const double* ap = As + (wm * WTM + (lane >> 2)) * LDA + (lane & 3);
  const double* bp = Bs + (lane & 3) * LDB + wn * WTN + (lane >> 2);
  double acc[FM][FN][2] = {};
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int kk = 0; kk < BK / 4; ++kk) {
      double af[FM], bf[FN];
#pragma unroll
      for (int fm = 0; fm < FM; ++fm) af[fm] = ap[fm * 8 * LDA + kk * 4];
#pragma unroll
      for (int fn = 0; fn < FN; ++fn) bf[fn] = bp[kk * 4 * LDB + fn * 8];
#pragma unroll
      for (int fm = 0; fm < FM; ++fm)
#pragma unroll
        for (int fn = 0; fn < FN; ++fn) dmma(acc[fm][fn][0], acc[fm][fn][1], af[fm], bf[fn]);
    }
    if (SYNC_EVERY) __syncthreads();
  }
  double s = 0;
#pragma unroll
  for (int fm = 0; fm < FM; ++fm)
#pragma unroll
    for (int fn = 0; fn < FN; ++fn) s += acc[fm][fn][0] + acc[fm][fn][1];
  if (s == 1234.5) out[threadIdx.x] = s;
}

template <int FM, int FN, int WM, int WN, int SYNC>
void run(const char* name, double* out, int sms) {
  constexpr int BK = 32, BM = WM * FM * 8, BN = WN * FN * 8;
  size_t smem = (BM * (BK + 4) + BK * (BN + 4)) * sizeof(double);
  auto k = kern<FM, FN, WM, WN, SYNC>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int occ = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, WM * WN * 32, smem);
  const int iters = 2000, grid = sms * occ;
  k<<<grid, WM * WN * 32, smem>>>(out, 10);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  float best = 1e30f;
  for (int r = 0; r < 3; ++r) {
    cudaEventRecord(e0); k<<<grid, WM * WN * 32, smem>>>(out, iters); cudaEventRecord(e1);
    cudaEventSynchronize(e1); float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
  }
  double flops = 2.0 * BM * BN * BK * (double)iters * grid;
  printf("{\"name\": \"%s\", \"sync\": %d, \"occ\": %d, \"tflops\": %.2f, \"err\": \"%s\"}\n", name, SYNC, occ,
         flops / best / 1e9, cudaGetErrorString(cudaGetLastError()));
}

int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* out; cudaMalloc(&out, 4096 * 8);
  run<8, 4, 2, 4, 0>("128x128 w8 warp64x32", out, sms);
  run<8, 4, 2, 4, 1>("128x128 w8 warp64x32", out, sms);
  run<4, 4, 4, 4, 0>("128x128 w16 warp32x32", out, sms);
  run<4, 4, 4, 4, 1>("128x128 w16 warp32x32", out, sms);
  run<4, 8, 2, 4, 0>("64x256 w8 warp32x64", out, sms);
  run<4, 8, 2, 4, 1>("64x256 w8 warp32x64", out, sms);
  run<4, 4, 1, 8, 0>("32x256 w8 warp32x32", out, sms);
  run<4, 4, 1, 8, 1>("32x256 w8 warp32x32", out, sms);
  run<4, 2, 1, 16, 1>("32x256 w16 warp32x16", out, sms);
  run<2, 8, 1, 8, 1>("16x512 w8 warp16x64", out, sms);
  run<8, 8, 2, 2, 1>("128x128 w4 warp64x64", out, sms);
  return 0;
}
