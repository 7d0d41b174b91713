// Dev probe: DMA-engine throughput of the row-run copies a symmetric-aware
// upload of BCSS diagonal blocks issues (b=32, m=4 blocks of 8 MB).
// Pattern "mid pair" (modes 1,2 equal): for fixed e2, rows e1 in [0, e2] of
// every e3 slab -> one 2D copy per e2 (width (e2+1)*256 B, height 32, pitch 256 KB),
// or one 3D copy per e2 spanning `depth` consecutive blocks.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/dma_pattern_probe tools/dma_pattern_probe.cu
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <chrono>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); exit(1);} } while (0)
int main() {
  const int b = 32; const size_t row = b * 8, slab = (size_t)b * b * row, blk = slab * b;  // 256 B, 256 KB, 8 MB
  const int nblk = 128;
  char *h, *d;
  CK(cudaHostAlloc((void**)&h, blk * nblk, 0));
  CK(cudaMalloc((void**)&d, blk * nblk));
  cudaStream_t s; CK(cudaStreamCreate(&s));
  cudaEvent_t e0, e1; CK(cudaEventCreate(&e0)); CK(cudaEventCreate(&e1));
  for (int depth : {1, 4, 16}) {
    for (int rep = 0; rep < 2; ++rep) {
      size_t useful = 0; int calls = 0;
      auto t0 = std::chrono::steady_clock::now();
      CK(cudaEventRecord(e0, s));
      for (int b0 = 0; b0 < nblk; b0 += depth)
        for (int e2 = 0; e2 < b; ++e2) {
          const size_t w = (size_t)(e2 + 1) * row;
          if (depth == 1) {
            CK(cudaMemcpy2DAsync(d + b0 * blk + e2 * slab / b * 0 + (size_t)e2 * b * row, slab, h + b0 * blk + (size_t)e2 * b * row, slab, w, b, cudaMemcpyHostToDevice, s));
          } else {
            cudaMemcpy3DParms p = {};
            p.srcPtr = make_cudaPitchedPtr(h + b0 * blk + (size_t)e2 * b * row, slab, w, b);
            p.dstPtr = make_cudaPitchedPtr(d + b0 * blk + (size_t)e2 * b * row, slab, w, b);
            p.extent = make_cudaExtent(w, b, depth);
            p.kind = cudaMemcpyHostToDevice;
            CK(cudaMemcpy3DAsync(&p, s));
          }
          useful += w * b * depth; ++calls;
        }
      CK(cudaEventRecord(e1, s));
      auto t1 = std::chrono::steady_clock::now();
      CK(cudaEventSynchronize(e1));
      float ms; CK(cudaEventElapsedTime(&ms, e0, e1));
      const double host_ms = std::chrono::duration<double, std::milli>(t1 - t0).count();
      if (rep) printf("{\"depth\": %d, \"calls\": %d, \"useful_GB\": %.3f, \"ms\": %.2f, \"useful_GBps\": %.2f, \"enqueue_ms\": %.2f}\n",
                      depth, calls, useful / 1e9, ms, useful / ms / 1e6, host_ms);
    }
  }
  // many plain 1D copies of one row run each (per-call overhead)
  for (size_t sz : {(size_t)65536, (size_t)262144, (size_t)1 << 20}) {
    const int n = (int)((blk * nblk / 2) / sz);
    CK(cudaEventRecord(e0, s));
    for (int i = 0; i < n; ++i) CK(cudaMemcpyAsync(d + i * sz * 2, h + i * sz * 2, sz, cudaMemcpyHostToDevice, s));
    CK(cudaEventRecord(e1, s)); CK(cudaEventSynchronize(e1));
    float ms; CK(cudaEventElapsedTime(&ms, e0, e1));
    printf("{\"memcpy1d_bytes\": %zu, \"calls\": %d, \"GBps\": %.2f}\n", sz, n, (double)sz * n / ms / 1e6);
  }
  return 0;
}
