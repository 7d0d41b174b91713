// Dev probe: host -> device read bandwidth of the ways a symmetric-aware
// upload could move only the unique elements of A's diagonal blocks.
//   (a) cudaMemcpyAsync of a contiguous range (DMA engine reference)
//   (b) zero-copy kernel: SMs read pinned host memory, 16 B per lane, contiguous
//   (c) zero-copy kernel, triangular runs: row r of 32 doubles, lanes < r+1 active
//   (d) cudaMemcpy2DAsync with 128 B rows at 256 B pitch / 256 B rows at 512 B pitch
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/zerocopy_probe tools/zerocopy_probe.cu
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>

#define CK(x)                                                                  \
  do {                                                                         \
    cudaError_t e = (x);                                                       \
    if (e != cudaSuccess) {                                                    \
      printf("%s: %s\n", #x, cudaGetErrorString(e));                           \
      exit(1);                                                                 \
    }                                                                          \
  } while (0)

__global__ void zc_contig(const double2* __restrict__ src, double2* __restrict__ dst, size_t n2) {
  size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  // 4 independent loads in flight per thread
  for (; i + 3 * stride < n2; i += 4 * stride) {
    double2 a = src[i], b = src[i + stride], c = src[i + 2 * stride], d = src[i + 3 * stride];
    dst[i] = a; dst[i + stride] = b; dst[i + 2 * stride] = c; dst[i + 3 * stride] = d;
  }
  for (; i < n2; i += stride) dst[i] = src[i];
}

// rows of 32 doubles; row r (mod 32) needs elements 0..r: one warp per row,
// lane l reads double l if l <= r (sector-granular predicated reads)
__global__ void zc_tri(const double* __restrict__ src, double* __restrict__ dst, size_t rows) {
  const int lane = threadIdx.x & 31;
  size_t w = (blockIdx.x * (size_t)blockDim.x + threadIdx.x) >> 5;
  const size_t nw = ((size_t)gridDim.x * blockDim.x) >> 5;
  for (; w + 3 * nw < rows; w += 4 * nw) {
    double v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const size_t r = w + u * nw;
      v[u] = lane <= (int)(r & 31) ? src[r * 32 + lane] : 0.0;
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const size_t r = w + u * nw;
      if (lane <= (int)(r & 31)) dst[r * 32 + lane] = v[u];
    }
  }
  for (; w < rows; w += nw)
    if (lane <= (int)(w & 31)) dst[w * 32 + lane] = src[w * 32 + lane];
}

int main(int argc, char** argv) {
  const size_t bytes = (size_t)(argc > 1 ? atof(argv[1]) : 4.0) * (1ull << 30);
  double* h;
  CK(cudaHostAlloc(&h, bytes, cudaHostAllocMapped));
  for (size_t i = 0; i < bytes / 8; i += 512) h[i] = (double)i;
  double* hd;
  CK(cudaHostGetDevicePointer((void**)&hd, h, 0));
  double* d;
  CK(cudaMalloc(&d, bytes));
  cudaStream_t s;
  CK(cudaStreamCreate(&s));
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  float ms;
  auto timeit = [&](auto fn) {
    fn();
    CK(cudaStreamSynchronize(s));
    CK(cudaEventRecord(e0, s));
    fn();
    CK(cudaEventRecord(e1, s));
    CK(cudaEventSynchronize(e1));
    CK(cudaEventElapsedTime(&ms, e0, e1));
    return ms;
  };
  ms = timeit([&] { CK(cudaMemcpyAsync(d, h, bytes, cudaMemcpyHostToDevice, s)); });
  printf("{\"probe\": \"memcpy\", \"GBps\": %.2f}\n", bytes / ms / 1e6);
  const int ctas[] = {2, 4, 8, 16, 32, 64, 148, 296};
  for (int threads : {256, 1024})
    for (int g : ctas) {
      ms = timeit([&] { zc_contig<<<g, threads, 0, s>>>((const double2*)hd, (double2*)d, bytes / 16); });
      printf("{\"probe\": \"zc_contig\", \"ctas\": %d, \"threads\": %d, \"GBps\": %.2f}\n", g, threads,
             bytes / ms / 1e6);
    }
  const size_t rows = bytes / 256;
  const double useful = (double)rows / 32 * (32 * 33 / 2) * 8;  // bytes of the triangle
  for (int g : ctas) {
    ms = timeit([&] { zc_tri<<<g, 1024, 0, s>>>(hd, d, rows); });
    printf("{\"probe\": \"zc_tri\", \"ctas\": %d, \"useful_GBps\": %.2f, \"span_GBps\": %.2f}\n", g,
           useful / ms / 1e6, bytes / ms / 1e6);
  }
  for (int w : {64, 128, 256, 512, 1024}) {
    const size_t h2 = bytes / (2 * w);
    ms = timeit([&] { CK(cudaMemcpy2DAsync(d, 2 * w, h, 2 * w, w, h2, cudaMemcpyHostToDevice, s)); });
    printf("{\"probe\": \"memcpy2d\", \"width\": %d, \"pitch\": %d, \"useful_GBps\": %.2f}\n", w, 2 * w,
           (double)w * h2 / ms / 1e6);
  }
  return 0;
}
