// PCIe bandwidth on the GPU box: pinned H2D / D2H, contiguous vs 2-D
// (row width w bytes, pitch 128 KB -- the B column slabs / C regions of the
// host-buffer pipeline), and H2D concurrent with D2H.
// Build: nvcc -O2 -o pcie_bw pcie_bw.cu
#include <cstdio>
#include <cuda_runtime.h>
int main() {
  const size_t n = 16384, bytes = n * n * 8;  // 2 GiB
  double *h1, *h2, *d1, *d2;
  cudaMallocHost(&h1, bytes); cudaMallocHost(&h2, bytes);
  cudaMalloc(&d1, bytes); cudaMalloc(&d2, bytes);
  cudaStream_t s1, s2; cudaStreamCreate(&s1); cudaStreamCreate(&s2);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  auto gbs = [&](float ms, size_t by) { return by / (ms * 1e-3) / 1e9; };
  float ms;
  for (int rep = 0; rep < 2; ++rep) {
    cudaEventRecord(a, s1); cudaMemcpyAsync(d1, h1, bytes, cudaMemcpyHostToDevice, s1); cudaEventRecord(b, s1);
    cudaEventSynchronize(b); cudaEventElapsedTime(&ms, a, b);
    printf("H2D contiguous 2 GiB: %.1f GB/s\n", gbs(ms, bytes));
    cudaEventRecord(a, s1); cudaMemcpyAsync(h1, d1, bytes, cudaMemcpyDeviceToHost, s1); cudaEventRecord(b, s1);
    cudaEventSynchronize(b); cudaEventElapsedTime(&ms, a, b);
    printf("D2H contiguous 2 GiB: %.1f GB/s\n", gbs(ms, bytes));
    for (size_t w : {2048, 4096, 8192, 32768}) {
      size_t rows = n, sub = bytes / (n * 8 * 8 / (w / 8 * 8)) ;
      (void)sub;
      cudaEventRecord(a, s1);
      size_t tot = 0;
      for (size_t c = 0; c + w <= n * 8; c += w) {
        cudaMemcpy2DAsync((char*)d1 + c, n * 8, (char*)h1 + c, n * 8, w, rows, cudaMemcpyHostToDevice, s1);
        tot += w * rows;
      }
      cudaEventRecord(b, s1); cudaEventSynchronize(b); cudaEventElapsedTime(&ms, a, b);
      printf("H2D 2-D width %zu B: %.1f GB/s\n", w, gbs(ms, tot));
      cudaEventRecord(a, s1);
      for (size_t c = 0; c + w <= n * 8; c += w)
        cudaMemcpy2DAsync((char*)h1 + c, n * 8, (char*)d1 + c, n * 8, w, rows, cudaMemcpyDeviceToHost, s1);
      cudaEventRecord(b, s1); cudaEventSynchronize(b); cudaEventElapsedTime(&ms, a, b);
      printf("D2H 2-D width %zu B: %.1f GB/s\n", w, gbs(ms, tot));
    }
    cudaDeviceSynchronize();
    cudaEvent_t c0, c1; cudaEventCreate(&c0); cudaEventCreate(&c1);
    cudaEventRecord(a, s1); cudaStreamWaitEvent(s2, a, 0);
    cudaMemcpyAsync(d1, h1, bytes, cudaMemcpyHostToDevice, s1);
    cudaMemcpyAsync(h2, d2, bytes, cudaMemcpyDeviceToHost, s2);
    cudaEventRecord(b, s1); cudaEventRecord(c1, s2);
    cudaEventSynchronize(b); cudaEventSynchronize(c1);
    float ms2; cudaEventElapsedTime(&ms, a, b); cudaEventElapsedTime(&ms2, a, c1);
    printf("concurrent H2D %.1f GB/s + D2H %.1f GB/s\n", gbs(ms, bytes), gbs(ms2, bytes));
  }
  return 0;
}
