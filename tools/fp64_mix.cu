// Do DMMA (mma.sync f64) and DFMA (fma.rn.f64) share one FP64 pipe on B200?
//
// Each CTA runs W warps; the first D of them issue DMMA.8x8x4 chains, the rest
// DFMA chains, for the same wall time (iteration counts scaled by the measured
// solo rates).  If the two ran on separate units the combined rate would exceed
// the solo DMMA peak (37.1 TF, profiles/peaks_fp64.json).
//
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_mix fp64_mix.cu
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  fprintf(stderr, "CUDA %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); exit(1);} } while (0)

__global__ void mix(double* out, int dmma_warps, int it_dmma, int it_dfma,
                    unsigned long long* cnt) {
  const int warp = threadIdx.x / 32;
  double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
  double s = 0;
  if (warp < dmma_warps) {
    double c[16][2];
#pragma unroll
    for (int i = 0; i < 16; ++i) { c[i][0] = 0.0; c[i][1] = 0.0; }
    for (int it = 0; it < it_dmma; ++it) {
#pragma unroll
      for (int i = 0; i < 16; ++i)
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                     : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
    }
#pragma unroll
    for (int i = 0; i < 16; ++i) s += c[i][0] + c[i][1];
    if ((threadIdx.x & 31) == 0) atomicAdd(&cnt[0], (unsigned long long)it_dmma * 16 * 256);  // FMA per warp-instruction
  } else {
    double c[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) c[i] = i;
    for (int it = 0; it < it_dfma; ++it) {
#pragma unroll
      for (int i = 0; i < 16; ++i) asm volatile("fma.rn.f64 %0, %1, %2, %0;" : "+d"(c[i]) : "d"(a), "d"(b));
    }
#pragma unroll
    for (int i = 0; i < 16; ++i) s += c[i];
    if ((threadIdx.x & 31) == 0) atomicAdd(&cnt[1], (unsigned long long)it_dfma * 16 * 32);
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
  cudaDeviceProp prop; CK(cudaGetDeviceProperties(&prop, 0));
  const int sms = prop.multiProcessorCount;
  double* out; CK(cudaMalloc(&out, sizeof(double) * sms * 4 * 512));
  unsigned long long* cnt; CK(cudaMalloc(&cnt, 16));
  cudaEvent_t e0, e1; CK(cudaEventCreate(&e0)); CK(cudaEventCreate(&e1));
  const int threads = 256, bps = 2;  // 16 warps per SM, 4 per sub-partition
  auto run = [&](int dw, int itm, int itf) {
    mix<<<sms * bps, threads>>>(out, dw, itm / 10, itf / 10, cnt);
    CK(cudaDeviceSynchronize());
    float best = 1e30f; unsigned long long h[2] = {0, 0};
    for (int r = 0; r < 5; ++r) {
      CK(cudaMemset(cnt, 0, 16));
      CK(cudaEventRecord(e0));
      mix<<<sms * bps, threads>>>(out, dw, itm, itf, cnt);
      CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1));
      float ms; CK(cudaEventElapsedTime(&ms, e0, e1));
      if (ms < best) { best = ms; CK(cudaMemcpy(h, cnt, 16, cudaMemcpyDeviceToHost)); }
    }
    double fl_m = 2.0 * h[0], fl_f = 2.0 * h[1];
    printf("{\"dmma_warps_per_cta\": %d, \"dfma_warps_per_cta\": %d, \"ms\": %.3f, \"dmma_tflops\": %.2f, "
           "\"dfma_tflops\": %.2f, \"total_tflops\": %.2f}\n",
           dw, threads / 32 - dw, best, fl_m / (best * 1e-3) / 1e12, fl_f / (best * 1e-3) / 1e12,
           (fl_m + fl_f) / (best * 1e-3) / 1e12);
    fflush(stdout);
  };
  // solo rates, then mixes with per-warp work balanced for equal duration
  run(8, 4000, 0);
  run(0, 0, 30000);
  for (int dw : {2, 4, 6}) {
    for (int itf : {10000, 20000, 30000}) run(dw, 4000, itf);
  }
  return 0;
}
