// Step-0 FP64 peak microbenchmarks for B200.
//
// MEASURED_PEAKS.json carries no FP64 figure, so the roofline denominators for
// the leaf DGEMM are measured here:
//   (1) DMMA: mma.sync.m8n8k4.f64 on register-resident fragments, all SMs;
//   (2) DFMA: scalar fma.rn.f64 chains, all SMs;
//   (3) cublasDgemm at several n (native FP64, default math mode).
// Each kernel also reports the SM clock it ran at (clock64 / globaltimer).
//
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o peaks_fp64 peaks_fp64.cu -lcublas
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <vector>
#include <cuda_runtime.h>
#include <cublas_v2.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  fprintf(stderr, "CUDA %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); exit(1);} } while (0)

__device__ __forceinline__ uint64_t gtimer() {
  uint64_t t; asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t)); return t;
}

template <int NACC>
__global__ void dmma_loop(double* out, int iters, unsigned long long* clk) {
  double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
  double c[NACC][2];
#pragma unroll
  for (int i = 0; i < NACC; ++i) { c[i][0] = 0.0; c[i][1] = 0.0; }
  uint64_t c0 = clock64(), t0 = gtimer();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NACC; ++i) {
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
    }
  }
  uint64_t c1 = clock64(), t1 = gtimer();
  double s = 0;
#pragma unroll
  for (int i = 0; i < NACC; ++i) s += c[i][0] + c[i][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (blockIdx.x == 0 && threadIdx.x == 0) { clk[0] = c1 - c0; clk[1] = t1 - t0; }
}

template <int NACC>
__global__ void dfma_loop(double* out, int iters, unsigned long long* clk) {
  double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
  double c[NACC];
#pragma unroll
  for (int i = 0; i < NACC; ++i) c[i] = i;
  uint64_t c0 = clock64(), t0 = gtimer();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NACC; ++i) asm volatile("fma.rn.f64 %0, %1, %2, %0;" : "+d"(c[i]) : "d"(a), "d"(b));
  }
  uint64_t c1 = clock64(), t1 = gtimer();
  double s = 0;
#pragma unroll
  for (int i = 0; i < NACC; ++i) s += c[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (blockIdx.x == 0 && threadIdx.x == 0) { clk[0] = c1 - c0; clk[1] = t1 - t0; }
}

int main(int argc, char** argv) {
  int dev = 0; CK(cudaSetDevice(dev));
  cudaDeviceProp prop; CK(cudaGetDeviceProperties(&prop, dev));
  int sms = prop.multiProcessorCount;
  printf("{\"gpu\": \"%s\", \"sms\": %d, \"cc\": \"%d.%d\"}\n", prop.name, sms, prop.major, prop.minor);
  double* out; CK(cudaMalloc(&out, sizeof(double) * sms * 32 * 1024));
  unsigned long long* clk; CK(cudaMalloc(&clk, 16));
  cudaEvent_t e0, e1; CK(cudaEventCreate(&e0)); CK(cudaEventCreate(&e1));

  auto run = [&](const char* name, auto kern, int threads, int blocks_per_sm, int iters, double flop_per_thread_iter) {
    int blocks = sms * blocks_per_sm;
    kern<<<blocks, threads>>>(out, iters / 10, clk);  // warm-up
    CK(cudaDeviceSynchronize());
    // sustained: repeat for ~2 s
    float best_ms = 1e30f; double total_ms = 0; int reps = 0;
    while (total_ms < 2000.0) {
      CK(cudaEventRecord(e0));
      kern<<<blocks, threads>>>(out, iters, clk);
      CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1));
      float ms; CK(cudaEventElapsedTime(&ms, e0, e1));
      best_ms = ms < best_ms ? ms : best_ms; total_ms += ms; ++reps;
    }
    unsigned long long h[2]; CK(cudaMemcpy(h, clk, 16, cudaMemcpyDeviceToHost));
    double flops = (double)blocks * threads * iters * flop_per_thread_iter;
    printf("{\"bench\": \"%s\", \"threads\": %d, \"blocks_per_sm\": %d, \"tflops_best\": %.3f, \"tflops_mean\": %.3f, "
           "\"sm_mhz_last\": %.0f, \"reps\": %d}\n",
           name, threads, blocks_per_sm, flops / (best_ms * 1e-3) / 1e12, flops * reps / (total_ms * 1e-3) / 1e12,
           (double)h[0] / (double)h[1] * 1e3, reps);
    fflush(stdout);
  };
  // DMMA m8n8k4: 8*8*4 FMA = 512 flop per warp-instruction = 16 flop per thread
  for (int bps : {1, 2, 4}) {
    run("dmma_m8n8k4_nacc8", dmma_loop<8>, 128, bps, 20000, 8 * 16.0);
    run("dmma_m8n8k4_nacc16", dmma_loop<16>, 128, bps, 10000, 16 * 16.0);
  }
  run("dmma_m8n8k4_nacc8_256t", dmma_loop<8>, 256, 2, 20000, 8 * 16.0);
  for (int bps : {2, 4}) {
    run("dfma_nacc8", dfma_loop<8>, 256, bps, 20000, 8 * 2.0);
  }

  // cuBLAS DGEMM
  cublasHandle_t h; cublasCreate(&h);
  int ver; cublasGetVersion(h, &ver);
  cublasMath_t mm; cublasGetMathMode(h, &mm);
  printf("{\"cublas_version\": %d, \"math_mode\": %d}\n", ver, (int)mm);
  for (int n : {2048, 4096, 8192, 16384}) {
    size_t bytes = (size_t)n * n * sizeof(double);
    double *A, *B, *C; CK(cudaMalloc(&A, bytes)); CK(cudaMalloc(&B, bytes)); CK(cudaMalloc(&C, bytes));
    CK(cudaMemset(A, 0, bytes)); CK(cudaMemset(B, 0, bytes));
    double one = 1.0, zero = 0.0;
    for (int w = 0; w < 3; ++w) cublasDgemm(h, CUBLAS_OP_N, CUBLAS_OP_N, n, n, n, &one, A, n, B, n, &zero, C, n);
    CK(cudaDeviceSynchronize());
    int reps = n <= 4096 ? 20 : (n <= 8192 ? 8 : 4);
    std::vector<float> t;
    for (int r = 0; r < reps; ++r) {
      CK(cudaEventRecord(e0));
      cublasDgemm(h, CUBLAS_OP_N, CUBLAS_OP_N, n, n, n, &one, A, n, B, n, &zero, C, n);
      CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1));
      float ms; CK(cudaEventElapsedTime(&ms, e0, e1)); t.push_back(ms);
    }
    float best = 1e30f; double sum = 0; for (float x : t) { best = x < best ? x : best; sum += x; }
    double fl = 2.0 * n * (double)n * n;
    printf("{\"bench\": \"cublasDgemm\", \"n\": %d, \"ms_best\": %.3f, \"tflops_best\": %.3f, \"tflops_mean\": %.3f}\n",
           n, best, fl / (best * 1e-3) / 1e12, fl * t.size() / (sum * 1e-3) / 1e12);
    fflush(stdout);
    // strided batched: 7 products of (n/2)^3 (the SW^1 leaf batch)
    int m = n / 2;
    for (int w = 0; w < 2; ++w)
      cublasDgemmStridedBatched(h, CUBLAS_OP_N, CUBLAS_OP_N, m, m, m, &one, A, m, (long long)m * m, B, m,
                                (long long)m * m, &zero, C, m, (long long)m * m, 4);
    CK(cudaDeviceSynchronize());
    CK(cudaEventRecord(e0));
    for (int r = 0; r < 5; ++r)
      cublasDgemmStridedBatched(h, CUBLAS_OP_N, CUBLAS_OP_N, m, m, m, &one, A, m, (long long)m * m, B, m,
                                (long long)m * m, &zero, C, m, (long long)m * m, 4);
    CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1));
    float ms; CK(cudaEventElapsedTime(&ms, e0, e1));
    printf("{\"bench\": \"cublasDgemmStridedBatched\", \"m\": %d, \"batch\": 4, \"tflops\": %.3f}\n", m,
           5 * 4 * 2.0 * m * (double)m * m / (ms * 1e-3) / 1e12);
    CK(cudaFree(A)); CK(cudaFree(B)); CK(cudaFree(C));
  }
  cublasDestroy(h);
  return 0;
}
