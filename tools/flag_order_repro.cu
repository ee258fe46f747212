// flag_order_repro.cu -- minimal reproducer for the ordered fold's protocol
// (mf_leaf.cu, FUSE == 2) outside the leaf kernel: J "products" update the same
// T tile positions of a C array in job order.  CTA (j, t), in ticket order:
//   thread 0 spins on flag[t] >= j (ld.acquire.gpu), __syncthreads, every
//   thread loads its 4 x ROWS doubles, adds (j + 1), stores, __syncthreads,
//   thread 0 fence + st.release.gpu flag[t] = j + 1.
// Expected: C = sum_{j<J} (j + 1) everywhere.  Run with 1 or 2 CTAs per SM
// (dynamic smem padding) and with / without a co-resident DMMA busy loop.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/repro tools/flag_order_repro.cu
//   /tmp/repro <ctas_per_sm 1|2> <busy 0|1|2 (2: bulk copies + mbarrier ring + DMMA)> <tiles> <jobs>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include <cuda_runtime.h>

constexpr int THREADS = 128, COLS = 64, ROWS = 128;  // one 128 x 64 tile per CTA

__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(unsigned* p, unsigned v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" :: "l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}

__global__ void __launch_bounds__(THREADS, 2)
repro(double* C, unsigned* sync, int tiles, int busy, const double* src) {
  extern __shared__ __align__(128) unsigned char ring[];
  __shared__ int s_ticket;
  if (threadIdx.x == 0) s_ticket = (int)atomicAdd(sync + tiles, 1u);
  __syncthreads();
  const int ticket = s_ticket, j = ticket / tiles, t = ticket % tiles;
  double acc = 0.0;
  if (busy == 2) {  // bulk async copies (the async proxy) into a 2-stage smem ring with mbarriers,
                   // fragments read from it into DMMAs -- the leaf's k loop in miniature
    __shared__ __align__(8) unsigned long long full[2];
    if (threadIdx.x == 0) {
      for (int i = 0; i < 2; ++i)
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(smem_u32(&full[i])) : "memory");
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const unsigned stage = 48 * 1024;
    double d0 = 0.0, d1 = 0.0;
    for (int it = 0; it < 64; ++it) {
      const int sl = it & 1;
      if (threadIdx.x == 0) {
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(smem_u32(&full[sl])),
                     "r"(stage) : "memory");
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                     :: "r"(smem_u32(ring + sl * stage)), "l"(src + (size_t)(it % 8) * (stage / 8)), "r"(stage),
                        "r"(smem_u32(&full[sl])) : "memory");
      }
      unsigned done = 0;
      while (!done)
        asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
                     "selp.u32 %0, 1, 0, p;\n\t}" : "=r"(done) : "r"(smem_u32(&full[sl])), "r"((it >> 1) & 1) : "memory");
      const double* f = reinterpret_cast<const double*>(ring + sl * stage);
      for (int k = 0; k < 32; ++k) {
        const double a = f[(threadIdx.x * 3 + k) % 6144], b = f[(threadIdx.x * 7 + k * 5) % 6144];
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                     : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
      }
      __syncthreads();
    }
    acc = (d0 + d1) * 0.0;
  } else if (busy) {  // some FP64 tensor work first, like the leaf's k loop
    double d0 = 1.0, d1 = 1.0;
    for (int k = 0; k < 4096; ++k)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(d0), "+d"(d1) : "d"(1e-9), "d"(1e-9));
    acc = (d0 + d1) * 0.0;
  }
  if (threadIdx.x == 0 && j > 0)
    while (ld_acquire(sync + t) < (unsigned)j) __nanosleep(64);
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int wm = warp / 2, wn = warp % 2;  // the leaf's 2 x 2 warp grid, 64 x 32 per warp
  double* base = C + (size_t)t * ROWS * COLS;
  for (int mi = 0; mi < 8; ++mi) {
    const int row = wm * 64 + mi * 8 + (lane >> 2);
    for (int nj = 0; nj < 2; ++nj) {
      const int col = wn * 32 + nj * 16 + 4 * (lane & 3);
      double* p = base + row * COLS + col;
      double v[4];
      asm volatile("ld.global.v2.f64 {%0, %1}, [%2];" : "=d"(v[0]), "=d"(v[1]) : "l"(p) : "memory");
      asm volatile("ld.global.v2.f64 {%0, %1}, [%2];" : "=d"(v[2]), "=d"(v[3]) : "l"(p + 2) : "memory");
      for (int u = 0; u < 4; ++u) v[u] += (double)(j + 1) + acc;
      asm volatile("st.global.v4.f64 [%0], {%1,%2,%3,%4};" :: "l"(p), "d"(v[0]), "d"(v[1]), "d"(v[2]),
                   "d"(v[3]) : "memory");
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    st_release(sync + t, (unsigned)j + 1);
  }
}

int main(int argc, char** argv) {
  const int per_sm = argc > 1 ? atoi(argv[1]) : 2, busy = argc > 2 ? atoi(argv[2]) : 0;
  const int tiles = argc > 3 ? atoi(argv[3]) : 128, jobs = argc > 4 ? atoi(argv[4]) : 49;
  const size_t n = (size_t)tiles * ROWS * COLS;
  double* C;
  unsigned* sync;
  double* src;
  cudaMalloc(&src, 1 << 20);
  cudaMemset(src, 0, 1 << 20);
  cudaMalloc(&C, n * 8);
  cudaMalloc(&sync, (tiles + 1) * 4);
  const int smem = per_sm == 1 ? 160 * 1024 : 96 * 1024;
  cudaFuncSetAttribute(repro, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  int bad_runs = 0;
  long long bad_total = 0;
  std::vector<double> h(n);
  for (int run = 0; run < 20; ++run) {
    cudaMemset(C, 0, n * 8);
    cudaMemset(sync, 0, (tiles + 1) * 4);
    repro<<<tiles * jobs, THREADS, smem>>>(C, sync, tiles, busy, src);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
    cudaMemcpy(h.data(), C, n * 8, cudaMemcpyDeviceToHost);
    const double expect = (double)jobs * (jobs + 1) / 2;
    long long bad = 0;
    for (size_t i = 0; i < n; ++i) bad += h[i] != expect;
    bad_runs += bad > 0;
    bad_total += bad;
  }
  printf("per_sm=%d busy=%d tiles=%d jobs=%d: %d of 20 runs wrong, %lld wrong elements\n", per_sm, busy,
         tiles, jobs, bad_runs, bad_total);
  return 0;
}
