// mf_tiny.cu -- the whole level of Eq. "strassen" in ONE
// launch for small problems (n <= 64, R^L <= 64): one thread-block cluster of
// up to 8 CTAs.  At these sizes the four launches of the general path (K4, K4,
// K5, K6) cost more than their work; here:
//   1. every CTA stages A and B in its shared memory;
//   2. CTA c computes the products q = c, c + CS, ...: T_q and S_q (ascending
//      k, the oracle's combination rule, as K4), then P_q = T_q S_q (fma,
//      k ascending) into its shared memory;
//   3. cluster barrier; every CTA pushes its products into every CTA's
//      gather area with bulk shared::cta -> shared::cluster copies that
//      complete on the receiver's mbarrier (distributed shared memory);
//   4. every thread of the cluster computes C elements
//      C_i = alpha * sum_q W[i][q] P_q (ascending q, as K6).
// The pre-/post-additions keep the oracle's per-element order (bit-exact like
// K4/K6); the leaf dot products are fma chains (pinned, like the DMMA leaf,
// by integer exactness and the error bound).
#include <cooperative_groups.h>

#include <algorithm>
#include <atomic>
#include <cstdlib>

#include "mf_internal.h"

namespace cg = cooperative_groups;

namespace mf {
namespace {

constexpr int TINY_THREADS = 256;

#ifdef MF_TINY_TRACE
// diagnostic build only (-DMF_TINY_TRACE): globaltimer stamps of CTA c's thread 0
__device__ unsigned long long g_tiny_trace[8][12];
__device__ __forceinline__ void tstamp(int i) {
  if (threadIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    g_tiny_trace[blockIdx.x & 7][i] = t;
  }
}
#define TSTAMP(i) tstamp(i)
#else
#define TSTAMP(i)
#endif

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// one term of an ascending combination, the oracle's rule (DESIGN R7):
// acc starts at -0.0; +-1 terms add / subtract, others multiply then add
// the same rule with the coefficient's kind decided outside the element loop
// (0 absent, 1: +x, 2: -x, 3: c*x): no floating-point compares per element
__device__ __forceinline__ int coef_kind(double c) {
  return c == 0.0 ? 0 : (c == 1.0 ? 1 : (c == -1.0 ? 2 : 3));
}
__device__ __forceinline__ double kterm(double acc, int kind, double c, double x) {
  return kind == 1 ? __dadd_rn(acc, x) : (kind == 2 ? __dadd_rn(acc, -x) : __dadd_rn(acc, __dmul_rn(c, x)));
}


__global__ void __launch_bounds__(TINY_THREADS)
tiny_kernel(const double* __restrict__ A, int64_t lda, const double* __restrict__ B, int64_t ldb,
            double* __restrict__ C, int64_t ldc, int n, int P, int R, const double* __restrict__ U,
            const double* __restrict__ V, const double* __restrict__ W, double alpha) {
  cg::cluster_group cluster = cg::this_cluster();
  const int cs = (int)cluster.num_blocks();
  const int me = (int)cluster.block_rank();
  const int m = n / P, mm = m * m, NB = P * P;
  const int per = (R + cs - 1) / cs;  // product slots per CTA
  extern __shared__ __align__(128) double sm[];
  // buffers start on 16-doubles (128-byte) boundaries: async / bulk copies
  auto up = [](int x) { return (x + 15) & ~15; };
  double* sU = sm;                      // NB x R coefficient tables
  double* sV = sU + up(NB * R);
  double* sW = sV + up(NB * R);
  double* sA = sW + up(NB * R);         // n x n
  double* sB = sA + up(n * n);          // n x n
  double* sT = sB + up(n * n);          // m x m
  double* sS = sT + up(mm);             // m x m
  double* sP = sS + up(mm);             // this CTA's products, slot j = product me + j*cs
  double* sAll = sP + per * up(mm);     // every product, gathered for the post-addition
  const int mmp = up(mm);               // product stride in sP / sAll

  TSTAMP(0);
  __shared__ __align__(8) uint64_t s_bar;  // gathered products landed
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(smem_addr(&s_bar)) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  // A, B: 16-byte asynchronous copies, all in flight at once, when rows allow
  const bool v2 = !(n & 1) && !(lda & 1) && !(ldb & 1) &&
                  !(reinterpret_cast<uintptr_t>(A) & 15) && !(reinterpret_cast<uintptr_t>(B) & 15);
  if (v2) {
    const int h = n / 2;
    for (int e = threadIdx.x; e < n * h; e += blockDim.x) {
      const int r = e / h, c = 2 * (e - r * h);
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;"
                   :: "r"(smem_addr(sA + r * n + c)), "l"(A + (int64_t)r * lda + c) : "memory");
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;"
                   :: "r"(smem_addr(sB + r * n + c)), "l"(B + (int64_t)r * ldb + c) : "memory");
    }
    for (int e = threadIdx.x; e < NB * R; e += blockDim.x) {
      sU[e] = U[e]; sV[e] = V[e]; sW[e] = W[e];
    }
    asm volatile("cp.async.wait_all;" ::: "memory");
  } else {
    for (int e = threadIdx.x; e < NB * R; e += blockDim.x) {
      sU[e] = U[e]; sV[e] = V[e]; sW[e] = W[e];
    }
    for (int e = threadIdx.x; e < n * n; e += blockDim.x) {
      const int r = e / n, c = e - r * n;
      sA[e] = A[(int64_t)r * lda + c];
      sB[e] = B[(int64_t)r * ldb + c];
    }
  }
  __syncthreads();
  TSTAMP(1);
  for (int q = me, j = 0; q < R; q += cs, ++j) {
    // T_q, S_q: block k of X is rows (k/P)*m.., cols (k%P)*m..;
    // the product's coefficients, their kinds and the block offsets sit in
    // registers while the threads sweep its elements (NB <= 16 here)
    double cu[16], cv[16];
    int ku[16], kv[16], boff[16];
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      cu[k] = k < NB ? sU[k * R + q] : 0.0;
      cv[k] = k < NB ? sV[k * R + q] : 0.0;
      ku[k] = coef_kind(cu[k]);
      kv[k] = coef_kind(cv[k]);
      boff[k] = k < NB ? (k / P) * m * n + (k % P) * m : 0;
    }
    for (int e = threadIdx.x; e < mm; e += blockDim.x) {
      const int r = e / m, c = e - r * m, rcn = r * n + c;
      double t = -0.0, s = -0.0;
#pragma unroll
      for (int k = 0; k < 16; ++k) {
        if (k >= NB) break;
        if (ku[k]) t = kterm(t, ku[k], cu[k], sA[boff[k] + rcn]);
        if (kv[k]) s = kterm(s, kv[k], cv[k], sB[boff[k] + rcn]);
      }
      sT[e] = t;
      sS[e] = s;
    }
    __syncthreads();
    if (j == 0) TSTAMP(2);
    double* Pq = sP + (size_t)j * mmp;
    if (!(m & 7)) {
      // P_q = T_q S_q on the FP64 tensor path: 8x8 tiles over the warps,
      // mma.sync.m8n8k4.f64 (DMMA) over k in steps of 4
      const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
      const int g = lane >> 2, tq = lane & 3, tiles = (m / 8) * (m / 8);
      for (int tile = warp; tile < tiles; tile += blockDim.x >> 5) {
        const int r0 = (tile / (m / 8)) * 8, c0 = (tile % (m / 8)) * 8;
        double d0 = 0.0, d1 = 0.0;
        for (int k = 0; k < m; k += 4) {
          const double a = sT[(r0 + g) * m + k + tq];
          const double b = sS[(k + tq) * m + c0 + g];
          asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
              : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
        }
        Pq[(r0 + g) * m + c0 + 2 * tq] = d0;
        Pq[(r0 + g) * m + c0 + 2 * tq + 1] = d1;
      }
      __syncthreads();
      continue;
    }
    // other m: up to 4 outputs per thread, four independent fma chains over
    // ascending k
    for (int e0 = threadIdx.x; e0 < mm; e0 += 4 * blockDim.x) {
      double acc[4] = {0.0, 0.0, 0.0, 0.0};
      int rr[4], cc[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int e = e0 + i * blockDim.x;
        rr[i] = e < mm ? e / m : 0;
        cc[i] = e < mm ? e - rr[i] * m : 0;
      }
      for (int k = 0; k < m; ++k) {
#pragma unroll
        for (int i = 0; i < 4; ++i) acc[i] = fma(sT[rr[i] * m + k], sS[k * m + cc[i]], acc[i]);
      }
#pragma unroll
      for (int i = 0; i < 4; ++i)
        if (e0 + i * (int)blockDim.x < mm) Pq[e0 + i * blockDim.x] = acc[i];
    }
    __syncthreads();
  }
  TSTAMP(3);
  // the products (generic-proxy stores) are read by bulk copies (async proxy)
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  cluster.sync();  // every CTA's products are complete and every barrier initialised
  TSTAMP(4);
  const uint32_t bytes = (uint32_t)mm * 8;
  if (!(bytes & 15)) {
    // push: thread d sends this CTA's products to CTA d's gather area with
    // bulk shared::cta -> shared::cluster copies, completing on d's barrier
    if (threadIdx.x == 0)
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;"
                   :: "r"(smem_addr(&s_bar)), "r"(bytes * (uint32_t)R) : "memory");
    if ((int)threadIdx.x < cs) {
      const uint32_t d = threadIdx.x;
      uint32_t rbar, rdst;
      asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(rbar) : "r"(smem_addr(&s_bar)), "r"(d));
      for (int q = me, j = 0; q < R; q += cs, ++j) {
        asm volatile("mapa.shared::cluster.u32 %0, %1, %2;"
                     : "=r"(rdst) : "r"(smem_addr(sAll + (size_t)q * mmp)), "r"(d));
        asm volatile(
            "cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
            :: "r"(rdst), "r"(smem_addr(sP + (size_t)j * mmp)), "r"(bytes), "r"(rbar) : "memory");
      }
    }
    uint32_t done = 0;
    while (!done)
      asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\t"
                   "selp.u32 %0, 1, 0, p;\n\t}" : "=r"(done) : "r"(smem_addr(&s_bar)) : "memory");
    // every CTA received everything, so every copy out of this CTA has been read
  } else {
    for (int q = 0; q < R; ++q) {
      const double* src = cluster.map_shared_rank(sP + (size_t)(q / cs) * mmp, q % cs);
      for (int e = threadIdx.x; e < mm; e += blockDim.x) sAll[(size_t)q * mmp + e] = src[e];
    }
  }
  TSTAMP(5);
  cluster.sync();  // no CTA leaves while another may still read its products
  TSTAMP(6);
  // C: element (i, r, c) of block i, ascending q (K6's order), alpha last
  const int tid = me * blockDim.x + threadIdx.x, nth = cs * blockDim.x;
  for (int e = tid; e < NB * mm; e += nth) {
    const int i = e / mm, rc = e - i * mm;
    double acc = -0.0;
    const double* wi = sW + i * R;
    for (int q = 0; q < R; ++q) {
      const double w = wi[q];
      const int kw = coef_kind(w);
      if (kw) acc = kterm(acc, kw, w, sAll[(size_t)q * mmp + rc]);
    }
    if (alpha != 1.0) acc = __dmul_rn(alpha, acc);
    const int r = rc / m, c = rc - r * m;
    C[(int64_t)((i / P) * m + r) * ldc + (i % P) * m + c] = acc;
  }
  TSTAMP(7);
}

}  // namespace

#ifdef MF_TINY_TRACE
extern "C" int mf_debug_tiny_trace(unsigned long long* out) {
  return (int)cudaMemcpyFromSymbol(out, g_tiny_trace, sizeof(unsigned long long) * 8 * 12);
}
#endif

size_t tiny_smem(const Plan& pl);

bool tiny_eligible(const Plan& pl) {
  return pl.levels > 0 && pl.n <= 64 && pl.RL <= 64 && !pl.child && pl.batches.empty() &&
         !pl.fuse && pl.shard_count == 1 && !pl.comm && pl.leaf == MF_LEAF_DMMA &&
         pl.d_tinyU != nullptr && (int64_t)pl.P * pl.P <= 16 && tiny_smem(pl) <= 200 * 1024;
}

static int tiny_cluster(const Plan& pl) {
  int cs = (int)std::min<int64_t>(8, pl.RL);
  if (const char* e = getenv("MF_TINY_CS")) cs = std::max(1, std::min(cs, atoi(e)));  // experiment
  return cs;
}

size_t tiny_smem(const Plan& pl) {
  const int cs = tiny_cluster(pl);
  auto up = [](int64_t x) { return (x + 15) & ~int64_t(15); };
  const int64_t mm = up(pl.m * pl.m), NB = (int64_t)pl.P * pl.P;
  return sizeof(double) * (3 * up(NB * pl.RL) + 2 * up(pl.n * pl.n) + 2 * mm +
                           ((pl.RL + cs - 1) / cs) * mm + pl.RL * mm);
}

cudaError_t launch_tiny(const Plan& pl, double alpha, const double* A, int64_t lda, const double* B,
                        int64_t ldb, double* C, int64_t ldc, cudaStream_t s) {
  const int cs = tiny_cluster(pl);
  const size_t smem = tiny_smem(pl);
  static std::atomic<uint64_t> opted{0};  // >48 KB opt-in, once per device
  int dev = 0;
  cudaGetDevice(&dev);
  if (!(opted.load() & (1ull << (dev & 63)))) {
    cudaError_t e = cudaFuncSetAttribute(tiny_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         200 * 1024);
    if (e != cudaSuccess) return e;
    opted.fetch_or(1ull << (dev & 63));
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(cs, 1, 1);
  cfg.blockDim = dim3(TINY_THREADS, 1, 1);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = cs;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, tiny_kernel, A, lda, B, ldb, C, ldc, (int)pl.n, pl.P, (int)pl.RL,
                            (const double*)pl.d_tinyU, (const double*)pl.d_tinyV,
                            (const double*)pl.d_tinyW, alpha);
}

}  // namespace mf
