// mf_mix.cu -- K4 (fused pre-addition) and K6 (fused post-addition).
//
// Both are the linear-combination steps of Eq. "strassen":
//   K4:  X_s = sum_k M[k][q_s] * Blk_k(X)      (T_q from A with U, S_q from B with V)
//   K6:  C_i = alpha * sum_q W'[i][q] * P_q'     (W' = W with aliased signs folded in)
// computed for ALL outputs of a level in ONE pass over HBM: each thread owns
// one VW-wide vector position (r, c) inside an m x m block, loads that
// position of every input block once (256-bit ld.global.nc.v4.f64 on
// sm_100a), and writes that position of every output.  HBM-bound: the
// algorithmic traffic is (#inputs read + #outputs written) * 8 * m^2 bytes.
//
// Summation order is fixed -- first nonzero term c0*X_{k0}, then
// acc = acc + c*X_k in ascending k (q for K6), separate multiply and add
// (__dmul_rn/__dadd_rn, never contracted), alpha applied last -- the order
// the oracle uses (reading R7/R8), so K4/K6 are bit-exact with it.
#include "mf_internal.h"

namespace mf {
namespace {

template <int VW> struct Vec { double v[VW]; };

template <int VW>
__device__ __forceinline__ Vec<VW> load_vec(const double* p) {
  Vec<VW> r;
  if constexpr (VW == 4) {
    asm volatile("ld.global.nc.L1::no_allocate.v4.f64 {%0,%1,%2,%3}, [%4];"
                 : "=d"(r.v[0]), "=d"(r.v[1]), "=d"(r.v[2]), "=d"(r.v[3]) : "l"(p));
  } else if constexpr (VW == 2) {
    asm volatile("ld.global.nc.L1::no_allocate.v2.f64 {%0,%1}, [%2];"
                 : "=d"(r.v[0]), "=d"(r.v[1]) : "l"(p));
  } else {
    r.v[0] = __ldg(p);
  }
  return r;
}

template <int VW>
__device__ __forceinline__ void store_vec(double* p, const Vec<VW>& x) {
  if constexpr (VW == 4) {
    asm volatile("st.global.v4.f64 [%0], {%1,%2,%3,%4};"
                 :: "l"(p), "d"(x.v[0]), "d"(x.v[1]), "d"(x.v[2]), "d"(x.v[3]) : "memory");
  } else if constexpr (VW == 2) {
    asm volatile("st.global.v2.f64 [%0], {%1,%2};" :: "l"(p), "d"(x.v[0]), "d"(x.v[1]) : "memory");
  } else {
    p[0] = x.v[0];
  }
}

// K4: pre-addition.  coef: nout x (P*P) (row o = output o), slot[o] = the
// workspace block output o writes (out + slot[o]*m*m, ld m).
template <int P, int VW>
__global__ void __launch_bounds__(256) premix_kernel(const double* __restrict__ X, int64_t ldx,
                                                     int64_t m, const double* __restrict__ coef,
                                                     const int32_t* __restrict__ slot, int nout,
                                                     double* __restrict__ out) {
  constexpr int NB = P * P;
  extern __shared__ double s_coef[];
  for (int i = threadIdx.x; i < nout * NB; i += blockDim.x) s_coef[i] = coef[i];
  __syncthreads();
  const int64_t vpr = m / VW;  // vectors per row
  const int64_t total = m * vpr;
  const int64_t mm = m * m;
  for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = idx / vpr;
    const int64_t c = (idx - r * vpr) * VW;
    Vec<VW> x[NB];
#pragma unroll
    for (int k = 0; k < NB; ++k)
      x[k] = load_vec<VW>(X + ((k / P) * m + r) * ldx + (k % P) * m + c);
    for (int o = 0; o < nout; ++o) {
      Vec<VW> acc;
      bool first = true;
#pragma unroll
      for (int k = 0; k < NB; ++k) {
        const double cf = s_coef[o * NB + k];
        if (cf != 0.0) {
#pragma unroll
          for (int e = 0; e < VW; ++e)
            acc.v[e] = first ? __dmul_rn(cf, x[k].v[e]) : __dadd_rn(acc.v[e], __dmul_rn(cf, x[k].v[e]));
          first = false;
        }
      }
      store_vec<VW>(out + (int64_t)slot[o] * mm + r * m + c, acc);
    }
  }
}

// K6: post-addition.  w: (P*P) x RL (row i = C block i); column q is zero
// for products outside this plan's shard.  active[q] != 0 iff column q has
// a nonzero.  C_i = alpha * sum_q w[i][q] * P_q (a C block without terms is 0).
template <int P, int VW>
__global__ void __launch_bounds__(256) postmix_kernel(const double* __restrict__ Pw, int64_t m,
                                                      int64_t RL, const double* __restrict__ w,
                                                      double alpha, double* __restrict__ C,
                                                      int64_t ldc) {
  constexpr int NB = P * P;
  extern __shared__ double s_w[];  // NB x RL, then RL activity flags (as doubles)
  for (int64_t i = threadIdx.x; i < NB * RL; i += blockDim.x) s_w[i] = w[i];
  __syncthreads();
  const int64_t vpr = m / VW;
  const int64_t total = m * vpr;
  const int64_t mm = m * m;
  for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = idx / vpr;
    const int64_t c = (idx - r * vpr) * VW;
    Vec<VW> acc[NB];
    bool first[NB];
#pragma unroll
    for (int i = 0; i < NB; ++i) {
      first[i] = true;
#pragma unroll
      for (int e = 0; e < VW; ++e) acc[i].v[e] = 0.0;
    }
    for (int64_t q = 0; q < RL; ++q) {
      bool any = false;
#pragma unroll
      for (int i = 0; i < NB; ++i) any |= (s_w[i * RL + q] != 0.0);
      if (!any) continue;
      const Vec<VW> x = load_vec<VW>(Pw + q * mm + r * m + c);
#pragma unroll
      for (int i = 0; i < NB; ++i) {
        const double cf = s_w[i * RL + q];
        if (cf != 0.0) {
#pragma unroll
          for (int e = 0; e < VW; ++e)
            acc[i].v[e] = first[i] ? __dmul_rn(cf, x.v[e]) : __dadd_rn(acc[i].v[e], __dmul_rn(cf, x.v[e]));
          first[i] = false;
        }
      }
    }
#pragma unroll
    for (int i = 0; i < NB; ++i) {
      if (alpha != 1.0) {
#pragma unroll
        for (int e = 0; e < VW; ++e) acc[i].v[e] = __dmul_rn(alpha, acc[i].v[e]);
      }
      store_vec<VW>(C + ((i / P) * m + r) * ldc + (i % P) * m + c, acc[i]);
    }
  }
}

int grid_for(int64_t work) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  int64_t blocks = (work + 255) / 256;
  int64_t cap = (int64_t)sms * 8;  // 8 x 256 threads resident per SM
  return (int)(blocks < cap ? (blocks < 1 ? 1 : blocks) : cap);
}

bool aligned(const void* p, int bytes) { return ((uintptr_t)p % bytes) == 0; }

template <int P, int VW>
cudaError_t premix_launch(const MixTable& t, const double* X, int64_t ldx, int64_t m, double* out,
                          const int32_t* d_slot, cudaStream_t s) {
  constexpr int NB = P * P;
  size_t smem = sizeof(double) * (size_t)t.nout * NB;
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(premix_kernel<P, VW>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
  }
  premix_kernel<P, VW><<<grid_for(m * (m / VW)), 256, smem, s>>>(X, ldx, m, t.d_coef, d_slot,
                                                                  t.nout, out);
  return cudaGetLastError();
}

template <int P, int VW>
cudaError_t postmix_launch(const Plan& pl, double alpha, const double* Pw, double* C, int64_t ldc,
                           cudaStream_t s) {
  constexpr int NB = P * P;
  size_t smem = sizeof(double) * (size_t)NB * pl.RL;
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(postmix_kernel<P, VW>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
  }
  postmix_kernel<P, VW><<<grid_for(pl.m * (pl.m / VW)), 256, smem, s>>>(
      Pw, pl.m, pl.RL, pl.mixC.d_coef, alpha, C, ldc);
  return cudaGetLastError();
}

}  // namespace

// Vector width: 256-bit when every row start is 32-byte aligned, else 128/64-bit.
static int pick_vw(int P, int64_t m, std::initializer_list<std::pair<const void*, int64_t>> views) {
  int max_vw = P <= 4 ? 4 : (P <= 6 ? 2 : 1);
  for (int vw = max_vw; vw > 1; vw /= 2) {
    bool ok = (m % vw) == 0;
    for (auto& v : views) ok = ok && aligned(v.first, 8 * vw) && (v.second % vw) == 0;
    if (ok) return vw;
  }
  return 1;
}

#define MF_DISPATCH_P(P_, VW_, CALL)                                   \
  switch (P_) {                                                        \
    case 1: CALL(1, VW_); break;                                       \
    case 2: CALL(2, VW_); break;                                       \
    case 3: CALL(3, VW_); break;                                       \
    case 4: CALL(4, VW_); break;                                       \
    default: return cudaErrorInvalidValue;                             \
  }

cudaError_t launch_premix(const Plan& pl, const MixTable& t, const double* X, int64_t ldx,
                          double* out, cudaStream_t s) {
  if (t.nout == 0) return cudaSuccess;
  const int32_t* d_slot = reinterpret_cast<const int32_t*>(t.d_coef + (size_t)t.nout * t.nin);
  int vw = pick_vw(pl.P, pl.m, {{X, ldx}, {out, pl.m}});
#define PRE(P_, VW_) return premix_launch<P_, VW_>(t, X, ldx, pl.m, out, d_slot, s)
  if (pl.P == 6) { if (vw >= 2) PRE(6, 2); PRE(6, 1); }
  if (pl.P == 8) PRE(8, 1);
  if (pl.P == 9) PRE(9, 1);
  if (vw == 4) { MF_DISPATCH_P(pl.P, 4, PRE); }
  else if (vw == 2) { MF_DISPATCH_P(pl.P, 2, PRE); }
  else { MF_DISPATCH_P(pl.P, 1, PRE); }
#undef PRE
  return cudaErrorInvalidValue;
}

cudaError_t launch_postmix(const Plan& pl, double alpha, const double* Pw, double* C, int64_t ldc,
                           cudaStream_t s) {
  int vw = pick_vw(pl.P, pl.m, {{Pw, pl.m}, {C, ldc}});
#define POST(P_, VW_) return postmix_launch<P_, VW_>(pl, alpha, Pw, C, ldc, s)
  if (pl.P == 6) { if (vw >= 2) POST(6, 2); POST(6, 1); }
  if (pl.P == 8) POST(8, 1);
  if (pl.P == 9) POST(9, 1);
  if (vw == 4) { MF_DISPATCH_P(pl.P, 4, POST); }
  else if (vw == 2) { MF_DISPATCH_P(pl.P, 2, POST); }
  else { MF_DISPATCH_P(pl.P, 1, POST); }
#undef POST
  return cudaErrorInvalidValue;
}

}  // namespace mf
