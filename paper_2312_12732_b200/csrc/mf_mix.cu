// mf_mix.cu -- K4 (fused pre-addition) and K6 (fused post-addition).
//
// Both are the linear-combination steps of Eq. "strassen":
//   K4:  X_s = sum_k M[k][q_s] * Blk_k(X)      (T_q from A with U, S_q from B with V)
//   K6:  C_i = alpha * sum_q W'[i][q] * P_q'     (W' = W with aliased signs folded in)
// computed for ALL outputs of a level in ONE launch: a CTA owns a segment of
// positions and produces every output for it, so each input element comes
// from HBM once (re-reads by other outputs hit L1) and each output is written
// once (256-bit ld/st.global.v4.f64 on sm_100a).  HBM-bound: the algorithmic
// traffic is (#inputs read + #outputs written) * 8 * m^2 bytes.
//
// Summation order is fixed -- first nonzero term c0*X_{k0}, then
// acc = acc + c*X_k in ascending k (q for K6), separate multiply and add
// (__dmul_rn/__dadd_rn, never contracted), alpha applied last -- the order
// the oracle uses (reading R7/R8), so K4/K6 are bit-exact with it.
// Coefficients arrive as warp-uniform term lists: +-1 terms cost one add.
#include <algorithm>
#include <cstdlib>

#include "mf_internal.h"

namespace mf {
namespace {

template <int VW> struct Vec { double v[VW]; };

// Streaming 256/128-bit loads that bypass L1 (inputs read exactly once).
template <int VW>
__device__ __forceinline__ Vec<VW> load_stream(const double* p) {
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

// L1-allocating loads (inputs re-read by other warps of the CTA).
template <int VW>
__device__ __forceinline__ Vec<VW> load_vec(const double* p) {
  Vec<VW> r;
  if constexpr (VW == 4) {
    asm volatile("ld.global.nc.v4.f64 {%0,%1,%2,%3}, [%4];"
                 : "=d"(r.v[0]), "=d"(r.v[1]), "=d"(r.v[2]), "=d"(r.v[3]) : "l"(p));
  } else if constexpr (VW == 2) {
    asm volatile("ld.global.nc.v2.f64 {%0,%1}, [%2];"
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

// One term of a combination: acc = acc + c*x.  c = +-1 is a single
// (negated) add -- bitwise the oracle's separate mul-then-add, since (+-1)*x
// is exact; other c multiply first (__dmul_rn, never contracted).
// Accumulators start at -0.0: (-0.0) + v == v for every v (signed zeros
// included), so the first term needs no special case.
template <int VW>
__device__ __forceinline__ void add_term(Vec<VW>& acc, const Vec<VW>& x, int kind, double cf) {
#pragma unroll
  for (int e = 0; e < VW; ++e) {
    const double v = kind == MIX_GEN ? __dmul_rn(cf, x.v[e]) : (kind == MIX_NEG ? -x.v[e] : x.v[e]);
    acc.v[e] = __dadd_rn(acc.v[e], v);
  }
}

// Address of element (r, c) of block/slot `id` in a view: a block view is the
// P x P partition of a matrix with leading dimension ld (id = br*P + bc); a
// slot view is a [slots][m][m] workspace.
struct View {
  double* base;
  int64_t ld;
  int P;         // 0 => slot view
  __device__ __forceinline__ double* at(int id, int64_t m, int64_t r, int64_t c) const {
    if (P == 0) return base + (int64_t)id * m * m + r * m + c;
    return base + ((int64_t)(id / P) * m + r) * ld + (int64_t)(id % P) * m + c;
  }
};

// General K4/K6: out_o = alpha * sum_t coef_t * in_{src_t}, for every output
// row o of the MixRow table, over every position of the m x m blocks.  A CTA
// owns a segment of 32*VW consecutive positions of one row r; warp w
// computes outputs w, w+8, ... for that segment along warp-uniform term
// lists (coalesced 1 KB loads/stores per warp; no data-dependent register
// indexing, no divergence).  Inputs are loaded with L1 allocation so the
// re-reads of an input block by the CTA's other outputs hit L1.  Any split
// factor, any number of terms.
template <int VW>
__global__ void __launch_bounds__(256) mix_kernel(View in, View out, int64_t m,
                                                  const void* __restrict__ table, int nrow,
                                                  int nterm, double alpha, int64_t r0,
                                                  int64_t r1, int64_t c0, int64_t c1,
                                                  int accumulate) {
  extern __shared__ __align__(16) uint8_t s_raw[];
  const size_t tbytes = sizeof(MixRow) * nrow + sizeof(MixTerm) * nterm;
  for (size_t i = threadIdx.x; i < tbytes / 8; i += blockDim.x)
    reinterpret_cast<uint64_t*>(s_raw)[i] = reinterpret_cast<const uint64_t*>(table)[i];
  __syncthreads();
  const MixRow* rows = reinterpret_cast<const MixRow*>(s_raw);
  const MixTerm* terms = reinterpret_cast<const MixTerm*>(rows + nrow);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  constexpr int SEG = 32 * VW;
  const int64_t segs_per_row = (c1 - c0 + SEG - 1) / SEG;
  const int64_t total = (r1 - r0) * segs_per_row;
  for (int64_t seg = blockIdx.x; seg < total; seg += gridDim.x) {
    const int64_t rr = seg / segs_per_row;
    const int64_t r = r0 + rr;
    const int64_t c = c0 + (seg - rr * segs_per_row) * SEG + lane * VW;
    if (c >= c1) continue;
    for (int o = warp; o < nrow; o += 8) {
      const MixRow row = rows[o];
      Vec<VW> acc;
#pragma unroll
      for (int e = 0; e < VW; ++e) acc.v[e] = -0.0;
      int t = row.first;
      const int tend = row.first + row.count;
      for (; t + 1 < tend; t += 2) {  // two loads in flight per step
        const MixTerm t0 = terms[t], t1 = terms[t + 1];
        const Vec<VW> x0 = load_vec<VW>(in.at(t0.src, m, r, c));
        const Vec<VW> x1 = load_vec<VW>(in.at(t1.src, m, r, c));
        add_term<VW>(acc, x0, t0.kind, t0.coef);
        add_term<VW>(acc, x1, t1.kind, t1.coef);
      }
      if (t < tend) {
        const MixTerm t0 = terms[t];
        add_term<VW>(acc, load_vec<VW>(in.at(t0.src, m, r, c)), t0.kind, t0.coef);
      }
      if (alpha != 1.0) {
#pragma unroll
        for (int e = 0; e < VW; ++e) acc.v[e] = __dmul_rn(alpha, acc.v[e]);
      }
      double* dst = out.at(row.target, m, r, c);
      if (accumulate) {  // bounded-workspace batches after the first: C += batch sum
        const Vec<VW> old = load_vec<VW>(dst);
#pragma unroll
        for (int e = 0; e < VW; ++e) acc.v[e] = __dadd_rn(old.v[e], acc.v[e]);
      }
      store_vec<VW>(dst, acc);
    }
  }
}

// Grouped K4/K6 (default when the table fits): warp w owns output groups
// w, w+8, ...; for each input in its group's union (ascending), it loads the
// input once and adds it into every member that uses it (warp-uniform
// coefficients from shared memory, zero = absent).  Each output still sums
// its own terms in ascending input order -- the oracle's order, bit-exact --
// but a CTA now reads each input about once per group instead of once per
// term, which is what bounded the term-list kernel (on-chip traffic, not HBM).
template <int VW, int G>
__global__ void __launch_bounds__(256) mix_group_kernel(View in, View out, int64_t m,
                                                        const void* __restrict__ table,
                                                        int ngroup, int tbytes, double alpha,
                                                        int64_t r0, int64_t r1, int64_t c0,
                                                        int64_t c1, int accumulate) {
  extern __shared__ __align__(16) uint8_t s_raw[];
  for (int i = threadIdx.x; i < tbytes / 8; i += blockDim.x)
    reinterpret_cast<uint64_t*>(s_raw)[i] = reinterpret_cast<const uint64_t*>(table)[i];
  __syncthreads();
  const MixGroup* groups = reinterpret_cast<const MixGroup*>(s_raw);
  const uint8_t* ents = reinterpret_cast<const uint8_t*>(groups + ngroup);
  constexpr int STRIDE = 8 + 8 * G;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  constexpr int SEG = 32 * VW;
  const int64_t segs_per_row = (c1 - c0 + SEG - 1) / SEG;
  const int64_t total = (r1 - r0) * segs_per_row;
  for (int64_t seg = blockIdx.x; seg < total; seg += gridDim.x) {
    const int64_t rr = seg / segs_per_row;
    const int64_t r = r0 + rr;
    const int64_t c = c0 + (seg - rr * segs_per_row) * SEG + lane * VW;
    if (c >= c1) continue;
    for (int g = warp; g < ngroup; g += 8) {
      const int first = groups[g].first, count = groups[g].count;
      Vec<VW> acc[G];
#pragma unroll
      for (int j = 0; j < G; ++j)
#pragma unroll
        for (int e = 0; e < VW; ++e) acc[j].v[e] = -0.0;
      auto apply = [&](const uint8_t* en, const Vec<VW>& x) {
        const double* cf = reinterpret_cast<const double*>(en + 8);
#pragma unroll
        for (int j = 0; j < G; ++j) {
          const double cj = cf[j];
          if (cj == 1.0) {
            add_term<VW>(acc[j], x, MIX_POS, cj);
          } else if (cj == -1.0) {
            add_term<VW>(acc[j], x, MIX_NEG, cj);
          } else if (cj != 0.0) {
            add_term<VW>(acc[j], x, MIX_GEN, cj);
          }
        }
      };
      int e = 0;
      for (; e + 1 < count; e += 2) {  // two loads in flight per step
        const uint8_t* e0 = ents + (size_t)(first + e) * STRIDE;
        const uint8_t* e1 = e0 + STRIDE;
        const Vec<VW> x0 = load_vec<VW>(in.at(*reinterpret_cast<const int32_t*>(e0), m, r, c));
        const Vec<VW> x1 = load_vec<VW>(in.at(*reinterpret_cast<const int32_t*>(e1), m, r, c));
        apply(e0, x0);
        apply(e1, x1);
      }
      if (e < count) {
        const uint8_t* e0 = ents + (size_t)(first + e) * STRIDE;
        apply(e0, load_vec<VW>(in.at(*reinterpret_cast<const int32_t*>(e0), m, r, c)));
      }
#pragma unroll
      for (int j = 0; j < G; ++j) {
        const int target = groups[g].target[j];
        if (target < 0) continue;
        Vec<VW> v = acc[j];
        if (alpha != 1.0) {
#pragma unroll
          for (int q = 0; q < VW; ++q) v.v[q] = __dmul_rn(alpha, v.v[q]);
        }
        double* dst = out.at(target, m, r, c);
        if (accumulate) {
          const Vec<VW> old = load_vec<VW>(dst);
#pragma unroll
          for (int q = 0; q < VW; ++q) v.v[q] = __dadd_rn(old.v[q], v.v[q]);
        }
        store_vec<VW>(dst, v);
      }
    }
  }
}

bool aligned(const void* p, int bytes) { return ((uintptr_t)p % bytes) == 0; }

// Grid: `work` items of `per_block` each, capped at 8 CTAs (of 256 threads) per SM.
int grid_for(int64_t work, int per_block) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t blocks = (work + per_block - 1) / per_block;
  const int64_t cap = (int64_t)sms * 8;
  return (int)(blocks < cap ? (blocks < 1 ? 1 : blocks) : cap);
}

template <int VW>
cudaError_t mix_launch(const MixTable& t, View in, View out, int64_t m, double alpha, cudaStream_t s,
                       int64_t r0, int64_t r1, int64_t c0, int64_t c1, int accumulate) {
  const size_t smem = sizeof(MixRow) * t.nrow + sizeof(MixTerm) * t.nterm;
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(mix_kernel<VW>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem);
    if (e != cudaSuccess) return e;
  }
  mix_kernel<VW><<<grid_for((r1 - r0) * ((c1 - c0 + 32 * VW - 1) / (32 * VW)), 1), 256, smem, s>>>(
      in, out, m, t.d_table, t.nrow, t.nterm, alpha, r0, r1, c0, c1, accumulate);
  return cudaGetLastError();
}

}  // namespace

// Vector width: 256-bit when every row start is 32-byte aligned, else 128/64-bit.
static int pick_vw(int64_t m, std::initializer_list<std::pair<const void*, int64_t>> views) {
  int max_vw = 4;
  if (const char* e = getenv("MF_MIX_VW")) {  // tuning knob for experiments: 1, 2 or 4
    const int v = atoi(e);
    if (v == 1 || v == 2 || v == 4) max_vw = v;
  }
  for (int vw = max_vw; vw > 1; vw /= 2) {
    bool ok = (m % vw) == 0;
    for (auto& v : views) ok = ok && aligned(v.first, 8 * vw) && (v.second % vw) == 0;
    if (ok) return vw;
  }
  return 1;
}

template <int VW, int G>
static cudaError_t group_launch(const MixTable& t, View in, View out, int64_t m, double alpha,
                               cudaStream_t s, int64_t r0, int64_t r1, int64_t c0, int64_t c1,
                               int accumulate) {
  const int smem = (int)t.gbytes;
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(mix_group_kernel<VW, G>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
  }
  mix_group_kernel<VW, G><<<grid_for((r1 - r0) * ((c1 - c0 + 32 * VW - 1) / (32 * VW)), 1), 256,
                            smem, s>>>(in, out, m, static_cast<const uint8_t*>(t.d_table) + t.goff,
                                       t.ngroup, smem, alpha, r0, r1, c0, c1, accumulate);
  return cudaGetLastError();
}

template <int VW>
static cudaError_t group_dispatch(const MixTable& t, View in, View out, int64_t m, double alpha,
                                  cudaStream_t s, int64_t r0, int64_t r1, int64_t c0, int64_t c1,
                                  int accumulate) {
  switch (t.gsize) {
    case 1: return group_launch<VW, 1>(t, in, out, m, alpha, s, r0, r1, c0, c1, accumulate);
    case 2: return group_launch<VW, 2>(t, in, out, m, alpha, s, r0, r1, c0, c1, accumulate);
    case 3: return group_launch<VW, 3>(t, in, out, m, alpha, s, r0, r1, c0, c1, accumulate);
    default: return group_launch<VW, 4>(t, in, out, m, alpha, s, r0, r1, c0, c1, accumulate);
  }
}

static cudaError_t mix_dispatch(int vw, const MixTable& t, View in, View out, int64_t m,
                                double alpha, cudaStream_t s, Rows rows, int accumulate = 0) {
  if (t.nrow == 0) return cudaSuccess;
  const int64_t r0 = rows.r0, r1 = rows.end(m), c0 = rows.c0, c1 = rows.cend(m);
  if (r1 <= r0 || c1 <= c0) return cudaSuccess;
  if (t.gsize > 0) {
    if (vw == 4) return group_dispatch<4>(t, in, out, m, alpha, s, r0, r1, c0, c1, accumulate);
    if (vw == 2) return group_dispatch<2>(t, in, out, m, alpha, s, r0, r1, c0, c1, accumulate);
    return group_dispatch<1>(t, in, out, m, alpha, s, r0, r1, c0, c1, accumulate);
  }
  if (vw == 4) return mix_launch<4>(t, in, out, m, alpha, s, r0, r1, c0, c1, accumulate);
  if (vw == 2) return mix_launch<2>(t, in, out, m, alpha, s, r0, r1, c0, c1, accumulate);
  return mix_launch<1>(t, in, out, m, alpha, s, r0, r1, c0, c1, accumulate);
}

cudaError_t launch_premix(const Plan& pl, const MixTable& t, const double* X, int64_t ldx,
                          double* out, cudaStream_t s, Rows rows) {
  if (t.nrow == 0 || rows.end(pl.m) <= rows.r0 || rows.cend(pl.m) <= rows.c0) return cudaSuccess;
  // specialised kernels serve the plan's own tables (unsharded plans: a shard's
  // tables use local slot numbering and run generated kernels)
  const bool own = &t == &pl.mixA || &t == &pl.mixA2 || &t == &pl.mixB;
  if (pl.fixed_id > 0 && own) {
    const int side = &t == &pl.mixB ? 1 : 0;
    const ProdMask& mask = &t == &pl.mixA ? pl.mask_whole : (&t == &pl.mixA2 ? pl.mask_part : pl.mask_all);
    if (pl.fixed_id >= 8)
      return ++pl.mix_launches[MIXK_KRON], launch_premix_kron(pl.fixed_id, side, X, ldx, pl.m, out, s, rows, mask);
    if (fixed_vw4_ok(pl.m, X, ldx, out, pl.m))
      return ++pl.mix_launches[MIXK_FIXED],
             launch_premix_fixed(pl.fixed_id, side, X, ldx, pl.m, out, s, rows, mask);
  }
  const cudaError_t j = jit_launch(t, X, ldx, out, pl.m, pl.m, 1.0, rows, 0, s);
  if (j != cudaErrorNotSupported) return ++pl.mix_launches[MIXK_JIT], j;
  ++pl.mix_launches[MIXK_TABLE];
  const int vw = pick_vw(pl.m, {{X, ldx}, {out, pl.m}});
  return mix_dispatch(vw, t, View{const_cast<double*>(X), ldx, pl.P}, View{out, pl.m, 0}, pl.m,
                      1.0, s, rows);
}

cudaError_t launch_postmix(const Plan& pl, const MixTable& t, double alpha, const double* Pw,
                           double* C, int64_t ldc, cudaStream_t s, Rows rows, bool accumulate) {
  if (rows.end(pl.m) <= rows.r0 || rows.cend(pl.m) <= rows.c0) return cudaSuccess;
  if (pl.fixed_id > 0 && !accumulate && (&t == &pl.mixC || &t == &pl.mixC2)) {
    const ProdMask& mask = &t == &pl.mixC ? pl.mask_whole : pl.mask_all;
    if (pl.fixed_id >= 8)
      return ++pl.mix_launches[MIXK_KRON], launch_postmix_kron(pl.fixed_id, Pw, pl.m, alpha, C, ldc, s, rows, mask);
    if (fixed_vw4_ok(pl.m, Pw, pl.m, C, ldc))
      return ++pl.mix_launches[MIXK_FIXED],
             launch_postmix_fixed(pl.fixed_id, Pw, pl.m, alpha, C, ldc, s, rows, mask);
  }
  const cudaError_t j = jit_launch(t, Pw, pl.m, C, ldc, pl.m, alpha, rows, accumulate ? 1 : 0, s);
  if (j != cudaErrorNotSupported) return ++pl.mix_launches[MIXK_JIT], j;
  ++pl.mix_launches[MIXK_TABLE];
  const int vw = pick_vw(pl.m, {{Pw, pl.m}, {C, ldc}});
  return mix_dispatch(vw, t, View{const_cast<double*>(Pw), pl.m, 0}, View{C, ldc, pl.P},
                      pl.m, alpha, s, rows, accumulate ? 1 : 0);
}

}  // namespace mf
