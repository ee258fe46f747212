// mf_kron.cu -- K4/K6 for Kronecker powers of a catalog triple, evaluated
// level by level (Kronecker-factored) instead of over the flattened table.
//
// For <U,V,W> = <u,v,w>^(x)L the flattened combination
//   T_(q1..qL) = sum_(k1..kL) u[k1][q1]...u[kL][qL] A_(k1..kL)
// factors into L small combinations.  Evaluated OUTER level first for K4
// and INNER level first for K6, this is exactly the order the paper's
// recursion uses ("compute the operands T_i and S_i first,
// recursively solve the result P_i and distribute it") -- so these kernels
// are bitwise the recursion interpreter's pre/post-additions (or_fmm), while
// the leaf products stay flattened (one launch over all R^L products).
//
// Work per element is sum over levels of R^l * nnz instead of R^L * nnz^L,
// and only the base table (p^2 x R) is needed at compile time, which keeps
// <8,8,8;343> and <9,9,9;529> compilable (the flattened fold of mf_fixed.cu
// is not).  Each thread owns one position (r, c) of the m x m blocks, loads
// that position of all p^(2L) input blocks into registers (VW = 1: 64 or 81
// registers), and walks the level tree with the intermediate sums in
// registers.  Accumulators start at -0.0 (bitwise the first-term rule).
#include <cstdint>
#include <utility>

#include "mf_internal.h"
#include "mf_tables.h"

namespace mf {
namespace kronmix {

using fixed::Tri;

template <int B, int E>
struct ipow { static constexpr int v = B * ipow<B, E - 1>::v; };
template <int B>
struct ipow<B, 0> { static constexpr int v = 1; };

// base coefficient (side 0: U, 1: V, 2: W) as a compile-time scalar
template <class Tag, int SIDE, int K, int Q>
inline constexpr int coef = SIDE == 0 ? Tag::T.U[K][Q] : (SIDE == 1 ? Tag::T.V[K][Q] : Tag::T.W[K][Q]);

template <int NB, int R>
constexpr bool single(const int8_t (&M)[NB][R], int q) {  // one +-1 entry
  int nz = 0, v = 0;
  for (int k = 0; k < NB; ++k)
    if (M[k][q]) { ++nz; v = M[k][q]; }
  return nz == 1 && (v == 1 || v == -1);
}
template <int NB, int R>
constexpr bool single_pos(const int8_t (&M)[NB][R], int q) {
  for (int k = 0; k < NB; ++k)
    if (M[k][q]) return M[k][q] == 1;
  return true;
}

// Flattened product q (base-R digits q1..qL, outer first) aliases its A (B)
// block iff every level's column is a single +-1 (mf_plan's rule).
template <class Tag, int SIDE, int L>
constexpr bool aliased(int q) {
  constexpr int R = Tag::R;
  for (int l = 0; l < L; ++l) {
    const int ql = q % R;
    q /= R;
    if (!single(SIDE == 0 ? Tag::T.U : Tag::T.V, ql)) return false;
  }
  return true;
}

template <class Tag, int SIDE, int L>
struct Slots {
  int slot[ipow<Tag::R, L>::v];
};
template <class Tag, int SIDE, int L>
constexpr Slots<Tag, SIDE, L> make_slots() {
  Slots<Tag, SIDE, L> s{};
  int next = 0;
  for (int q = 0; q < ipow<Tag::R, L>::v; ++q) s.slot[q] = aliased<Tag, SIDE, L>(q) ? -1 : next++;
  return s;
}
template <class Tag, int SIDE, int L>
inline constexpr Slots<Tag, SIDE, L> slots_v = make_slots<Tag, SIDE, L>();
template <class Tag, int SIDE, int L, int Q>
inline constexpr int slot_v = slots_v<Tag, SIDE, L>.slot[Q];

// the catalog triples fold no signs (every single-entry column is +1)
template <class Tag>
constexpr bool unsigned_aliases_f() {
  for (int q = 0; q < Tag::R; ++q) {
    if (single(Tag::T.U, q) && !single_pos(Tag::T.U, q)) return false;
    if (single(Tag::T.V, q) && !single_pos(Tag::T.V, q)) return false;
  }
  return true;
}
template <class Tag>
inline constexpr bool unsigned_aliases = unsigned_aliases_f<Tag>();

// flat block index of digit tuple idx (base NB1 digits k1..kL, outer first)
template <int P1, int L>
__host__ __device__ constexpr int flat_block(int idx) {
  int row = 0, col = 0, scale = 1;
  for (int l = 0; l < L; ++l) {  // innermost digit first
    const int k = idx % (P1 * P1);
    idx /= P1 * P1;
    row += (k / P1) * scale;
    col += (k % P1) * scale;
    scale *= P1;
  }
  return row * scale + col;  // scale == P1^L == P
}

template <int VW> struct V { double v[VW]; };

template <int C, int VW>
__device__ __forceinline__ void acc_term(V<VW>& acc, const V<VW>& x) {
  if constexpr (C == 1) {
#pragma unroll
    for (int e = 0; e < VW; ++e) acc.v[e] = __dadd_rn(acc.v[e], x.v[e]);
  } else if constexpr (C == -1) {
#pragma unroll
    for (int e = 0; e < VW; ++e) acc.v[e] = __dadd_rn(acc.v[e], -x.v[e]);
  } else if constexpr (C != 0) {
#pragma unroll
    for (int e = 0; e < VW; ++e) acc.v[e] = __dadd_rn(acc.v[e], __dmul_rn((double)C, x.v[e]));
  }
}

template <int VW>
__device__ __forceinline__ V<VW> ld1(const double* p) {
  V<VW> r;
  if constexpr (VW == 2) {
    asm("ld.global.nc.L1::no_allocate.v2.f64 {%0,%1}, [%2];" : "=d"(r.v[0]), "=d"(r.v[1]) : "l"(p));
  } else {
    r.v[0] = __ldg(p);
  }
  return r;
}
template <int VW>
__device__ __forceinline__ void st1(double* p, const V<VW>& x) {
  if constexpr (VW == 2) {
    asm volatile("st.global.v2.f64 [%0], {%1,%2};" :: "l"(p), "d"(x.v[0]), "d"(x.v[1]) : "memory");
  } else {
    p[0] = x.v[0];
  }
}

// ---------------------------------------------------------------- K4
// Level LEV (1-based) of the pre-addition tree under product prefix QP:
// in[] holds NB1^(L-LEV+1) values indexed (k_LEV, k_LEV+1..k_L).
template <class Tag, int L, int SIDE, int VW, int LEV, int QP, int NIN, int Q, int... Ks>
__device__ __forceinline__ void pre_q(const V<VW> (&in)[NIN], double* out, int64_t off, int64_t mm,
                                      std::integer_sequence<int, Ks...>);

template <class Tag, int L, int SIDE, int VW, int LEV, int QP, int NIN, int... Qs>
__device__ __forceinline__ void pre_stage(const V<VW> (&in)[NIN], double* out, int64_t off,
                                          int64_t mm, std::integer_sequence<int, Qs...>) {
  constexpr int NB1 = Tag::p * Tag::p;
  (pre_q<Tag, L, SIDE, VW, LEV, QP, NIN, Qs>(in, out, off, mm, std::make_integer_sequence<int, NB1>{}),
   ...);
}

template <class Tag, int L, int SIDE, int VW, int LEV, int QP, int NIN, int Q, int... Ks>
__device__ __forceinline__ void pre_q(const V<VW> (&in)[NIN], double* out, int64_t off, int64_t mm,
                                      std::integer_sequence<int, Ks...>) {
  constexpr int NB1 = Tag::p * Tag::p;
  constexpr int NOUT = NIN / NB1;
  constexpr int q = QP * Tag::R + Q;
  if constexpr (LEV == L) {
    if constexpr (slot_v<Tag, SIDE, L, q> >= 0) {
      V<VW> y;
#pragma unroll
      for (int e = 0; e < VW; ++e) y.v[e] = -0.0;
      (acc_term<coef<Tag, SIDE, Ks, Q>, VW>(y, in[Ks]), ...);
      st1<VW>(out + (int64_t)slot_v<Tag, SIDE, L, q> * mm + off, y);
    }
  } else {
    V<VW> y[NOUT];
#pragma unroll
    for (int kk = 0; kk < NOUT; ++kk) {
#pragma unroll
      for (int e = 0; e < VW; ++e) y[kk].v[e] = -0.0;
      (acc_term<coef<Tag, SIDE, Ks, Q>, VW>(y[kk], in[Ks * NOUT + kk]), ...);
    }
    pre_stage<Tag, L, SIDE, VW, LEV + 1, q, NOUT>(y, out, off, mm,
                                                  std::make_integer_sequence<int, Tag::R>{});
  }
}

template <class Tag, int L, int SIDE, int VW>
__global__ void __launch_bounds__(256) premix_kron(const double* __restrict__ X, int64_t ldx,
                                                   int64_t m, double* __restrict__ out, int64_t r0,
                                                   int64_t r1, int64_t c0, int64_t c1) {
  static_assert(unsigned_aliases<Tag>, "sign folding not supported on this path");
  constexpr int NB1 = Tag::p * Tag::p;
  constexpr int NB = ipow<NB1, L>::v;
  constexpr int P = ipow<Tag::p, L>::v;
  const int64_t vpr = (c1 - c0) / VW;
  const int64_t total = (r1 - r0) * vpr;
  const int64_t mm = m * m;
  for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = r0 + idx / vpr;
    const int64_t c = c0 + (idx % vpr) * VW;
    V<VW> x[NB];
#pragma unroll
    for (int k = 0; k < NB; ++k) {
      const int b = flat_block<Tag::p, L>(k);
      x[k] = ld1<VW>(X + ((b / P) * m + r) * ldx + (b % P) * m + c);
    }
    pre_stage<Tag, L, SIDE, VW, 1, 0, NB>(x, out, r * m + c, mm,
                                           std::make_integer_sequence<int, Tag::R>{});
  }
}

// ---------------------------------------------------------------- K6
// Level LEV of the post-addition tree under prefix QP: acc[] holds
// NB1^(L-LEV+1) partial C values indexed (i_LEV, i_LEV+1..i_L); the deepest
// level combines leaf products over q_L, each shallower level combines the
// level below over its q (inner first, as the recursion distributes P_i).
template <class Tag, int L, int VW, int LEV, int QP, int NACC, int Q, int... Is>
__device__ __forceinline__ void post_q(V<VW> (&acc)[NACC], const double* __restrict__ Pw,
                                       int64_t off, int64_t mm, std::integer_sequence<int, Is...>);

template <class Tag, int L, int VW, int LEV, int QP, int NACC, int... Qs>
__device__ __forceinline__ void post_stage(V<VW> (&acc)[NACC], const double* __restrict__ Pw,
                                           int64_t off, int64_t mm,
                                           std::integer_sequence<int, Qs...>) {
  constexpr int NB1 = Tag::p * Tag::p;
  (post_q<Tag, L, VW, LEV, QP, NACC, Qs>(acc, Pw, off, mm, std::make_integer_sequence<int, NB1>{}),
   ...);
}

template <class Tag, int L, int VW, int LEV, int QP, int NACC, int Q, int... Is>
__device__ __forceinline__ void post_q(V<VW> (&acc)[NACC], const double* __restrict__ Pw,
                                       int64_t off, int64_t mm, std::integer_sequence<int, Is...>) {
  constexpr int NB1 = Tag::p * Tag::p;
  constexpr int NSUB = NACC / NB1;
  constexpr int q = QP * Tag::R + Q;
  constexpr int nz = (0 + ... + (coef<Tag, 2, Is, Q> != 0));
  if constexpr (nz > 0) {
    if constexpr (LEV == L) {
      const V<VW> x = ld1<VW>(Pw + (int64_t)q * mm + off);
      (acc_term<coef<Tag, 2, Is, Q>, VW>(acc[Is], x), ...);
    } else {
      V<VW> y[NSUB];
#pragma unroll
      for (int rr = 0; rr < NSUB; ++rr)
#pragma unroll
        for (int e = 0; e < VW; ++e) y[rr].v[e] = -0.0;
      post_stage<Tag, L, VW, LEV + 1, q, NSUB>(y, Pw, off, mm,
                                               std::make_integer_sequence<int, Tag::R>{});
#pragma unroll
      for (int rr = 0; rr < NSUB; ++rr) (acc_term<coef<Tag, 2, Is, Q>, VW>(acc[Is * NSUB + rr], y[rr]), ...);
    }
  }
}

template <class Tag, int L, int VW>
__global__ void __launch_bounds__(256) postmix_kron(const double* __restrict__ Pw, int64_t m,
                                                    double alpha, double* __restrict__ C,
                                                    int64_t ldc, int64_t r0, int64_t r1, int64_t c0,
                                                    int64_t c1) {
  static_assert(unsigned_aliases<Tag>, "sign folding not supported on this path");
  constexpr int NB1 = Tag::p * Tag::p;
  constexpr int NB = ipow<NB1, L>::v;
  constexpr int P = ipow<Tag::p, L>::v;
  const int64_t vpr = (c1 - c0) / VW;
  const int64_t total = (r1 - r0) * vpr;
  const int64_t mm = m * m;
  for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = r0 + idx / vpr;
    const int64_t c = c0 + (idx % vpr) * VW;
    V<VW> acc[NB];
#pragma unroll
    for (int i = 0; i < NB; ++i)
#pragma unroll
      for (int e = 0; e < VW; ++e) acc[i].v[e] = -0.0;
    post_stage<Tag, L, VW, 1, 0, NB>(acc, Pw, r * m + c, mm,
                                      std::make_integer_sequence<int, Tag::R>{});
#pragma unroll
    for (int i = 0; i < NB; ++i) {
      if (alpha != 1.0) {
#pragma unroll
        for (int e = 0; e < VW; ++e) acc[i].v[e] = __dmul_rn(alpha, acc[i].v[e]);
      }
      const int b = flat_block<Tag::p, L>(i);
      st1<VW>(C + ((b / P) * m + r) * ldc + (b % P) * m + c, acc[i]);
    }
  }
}

int grid_for(int64_t work) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t blocks = (work + 255) / 256;
  const int64_t cap = (int64_t)sms * 8;
  return (int)(blocks < cap ? (blocks < 1 ? 1 : blocks) : cap);
}

// host-side Kronecker power of a base table, compared with the plan's
template <class Tag>
bool is_power(const Plan& pl, int L) {
  const int p = Tag::p, R = Tag::R, NB1 = p * p;
  int P = 1, RL = 1;
  for (int l = 0; l < L; ++l) { P *= p; RL *= R; }
  if (pl.P != P || pl.RL != RL) return false;
  for (int idx = 0; idx < P * P; ++idx) {
    // digits of flat block idx (row, col) -> per-level base blocks, outer first
    int row = idx / P, col = idx % P;
    int k[8];
    for (int l = L - 1; l >= 0; --l) { k[l] = (row % p) * p + (col % p); row /= p; col /= p; }
    (void)NB1;
    for (int q = 0; q < RL; ++q) {
      int qq = q, u = 1, v = 1, w = 1;
      for (int l = L - 1; l >= 0; --l) {
        const int ql = qq % R;
        qq /= R;
        u *= Tag::T.U[k[l]][ql];
        v *= Tag::T.V[k[l]][ql];
        w *= Tag::T.W[k[l]][ql];
      }
      const size_t at = (size_t)idx * RL + q;
      if (pl.U[at] != u || pl.V[at] != v || pl.W[at] != w) return false;
    }
  }
  return true;
}

}  // namespace kronmix

// ids 8.. : Kronecker-factored kernels (see mf_fixed.cu for 1..7)
int kron_match(const Plan& pl) {
  using namespace kronmix;
  if (pl.P == 8 && is_power<fixed::TagSW>(pl, 3)) return 8;
  if (pl.P == 8 && is_power<fixed::TagPS>(pl, 3)) return 9;
  if (pl.P == 8 && is_power<fixed::TagS69>(pl, 3)) return 10;
  if (pl.P == 9 && is_power<fixed::TagLD>(pl, 2)) return 11;
  return 0;
}

#define MF_KRON_SWITCH(ID, CALL)          \
  switch (ID) {                           \
    case 8: return CALL(fixed::TagSW, 3); \
    case 9: return CALL(fixed::TagPS, 3); \
    case 10: return CALL(fixed::TagS69, 3); \
    case 11: return CALL(fixed::TagLD, 2); \
    default: return cudaErrorInvalidValue; \
  }

cudaError_t launch_premix_kron(int id, int side, const double* X, int64_t ldx, int64_t m,
                               double* out, cudaStream_t s, Rows rows) {
  const int64_t r0 = rows.r0, r1 = rows.end(m), c0 = rows.c0, c1 = rows.cend(m);
  const int grid = kronmix::grid_for((r1 - r0) * (c1 - c0));
#define PRE(T_, L_)                                                                                \
  (side == 0 ? (kronmix::premix_kron<T_, L_, 0, 1><<<grid, 256, 0, s>>>(X, ldx, m, out, r0, r1, c0, c1), \
                cudaGetLastError())                                                                \
             : (kronmix::premix_kron<T_, L_, 1, 1><<<grid, 256, 0, s>>>(X, ldx, m, out, r0, r1, c0, c1), \
                cudaGetLastError()))
  MF_KRON_SWITCH(id, PRE)
#undef PRE
}

cudaError_t launch_postmix_kron(int id, const double* Pw, int64_t m, double alpha, double* C,
                                int64_t ldc, cudaStream_t s, Rows rows) {
  const int64_t r0 = rows.r0, r1 = rows.end(m), c0 = rows.c0, c1 = rows.cend(m);
  const int grid = kronmix::grid_for((r1 - r0) * (c1 - c0));
#define POST(T_, L_)                                                                              \
  (kronmix::postmix_kron<T_, L_, 1><<<grid, 256, 0, s>>>(Pw, m, alpha, C, ldc, r0, r1, c0, c1), \
   cudaGetLastError())
  MF_KRON_SWITCH(id, POST)
#undef POST
}

}  // namespace mf
