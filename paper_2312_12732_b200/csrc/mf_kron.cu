// mf_kron.cu -- K4/K6 for Kronecker powers of a catalog triple, evaluated
// level by level (Kronecker-factored) instead of over the flattened table.
//
// For <U,V,W> = <u1,v1,w1> (x) ... (x) <uL,vL,wL> (a power
// or a mixed chain such as SW (x) Laderman) the flattened combination
//   T_(q1..qL) = sum_(k1..kL) u1[k1][q1]...uL[kL][qL] A_(k1..kL)
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
#include <tuple>
#include <utility>

#include "mf_internal.h"
#include "mf_tables.h"

namespace mf {
namespace kronmix {

using fixed::Tri;

// A chain of base triples, outermost first: <u1,v1,w1> (x) <u2,v2,w2> (x) ...
// (a power is the chain of one triple repeated).
template <class... Ts>
struct Chain {
  static constexpr int L = sizeof...(Ts);
  // per-level p and R as pure functions (no static arrays: usable at run time
  // in device code, e.g. in flat_block's loop)
  __host__ __device__ static constexpr int p_of(int l) {
    int v = 0, i = 0;
    ((v = (i++ == l) ? Ts::p : v), ...);
    return v;
  }
  __host__ __device__ static constexpr int R_of(int l) {
    int v = 0, i = 0;
    ((v = (i++ == l) ? Ts::R : v), ...);
    return v;
  }
  template <int LEV>  // 0-based
  using tag = std::tuple_element_t<LEV, std::tuple<Ts...>>;
  __host__ __device__ static constexpr int NB(int lev) { return p_of(lev) * p_of(lev); }
  __host__ __device__ static constexpr int NB_from(int lev) {  // prod_{l >= lev} p_l^2
    int v = 1;
    for (int l = lev; l < L; ++l) v *= p_of(l) * p_of(l);
    return v;
  }
  __host__ __device__ static constexpr int R_from(int lev) {
    int v = 1;
    for (int l = lev; l < L; ++l) v *= R_of(l);
    return v;
  }
  __host__ __device__ static constexpr int P() {
    int v = 1;
    for (int l = 0; l < L; ++l) v *= p_of(l);
    return v;
  }
};

// base coefficient of level LEV's triple (side 0: U, 1: V, 2: W)
template <class Ch, int LEV, int SIDE, int K, int Q>
inline constexpr int coef = SIDE == 0   ? Ch::template tag<LEV>::T.U[K][Q]
                            : SIDE == 1 ? Ch::template tag<LEV>::T.V[K][Q]
                                        : Ch::template tag<LEV>::T.W[K][Q];

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

template <class Tag, int SIDE>
constexpr bool single_col(int q) { return single(SIDE == 0 ? Tag::T.U : Tag::T.V, q); }

template <class Ch, int SIDE, size_t... Ls>
constexpr bool aliased_impl(int q, std::index_sequence<Ls...>) {
  // digits of q, innermost last: q = (..((q0)*R1 + q1)*R2 + ..)
  int digits[Ch::L] = {};
  for (int l = Ch::L - 1; l >= 0; --l) { digits[l] = q % Ch::R_of(l); q /= Ch::R_of(l); }
  return (single_col<typename Ch::template tag<Ls>, SIDE>(digits[Ls]) && ...);
}
// flattened product q aliases its A (B) block iff every level's column is a
// single +-1 (mf_plan's rule)
template <class Ch, int SIDE>
constexpr bool aliased(int q) {
  return aliased_impl<Ch, SIDE>(q, std::make_index_sequence<Ch::L>{});
}

template <class Ch, int SIDE>
struct Slots {
  int slot[Ch::R_from(0)];
};
template <class Ch, int SIDE>
constexpr Slots<Ch, SIDE> make_slots() {
  Slots<Ch, SIDE> s{};
  int next = 0;
  for (int q = 0; q < Ch::R_from(0); ++q) s.slot[q] = aliased<Ch, SIDE>(q) ? -1 : next++;
  return s;
}
template <class Ch, int SIDE>
inline constexpr Slots<Ch, SIDE> slots_v = make_slots<Ch, SIDE>();
template <class Ch, int SIDE, int Q>
inline constexpr int slot_v = slots_v<Ch, SIDE>.slot[Q];

template <class Tag>
constexpr bool unsigned_aliases_f() {
  for (int q = 0; q < Tag::R; ++q) {
    if (single(Tag::T.U, q) && !single_pos(Tag::T.U, q)) return false;
    if (single(Tag::T.V, q) && !single_pos(Tag::T.V, q)) return false;
  }
  return true;
}
// the catalog triples fold no signs (every single-entry column is +1)
template <class... Ts>
constexpr bool chain_unsigned(Chain<Ts...>*) { return (unsigned_aliases_f<Ts>() && ...); }
template <class Ch>
inline constexpr bool unsigned_aliases = chain_unsigned(static_cast<Ch*>(nullptr));

// flat block index (row * P + col) of the digit tuple idx = (k1..kL), k_l in
// [0, p_l^2), outer first (SPEC.md L244's interleave, applied per level)
template <class Ch>
__host__ __device__ constexpr int flat_block(int idx) {
  int row = 0, col = 0, scale = 1;
  for (int l = Ch::L - 1; l >= 0; --l) {  // innermost digit first
    const int p = Ch::p_of(l);
    const int k = idx % (p * p);
    idx /= p * p;
    row += (k / p) * scale;
    col += (k % p) * scale;
    scale *= p;
  }
  return row * scale + col;
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
// Level LEV (0-based) of the pre-addition tree under product prefix QP:
// in[] holds NB_from(LEV) values indexed (k_LEV, k_LEV+1..k_L-1).
template <class Ch, int SIDE, int VW, int LEV, int QP, int NIN, int Q, int... Ks>
__device__ __forceinline__ void pre_q(const V<VW> (&in)[NIN], double* out, int64_t off, int64_t mm,
                                      const ProdMask& mask, std::integer_sequence<int, Ks...>);

template <class Ch, int SIDE, int VW, int LEV, int QP, int NIN, int... Qs>
__device__ __forceinline__ void pre_stage(const V<VW> (&in)[NIN], double* out, int64_t off,
                                          int64_t mm, const ProdMask& mask,
                                          std::integer_sequence<int, Qs...>) {
  (pre_q<Ch, SIDE, VW, LEV, QP, NIN, Qs>(in, out, off, mm, mask,
                                         std::make_integer_sequence<int, Ch::NB(LEV)>{}),
   ...);
}

template <class Ch, int SIDE, int VW, int LEV, int QP, int NIN, int Q, int... Ks>
__device__ __forceinline__ void pre_q(const V<VW> (&in)[NIN], double* out, int64_t off, int64_t mm,
                                      const ProdMask& mask, std::integer_sequence<int, Ks...>) {
  constexpr int NOUT = NIN / Ch::NB(LEV);
  constexpr int q = QP * Ch::R_of(LEV) + Q;
  if constexpr (LEV == Ch::L - 1) {
    if constexpr (slot_v<Ch, SIDE, q> >= 0) {
      if (!mask.has(q)) return;  // product of another shard
      V<VW> y;
#pragma unroll
      for (int e = 0; e < VW; ++e) y.v[e] = -0.0;
      (acc_term<coef<Ch, LEV, SIDE, Ks, Q>, VW>(y, in[Ks]), ...);
      st1<VW>(out + (int64_t)slot_v<Ch, SIDE, q> * mm + off, y);
    }
  } else {
    V<VW> y[NOUT];
#pragma unroll
    for (int kk = 0; kk < NOUT; ++kk) {
#pragma unroll
      for (int e = 0; e < VW; ++e) y[kk].v[e] = -0.0;
      (acc_term<coef<Ch, LEV, SIDE, Ks, Q>, VW>(y[kk], in[Ks * NOUT + kk]), ...);
    }
    pre_stage<Ch, SIDE, VW, LEV + 1, q, NOUT>(y, out, off, mm, mask,
                                              std::make_integer_sequence<int, Ch::R_of(LEV + 1)>{});
  }
}

template <class Ch, int SIDE, int VW>
__global__ void __launch_bounds__(256) premix_kron(const double* __restrict__ X, int64_t ldx,
                                                   int64_t m, double* __restrict__ out, int64_t r0,
                                                   int64_t r1, int64_t c0, int64_t c1,
                                                   const ProdMask mask) {
  static_assert(unsigned_aliases<Ch>, "sign folding not supported on this path");
  constexpr int NB = Ch::NB_from(0);
  constexpr int P = Ch::P();
  const int64_t vpr = (c1 - c0) / VW;
  const int64_t total = (r1 - r0) * vpr;
  const int64_t mm = m * m;
  // grid-stride over (row, vector) positions, advanced without divisions
  const int64_t start = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t sd = stride / vpr, sm = stride - sd * vpr;
  int64_t rr = start / vpr, cv = start - rr * vpr;
  (void)total;
  for (; rr < r1 - r0; rr += sd, cv += sm, (cv >= vpr ? (cv -= vpr, ++rr) : 0)) {
    const int64_t r = r0 + rr;
    const int64_t c = c0 + cv * VW;
    V<VW> x[NB];
#pragma unroll
    for (int k = 0; k < NB; ++k) {
      const int b = flat_block<Ch>(k);
      x[k] = ld1<VW>(X + ((b / P) * m + r) * ldx + (b % P) * m + c);
    }
    pre_stage<Ch, SIDE, VW, 0, 0, NB>(x, out, r * m + c, mm, mask,
                                      std::make_integer_sequence<int, Ch::R_of(0)>{});
  }
}

// ---------------------------------------------------------------- K6
// Level LEV of the post-addition tree under prefix QP: acc[] holds NB_from(LEV)
// partial C values indexed (i_LEV, i_LEV+1..); the deepest level combines leaf
// products over its q, each shallower level combines the level below (inner
// first, as the recursion distributes P_i).
template <class Ch, int VW, bool MASKED, int LEV, int QP, int NACC, int Q, int... Is>
__device__ __forceinline__ void post_q(V<VW> (&acc)[NACC], const double* __restrict__ Pw,
                                       int64_t off, int64_t mm, const ProdMask& mask,
                                       std::integer_sequence<int, Is...>);

template <class Ch, int VW, bool MASKED, int LEV, int QP, int NACC, int... Qs>
__device__ __forceinline__ void post_stage(V<VW> (&acc)[NACC], const double* __restrict__ Pw,
                                           int64_t off, int64_t mm, const ProdMask& mask,
                                           std::integer_sequence<int, Qs...>) {
  (post_q<Ch, VW, MASKED, LEV, QP, NACC, Qs>(acc, Pw, off, mm, mask,
                                     std::make_integer_sequence<int, Ch::NB(LEV)>{}),
   ...);
}

template <class Ch, int VW, bool MASKED, int LEV, int QP, int NACC, int Q, int... Is>
__device__ __forceinline__ void post_q(V<VW> (&acc)[NACC], const double* __restrict__ Pw,
                                       int64_t off, int64_t mm, const ProdMask& mask,
                                       std::integer_sequence<int, Is...>) {
  constexpr int NSUB = NACC / Ch::NB(LEV);
  constexpr int q = QP * Ch::R_of(LEV) + Q;
  constexpr int nz = (0 + ... + (coef<Ch, LEV, 2, Is, Q> != 0));
  if constexpr (nz > 0) {
    if constexpr (LEV == Ch::L - 1) {
      if constexpr (MASKED)
        if (!mask.has(q)) return;  // product of another shard
      const V<VW> x = ld1<VW>(Pw + (int64_t)q * mm + off);
      (acc_term<coef<Ch, LEV, 2, Is, Q>, VW>(acc[Is], x), ...);
    } else {
      V<VW> y[NSUB];
#pragma unroll
      for (int rr = 0; rr < NSUB; ++rr)
#pragma unroll
        for (int e = 0; e < VW; ++e) y[rr].v[e] = -0.0;
      post_stage<Ch, VW, MASKED, LEV + 1, q, NSUB>(y, Pw, off, mm, mask,
                                           std::make_integer_sequence<int, Ch::R_of(LEV + 1)>{});
#pragma unroll
      for (int rr = 0; rr < NSUB; ++rr)
        (acc_term<coef<Ch, LEV, 2, Is, Q>, VW>(acc[Is * NSUB + rr], y[rr]), ...);
    }
  }
}

template <class Ch, int VW, bool MASKED>
__global__ void __launch_bounds__(256) postmix_kron(const double* __restrict__ Pw, int64_t m,
                                                    double alpha, double* __restrict__ C,
                                                    int64_t ldc, int64_t r0, int64_t r1, int64_t c0,
                                                    int64_t c1, const ProdMask mask) {
  static_assert(unsigned_aliases<Ch>, "sign folding not supported on this path");
  constexpr int NB = Ch::NB_from(0);
  constexpr int P = Ch::P();
  const int64_t vpr = (c1 - c0) / VW;
  const int64_t total = (r1 - r0) * vpr;
  const int64_t mm = m * m;
  // grid-stride over (row, vector) positions, advanced without divisions
  const int64_t start = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t sd = stride / vpr, sm = stride - sd * vpr;
  int64_t rr = start / vpr, cv = start - rr * vpr;
  (void)total;
  for (; rr < r1 - r0; rr += sd, cv += sm, (cv >= vpr ? (cv -= vpr, ++rr) : 0)) {
    const int64_t r = r0 + rr;
    const int64_t c = c0 + cv * VW;
    V<VW> acc[NB];
#pragma unroll
    for (int i = 0; i < NB; ++i)
#pragma unroll
      for (int e = 0; e < VW; ++e) acc[i].v[e] = -0.0;
    post_stage<Ch, VW, MASKED, 0, 0, NB>(acc, Pw, r * m + c, mm, mask,
                                 std::make_integer_sequence<int, Ch::R_of(0)>{});
#pragma unroll
    for (int i = 0; i < NB; ++i) {
      if (alpha != 1.0) {
#pragma unroll
        for (int e = 0; e < VW; ++e) acc[i].v[e] = __dmul_rn(alpha, acc[i].v[e]);
      }
      const int b = flat_block<Ch>(i);
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

// host side: is the plan's flattened triple the chain's Kronecker product?
template <class Tag>
int base_coef(int side, int k, int q) {
  return side == 0 ? Tag::T.U[k][q] : (side == 1 ? Tag::T.V[k][q] : Tag::T.W[k][q]);
}
template <class... Ts>
bool is_chain(const Plan& pl) {
  using Ch = Chain<Ts...>;
  constexpr int L = Ch::L;
  if (pl.P != Ch::P() || pl.RL != Ch::R_from(0)) return false;
  int (*coefs[L])(int, int, int) = {&base_coef<Ts>...};
  const int P = Ch::P(), RL = Ch::R_from(0);
  for (int idx = 0; idx < P * P; ++idx) {
    int row = idx / P, col = idx % P, k[L];
    for (int l = L - 1; l >= 0; --l) {
      const int p = Ch::p_of(l);
      k[l] = (row % p) * p + (col % p);
      row /= p;
      col /= p;
    }
    for (int q = 0; q < RL; ++q) {
      int qq = q, c[3] = {1, 1, 1};
      for (int l = L - 1; l >= 0; --l) {
        const int ql = qq % Ch::R_of(l);
        qq /= Ch::R_of(l);
        for (int sd = 0; sd < 3; ++sd) c[sd] *= coefs[l](sd, k[l], ql);
      }
      const size_t at = (size_t)idx * RL + q;
      if (pl.U[at] != c[0] || pl.V[at] != c[1] || pl.W[at] != c[2]) return false;
    }
  }
  return true;
}

using fixed::TagLD;
using fixed::TagPS;
using fixed::TagS69;
using fixed::TagSW;
using ChSW3 = Chain<TagSW, TagSW, TagSW>;
using ChPS3 = Chain<TagPS, TagPS, TagPS>;
using ChS693 = Chain<TagS69, TagS69, TagS69>;
using ChLD2 = Chain<TagLD, TagLD>;
using ChSWLD = Chain<TagSW, TagLD>;
using ChLDSW = Chain<TagLD, TagSW>;

}  // namespace kronmix

// ids 8.. : Kronecker-factored kernels (see mf_fixed.cu for 1..7)
int kron_match(const Plan& pl) {
  using namespace kronmix;
  if (is_chain<TagSW, TagSW, TagSW>(pl)) return 8;
  if (is_chain<TagPS, TagPS, TagPS>(pl)) return 9;
  if (is_chain<TagS69, TagS69, TagS69>(pl)) return 10;
  if (is_chain<TagLD, TagLD>(pl)) return 11;
  if (is_chain<TagSW, TagLD>(pl)) return 12;
  if (is_chain<TagLD, TagSW>(pl)) return 13;
  return 0;
}

#define MF_KRON_SWITCH(ID, CALL)             \
  switch (ID) {                              \
    case 8: return CALL(kronmix::ChSW3);     \
    case 9: return CALL(kronmix::ChPS3);     \
    case 10: return CALL(kronmix::ChS693);   \
    case 11: return CALL(kronmix::ChLD2);    \
    case 12: return CALL(kronmix::ChSWLD);   \
    case 13: return CALL(kronmix::ChLDSW);   \
    default: return cudaErrorInvalidValue;   \
  }

// number of products of chain id (for the mask-is-full test)
static int pl_products(int id) {
  switch (id) {
    case 8: case 9: case 10: return 343;
    case 11: return 529;
    case 12: case 13: return 161;
    default: return 0;
  }
}

cudaError_t launch_premix_kron(int id, int side, const double* X, int64_t ldx, int64_t m,
                               double* out, cudaStream_t s, Rows rows, const ProdMask& mask) {
  const int64_t r0 = rows.r0, r1 = rows.end(m), c0 = rows.c0, c1 = rows.cend(m);
  const int grid = kronmix::grid_for((r1 - r0) * (c1 - c0));
#define PRE(CH_)                                                                                  \
  (side == 0 ? (kronmix::premix_kron<CH_, 0, 1><<<grid, 256, 0, s>>>(X, ldx, m, out, r0, r1, c0, c1, mask), \
                cudaGetLastError())                                                               \
             : (kronmix::premix_kron<CH_, 1, 1><<<grid, 256, 0, s>>>(X, ldx, m, out, r0, r1, c0, c1, mask), \
                cudaGetLastError()))
  MF_KRON_SWITCH(id, PRE)
#undef PRE
}

cudaError_t launch_postmix_kron(int id, const double* Pw, int64_t m, double alpha, double* C,
                                int64_t ldc, cudaStream_t s, Rows rows, const ProdMask& mask) {
  const int64_t r0 = rows.r0, r1 = rows.end(m), c0 = rows.c0, c1 = rows.cend(m);
  const int grid = kronmix::grid_for((r1 - r0) * (c1 - c0));
  bool full = true;
  for (int q = 0; q < 576; ++q) full = full && (q >= pl_products(id) || mask.has(q));
#define POST(CH_)                                                                                 \
  (full ? kronmix::postmix_kron<CH_, 1, false><<<grid, 256, 0, s>>>(Pw, m, alpha, C, ldc, r0, r1, c0, \
                                                                    c1, mask)                      \
        : kronmix::postmix_kron<CH_, 1, true><<<grid, 256, 0, s>>>(Pw, m, alpha, C, ldc, r0, r1, c0,  \
                                                                   c1, mask),                      \
   cudaGetLastError())
  MF_KRON_SWITCH(id, POST)
#undef POST
}

}  // namespace mf
