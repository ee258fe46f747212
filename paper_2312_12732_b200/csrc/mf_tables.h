// mf_tables.h -- compile-time coefficient tables of the catalog triples, shared
// by the specialised K4/K6 kernels (mf_fixed.cu: flattened; mf_kron.cu:
// Kronecker-factored).  Product side only (the oracle types its own tables).
#pragma once
#include <cstdint>

namespace mf {
namespace fixed {

template <int NB, int R>
struct Tri {
  int8_t U[NB][R], V[NB][R], W[NB][R];
};

// Blocks 0=(1,1) 1=(1,2) 2=(2,1) 3=(2,2); W rows in natural C order.
inline constexpr Tri<4, 7> kSW = {
    {{1, 0, 1, 0, 0, -1, 1}, {0, 1, 1, 0, 0, 0, 0}, {0, 0, -1, 0, 1, 1, -1}, {0, 0, -1, 1, 1, 1, 0}},
    {{1, 0, 0, 1, -1, 1, 0}, {0, 0, 0, -1, 1, -1, -1}, {0, 1, 0, -1, 0, 0, 0}, {0, 0, 1, 1, 0, 1, 1}},
    {{1, 1, 0, 0, 0, 0, 0}, {1, 0, 1, 0, 1, 1, 0}, {1, 0, 0, -1, 0, 1, 1}, {1, 0, 0, 0, 1, 1, 1}}};
inline constexpr Tri<4, 7> kPS = {
    {{0, 1, 1, 0, 1, 1, 0}, {0, 0, -1, 1, 0, 0, 0}, {1, 1, 1, 0, 1, 0, 0}, {-1, -1, -1, 0, 0, 0, 1}},
    {{0, 0, 0, 0, 1, 1, 0}, {1, 1, 0, 0, 1, 0, 1}, {0, 1, 1, 1, 1, 0, 0}, {0, 1, 1, 0, 1, 0, 1}},
    {{0, 0, 0, 1, 0, 1, 0}, {-1, 1, -1, -1, 0, 0, 0}, {0, -1, 0, 0, 1, -1, -1}, {1, 0, 0, 0, 0, 0, 1}}};
inline constexpr Tri<4, 7> kS69 = {
    {{1, 0, 1, 0, 1, -1, 0}, {0, 0, 0, 0, 1, 0, 1}, {0, 1, 0, 0, 0, 1, 0}, {1, 1, 0, 1, 0, 0, -1}},
    {{1, 1, 0, -1, 0, 1, 0}, {0, 0, 1, 0, 0, 1, 0}, {0, 0, 0, 1, 0, 0, 1}, {1, 0, -1, 0, 1, 0, 1}},
    {{1, 0, 0, 1, -1, 0, 1}, {0, 0, 1, 0, 1, 0, 0}, {0, 1, 0, 1, 0, 0, 0}, {1, -1, 1, 0, 0, 1, 0}}};
// Laderman 1976, blocks 0..8 row-major over the 3x3 grid.
inline constexpr Tri<9, 23> kLD = {
    {{1, 1, 0, -1, 0, 1, -1, -1, 0, 1, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0},
     {1, 0, 0, 0, 0, 0, 0, 0, 0, 1, 0, 0, 0, 0, 0, 0, 0, 0, 1, 0, 0, 0, 0},
     {1, 0, 0, 0, 0, 0, 0, 0, 0, 1, 0, -1, 1, 1, 0, -1, 1, 0, 0, 0, 0, 0, 0},
     {-1, -1, 0, 1, 1, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 1, 0, 0},
     {-1, 0, 1, 1, 1, 0, 0, 0, 0, -1, 0, 0, 0, 0, 0, 1, 0, 1, 0, 0, 0, 0, 0},
     {0, 0, 0, 0, 0, 0, 0, 0, 0, -1, 0, 0, 0, 0, 0, 1, -1, 1, 0, 1, 0, 0, 0},
     {0, 0, 0, 0, 0, 0, 1, 1, 1, -1, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 1, 0},
     {-1, 0, 0, 0, 0, 0, 1, 0, 1, -1, 1, 1, 0, 0, 1, 0, 0, 0, 0, 0, 0, 0, 0},
     {-1, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 1, -1, 0, 1, 0, 0, 0, 0, 0, 0, 0, 1}},
    {{0, 0, -1, 1, -1, 1, 1, 0, -1, 0, -1, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0},
     {0, -1, 1, -1, 1, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 1, 0},
     {0, 0, 0, 0, 0, 0, -1, 1, 1, 0, 1, 0, 0, 0, 0, 0, 0, 0, 0, 0, 1, 0, 0},
     {0, 0, 1, 0, 0, 0, 0, 0, 0, 0, 1, 0, 0, 0, 0, 0, 0, 0, 1, 0, 0, 0, 0},
     {1, 1, -1, 1, 0, 0, 0, 0, 0, 0, -1, 1, 1, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0},
     {0, 0, -1, 0, 0, 0, 1, -1, 0, 1, -1, 0, 0, 0, 0, 1, 1, 0, 0, 0, 0, 0, 0},
     {0, 0, -1, 0, 0, 0, 0, 0, 0, 0, -1, 1, 0, 1, -1, 1, 0, -1, 0, 0, 0, 0, 0},
     {0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 1, -1, -1, 0, 1, 0, 0, 0, 0, 1, 0, 0, 0},
     {0, 0, 1, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, -1, -1, 1, 0, 0, 0, 0, 1}},
    {{0, 0, 0, 0, 0, 1, 0, 0, 0, 0, 0, 0, 0, 1, 0, 0, 0, 0, 1, 0, 0, 0, 0},
     {1, 0, 0, 1, 1, 1, 0, 0, 0, 0, 0, 1, 0, 1, 1, 0, 0, 0, 0, 0, 0, 0, 0},
     {0, 0, 0, 0, 0, 1, 1, 0, 1, 1, 0, 0, 0, 1, 0, 1, 0, 1, 0, 0, 0, 0, 0},
     {0, 1, 1, 1, 0, 1, 0, 0, 0, 0, 0, 0, 0, 1, 0, 1, 1, 0, 0, 0, 0, 0, 0},
     {0, 1, 0, 1, 1, 1, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 1, 0, 0, 0},
     {0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 1, 0, 1, 1, 1, 0, 0, 1, 0, 0},
     {0, 0, 0, 0, 0, 1, 1, 1, 0, 0, 1, 1, 1, 1, 0, 0, 0, 0, 0, 0, 0, 0, 0},
     {0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 1, 1, 1, 1, 0, 0, 0, 0, 0, 0, 1, 0},
     {0, 0, 0, 0, 0, 1, 1, 1, 1, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 1}}};

// PAPER.md L303-309 with SPEC.md L244's row interleave; q = qo*Ri + qi.
template <int Po, int NBo, int Ro, int Pi, int NBi, int Ri>
constexpr Tri<NBo * NBi, Ro * Ri> kron(const Tri<NBo, Ro>& o, const Tri<NBi, Ri>& in) {
  Tri<NBo * NBi, Ro * Ri> t{};
  constexpr int P = Po * Pi;
  for (int b = 0; b < NBo; ++b)
    for (int s = 0; s < NBi; ++s) {
      const int row = ((b / Po) * Pi + s / Pi) * P + (b % Po) * Pi + s % Pi;
      for (int qo = 0; qo < Ro; ++qo)
        for (int qi = 0; qi < Ri; ++qi) {
          const int q = qo * Ri + qi;
          t.U[row][q] = (int8_t)(o.U[b][qo] * in.U[s][qi]);
          t.V[row][q] = (int8_t)(o.V[b][qo] * in.V[s][qi]);
          t.W[row][q] = (int8_t)(o.W[b][qo] * in.W[s][qi]);
        }
    }
  return t;
}


// Base-triple tags for kernels parameterised by a TYPE (nvcc host stubs cannot
// name reference template arguments).
struct TagSW { static constexpr const auto& T = kSW; static constexpr int p = 2, R = 7; };
struct TagPS { static constexpr const auto& T = kPS; static constexpr int p = 2, R = 7; };
struct TagS69 { static constexpr const auto& T = kS69; static constexpr int p = 2, R = 7; };
struct TagLD { static constexpr const auto& T = kLD; static constexpr int p = 3, R = 23; };

}  // namespace fixed
}  // namespace mf
