// mf_api.cpp -- the C ABI of include/mf.h: plan construction (host logic of
// SURVEY.md §3 step 1), the stream-ordered scheduler of mf_dgemm, the
// host-buffer entry point and the NCCL bootstrap.  Kernels live in
// mf_mix.cu (K4/K6) and mf_leaf.cu (K5).
#include <dlfcn.h>
#include <nvtx3/nvToolsExt.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <memory>
#include <mutex>
#include <new>

#include "mf_internal.h"

using namespace mf;

struct mf_plan_st : public Plan {};

namespace mf {

thread_local std::string g_err;

mf_status fail(mf_status st, const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = buf;
  return st;
}

}  // namespace mf

namespace {

// NVTX ranges of mf_dgemm's phases (SURVEY §5 tracing): "mf:K4 A", "mf:K4 B",
// "mf:K5 leaf", "mf:K6", "mf:exchange" on the calling host thread, nested in
// "mf_dgemm".  Header-only NVTX v3: no-ops unless a tool (nsys, ncu --nvtx)
// injects itself.  The guard closes whatever is open on every return path.
struct NvtxPhases {
  int depth = 0;
  NvtxPhases() { nvtxRangePushA("mf_dgemm"); depth = 1; }
  void to(const char* name) {
    if (depth > 1) { nvtxRangePop(); --depth; }
    if (name) { nvtxRangePushA(name); ++depth; }
  }
  ~NvtxPhases() { while (depth-- > 0) nvtxRangePop(); }
};

mf_status cuda_fail(cudaError_t e, const char* what) {
  return fail(MF_ERR_CUDA, "%s: %s (%s)", what, cudaGetErrorName(e), cudaGetErrorString(e));
}

#define MF_CUDA(call, what)                           \
  do {                                                \
    cudaError_t e_ = (call);                          \
    if (e_ != cudaSuccess) return cuda_fail(e_, what); \
  } while (0)

struct DeviceGuard {
  int prev = -1;
  bool ok = true;
  explicit DeviceGuard(int dev) {
    if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
    if (dev >= 0 && dev != prev) ok = cudaSetDevice(dev) == cudaSuccess;
  }
  ~DeviceGuard() {
    int cur = -1;
    if (prev >= 0 && cudaGetDevice(&cur) == cudaSuccess && cur != prev) cudaSetDevice(prev);
  }
};

// ------------------------------------------------- cuBLAS (dlopen; MF_LEAF_CUBLAS)
// The leaf ablation only: the library DGEMM on the same K4/K6 pipeline.
struct Cublas {
  void* h = nullptr;
  int (*Create)(void**) = nullptr;
  int (*Destroy)(void*) = nullptr;
  int (*SetStream)(void*, cudaStream_t) = nullptr;
  int (*DgemmBatched)(void*, int, int, int, int, int, const double*, const double* const*, int,
                      const double* const*, int, const double*, double* const*, int, int) = nullptr;
};

Cublas* cublas() {
  static Cublas c;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libcublas.so.12", RTLD_NOW | RTLD_NOLOAD);
    if (!h) h = dlopen("libcublas.so.12", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return;
    c.h = h;
    c.Create = (decltype(c.Create))dlsym(h, "cublasCreate_v2");
    c.Destroy = (decltype(c.Destroy))dlsym(h, "cublasDestroy_v2");
    c.SetStream = (decltype(c.SetStream))dlsym(h, "cublasSetStream_v2");
    c.DgemmBatched = (decltype(c.DgemmBatched))dlsym(h, "cublasDgemmBatched");
  });
  return c.h && c.Create && c.Destroy && c.SetStream && c.DgemmBatched ? &c : nullptr;
}

// ---------------------------------------------------------------- triple algebra
// Exact Brent check of <U,V,W> (p^2 x R each).  Dyadic
// coefficients are scaled to integers by 2^d per matrix; the identity becomes
// sum_q U'V'W' = 2^(dU+dV+dW) * [k==k' && i==i' && j==j'], checked in __int128.
mf_status brent_check(int p, int R, const double* U, const double* V, const double* W) {
  const int P2 = p * p;
  int dexp[3] = {0, 0, 0};
  const double* mats[3] = {U, V, W};
  for (int t = 0; t < 3; ++t)
    for (int i = 0; i < P2 * R; ++i) {
      double x = mats[t][i];
      if (!std::isfinite(x)) return fail(MF_ERR_BAD_TRIPLE, "non-finite coefficient");
      int d = 0;
      while (x != std::floor(x) && d < 30) { x *= 2.0; ++d; }
      if (x != std::floor(x) || std::fabs(x) > 1e6)
        return fail(MF_ERR_UNSUPPORTED,
                    "coefficient %g is not an integer or a dyadic rational of modest size",
                    mats[t][i]);
      dexp[t] = std::max(dexp[t], d);
    }
  std::vector<int64_t> Ui(P2 * R), Vi(P2 * R), Wi(P2 * R);
  for (int i = 0; i < P2 * R; ++i) {
    Ui[i] = (int64_t)std::ldexp(U[i], dexp[0]);
    Vi[i] = (int64_t)std::ldexp(V[i], dexp[1]);
    Wi[i] = (int64_t)std::ldexp(W[i], dexp[2]);
  }
  // every sum of R terms |U'V'W'| must stay inside __int128 (signed overflow
  // would be undefined and could accept a wrong triple)
  {
    double mx[3] = {0, 0, 0};
    const std::vector<int64_t>* sc[3] = {&Ui, &Vi, &Wi};
    for (int t = 0; t < 3; ++t)
      for (int64_t x : *sc[t]) mx[t] = std::max(mx[t], std::fabs((double)x));
    if (mx[0] * mx[1] * mx[2] * (double)R >= std::ldexp(1.0, 125))
      return fail(MF_ERR_UNSUPPORTED,
                  "coefficients too large for the exact Brent check (scaled |U||V||W|R >= 2^125)");
  }
  const __int128 one = (__int128)1 << (dexp[0] + dexp[1] + dexp[2]);
  int64_t bad = 0;
  int fx = -1, fy = -1, fz = -1;
  for (int x = 0; x < P2; ++x)
    for (int y = 0; y < P2; ++y)
      for (int z = 0; z < P2; ++z) {
        __int128 s = 0;
        for (int q = 0; q < R; ++q)
          s += (__int128)Ui[x * R + q] * Vi[y * R + q] * Wi[z * R + q];
        const int i = x / p, k = x % p, k2 = y / p, j = y % p, i2 = z / p, j2 = z % p;
        const __int128 expect = (k == k2 && i == i2 && j == j2) ? one : 0;
        if (s != expect) {
          if (bad == 0) { fx = x; fy = y; fz = z; }
          ++bad;
        }
      }
  if (bad)
    return fail(MF_ERR_BAD_TRIPLE,
                "Brent equations violated: %lld of %lld fail; first (x,y,z) = (%d,%d,%d)",
                (long long)bad, (long long)P2 * P2 * P2, fx, fy, fz);
  for (int q = 0; q < R; ++q) {
    bool u = false, v = false;
    for (int k = 0; k < P2; ++k) { u |= U[k * R + q] != 0.0; v |= V[k * R + q] != 0.0; }
    if (!u || !v) return fail(MF_ERR_BAD_TRIPLE, "product column %d has an all-zero operand", q);
  }
  return MF_OK;
}

// Kronecker composition outer (x) inner with the
// row interleave of SPEC.md L244: outer block b, inner block s ->
// row ((b/po)*pi + s/pi) * (po*pi) + (b%po)*pi + s%pi; product q = qo*Ri + qi.
void kron(int po, int64_t Ro, const std::vector<double>& Uo, const std::vector<double>& Vo,
          const std::vector<double>& Wo, int pi, int64_t Ri, const double* Ui, const double* Vi,
          const double* Wi, std::vector<double>& U, std::vector<double>& V, std::vector<double>& W) {
  const int P = po * pi;
  const int64_t R = Ro * Ri;
  U.assign((size_t)P * P * R, 0.0);
  V.assign(U.size(), 0.0);
  W.assign(U.size(), 0.0);
  for (int b = 0; b < po * po; ++b)
    for (int s = 0; s < pi * pi; ++s) {
      const int row = ((b / po) * pi + s / pi) * P + (b % po) * pi + s % pi;
      for (int64_t qo = 0; qo < Ro; ++qo)
        for (int64_t qi = 0; qi < Ri; ++qi) {
          const int64_t q = qo * Ri + qi;
          U[row * R + q] = Uo[b * Ro + qo] * Ui[s * Ri + qi];
          V[row * R + q] = Vo[b * Ro + qo] * Vi[s * Ri + qi];
          W[row * R + q] = Wo[b * Ro + qo] * Wi[s * Ri + qi];
        }
    }
}

// Greedy output grouping for the grouped mix kernel: each group is seeded with
// the first unassigned output and grown with the unassigned output sharing the
// most inputs with the group (lowest index on ties), so a warp's loads serve as
// many of its outputs as possible.  ngroup = ceil(nout / gsize), sizes differ
// by at most one.
static std::vector<std::vector<int>> group_outputs(const MixTable& t, int gsize) {
  const int ng = (t.nout + gsize - 1) / gsize;
  std::vector<std::vector<int>> groups;
  std::vector<char> used(t.nout, 0);
  auto uses = [&](int o, int k) { return t.coef[(size_t)o * t.nin + k] != 0.0; };
  for (int g = 0; g < ng; ++g) {
    const int size = t.nout / ng + (g < t.nout % ng ? 1 : 0);
    std::vector<int> grp;
    std::vector<char> in_union(t.nin, 0);
    for (int o = 0; o < t.nout && grp.empty(); ++o)
      if (!used[o]) { grp.push_back(o); used[o] = 1; }
    if (grp.empty()) break;
    for (int k = 0; k < t.nin; ++k) in_union[k] = uses(grp[0], k);
    while ((int)grp.size() < size) {
      int best = -1, best_shared = -1;
      for (int o = 0; o < t.nout; ++o) {
        if (used[o]) continue;
        int shared = 0;
        for (int k = 0; k < t.nin; ++k) shared += in_union[k] && uses(o, k);
        if (shared > best_shared) { best = o; best_shared = shared; }
      }
      if (best < 0) break;
      grp.push_back(best);
      used[best] = 1;
      for (int k = 0; k < t.nin; ++k) in_union[k] = in_union[k] || uses(best, k);
    }
    groups.push_back(grp);
  }
  return groups;
}

// Device table: MixRow[nout] then MixTerm[...] -- each output's nonzero
// terms in ascending input order (the oracle's combination order) -- then the
// grouped form (MixGroup[ngroup], entries) when it fits in shared memory.
mf_status upload_table(MixTable& t) {
  std::vector<MixRow> rows;
  std::vector<MixTerm> terms;
  for (int o = 0; o < t.nout; ++o) {
    MixRow r{};
    r.first = (int32_t)terms.size();
    r.target = t.out_map[o];
    for (int k = 0; k < t.nin; ++k) {
      const double v = t.coef[(size_t)o * t.nin + k];
      if (v == 0.0) continue;
      MixTerm term{};
      term.src = k;
      term.kind = v == 1.0 ? MIX_POS : (v == -1.0 ? MIX_NEG : MIX_GEN);
      term.coef = v;
      terms.push_back(term);
    }
    r.count = (int32_t)terms.size() - r.first;
    rows.push_back(r);
  }
  t.nrow = (int)rows.size();
  t.nterm = (int)terms.size();
  const size_t bytes = sizeof(MixRow) * rows.size() + sizeof(MixTerm) * terms.size();
  if (bytes == 0) return MF_OK;
  if (bytes > 200 * 1024) return fail(MF_ERR_UNSUPPORTED, "mix table of %zu bytes exceeds shared memory", bytes);
  // grouped form: one group per warp of a 256-thread CTA.  Measured against
  // the term-list kernel it wins up to 4 outputs per warp (LD K4, every K6)
  // and loses beyond (SW^2 K4: 5 per warp, 4.2 vs 3.4 ms; profiles/mix_r01.json)
  std::vector<uint8_t> gtab;
  t.gsize = t.ngroup = 0;
  const int gsize = std::max(1, (t.nout + 7) / 8);
  if (!getenv("MF_MIX_UNGROUPED") && gsize <= 4) {
    const auto groups = group_outputs(t, gsize);
    std::vector<MixGroup> hdr;
    std::vector<uint8_t> ent;
    const size_t stride = 8 + 8 * (size_t)gsize;
    for (const auto& grp : groups) {
      MixGroup h{};
      h.first = (int32_t)(ent.size() / stride);
      for (int j = 0; j < MIX_GMAX; ++j) h.target[j] = j < (int)grp.size() ? t.out_map[grp[j]] : -1;
      for (int k = 0; k < t.nin; ++k) {
        bool any = false;
        for (int o : grp) any = any || t.coef[(size_t)o * t.nin + k] != 0.0;
        if (!any) continue;
        std::vector<uint8_t> e(stride, 0);
        const int32_t src = k;
        memcpy(e.data(), &src, 4);
        for (int j = 0; j < (int)grp.size(); ++j) {
          const double v = t.coef[(size_t)grp[j] * t.nin + k];
          memcpy(e.data() + 8 + 8 * j, &v, 8);
        }
        ent.insert(ent.end(), e.begin(), e.end());
      }
      h.count = (int32_t)(ent.size() / stride) - h.first;
      hdr.push_back(h);
    }
    const size_t gb = sizeof(MixGroup) * hdr.size() + ent.size();
    if (gb <= 96 * 1024) {
      gtab.resize(gb);
      memcpy(gtab.data(), hdr.data(), sizeof(MixGroup) * hdr.size());
      memcpy(gtab.data() + sizeof(MixGroup) * hdr.size(), ent.data(), ent.size());
      t.gsize = gsize;
      t.ngroup = (int)hdr.size();
    }
  }
  t.goff = (bytes + 15) / 16 * 16;
  t.gbytes = gtab.size();
  MF_CUDA(cudaMalloc(&t.d_table, t.goff + t.gbytes), "cudaMalloc(coefficient table)");
  MF_CUDA(cudaMemcpy(t.d_table, rows.data(), sizeof(MixRow) * rows.size(), cudaMemcpyHostToDevice),
          "upload table");
  if (!terms.empty())
    MF_CUDA(cudaMemcpy(static_cast<uint8_t*>(t.d_table) + sizeof(MixRow) * rows.size(), terms.data(),
                       sizeof(MixTerm) * terms.size(), cudaMemcpyHostToDevice),
            "upload table");
  if (!gtab.empty())
    MF_CUDA(cudaMemcpy(static_cast<uint8_t*>(t.d_table) + t.goff, gtab.data(), gtab.size(),
                       cudaMemcpyHostToDevice),
            "upload grouped table");
  return MF_OK;
}

void free_plan(Plan* pl) {
  if (!pl || pl->opt.host_only) return;
  DeviceGuard g(pl->device);
  cudaDeviceSynchronize();
  for (void* p : {(void*)pl->T, (void*)pl->S, (void*)pl->Pw, (void*)pl->d_jobs, (void*)pl->mixA.d_table,
                  (void*)pl->mixB.d_table, (void*)pl->mixC.d_table, (void*)pl->mixA2.d_table,
                  (void*)pl->mixC2.d_table, (void*)pl->hA, (void*)pl->hB,
                  (void*)pl->d_post_off, (void*)pl->d_post, (void*)pl->d_ptrs, (void*)pl->Cfull,
                  (void*)pl->split_ws, (void*)pl->split_cnt, (void*)pl->d_tinyU, (void*)pl->d_tinyV,
                  (void*)pl->rA, (void*)pl->rB, (void*)pl->fuse_sync,
                  (void*)pl->d_tinyW, (void*)pl->hA2, (void*)pl->hB2,
                  (void*)pl->hC2,
                  (void*)pl->hC})
    if (p) cudaFree(p);
  if (pl->done) cudaEventDestroy(pl->done);
  if (pl->cublas) cublas()->Destroy(pl->cublas);
  if (pl->g_exec) cudaGraphExecDestroy(pl->g_exec);
  for (auto& set : pl->prof_events)
    for (cudaEvent_t e : set) cudaEventDestroy(e);
  for (cudaEvent_t e : pl->pipe_events) cudaEventDestroy(e);
  for (cudaEvent_t e : pl->comm_events) cudaEventDestroy(e);
  for (cudaEvent_t e : pl->in_events) cudaEventDestroy(e);
  for (cudaEvent_t e : {pl->set_free[0], pl->set_free[1], pl->compute_done, pl->ser_in[0],
                        pl->ser_in[1], pl->ser_done[0], pl->ser_done[1]})
    if (e) cudaEventDestroy(e);
  for (auto& b : pl->batches) {
    for (void* p : {b.mixA.d_table, b.mixB.d_table, b.mixC.d_table})
      if (p) cudaFree(p);
    for (MixTable* t : {&b.mixA, &b.mixB, &b.mixC}) jit_free(*t);
  }
  for (MixTable* t : {&pl->mixA, &pl->mixB, &pl->mixC, &pl->mixA2, &pl->mixC2}) jit_free(*t);
  for (cudaStream_t st : {pl->h2d, pl->d2h, pl->mixs, pl->s2, pl->comm_s, pl->cs1})
    if (st) cudaStreamDestroy(st);
}

// Events of the current call when profiling is on (nullptr otherwise).  At
// most kMaxProfSets sets are kept between reads; later calls are not recorded.
constexpr size_t kMaxProfSets = 4096;
cudaEvent_t* prof_slot(Plan* pl) {
  if (!pl->opt.profile || pl->prof_used >= kMaxProfSets) return nullptr;
  if (pl->prof_used == pl->prof_events.size()) {
    std::vector<cudaEvent_t> set(6, nullptr);
    for (auto& e : set)
      if (cudaEventCreate(&e) != cudaSuccess) return nullptr;
    pl->prof_events.push_back(set);
  }
  return pl->prof_events[pl->prof_used++].data();
}

// do the address ranges of X (rx rows) and Y (ry rows), n columns each, intersect?
bool overlaps(const double* X, int64_t ldx, int64_t rx, const double* Y, int64_t ldy, int64_t ry,
              int64_t n) {
  auto lo1 = reinterpret_cast<uintptr_t>(X), hi1 = lo1 + 8 * ((rx - 1) * ldx + n);
  auto lo2 = reinterpret_cast<uintptr_t>(Y), hi2 = lo2 + 8 * ((ry - 1) * ldy + n);
  return lo1 < hi2 && lo2 < hi1;
}

// MF_LEAF_CUBLAS: row-major P = X*Y is column-major P^T = Y^T X^T, so each
// product is cublasDgemm(N, N, cols, rows, m, Y, ldy, X, ldx, P, ldo); jobs are
// grouped by (ldx, ldy) (aliased operands have ld n, workspace slots ld m).
mf_status run_leaf_cublas(Plan& pl, const double* A, int64_t lda, const double* B, int64_t ldb,
                          const double* T, const double* S, double* out, int64_t ldo,
                          int64_t stride, double alpha, cudaStream_t s, Rows rows, int j0, int nj) {
  Cublas* cb = cublas();
  if (!cb) return fail(MF_ERR_CUDA, "MF_LEAF_CUBLAS: libcublas.so.12 could not be loaded");
  if (!pl.cublas && cb->Create(&pl.cublas) != 0) return fail(MF_ERR_CUDA, "cublasCreate failed");
  if (cb->SetStream(pl.cublas, s) != 0) return fail(MF_ERR_CUDA, "cublasSetStream failed");
  const int64_t m = pl.m, mm = m * m;
  const int64_t r0 = rows.r0, r1 = rows.end(m), c0 = rows.c0, c1 = rows.cend(m);
  if (nj == 0 || r1 <= r0 || c1 <= c0) return MF_OK;
  if (m > INT32_MAX || lda > INT32_MAX || ldb > INT32_MAX || ldo > INT32_MAX)
    return fail(MF_ERR_UNSUPPORTED, "MF_LEAF_CUBLAS: dimensions exceed int32");
  struct Group { int64_t ldx, ldy; std::vector<const double*> x, y, p; };
  std::vector<Group> groups;
  for (int j = j0; j < j0 + nj; ++j) {
    const LeafJob& jb = pl.h_jobs[j];
    const bool aw = jb.flags & 1, bw = jb.flags & 2;
    const double* X = aw ? T + (int64_t)jb.a_coord * mm
                         : A + (int64_t)(jb.a_coord >> 16) * m * lda + (int64_t)(jb.a_coord & 0xffff) * m;
    const double* Y = bw ? S + (int64_t)jb.b_coord * mm
                         : B + (int64_t)(jb.b_coord >> 16) * m * ldb + (int64_t)(jb.b_coord & 0xffff) * m;
    const int64_t ldx = aw ? m : lda, ldy = bw ? m : ldb;
    Group* g = nullptr;
    for (auto& e : groups)
      if (e.ldx == ldx && e.ldy == ldy) g = &e;
    if (!g) { groups.push_back(Group{ldx, ldy, {}, {}, {}}); g = &groups.back(); }
    g->x.push_back(X + r0 * ldx);
    g->y.push_back(Y + c0);
    g->p.push_back(out + (int64_t)jb.out_idx * stride + r0 * ldo + c0);
  }
  const size_t need = 3 * (size_t)nj;
  if (pl.d_ptrs_cap < need) {
    if (pl.d_ptrs) cudaFree(pl.d_ptrs);
    pl.d_ptrs = nullptr; pl.d_ptrs_cap = 0;
    MF_CUDA(cudaMalloc(&pl.d_ptrs, need * sizeof(double*)), "cudaMalloc(pointer arrays)");
    pl.d_ptrs_cap = need;
  }
  std::vector<const double*> host;
  host.reserve(need);
  for (auto& g : groups) {
    host.insert(host.end(), g.y.begin(), g.y.end());
    host.insert(host.end(), g.x.begin(), g.x.end());
    host.insert(host.end(), g.p.begin(), g.p.end());
  }
  // pageable source: the copy is staged before the call returns
  MF_CUDA(cudaMemcpyAsync(pl.d_ptrs, host.data(), host.size() * sizeof(double*),
                          cudaMemcpyHostToDevice, s), "H2D pointer arrays");
  const double beta = 0.0;
  size_t off = 0;
  for (auto& g : groups) {
    const int cnt = (int)g.x.size();
    const double* const* dy = pl.d_ptrs + off;
    const double* const* dx = dy + cnt;
    double* const* dp = const_cast<double* const*>(dx + cnt);
    if (cb->DgemmBatched(pl.cublas, 0, 0, (int)(c1 - c0), (int)(r1 - r0), (int)m, &alpha, dy,
                         (int)g.ldy, dx, (int)g.ldx, &beta, dp, (int)ldo, cnt) != 0)
      return fail(MF_ERR_CUDA, "cublasDgemmBatched failed");
    off += 3 * (size_t)cnt;
  }
  return MF_OK;
}

mf_status run_leaf(const Plan& pl, const double* A, int64_t lda, const double* B, int64_t ldb,
                   const double* T, const double* S, double* out, int64_t ldo, int64_t stride,
                   double alpha, cudaStream_t s, Rows rows = Rows(), bool part = false,
                   const Plan::Batch* batch = nullptr) {
  if (pl.leaf == MF_LEAF_CUBLAS)
    return run_leaf_cublas(const_cast<Plan&>(pl), A, lda, B, ldb, T, S, out, ldo, stride, alpha, s,
                           rows, batch ? batch->job0 : (part ? pl.n_jobs : 0),
                           batch ? batch->n_jobs : (part ? pl.n_jobs_part : pl.n_jobs));
  LeafArgs a;
  a.A = A; a.lda = lda; a.B = B; a.ldb = ldb; a.T = T; a.S = S;
  a.n_slots_a = pl.n_loc_a; a.n_slots_b = pl.n_loc_b;
  a.P = pl.P; a.m = pl.m;
  a.out = out; a.ldo = ldo; a.out_block_stride = stride; a.alpha = alpha;
  a.jobs = batch ? pl.d_jobs + batch->job0 : (part ? pl.d_jobs + pl.n_jobs : pl.d_jobs);
  a.n_jobs = batch ? batch->n_jobs : (part ? pl.n_jobs_part : pl.n_jobs);
  if (batch) { a.n_slots_a = batch->n_a; a.n_slots_b = batch->n_b; }
  a.rows = rows;
  if (pl.fuse && !batch && pl.levels > 0) {
    a.post_off = pl.d_post_off;
    a.post = pl.d_post;
    if (pl.fuse_ordered) { a.fuse_sync = pl.fuse_sync; a.fuse_sync_len = pl.fuse_sync_len; }
  }
  if (pl.leaf == MF_LEAF_DMMA) {
    // split-K tail workspace: grown to what this launch's tiling needs
    const LeafTiles cfg = leaf_tiles(a);
    Plan& mp = const_cast<Plan&>(pl);
    if (cfg.split > 1 && (mp.split_ws_elems < cfg.ws_elems || mp.split_cnt_len < cfg.n_tail)) {
      MF_CUDA(cudaStreamSynchronize(s), "sync before workspace growth");
      if (mp.split_ws) cudaFree(mp.split_ws);
      if (mp.split_cnt) cudaFree(mp.split_cnt);
      mp.split_ws = nullptr; mp.split_cnt = nullptr; mp.split_ws_elems = mp.split_cnt_len = 0;
      MF_CUDA(cudaMalloc(&mp.split_ws, sizeof(double) * cfg.ws_elems), "cudaMalloc(split-K workspace)");
      MF_CUDA(cudaMalloc(&mp.split_cnt, sizeof(int) * cfg.n_tail), "cudaMalloc(split-K counters)");
      MF_CUDA(cudaMemset(mp.split_cnt, 0, sizeof(int) * cfg.n_tail), "zero split-K counters");
      mp.split_ws_elems = cfg.ws_elems;
      mp.split_cnt_len = cfg.n_tail;
    }
    a.split_ws = mp.split_ws; a.split_ws_elems = mp.split_ws_elems;
    a.split_cnt = mp.split_cnt; a.split_cnt_len = mp.split_cnt_len;
  }
  MF_CUDA(launch_leaf(a, pl.leaf, s), "leaf kernel launch");
  return MF_OK;
}

}  // namespace

// =========================================================================== ABI
extern "C" {

const char* mf_last_error(void) { return g_err.c_str(); }

const char* mf_version(void) { return "mf 0.1.0 sm_100a"; }

static mf_status mf_plan_impl(mf_plan_t* out, int32_t p, int32_t R, const double* U,
                              const double* V, const double* W, int32_t levels, int64_t n,
                              const mf_options* opt, bool allow_split);

mf_status mf_plan(mf_plan_t* out, int32_t p, int32_t R, const double* U, const double* V,
                  const double* W, int32_t levels, int64_t n, const mf_options* opt) {
  return mf_plan_impl(out, p, R, U, V, W, levels, n, opt, true);
}

static mf_status mf_plan_impl(mf_plan_t* out, int32_t p, int32_t R, const double* U,
                              const double* V, const double* W, int32_t levels, int64_t n,
                              const mf_options* opt, bool allow_split) {
  g_err.clear();
  if (!out) return fail(MF_ERR_INVALID_ARG, "out is NULL");
  *out = nullptr;
  if (n < 1) return fail(MF_ERR_INVALID_ARG, "n must be >= 1 (got %lld)", (long long)n);
  if (levels < 0) return fail(MF_ERR_INVALID_ARG, "levels must be >= 0 (got %d)", levels);
  if (levels > 0 && (p < 1 || R < 1 || !U || !V || !W))
    return fail(MF_ERR_INVALID_ARG, "levels > 0 needs p >= 1, R >= 1 and U, V, W");
  mf_options o{};
  o.device = -1;
  if (opt) {
    if (opt->struct_size != 0 && opt->struct_size != (int32_t)sizeof(mf_options))
      return fail(MF_ERR_INVALID_ARG, "mf_options.struct_size %d != %d", opt->struct_size,
                  (int)sizeof(mf_options));
    o = *opt;
  }
  if (o.leaf != MF_LEAF_DMMA && o.leaf != MF_LEAF_SIMPLE && o.leaf != MF_LEAF_CUBLAS)
    return fail(MF_ERR_INVALID_ARG, "unknown leaf kind %d", o.leaf);
  if (o.output_mode != MF_OUT_ROOT && o.output_mode != MF_OUT_ALL && o.output_mode != MF_OUT_ROWSLAB)
    return fail(MF_ERR_INVALID_ARG, "unknown output_mode %d", o.output_mode);
  if (o.input_mode != MF_IN_ROOT && o.input_mode != MF_IN_REPLICATED)
    return fail(MF_ERR_INVALID_ARG, "unknown input_mode %d", o.input_mode);
  if (o.output_mode == MF_OUT_ROWSLAB && o.shard_count > 1 && n % o.shard_count != 0)
    return fail(MF_ERR_INVALID_ARG, "MF_OUT_ROWSLAB needs n %% shard_count == 0 (n = %lld, N = %d)",
                (long long)n, o.shard_count);
  if (o.fuse_postadd && o.leaf == MF_LEAF_CUBLAS)
    return fail(MF_ERR_UNSUPPORTED, "fuse_postadd needs the DMMA or simple leaf");
  if (o.comm_regions < 0)
    return fail(MF_ERR_INVALID_ARG, "comm_regions must be >= 0 (got %d)", o.comm_regions);
  if (o.recurse_levels < 0)
    return fail(MF_ERR_INVALID_ARG, "recurse_levels must be >= 0 (got %d)", o.recurse_levels);
  if (o.fuse_postadd && levels < 1)
    return fail(MF_ERR_UNSUPPORTED, "fuse_postadd needs levels >= 1");
  if (o.fuse_postadd && o.level_by_level && levels >= 2)
    return fail(MF_ERR_UNSUPPORTED, "fuse_postadd with level_by_level is not supported");
  if (o.fuse_postadd < 0 || o.fuse_postadd > 2)
    return fail(MF_ERR_INVALID_ARG, "fuse_postadd must be 0, 1 (ordered) or 2 (bulk reductions)");
  if (o.fuse_postadd == 1 && o.shard_count > 1)
    return fail(MF_ERR_UNSUPPORTED,
                "fuse_postadd = 1 (ordered fold) needs an unsharded plan; sharded plans take 2");
  const int shard_count = o.shard_count > 1 ? o.shard_count : 1;
  if (o.shard_rank < 0 || o.shard_rank >= shard_count)
    return fail(MF_ERR_INVALID_ARG, "shard_rank %d outside [0, %d)", o.shard_rank, shard_count);
  if (o.comm) {
    // the communicator fixes the sharding: rank r of N computes shard r of N
    const Comm* xc = comm_from(o.comm);
    if (!xc)
      return fail(MF_ERR_INVALID_ARG,
                  "mf_options.comm is not a handle from mf_nccl_comm_create / mf_loop_comm_create");
    if (xc->size != shard_count || xc->rank != o.shard_rank)
      return fail(MF_ERR_INVALID_ARG,
                  "shard_rank / shard_count (%d / %d) differ from the communicator's rank / size (%d / %d)",
                  o.shard_rank, shard_count, xc->rank, xc->size);
  }

  if (levels > 0) {
    mf_status st = brent_check(p, R, U, V, W);
    if (st != MF_OK) return st;
  }
  int64_t P = 1, RL = 1;
  for (int l = 0; l < levels; ++l) {
    if (n % (P * p) != 0)
      return fail(MF_ERR_INDIVISIBLE,
                  "n = %lld is not divisible by p^%d = %lld (p = %d, levels = %d)", (long long)n,
                  l + 1, (long long)(P * p), p, levels);
    P *= p;
    RL *= R;
  }
  if (o.level_by_level && levels >= 2) {
    // the paper's recursion: this plan = one level; each of its R products is
    // computed by a child plan of levels - 1 levels at n / p
    // top `r` levels one at a time; below them one flattened child plan
    const int r = (o.recurse_levels <= 0 || o.recurse_levels >= levels) ? levels - 1 : o.recurse_levels;
    mf_options top = o, sub = o;
    top.level_by_level = 0;
    top.recurse_levels = 0;
    sub.graph = 0;
    sub.level_by_level = r > 1 ? 1 : 0;
    sub.recurse_levels = r > 1 ? r - 1 : 0;
    sub.shard_rank = 0; sub.shard_count = 1; sub.comm = nullptr; sub.profile = 0;
    sub.input_mode = MF_IN_REPLICATED;
    mf_plan_t parent = nullptr, child = nullptr;
    mf_status st = mf_plan_impl(&parent, p, R, U, V, W, 1, n, &top, false);
    if (st != MF_OK) return st;
    st = mf_plan(&child, p, R, U, V, W, levels - 1, n / p, &sub);
    if (st != MF_OK) {
      std::string msg = g_err;
      mf_destroy(parent);
      g_err = msg;
      return st;
    }
    parent->child = child;
    parent->opt.level_by_level = 1;
    *out = parent;
    return MF_OK;
  }
  if (P > 256 || RL > (1 << 20))
    return fail(MF_ERR_UNSUPPORTED, "flattened triple too large (p^levels = %lld, R^levels = %lld)",
                (long long)P, (long long)RL);
  if (shard_count > RL)
    return fail(MF_ERR_INVALID_ARG, "shard_count %d exceeds the %lld leaf products", shard_count,
                (long long)RL);

  const bool host_only = o.host_only != 0;
  DeviceGuard guard(host_only ? -1 : o.device);
  if (!guard.ok) return fail(MF_ERR_CUDA, "cannot select device %d", o.device);
  std::unique_ptr<mf_plan_st> pl(new (std::nothrow) mf_plan_st());
  if (!pl) return fail(MF_ERR_OUT_OF_MEMORY, "host allocation");
  if (!host_only) MF_CUDA(cudaGetDevice(&pl->device), "cudaGetDevice");
  else pl->device = -1;
  pl->p = p; pl->R = R; pl->levels = levels; pl->n = n;
  pl->P = (int)P; pl->RL = RL; pl->m = n / P;
  pl->opt = o; pl->leaf = o.leaf; pl->fuse = o.fuse_postadd != 0;
  pl->fuse_ordered = o.fuse_postadd == 1;
  pl->shard_rank = o.shard_rank; pl->shard_count = shard_count;
  pl->comm = comm_from(o.comm);

  // ---- flatten: U^(x)L etc. (a5 of SURVEY.md §8a executed as one level) ----
  if (levels == 0) {
    pl->U = {1.0}; pl->V = {1.0}; pl->W = {1.0};
  } else {
    std::vector<double> u(U, U + p * p * R), v(V, V + p * p * R), w(W, W + p * p * R);
    int64_t pc = p, rc = R;
    for (int l = 1; l < levels; ++l) {
      std::vector<double> u2, v2, w2;
      kron((int)pc, rc, u, v, w, p, R, U, V, W, u2, v2, w2);
      u.swap(u2); v.swap(v2); w.swap(w2);
      pc *= p; rc *= R;
    }
    pl->U.swap(u); pl->V.swap(v); pl->W.swap(w);
  }

  // ---- classify operand columns: single +-1 entry => alias ----
  const int NB = pl->P * pl->P;
  // Sharding: base = RL / N whole products per rank in contiguous
  // ranges; the RL mod N leftovers are split by tile-aligned row slabs, rank r
  // taking slab r of each (shard = -1).  Without enough tile rows, or for the
  // parent of a level-by-level plan, the leftovers go whole to ranks instead.
  const int64_t base = RL / shard_count, left = RL % shard_count;
  const bool split = allow_split && levels > 0 && shard_count > 1 && left > 0 &&
                     (pl->m + 127) / 128 >= shard_count;
  if (split) {
    const int64_t tiles = (pl->m + 127) / 128;
    pl->part_r0 = std::min<int64_t>(pl->m, 128 * (pl->shard_rank * tiles / shard_count));
    pl->part_r1 = std::min<int64_t>(pl->m, 128 * ((pl->shard_rank + 1) * tiles / shard_count));
  }
  pl->prods.resize(RL);
  for (int64_t q = 0; q < RL; ++q) {
    Product& pr = pl->prods[q];
    pr.sign = 1;
    pr.shard = split ? (q < base * shard_count ? (int32_t)(q / base) : -1)
                     : (int32_t)((q * shard_count) / RL);
    for (int side = 0; side < 2; ++side) {
      const std::vector<double>& M = side == 0 ? pl->U : pl->V;
      int nnz = 0, k0 = -1;
      for (int k = 0; k < NB; ++k)
        if (M[k * RL + q] != 0.0) { ++nnz; if (k0 < 0) k0 = k; }
      const bool alias = nnz == 1 && std::fabs(M[k0 * RL + q]) == 1.0;
      int32_t& src = side == 0 ? pr.a_src : pr.b_src;
      int32_t& idx = side == 0 ? pr.a_idx : pr.b_idx;
      if (alias) {
        src = SRC_INPUT;
        idx = k0;
        if (M[k0 * RL + q] < 0) pr.sign = -pr.sign;
      } else {
        src = SRC_WORKSPACE;
        std::vector<int32_t>& cols = side == 0 ? pl->mat_a_col : pl->mat_b_col;
        idx = (int32_t)cols.size();
        cols.push_back((int32_t)q);
      }
    }
  }
  pl->n_mat_a = (int)pl->mat_a_col.size();
  pl->n_mat_b = (int)pl->mat_b_col.size();
  for (int64_t q = 0; q < RL; ++q) {
    if (pl->prods[q].shard == pl->shard_rank) pl->my_prods.push_back((int32_t)q);
    if (pl->prods[q].shard < 0) pl->my_part.push_back((int32_t)q);
  }

  // shard-local numbering (sharded per-rank workspace ~ 1/N): a
  // rank allocates and addresses only the T / S slots and P blocks of its own
  // products -- whole ones, then split ones (the leaf job order) -- slots in
  // ascending q.  The identity for unsharded plans.
  {
    std::vector<int32_t> jq = pl->my_prods;
    jq.insert(jq.end(), pl->my_part.begin(), pl->my_part.end());
    pl->loc_q.assign(RL, -1);
    for (size_t j = 0; j < jq.size(); ++j) pl->loc_q[jq[j]] = (int32_t)j;
    pl->n_loc_q = (int)jq.size();
    std::sort(jq.begin(), jq.end());
    pl->loc_a.assign(pl->n_mat_a, -1);
    pl->loc_b.assign(pl->n_mat_b, -1);
    for (int32_t q : jq) {
      const Product& pr = pl->prods[q];
      if (pr.a_src == SRC_WORKSPACE && pl->loc_a[pr.a_idx] < 0) pl->loc_a[pr.a_idx] = pl->n_loc_a++;
      if (pr.b_src == SRC_WORKSPACE && pl->loc_b[pr.b_idx] < 0) pl->loc_b[pr.b_idx] = pl->n_loc_b++;
    }
  }

  // plans of a compiled-in triple use the specialised K4/K6 (their slot and
  // product numbering is the whole triple's: unsharded plans only; a shard's
  // K4 / K6 are generated over its own slots and products)
  if (levels > 0 && RL <= 576 && shard_count == 1 && !getenv("MF_MIX_GENERIC")) {
    pl->fixed_id = fixed_match(*pl);
    if (pl->fixed_id == 0) pl->fixed_id = kron_match(*pl);
  }
  // the masks exist for the specialised K4/K6 only (RL <= 576 = 9 x 64 bits;
  // larger flattened plans run generated or table kernels and leave them empty)
  if (RL <= 64 * (int64_t)(sizeof(ProdMask::w) / sizeof(uint64_t))) {
    for (int32_t q : pl->my_prods) pl->mask_whole.w[q >> 6] |= 1ull << (q & 63);
    for (int32_t q : pl->my_part) pl->mask_part.w[q >> 6] |= 1ull << (q & 63);
    for (int i = 0; i < 9; ++i) pl->mask_all.w[i] = pl->mask_whole.w[i] | pl->mask_part.w[i];
  }

  // ---- mix tables for this shard ----
  auto add_slots = [&](MixTable& t, int side, const std::vector<int32_t>& qs) {
    const std::vector<double>& M = side == 0 ? pl->U : pl->V;
    t.nin = NB;
    for (int32_t q : qs) {
      const Product& pr = pl->prods[q];
      if ((side == 0 ? pr.a_src : pr.b_src) != SRC_WORKSPACE) continue;
      for (int k = 0; k < NB; ++k) t.coef.push_back(M[k * RL + q]);
      t.out_map.push_back(side == 0 ? pl->loc_a[pr.a_idx] : pl->loc_b[pr.b_idx]);
      ++t.nout;
    }
  };
  // K6 over the shard's P blocks (local product index = input index)
  auto post_table = [&](MixTable& c, bool with_part) {
    const int nq = pl->n_loc_q;
    c.nin = nq;
    c.nout = NB;
    c.coef.assign((size_t)NB * nq, 0.0);
    for (int i = 0; i < NB; ++i) c.out_map.push_back(i);
    for (int32_t q : pl->my_prods)
      for (int i = 0; i < NB; ++i) c.coef[(size_t)i * nq + pl->loc_q[q]] = pl->W[i * RL + q] * pl->prods[q].sign;
    if (with_part)
      for (int32_t q : pl->my_part)
        for (int i = 0; i < NB; ++i)
          c.coef[(size_t)i * nq + pl->loc_q[q]] = pl->W[i * RL + q] * pl->prods[q].sign;
  };
  if (levels > 0) {
    std::vector<int32_t> all = pl->my_prods;
    all.insert(all.end(), pl->my_part.begin(), pl->my_part.end());
    std::sort(all.begin(), all.end());
    add_slots(pl->mixA, 0, pl->my_prods);
    add_slots(pl->mixA2, 0, pl->my_part);
    add_slots(pl->mixB, 1, all);
    post_table(pl->mixC, false);
    if (!pl->my_part.empty()) post_table(pl->mixC2, true);
  }

  // ---- bounded workspace: batches of products whose T/S/P fit the cap ----
  const int64_t blk = (int64_t)sizeof(double) * pl->m * pl->m;
  if (levels > 0 && o.max_workspace > 0 &&
      (int64_t)(pl->n_mat_a + pl->n_mat_b + (pl->fuse ? 0 : RL)) * blk > o.max_workspace) {
    if (pl->fuse)
      return fail(MF_ERR_UNSUPPORTED, "fuse_postadd: T/S workspace exceeds max_workspace (no batching)");
    if (shard_count > 1)
      return fail(MF_ERR_UNSUPPORTED, "max_workspace with product sharding is not supported");
    const int64_t g = o.max_workspace / (3 * blk);
    if (g < 1)
      return fail(MF_ERR_OUT_OF_MEMORY, "max_workspace %lld < 3 leaf blocks (%lld bytes)",
                  (long long)o.max_workspace, (long long)(3 * blk));
    pl->fixed_id = 0;  // batches use the table-driven K4/K6
    const int nq = (int)pl->my_prods.size();
    for (int q0 = 0; q0 < nq; q0 += (int)g) {
      Plan::Batch b;
      const int q1 = std::min<int>(nq, q0 + (int)g);
      const int gb = q1 - q0;
      b.mixA.nin = b.mixB.nin = NB;
      b.mixC.nin = gb;
      b.mixC.nout = NB;
      b.mixC.coef.assign((size_t)NB * gb, 0.0);
      for (int i = 0; i < NB; ++i) b.mixC.out_map.push_back(i);
      for (int j = 0; j < gb; ++j) {
        const int32_t q = pl->my_prods[q0 + j];
        const Product& pr = pl->prods[q];
        for (int side = 0; side < 2; ++side) {
          if ((side == 0 ? pr.a_src : pr.b_src) != SRC_WORKSPACE) continue;
          MixTable& t = side == 0 ? b.mixA : b.mixB;
          const std::vector<double>& M = side == 0 ? pl->U : pl->V;
          for (int k = 0; k < NB; ++k) t.coef.push_back(M[k * RL + q]);
          t.out_map.push_back(side == 0 ? b.n_a++ : b.n_b++);
          ++t.nout;
        }
        for (int i = 0; i < NB; ++i) b.mixC.coef[(size_t)i * gb + j] = pl->W[i * RL + q] * pr.sign;
      }
      b.n_jobs = gb;
      pl->batches.push_back(std::move(b));
    }
  }

  if (host_only) {  // host logic only: no device work, no workspace
    pl->n_jobs = (int)pl->my_prods.size();
    pl->n_jobs_part = (int)pl->my_part.size();
    *out = pl.release();
    return MF_OK;
  }

  // ---- device allocations ----
  const int64_t mm = pl->m * pl->m;
  if (levels > 0) {
    size_t tb = sizeof(double) * mm * pl->n_loc_a, sb = sizeof(double) * mm * pl->n_loc_b,
           pb = sizeof(double) * mm * pl->n_loc_q;
    if (!pl->batches.empty()) {
      int na = 0, nb = 0, np = 0;
      for (auto& b : pl->batches) {
        na = std::max(na, b.n_a); nb = std::max(nb, b.n_b); np = std::max(np, b.n_jobs);
      }
      tb = sizeof(double) * mm * na; sb = sizeof(double) * mm * nb; pb = sizeof(double) * mm * np;
    }
    if (tb && cudaMalloc(&pl->T, tb) != cudaSuccess) { free_plan(pl.get()); return fail(MF_ERR_OUT_OF_MEMORY, "workspace T (%zu bytes)", tb); }
    if (sb && cudaMalloc(&pl->S, sb) != cudaSuccess) { free_plan(pl.get()); return fail(MF_ERR_OUT_OF_MEMORY, "workspace S (%zu bytes)", sb); }
    if (pl->fuse) pb = 0;  // leaf tiles are added straight into C
    if (pb && cudaMalloc(&pl->Pw, pb) != cudaSuccess) { free_plan(pl.get()); return fail(MF_ERR_OUT_OF_MEMORY, "workspace P (%zu bytes)", pb); }
    pl->ws_bytes = tb + sb + pb;
    mf_status st;
    if ((st = upload_table(pl->mixA)) != MF_OK || (st = upload_table(pl->mixB)) != MF_OK ||
        (st = upload_table(pl->mixC)) != MF_OK || (st = upload_table(pl->mixA2)) != MF_OK ||
        (st = upload_table(pl->mixC2)) != MF_OK) {
      free_plan(pl.get());
      return st;
    }
    for (auto& b : pl->batches)
      if ((st = upload_table(b.mixA)) != MF_OK || (st = upload_table(b.mixB)) != MF_OK ||
          (st = upload_table(b.mixC)) != MF_OK) {
      free_plan(pl.get());
      return st;
    }
    // small problems run the whole level as one cluster launch (mf_tiny.cu)
    if (levels > 0 && n <= 64 && pl->RL <= 64) {
      const size_t tb2 = sizeof(double) * pl->U.size();
      bool ok = cudaMalloc(&pl->d_tinyU, tb2) == cudaSuccess && cudaMalloc(&pl->d_tinyV, tb2) == cudaSuccess &&
                cudaMalloc(&pl->d_tinyW, tb2) == cudaSuccess;
      ok = ok && cudaMemcpy(pl->d_tinyU, pl->U.data(), tb2, cudaMemcpyHostToDevice) == cudaSuccess &&
           cudaMemcpy(pl->d_tinyV, pl->V.data(), tb2, cudaMemcpyHostToDevice) == cudaSuccess &&
           cudaMemcpy(pl->d_tinyW, pl->W.data(), tb2, cudaMemcpyHostToDevice) == cudaSuccess;
      if (!ok) { free_plan(pl.get()); return fail(MF_ERR_OUT_OF_MEMORY, "small-problem tables"); }
    }
    // triples without compiled-in K4/K6, and the local tables of batches:
    // generate and compile their kernels now (mf_jit.cpp)
    std::vector<JitJob> jj;
    if (pl->fixed_id == 0 && levels > 0) {
      // (a shard's K4 reads just the input blocks its slots use)
      for (MixTable* t : {&pl->mixA, &pl->mixA2, &pl->mixB}) jj.push_back({t, pl->P, 0});
      for (MixTable* t : {&pl->mixC, &pl->mixC2}) jj.push_back({t, 0, pl->P});
    }
    for (auto& b : pl->batches) {
      jj.push_back({&b.mixA, pl->P, 0});
      jj.push_back({&b.mixB, pl->P, 0});
      jj.push_back({&b.mixC, 0, pl->P});
    }
    for (const JitJob& j : jj) pl->jit_tables += j.t->nout > 0 && jit_shape(*j.t).vw > 0;
    pl->jit_built = jit_build_all(jj);
  }
  std::vector<LeafJob> jobs;
  std::vector<int32_t> job_q = pl->my_prods;
  job_q.insert(job_q.end(), pl->my_part.begin(), pl->my_part.end());
  for (int32_t q : job_q) {
    const Product& pr = pl->prods[q];
    LeafJob j;
    j.a_coord = pr.a_src == SRC_INPUT ? ((pr.a_idx / pl->P) << 16) | (pr.a_idx % pl->P) : pl->loc_a[pr.a_idx];
    j.b_coord = pr.b_src == SRC_INPUT ? ((pr.b_idx / pl->P) << 16) | (pr.b_idx % pl->P) : pl->loc_b[pr.b_idx];
    j.flags = (pr.a_src == SRC_WORKSPACE ? 1 : 0) | (pr.b_src == SRC_WORKSPACE ? 2 : 0);
    j.out_idx = levels > 0 ? pl->loc_q[q] : 0;
    jobs.push_back(j);
  }
  pl->n_jobs = (int)pl->my_prods.size();
  pl->n_jobs_part = (int)pl->my_part.size();
  {  // batch-local jobs: local slot indices, output into the batch's P block j
    int base = (int)jobs.size(), nq = 0;
    for (auto& b : pl->batches) {
      b.job0 = base;
      int la = 0, lb = 0;
      for (int j = 0; j < b.n_jobs; ++j) {
        const Product& pr = pl->prods[pl->my_prods[nq + j]];
        LeafJob jb;
        jb.a_coord = pr.a_src == SRC_INPUT ? ((pr.a_idx / pl->P) << 16) | (pr.a_idx % pl->P) : la++;
        jb.b_coord = pr.b_src == SRC_INPUT ? ((pr.b_idx / pl->P) << 16) | (pr.b_idx % pl->P) : lb++;
        jb.flags = (pr.a_src == SRC_WORKSPACE ? 1 : 0) | (pr.b_src == SRC_WORKSPACE ? 2 : 0);
        jb.out_idx = j;
        jobs.push_back(jb);
      }
      nq += b.n_jobs;
      base += b.n_jobs;
    }
  }
  if (!jobs.empty()) {
    if (cudaMalloc(&pl->d_jobs, sizeof(LeafJob) * jobs.size()) != cudaSuccess) {
      free_plan(pl.get());
      return fail(MF_ERR_OUT_OF_MEMORY, "job table");
    }
    const cudaError_t e = cudaMemcpy(pl->d_jobs, jobs.data(), sizeof(LeafJob) * jobs.size(),
                                     cudaMemcpyHostToDevice);
    if (e != cudaSuccess) {
      free_plan(pl.get());
      return cuda_fail(e, "upload job table");
    }
  }
  pl->h_jobs = jobs;
  if (pl->fuse) {
    // fused post-addition: product q feeds C block i with W'[i][q] (alias sign
    // folded in); terms sorted by coefficient so each value is staged once
    // indexed by the local product index (the leaf job's out_idx)
    const int nq = pl->n_loc_q;
    std::vector<int32_t> off(nq + 1, 0);
    std::vector<PostTerm> terms;
    std::vector<char> mine(RL, 0);
    for (int32_t q : job_q) mine[q] = 1;
    // ordered fold: the first and last product (ascending q) feeding each C block
    std::vector<int64_t> q_first(NB, -1), q_last(NB, -1);
    for (int64_t q = 0; q < RL; ++q)
      if (mine[q])
        for (int i = 0; i < NB; ++i)
          if (pl->W[i * RL + q] != 0.0) {
            if (q_first[i] < 0) q_first[i] = q;
            q_last[i] = q;
          }
    for (int i = 0; i < NB && pl->fuse_ordered; ++i)
      if (q_first[i] < 0) {  // (a valid triple feeds every C block)
        free_plan(pl.get());
        return fail(MF_ERR_BAD_TRIPLE, "C block %d has no product (ordered fold)", i);
      }
    std::vector<int32_t> n_seen(NB, 0);
    std::vector<std::vector<PostTerm>> per(nq);
    for (int64_t q = 0; q < RL; ++q) {
      if (!mine[q]) continue;
      std::vector<PostTerm>& tq = per[pl->loc_q[q]];
      for (int i = 0; i < NB; ++i) {
        const double w = pl->W[i * RL + q] * pl->prods[q].sign;
        if (w == 0.0) continue;
        const int32_t fl = (q == q_first[i] ? POST_FIRST : 0) | (q == q_last[i] ? POST_LAST : 0) |
                           (n_seen[i]++ << 8);  // ordered fold: the product's rank in block i
        tq.push_back(PostTerm{(int32_t)(((i / pl->P) << 16) | (i % pl->P)), fl, w});
      }
      // the bulk-reduction fold restages its tile once per coefficient value
      if (!pl->fuse_ordered)
        std::stable_sort(tq.begin(), tq.end(),
                         [](const PostTerm& x, const PostTerm& y) { return x.coef < y.coef; });
    }
    for (int j = 0; j < nq; ++j) {
      off[j] = (int32_t)terms.size();
      terms.insert(terms.end(), per[j].begin(), per[j].end());
    }
    off[nq] = (int32_t)terms.size();
    if (pl->fuse_ordered) {
      // per-tile-position flags of the widest tiling (64-wide tiles), then the
      // ticket and done counters; zero between launches
      const int64_t tiles = (int64_t)NB * ((pl->m + 127) / 128) * ((pl->m + 63) / 64);
      pl->fuse_sync_len = tiles;
      if (cudaMalloc(&pl->fuse_sync, sizeof(uint32_t) * (tiles + 8)) != cudaSuccess ||
          cudaMemset(pl->fuse_sync, 0, sizeof(uint32_t) * (tiles + 8)) != cudaSuccess) {
        free_plan(pl.get());
        return fail(MF_ERR_OUT_OF_MEMORY, "ordered fold flags");
      }
    }
    if (cudaMalloc(&pl->d_post_off, sizeof(int32_t) * off.size()) != cudaSuccess ||
        (!terms.empty() && cudaMalloc(&pl->d_post, sizeof(PostTerm) * terms.size()) != cudaSuccess)) {
      free_plan(pl.get());
      return fail(MF_ERR_OUT_OF_MEMORY, "fused post-addition table");
    }
    cudaError_t e = cudaMemcpy(pl->d_post_off, off.data(), sizeof(int32_t) * off.size(),
                               cudaMemcpyHostToDevice);
    if (e == cudaSuccess && !terms.empty())
      e = cudaMemcpy(pl->d_post, terms.data(), sizeof(PostTerm) * terms.size(), cudaMemcpyHostToDevice);
    if (e != cudaSuccess) {
      free_plan(pl.get());
      return cuda_fail(e, "upload fused post-addition table");
    }
  }
  if (cudaEventCreateWithFlags(&pl->done, cudaEventDisableTiming) != cudaSuccess) {
    free_plan(pl.get());
    return fail(MF_ERR_CUDA, "cudaEventCreate");
  }
  *out = pl.release();
  return MF_OK;
}

mf_status mf_destroy(mf_plan_t plan) {
  g_err.clear();
  if (!plan) return MF_OK;
  if (plan->child) mf_destroy(static_cast<mf_plan_t>(plan->child));
  free_plan(plan);
  delete plan;
  return MF_OK;
}

mf_status mf_plan_info(mf_plan_t pl, size_t* ws, int64_t* leaf_n, int64_t* n_products,
                       int32_t* n_mat_a, int32_t* n_mat_b) {
  if (!pl) return fail(MF_ERR_INVALID_ARG, "plan is NULL");
  if (ws) *ws = pl->ws_bytes;
  if (leaf_n) *leaf_n = pl->m;
  if (n_products) *n_products = pl->RL;
  if (n_mat_a) *n_mat_a = pl->n_mat_a;
  if (n_mat_b) *n_mat_b = pl->n_mat_b;
  return MF_OK;
}

mf_status mf_triple_kron(int32_t po, int32_t Ro, const double* Uo, const double* Vo,
                         const double* Wo, int32_t pi, int32_t Ri, const double* Ui,
                         const double* Vi, const double* Wi, double* U, double* V, double* W) {
  g_err.clear();
  if (po < 1 || pi < 1 || Ro < 1 || Ri < 1 || !Uo || !Vo || !Wo || !Ui || !Vi || !Wi || !U || !V || !W)
    return fail(MF_ERR_INVALID_ARG, "bad argument");
  if ((int64_t)po * pi > 256 || (int64_t)Ro * Ri > (1 << 20))
    return fail(MF_ERR_UNSUPPORTED, "composed triple too large");
  const size_t no = (size_t)po * po * Ro;
  std::vector<double> uo(Uo, Uo + no), vo(Vo, Vo + no), wo(Wo, Wo + no), u, v, w;
  kron(po, Ro, uo, vo, wo, pi, Ri, Ui, Vi, Wi, u, v, w);
  std::copy(u.begin(), u.end(), U);
  std::copy(v.begin(), v.end(), V);
  std::copy(w.begin(), w.end(), W);
  return MF_OK;
}

mf_status mf_plan_kernels(mf_plan_t pl, int32_t* jit_tables, int32_t* jit_built, int64_t* launches) {
  if (!pl) return fail(MF_ERR_INVALID_ARG, "plan is NULL");
  int32_t jt = 0, jb = 0;
  int64_t l[4] = {0, 0, 0, 0};
  for (const Plan* q = pl; q; q = q->child) {
    jt += q->jit_tables;
    jb += q->jit_built;
    for (int i = 0; i < 4; ++i) l[i] += q->mix_launches[i];
  }
  if (jit_tables) *jit_tables = jt;
  if (jit_built) *jit_built = jb;
  if (launches)
    for (int i = 0; i < 4; ++i) launches[i] = l[i];
  return MF_OK;
}

mf_status mf_plan_shard_rows(mf_plan_t pl, int64_t* r0, int64_t* r1) {
  if (!pl) return fail(MF_ERR_INVALID_ARG, "plan is NULL");
  if (r0) *r0 = pl->my_part.empty() ? 0 : pl->part_r0;
  if (r1) *r1 = pl->my_part.empty() ? 0 : pl->part_r1;
  return MF_OK;
}

mf_status mf_plan_products(mf_plan_t pl, int32_t* a_src, int32_t* a_idx, int32_t* b_src,
                           int32_t* b_idx, int32_t* sign, int32_t* shard) {
  if (!pl) return fail(MF_ERR_INVALID_ARG, "plan is NULL");
  for (int64_t q = 0; q < pl->RL; ++q) {
    const Product& pr = pl->prods[q];
    if (a_src) a_src[q] = pr.a_src;
    if (a_idx) a_idx[q] = pr.a_idx;
    if (b_src) b_src[q] = pr.b_src;
    if (b_idx) b_idx[q] = pr.b_idx;
    if (sign) sign[q] = pr.sign;
    if (shard) shard[q] = pr.shard;
  }
  return MF_OK;
}

static mf_status check_mat(const char* name, const void* X, int64_t ld, int64_t n) {
  if (!X) return fail(MF_ERR_INVALID_ARG, "%s is NULL", name);
  if (ld < n) return fail(MF_ERR_INVALID_ARG, "ld%s = %lld < n = %lld", name, (long long)ld, (long long)n);
  if (reinterpret_cast<uintptr_t>(X) % 8) return fail(MF_ERR_INVALID_ARG, "%s is not 8-byte aligned", name);
  return MF_OK;
}

static mf_status dgemm_eager(mf_plan_t pl, double alpha, const double* A, int64_t lda,
                             const double* B, int64_t ldb, double* C, int64_t ldc, void* stream);
static std::pair<int64_t, int64_t> tile_piece(int64_t m, int i, int n);

// Row regions of the region-overlapped exchange (mf_options.comm_regions).
// Without a communicator only an explicit comm_regions > 1 applies (the regions
// are computed, nothing is reduced: the emulated ranks' partial C, for tests).
static int comm_regions(const Plan& pl, bool with_comm) {
  if (pl.child || pl.fuse || !pl.batches.empty() || pl.levels == 0 ||
      (!with_comm && pl.opt.comm_regions <= 1))
    return 1;
  const int want = pl.opt.comm_regions > 0 ? pl.opt.comm_regions
                                           : (with_comm && pl.shard_count > 1 ? 8 : 1);
  return (int)std::max<int64_t>(1, std::min<int64_t>(want, (pl.m + 127) / 128));
}

// mf_options.graph: eager on the first call with an argument tuple, captured on
// the second (every allocation and attribute set-up already happened), replayed
// from then on.  The graph holds the same launches with the same parameters.
mf_status mf_dgemm(mf_plan_t pl, double alpha, const double* A, int64_t lda, const double* B,
                   int64_t ldb, double* C, int64_t ldc, void* stream) {
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (!pl || !pl->opt.graph || pl->opt.profile || pl->opt.host_only || pl->comm || pl->child ||
      pl->leaf == MF_LEAF_CUBLAS || s == nullptr || s == cudaStreamLegacy || s == cudaStreamPerThread)
    return dgemm_eager(pl, alpha, A, lda, B, ldb, C, ldc, stream);
  Plan::GraphKey key;
  key.A = A; key.B = B; key.C = C; key.lda = lda; key.ldb = ldb; key.ldc = ldc; key.alpha = alpha;
  DeviceGuard guard(pl->device);
  if (pl->g_exec && pl->g_key == key) {
    g_err.clear();
    MF_CUDA(cudaGraphLaunch(pl->g_exec, s), "cudaGraphLaunch");
    return MF_OK;
  }
  if (!(pl->g_has_seen && pl->g_seen == key)) {
    pl->g_seen = key;
    pl->g_has_seen = true;
    return dgemm_eager(pl, alpha, A, lda, B, ldb, C, ldc, stream);
  }
  MF_CUDA(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal), "cudaStreamBeginCapture");
  mf_status st = dgemm_eager(pl, alpha, A, lda, B, ldb, C, ldc, stream);
  cudaGraph_t graph = nullptr;
  const cudaError_t ce = cudaStreamEndCapture(s, &graph);
  if (st != MF_OK) {
    if (graph) cudaGraphDestroy(graph);
    return st;
  }
  if (ce != cudaSuccess || !graph)
    return fail(MF_ERR_CUDA, "graph capture failed: %s", cudaGetErrorString(ce));
  if (pl->g_exec) { cudaGraphExecDestroy(pl->g_exec); pl->g_exec = nullptr; }
  const cudaError_t ie = cudaGraphInstantiate(&pl->g_exec, graph, 0);
  cudaGraphDestroy(graph);
  if (ie != cudaSuccess) {
    pl->g_exec = nullptr;
    return fail(MF_ERR_CUDA, "cudaGraphInstantiate: %s", cudaGetErrorString(ie));
  }
  pl->g_key = key;
  MF_CUDA(cudaGraphLaunch(pl->g_exec, s), "cudaGraphLaunch");
  return MF_OK;
}

// ---- exchange schedule (a6): the collectives a rank issues, in order ----
// One generator serves mf_dgemm (which executes the ops) and mf_plan_exchange
// (which returns them, so CPU tests can replay the schedule with gloo).
// Offsets / counts in doubles, relative to the buffer named by buf / recv_buf
// (XB_A, XB_B: the n x n inputs, ld n; XB_C: the partial C, ld n; XB_COUT: this
// rank's output slab under MF_OUT_ROWSLAB).  Ops with one `group` id are issued
// in one group; `event` >= 0: the input slab event recorded after the group.
static std::pair<int64_t, int64_t> tile_piece(int64_t m, int i, int n);

static void input_schedule(const Plan& pl, int KI, std::vector<XOp>& ops) {
  const int64_t m = pl.m, n = pl.n;
  int group = 0;
  // B first: every product needs all of S_q, while the leaf's row region k
  // needs only A's slab k -- so region k can start when A's slab k landed
  for (int side = 1; side >= 0; --side)
    for (int k = 0; k < KI; ++k, ++group) {
      const auto sr = tile_piece(m, k, KI);
      for (int br = 0; br < pl.P && sr.second > sr.first; ++br) {
        XOp o{};
        o.kind = XK_BCAST;
        o.buf = o.recv_buf = side == 0 ? XB_A : XB_B;
        o.off = o.recv_off = (br * m + sr.first) * n;
        o.count = (sr.second - sr.first) * n;
        o.root = 0;
        o.group = group;
        o.event = -1;
        ops.push_back(o);
      }
      if (!ops.empty() && ops.back().group == group) ops.back().event = side * KI + k;
    }
}

// region rows [r0, r1) of every block row of the partial C (MF_OUT_ROWSLAB:
// cut at the owners' output slabs and reduced onto each owner)
static void region_schedule(const Plan& pl, int64_t r0, int64_t r1, int group, std::vector<XOp>& ops) {
  const int64_t m = pl.m, n = pl.n, slab = n / pl.shard_count;
  for (int br = 0; br < pl.P; ++br) {
    const int64_t row0 = br * m + r0, row1 = br * m + r1;
    if (pl.opt.output_mode == MF_OUT_ROWSLAB) {
      for (int64_t o = row0 / slab; o * slab < row1; ++o) {
        const int64_t a = std::max<int64_t>(row0, o * slab), b = std::min<int64_t>(row1, (o + 1) * slab);
        XOp x{};
        x.kind = XK_REDUCE;
        x.buf = XB_C;
        x.off = a * n;
        x.count = (b - a) * n;
        x.root = (int32_t)o;
        x.recv_buf = o == pl.shard_rank ? XB_COUT : XB_C;
        x.recv_off = o == pl.shard_rank ? (a - o * slab) * n : a * n;
        x.group = group;
        x.event = -1;
        ops.push_back(x);
      }
    } else {
      XOp x{};
      x.kind = pl.opt.output_mode == MF_OUT_ALL ? XK_ALLREDUCE : XK_REDUCE;
      x.buf = x.recv_buf = XB_C;
      x.off = x.recv_off = row0 * n;
      x.count = (row1 - row0) * n;
      x.root = 0;
      x.group = group;
      x.event = -1;
      ops.push_back(x);
    }
  }
}

// one collective on the whole partial C (no region schedule)
static void final_schedule(const Plan& pl, int group, std::vector<XOp>& ops) {
  const int64_t n = pl.n;
  XOp x{};
  x.buf = XB_C;
  x.root = 0;
  x.group = group;
  x.event = -1;
  if (pl.opt.output_mode == MF_OUT_ROWSLAB) {
    x.kind = XK_REDUCE_SCATTER;
    x.count = (n / pl.shard_count) * n;  // per rank
    x.recv_buf = XB_COUT;
  } else {
    x.kind = pl.opt.output_mode == MF_OUT_ALL ? XK_ALLREDUCE : XK_REDUCE;
    x.count = n * n;
    x.recv_buf = XB_C;
  }
  ops.push_back(x);
}

// issue ops[i0, i1) (whole groups) on stream s; base[b] = the buffer of XB_* b
static mf_status exec_ops(Comm* xc, const std::vector<XOp>& ops, size_t i0, size_t i1, double* const base[4],
                          cudaStream_t s, const std::vector<cudaEvent_t>* events) {
  mf_status st = MF_OK;
  for (size_t i = i0; i < i1;) {
    const int g = ops[i].group;
    if ((st = xc->group_start()) != MF_OK) return st;
    int ev = -1;
    for (; i < i1 && ops[i].group == g; ++i) {
      const XOp& o = ops[i];
      double* src = base[o.buf] + o.off;
      double* dst = base[o.recv_buf] + o.recv_off;
      switch (o.kind) {
        case XK_BCAST: st = xc->bcast(src, (size_t)o.count, o.root, s); break;
        case XK_REDUCE: st = xc->reduce(src, dst, (size_t)o.count, o.root, s); break;
        case XK_ALLREDUCE: st = xc->allreduce(src, dst, (size_t)o.count, s); break;
        default: st = xc->reduce_scatter(src, dst, (size_t)o.count, s); break;
      }
      if (st != MF_OK) {
        xc->group_end();
        return st;
      }
      if (o.event >= 0) ev = o.event;
    }
    if ((st = xc->group_end()) != MF_OK) return st;
    if (ev >= 0 && events) MF_CUDA(cudaEventRecord((*events)[ev], s), "event");
  }
  return MF_OK;
}

static mf_status ensure_events(std::vector<cudaEvent_t>& v, size_t k) {
  while (v.size() < k) {
    cudaEvent_t e;
    MF_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "cudaEventCreate");
    v.push_back(e);
  }
  return MF_OK;
}

// the default flattened schedule (not level-by-level, fused or batched)
static bool levels_flat(const Plan& pl) {
  return pl.levels > 0 && !pl.child && !pl.fuse && pl.batches.empty();
}

// Input row slabs of the MF_IN_ROOT broadcast (and of the K4 launches that
// follow each slab): as many as the exchange regions, at least 1.
static int input_slabs(const Plan& pl) {
  const int want = pl.opt.comm_regions > 0 ? pl.opt.comm_regions : 8;
  return (int)std::max<int64_t>(1, std::min<int64_t>(want, (pl.m + 127) / 128));
}

static mf_status dgemm_eager(mf_plan_t pl, double alpha, const double* A, int64_t lda,
                             const double* B, int64_t ldb, double* C, int64_t ldc, void* stream) {
  g_err.clear();
  if (!pl) return fail(MF_ERR_INVALID_ARG, "plan is NULL");
  if (pl->opt.host_only) return fail(MF_ERR_INVALID_ARG, "host-only plan cannot compute");
  const int64_t n = pl->n;
  Comm* const xc = pl->comm;
  const bool root_inputs = xc && pl->opt.input_mode == MF_IN_ROOT;
  const bool is_root = pl->shard_rank == 0;
  mf_status st;
  if (!root_inputs || is_root) {
    if ((st = check_mat("A", A, lda, n)) != MF_OK || (st = check_mat("B", B, ldb, n)) != MF_OK)
      return st;
  }
  // MF_OUT_ROWSLAB: C is this rank's n/N x n row slab of the reduced product
  const bool rowslab = xc && pl->opt.output_mode == MF_OUT_ROWSLAB;
  const int64_t c_rows = rowslab ? n / pl->shard_count : n;
  if ((st = check_mat("C", C, ldc, n)) != MF_OK) return st;
  if ((A && overlaps(A, lda, n, C, ldc, c_rows, n)) || (B && overlaps(B, ldb, n, C, ldc, c_rows, n)))
    return fail(MF_ERR_INVALID_ARG, "C overlaps A or B");
  if (xc && ldc != n)
    return fail(MF_ERR_UNSUPPORTED, "multi-GPU reduction needs ldc == n (got %lld)", (long long)ldc);
  DeviceGuard guard(pl->device);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int64_t m = pl->m;
  if (xc && !pl->comm_s) MF_CUDA(cudaStreamCreateWithFlags(&pl->comm_s, cudaStreamNonBlocking), "stream");

  // a6, input side (MF_IN_ROOT): rank 0's A and B reach the other ranks as
  // broadcasts of row slabs on the exchange stream -- slab k = rows
  // [r0_k, r1_k) of every block row, one contiguous piece per block row -- and
  // each rank's K4 of slab k starts as soon as that slab landed, so K4(A) runs
  // under the broadcast of B.  Rank 0 sends straight from
  // its A and B when they are contiguous (ld == n) and computes without waiting.
  const int KI = root_inputs ? input_slabs(*pl) : 1;
  bool wait_inputs = false;  // this rank's K4 / leaf wait for the slabs
  if (root_inputs) {
    const size_t bytes = sizeof(double) * n * n;
    double* bufA = nullptr;
    double* bufB = nullptr;
    if (is_root) {
      bufA = const_cast<double*>(A);
      bufB = const_cast<double*>(B);
      if (lda != n) {
        if (!pl->rA && cudaMalloc(&pl->rA, bytes) != cudaSuccess) return fail(MF_ERR_OUT_OF_MEMORY, "replica A");
        MF_CUDA(cudaMemcpy2DAsync(pl->rA, n * 8, A, lda * 8, n * 8, n, cudaMemcpyDeviceToDevice, s), "pack A");
        bufA = pl->rA;
      }
      if (ldb != n) {
        if (!pl->rB && cudaMalloc(&pl->rB, bytes) != cudaSuccess) return fail(MF_ERR_OUT_OF_MEMORY, "replica B");
        MF_CUDA(cudaMemcpy2DAsync(pl->rB, n * 8, B, ldb * 8, n * 8, n, cudaMemcpyDeviceToDevice, s), "pack B");
        bufB = pl->rB;
      }
    } else {
      if (pl->recvA) bufA = pl->recvA;
      else if (!pl->rA && cudaMalloc(&pl->rA, bytes) != cudaSuccess) return fail(MF_ERR_OUT_OF_MEMORY, "replica A");
      if (pl->recvB) bufB = pl->recvB;
      else if (!pl->rB && cudaMalloc(&pl->rB, bytes) != cudaSuccess) return fail(MF_ERR_OUT_OF_MEMORY, "replica B");
      if (!bufA) bufA = pl->rA;
      if (!bufB) bufB = pl->rB;
      wait_inputs = true;
    }
    if ((st = ensure_events(pl->in_events, 2 * (size_t)KI + 2)) != MF_OK) return st;
    // the exchange stream starts after the caller's prior work (packing, and
    // the previous call's reads of the replicas)
    MF_CUDA(cudaEventRecord(pl->in_events[2 * KI + 1], s), "event");
    MF_CUDA(cudaStreamWaitEvent(pl->comm_s, pl->in_events[2 * KI + 1], 0), "wait");
    std::vector<XOp> ops;
    input_schedule(*pl, KI, ops);
    double* const base[4] = {bufA, bufB, nullptr, nullptr};
    if ((st = exec_ops(xc, ops, 0, ops.size(), base, pl->comm_s, &pl->in_events)) != MF_OK) return st;
    MF_CUDA(cudaEventRecord(pl->in_events[2 * KI], pl->comm_s), "event");  // all landed
    A = bufA; lda = n; B = bufB; ldb = n;
  }

  double* const C_out = C;
  if (rowslab) {  // compute the full partial C in a plan buffer, reduce-scatter it below
    if (!pl->Cfull && cudaMalloc(&pl->Cfull, sizeof(double) * n * n) != cudaSuccess)
      return fail(MF_ERR_OUT_OF_MEMORY, "partial C buffer (MF_OUT_ROWSLAB)");
    C = pl->Cfull;
  }

  cudaEvent_t* ev = prof_slot(pl);
  if (pl->opt.profile) ++pl->prof_calls;
  bool reduced = false;  // C already summed over ranks region by region
  NvtxPhases nvtx;
  static const char* kPhase[6] = {"mf:K4 A", "mf:K4 B", "mf:K5 leaf", "mf:K6", "mf:exchange", nullptr};
  auto mark = [&](int i) {
    if (ev) cudaEventRecord(ev[i], s);
    nvtx.to(kPhase[i]);
  };
  // K4(A) on rows r of every block: the whole products' slots, then the split
  // products' slots on the part of r inside the rank's row slab
  auto premix_a_rows = [&](Rows r) -> mf_status {
    MF_CUDA(launch_premix(*pl, pl->mixA, A, lda, pl->T, s, r), "pre-add A (K4)");
    if (!pl->my_part.empty()) {
      Rows pr;
      pr.r0 = std::max<int64_t>(r.r0, pl->part_r0);
      pr.r1 = std::min<int64_t>(r.end(m), pl->part_r1);
      if (pr.r0 < pr.r1) MF_CUDA(launch_premix(*pl, pl->mixA2, A, lda, pl->T, s, pr), "pre-add A (K4, split)");
    }
    return MF_OK;
  };
  // MF_IN_ROOT with the region schedule: K4(A) of slab k runs right before the
  // leaf's region k (same rows), so A's broadcast overlaps the leaf, not only K4
  const bool a_by_region = wait_inputs && levels_flat(*pl) && comm_regions(*pl, pl->comm != nullptr) == KI && KI > 1;
  // K4 of one side for this shard (whole products' slots, then the split
  // products' slots on the rank's row slab), slab by slab behind the input
  // broadcast when this rank receives its inputs
  auto premix_side = [&](int side) -> mf_status {
    const MixTable& whole = side == 0 ? pl->mixA : pl->mixB;
    const double* X = side == 0 ? A : B;
    const int64_t ldx = side == 0 ? lda : ldb;
    double* out = side == 0 ? pl->T : pl->S;
    const int nk = wait_inputs ? KI : 1;
    for (int k = 0; k < nk; ++k) {
      Rows r;
      if (wait_inputs) {
        MF_CUDA(cudaStreamWaitEvent(s, pl->in_events[side * KI + k], 0), "wait");
        const auto sr = tile_piece(m, k, KI);
        r.r0 = sr.first; r.r1 = sr.second;
        if (r.r1 <= r.r0) continue;
      }
      if (side == 0) {
        if ((st = premix_a_rows(r)) != MF_OK) return st;
      } else {
        MF_CUDA(launch_premix(*pl, whole, X, ldx, out, s, r), "pre-add B (K4)");
      }
    }
    return MF_OK;
  };
  mark(0);
  if (tiny_eligible(*pl) && !getenv("MF_TINY_OFF")) {
    // n <= 64: the whole level in one cluster launch (profile: the leaf phase)
    mark(1); mark(2);
    MF_CUDA(launch_tiny(*pl, alpha, A, lda, B, ldb, C, ldc, s), "small-problem kernel");
    mark(3);
  } else if (pl->levels == 0) {
    mark(1); mark(2);
    if (wait_inputs) MF_CUDA(cudaStreamWaitEvent(s, pl->in_events[2 * KI], 0), "wait");
    if ((st = run_leaf(*pl, A, lda, B, ldb, nullptr, nullptr, C, ldc, 0, alpha, s)) != MF_OK) return st;
    mark(3);
  } else if (!pl->batches.empty()) {
    // bounded workspace: per batch K4(A), K4(B), K5, K6 (adding into C after the first)
    // (profiling: each batch records its own event set; phases sum over batches)
    for (size_t bi = 0; bi < pl->batches.size(); ++bi) {
      const Plan::Batch& b = pl->batches[bi];
      if (bi > 0 && ev) {
        mark(4); mark(5);
        ev = prof_slot(pl);
        mark(0);
      }
      MF_CUDA(launch_premix(*pl, b.mixA, A, lda, pl->T, s), "pre-add A (K4, batch)");
      mark(1);
      MF_CUDA(launch_premix(*pl, b.mixB, B, ldb, pl->S, s), "pre-add B (K4, batch)");
      mark(2);
      if ((st = run_leaf(*pl, A, lda, B, ldb, pl->T, pl->S, pl->Pw, pl->m, pl->m * pl->m, 1.0, s,
                         Rows(), false, &b)) != MF_OK)
        return st;
      mark(3);
      MF_CUDA(launch_postmix(*pl, b.mixC, alpha, pl->Pw, C, ldc, s, Rows(), bi > 0), "post-add (K6, batch)");
    }
  } else if (pl->fuse) {
    // fused post-addition: K4(A), K4(B) and the leaf, whose epilogue folds
    // W'[i][q] * P_q into each C block i (no K6, no P workspace).  Ordered
    // (fuse_postadd = 1): each tile position's products update C in ascending
    // q -- store first, add, alpha last: bitwise K6.  Bulk reductions (2): C
    // is zeroed first (profile: timed with pre-add A), order not fixed.
    if (!pl->fuse_ordered) MF_CUDA(cudaMemset2DAsync(C, ldc * 8, 0, n * 8, n, s), "zero C");
    if ((st = premix_side(0)) != MF_OK) return st;
    mark(1);
    if ((st = premix_side(1)) != MF_OK) return st;
    mark(2);
    if (wait_inputs) MF_CUDA(cudaStreamWaitEvent(s, pl->in_events[2 * KI], 0), "wait");
    if ((st = run_leaf(*pl, A, lda, B, ldb, pl->T, pl->S, C, ldc, 0, alpha, s)) != MF_OK) return st;
    if (!pl->my_part.empty()) {
      Rows pr;
      pr.r0 = pl->part_r0; pr.r1 = pl->part_r1;
      if ((st = run_leaf(*pl, A, lda, B, ldb, pl->T, pl->S, C, ldc, 0, alpha, s, pr, true)) != MF_OK)
        return st;
    }
    mark(3);
  } else {
    // a1, a2: fused pre-additions (K4) for this shard's materialised operands
    // (a_by_region: K4(A) runs per region below -- profiled in the leaf phase)
    if (!a_by_region && (st = premix_side(0)) != MF_OK) return st;
    mark(1);
    if ((st = premix_side(1)) != MF_OK) return st;
    mark(2);
    // aliased operands are read by the leaf straight from the received inputs
    if (wait_inputs && !a_by_region) MF_CUDA(cudaStreamWaitEvent(s, pl->in_events[2 * KI], 0), "wait");
    if (pl->child) {
      // a5: level by level -- each product P_q' = X_q Y_q is itself computed by
      // the (levels-1)-level child plan ("recursively solve P_i")
      const int64_t mm = m * m;
      for (int32_t q : pl->my_prods) {
        const Product& pr = pl->prods[q];
        const double* X = pr.a_src == SRC_WORKSPACE
                              ? pl->T + (int64_t)pl->loc_a[pr.a_idx] * mm
                              : A + (int64_t)(pr.a_idx / pl->P) * m * lda + (pr.a_idx % pl->P) * m;
        const double* Y = pr.b_src == SRC_WORKSPACE
                              ? pl->S + (int64_t)pl->loc_b[pr.b_idx] * mm
                              : B + (int64_t)(pr.b_idx / pl->P) * m * ldb + (pr.b_idx % pl->P) * m;
        const int64_t ldx = pr.a_src == SRC_WORKSPACE ? m : lda;
        const int64_t ldy = pr.b_src == SRC_WORKSPACE ? m : ldb;
        if ((st = mf_dgemm(static_cast<mf_plan_t>(pl->child), 1.0, X, ldx, Y, ldy,
                           pl->Pw + (int64_t)pl->loc_q[q] * mm, m, stream)) != MF_OK)
          return st;
      }
    } else if (comm_regions(*pl, pl->comm != nullptr) > 1) {
      // a3 + a4 + a6 by row regions (NEXT-4): region k's leaf products and
      // post-addition, then its rows of the partial C (one contiguous piece per
      // block row) are summed on the exchange stream while region k+1
      // computes -- reduced onto rank 0 (MF_OUT_ROOT), onto every rank
      // (MF_OUT_ALL), or onto the rank whose output row slab holds them
      // (MF_OUT_ROWSLAB: a region-wise reduce-scatter).  Every rank issues the
      // same collectives in the same order.
      const int K = comm_regions(*pl, pl->comm != nullptr);
      if (!pl->comm_s) MF_CUDA(cudaStreamCreateWithFlags(&pl->comm_s, cudaStreamNonBlocking), "stream");
      if ((st = ensure_events(pl->comm_events, (size_t)K + 1)) != MF_OK) return st;
      const bool exchange = xc != nullptr;
      auto post = [&](int64_t a, int64_t b, const MixTable& t) -> mf_status {
        if (a >= b) return MF_OK;
        Rows q;
        q.r0 = a; q.r1 = b;
        MF_CUDA(launch_postmix(*pl, t, alpha, pl->Pw, C, ldc, s, q), "post-add (K6, region)");
        return MF_OK;
      };
      MF_CUDA(cudaEventRecord(pl->comm_events[K], s), "event");
      MF_CUDA(cudaStreamWaitEvent(pl->comm_s, pl->comm_events[K], 0), "wait");  // exchange after K4
      for (int k = 0; k < K; ++k) {
        const auto rg = tile_piece(m, k, K);
        if (rg.second <= rg.first) continue;
        Rows r;
        r.r0 = rg.first; r.r1 = rg.second;
        if (a_by_region) {  // A's slab k (= region k's rows) landed: its K4, then the leaf
          MF_CUDA(cudaStreamWaitEvent(s, pl->in_events[k], 0), "wait");
          if ((st = premix_a_rows(r)) != MF_OK) return st;
        }
        if ((st = run_leaf(*pl, A, lda, B, ldb, pl->T, pl->S, pl->Pw, m, m * m, 1.0, s, r)) != MF_OK)
          return st;
        if (!pl->my_part.empty()) {
          Rows pr;
          pr.r0 = std::max<int64_t>(rg.first, pl->part_r0);
          pr.r1 = std::min<int64_t>(rg.second, pl->part_r1);
          if (pr.r0 < pr.r1 &&
              (st = run_leaf(*pl, A, lda, B, ldb, pl->T, pl->S, pl->Pw, m, m * m, 1.0, s, pr, true)) != MF_OK)
            return st;
          if ((st = post(rg.first, std::min<int64_t>(rg.second, pl->part_r0), pl->mixC)) != MF_OK ||
              (st = post(std::max<int64_t>(rg.first, pl->part_r0), std::min<int64_t>(rg.second, pl->part_r1),
                         pl->mixC2)) != MF_OK ||
              (st = post(std::max<int64_t>(rg.first, pl->part_r1), rg.second, pl->mixC)) != MF_OK)
            return st;
        } else if ((st = post(rg.first, rg.second, pl->mixC)) != MF_OK) {
          return st;
        }
        if (!exchange) continue;
        MF_CUDA(cudaEventRecord(pl->comm_events[k], s), "event");
        MF_CUDA(cudaStreamWaitEvent(pl->comm_s, pl->comm_events[k], 0), "wait");
        std::vector<XOp> ops;
        region_schedule(*pl, rg.first, rg.second, k, ops);
        double* const base[4] = {nullptr, nullptr, C, C_out};
        if ((st = exec_ops(xc, ops, 0, ops.size(), base, pl->comm_s, nullptr)) != MF_OK) return st;
      }
      MF_CUDA(cudaEventRecord(pl->comm_events[K], pl->comm_s), "event");
      MF_CUDA(cudaStreamWaitEvent(s, pl->comm_events[K], 0), "wait");
      reduced = true;  // (without a communicator: the region K6 wrote the partial C)
    } else {
      // a3: all leaf products in one launch (K5); split products on this rank's slab
      if ((st = run_leaf(*pl, A, lda, B, ldb, pl->T, pl->S, pl->Pw, m, m * m, 1.0, s)) != MF_OK)
        return st;
      if (!pl->my_part.empty()) {
        Rows pr;
        pr.r0 = pl->part_r0; pr.r1 = pl->part_r1;
        if ((st = run_leaf(*pl, A, lda, B, ldb, pl->T, pl->S, pl->Pw, m, m * m, 1.0, s, pr, true)) != MF_OK)
          return st;
      }
    }
    mark(3);
    // a4: fused post-addition (K6); rows holding split-product slabs use mixC2
    if (reduced) {
      // done region by region above
    } else if (pl->my_part.empty()) {
      MF_CUDA(launch_postmix(*pl, pl->mixC, alpha, pl->Pw, C, ldc, s), "post-add (K6)");
    } else {
      Rows lo, mid, hi;
      lo.r1 = pl->part_r0;
      mid.r0 = pl->part_r0; mid.r1 = pl->part_r1;
      hi.r0 = pl->part_r1;
      MF_CUDA(launch_postmix(*pl, pl->mixC, alpha, pl->Pw, C, ldc, s, lo), "post-add (K6)");
      MF_CUDA(launch_postmix(*pl, pl->mixC2, alpha, pl->Pw, C, ldc, s, mid), "post-add (K6)");
      MF_CUDA(launch_postmix(*pl, pl->mixC, alpha, pl->Pw, C, ldc, s, hi), "post-add (K6)");
    }
  }
  mark(4);
  if (xc && !reduced) {
    // a6: sum the partial C over ranks (NCCL over NVLink/NVSwitch)
    std::vector<XOp> ops;
    final_schedule(*pl, 0, ops);
    double* const base[4] = {nullptr, nullptr, C, C_out};
    if ((st = exec_ops(xc, ops, 0, ops.size(), base, s, nullptr)) != MF_OK) return st;
  }
  // the call's stream ends after the input broadcast (rank 0 sends from the
  // caller's A and B, which must stay untouched until then)
  if (root_inputs) MF_CUDA(cudaStreamWaitEvent(s, pl->in_events[2 * KI], 0), "wait");
  mark(5);
  return MF_OK;
}

mf_status mf_plan_exchange(mf_plan_t pl, int32_t* kind, int32_t* buf, int64_t* off, int64_t* count,
                           int32_t* root, int32_t* recv_buf, int64_t* recv_off, int32_t* group,
                           int32_t* phase, int64_t cap, int64_t* n_ops) {
  g_err.clear();
  if (!pl || !n_ops) return fail(MF_ERR_INVALID_ARG, "plan or n_ops is NULL");
  if (pl->shard_count < 2) { *n_ops = 0; return MF_OK; }
  std::vector<XOp> ops;
  std::vector<int32_t> ph;
  if (pl->opt.input_mode == MF_IN_ROOT && pl->levels > 0) {
    input_schedule(*pl, input_slabs(*pl), ops);
    ph.assign(ops.size(), 0);
  }
  const int K = comm_regions(*pl, true);
  int g0 = ops.empty() ? 0 : ops.back().group + 1;
  if (K > 1) {
    for (int k = 0; k < K; ++k) {
      const auto rg = tile_piece(pl->m, k, K);
      if (rg.second <= rg.first) continue;
      region_schedule(*pl, rg.first, rg.second, g0 + k, ops);
      ph.resize(ops.size(), 1 + k);
    }
  } else {
    final_schedule(*pl, g0, ops);
    ph.resize(ops.size(), 1);
  }
  *n_ops = (int64_t)ops.size();
  for (size_t i = 0; i < ops.size() && (int64_t)i < cap; ++i) {
    const XOp& o = ops[i];
    if (kind) kind[i] = o.kind;
    if (buf) buf[i] = o.buf;
    if (off) off[i] = o.off;
    if (count) count[i] = o.count;
    if (root) root[i] = o.root;
    if (recv_buf) recv_buf[i] = o.recv_buf;
    if (recv_off) recv_off[i] = o.recv_off;
    if (group) group[i] = o.group;
    if (phase) phase[i] = ph[i];
  }
  return MF_OK;
}

mf_status mf_profile_read(mf_plan_t pl, double* ms, int32_t* calls, int32_t reset) {
  g_err.clear();
  if (!pl) return fail(MF_ERR_INVALID_ARG, "plan is NULL");
  if (!pl->opt.profile) return fail(MF_ERR_INVALID_ARG, "plan was created without profile = 1");
  DeviceGuard guard(pl->device);
  double sum[5] = {0, 0, 0, 0, 0};
  for (size_t c = 0; c < pl->prof_used; ++c) {
    auto& ev = pl->prof_events[c];
    MF_CUDA(cudaEventSynchronize(ev[5]), "cudaEventSynchronize");
    for (int i = 0; i < 5; ++i) {
      float t = 0.f;
      MF_CUDA(cudaEventElapsedTime(&t, ev[i], ev[i + 1]), "cudaEventElapsedTime");
      sum[i] += t;
    }
  }
  if (ms)
    for (int i = 0; i < 5; ++i) ms[i] = sum[i];
  if (calls) *calls = (int32_t)pl->prof_calls;
  if (reset) { pl->prof_used = 0; pl->prof_calls = 0; }
  return MF_OK;
}

// Host-buffer pipeline.  Output region (i, j) -- rows of slab
// i, columns of slab j of every block -- needs A's row slab i and B's column
// slab j only (K4(A) on rows i, K4(B) on columns j, then K5 and K6 on the
// region).  Schedule:
//   h2d  : A_0, B_0, A_1, B_1, ... (interleaved, 1/NS and 1/NC of each)
//   mixs : (high priority) K4(A_i) / K4(B_j) as soon as the slab has landed
//   s, s2: regions in "shells" k = max(i, j) -- (k,0..k-1) then (0..k, k) --
//          alternating between two streams so one region's last wave overlaps
//          the next region's first
//   d2h  : each finished C region
// Compute starts after 1/NS + 1/NC of an input crossed PCIe; everything else
// overlaps.  Results are bitwise those of mf_dgemm (same kernels, same order
// per element) unless mf_dgemm's leaf cut a few-wave launch's tail into
// split-K pieces (region launches never split); then they agree to rounding.
static int pipeline_slabs(const Plan& pl) {
  if (pl.comm || pl.shard_count > 1 || pl.leaf != MF_LEAF_DMMA || pl.child ||
      !pl.batches.empty() || pl.fuse)
    return 1;
  // as many slabs as keep every region launch above 1.3 waves of 128x128
  // tiles (products x (tile rows per slab)^2 >= 1.3 SMs), up to 16 slabs
  // of >= 2 tile rows: fewer bytes must land before the first region starts
  // (n=16384 SW^2: sync call 202.7 -> 199.0 ms at 16 slabs vs 8), while a
  // sub-wave region would leave SMs idle (n=16384 SW^1 at 16 slabs: 112 tiles)
  const int64_t tiles = (pl.m + 127) / 128;
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, pl.device);
  const int64_t prods = std::max<int64_t>(1, (int64_t)pl.my_prods.size());
  int64_t want = 2;
  for (int64_t ns = 16; ns >= 2; --ns) {
    const int64_t per = tiles / ns;  // the smaller slabs
    if (per >= 2 && 10 * prods * per * per >= 13 * (int64_t)sms) { want = ns; break; }
  }
  if (const char* e = getenv("MF_HOST_SLABS")) want = std::max(2, atoi(e));
  return (int)std::min<int64_t>(want, tiles);
}

// piece i of n over the 128-aligned tiles of [0, m)
static std::pair<int64_t, int64_t> tile_piece(int64_t m, int i, int n) {
  const int64_t tiles = (m + 127) / 128;
  return {std::min<int64_t>(m, 128 * (i * tiles / n)), std::min<int64_t>(m, 128 * ((i + 1) * tiles / n))};
}

// Wait for every enqueued mf_dgemm_host_async call of the plan.
static mf_status host_drain(Plan* pl) {
  for (int b = 0; b < 2; ++b)
    if (pl->set_busy[b]) {
      MF_CUDA(cudaEventSynchronize(pl->set_free[b]), "cudaEventSynchronize");
      pl->set_busy[b] = false;
    }
  pl->compute_pending = false;
  return MF_OK;
}

static mf_status host_call(mf_plan_t pl, double alpha, const double* A, int64_t lda,
                           const double* B, int64_t ldb, double* C, int64_t ldc, void* stream,
                           bool async);

mf_status mf_dgemm_host(mf_plan_t pl, double alpha, const double* A, int64_t lda, const double* B,
                        int64_t ldb, double* C, int64_t ldc, void* stream) {
  return host_call(pl, alpha, A, lda, B, ldb, C, ldc, stream, false);
}

mf_status mf_dgemm_host_async(mf_plan_t pl, double alpha, const double* A, int64_t lda,
                              const double* B, int64_t ldb, double* C, int64_t ldc, void* stream) {
  return host_call(pl, alpha, A, lda, B, ldb, C, ldc, stream, true);
}

mf_status mf_host_sync(mf_plan_t pl) {
  g_err.clear();
  if (!pl) return fail(MF_ERR_INVALID_ARG, "plan is NULL");
  if (pl->opt.host_only) return MF_OK;
  DeviceGuard guard(pl->device);
  return host_drain(pl);
}

static mf_status host_call(mf_plan_t pl, double alpha, const double* A, int64_t lda,
                           const double* B, int64_t ldb, double* C, int64_t ldc, void* stream,
                           bool async) {
  g_err.clear();
  if (!pl) return fail(MF_ERR_INVALID_ARG, "plan is NULL");
  if (pl->opt.host_only) return fail(MF_ERR_INVALID_ARG, "host-only plan cannot compute");
  const int64_t n = pl->n;
  mf_status st;
  // MF_IN_ROOT: only rank 0's host A and B are read (the others may pass NULL)
  const bool root_in = pl->comm && pl->opt.input_mode == MF_IN_ROOT;
  const bool reads_inputs = !root_in || pl->shard_rank == 0;
  if (reads_inputs &&
      ((st = check_mat("A", A, lda, n)) != MF_OK || (st = check_mat("B", B, ldb, n)) != MF_OK))
    return st;
  if ((st = check_mat("C", C, ldc, n)) != MF_OK) return st;
  DeviceGuard guard(pl->device);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const size_t bytes = sizeof(double) * n * n;
  if (!pl->hA && cudaMalloc(&pl->hA, bytes) != cudaSuccess) return fail(MF_ERR_OUT_OF_MEMORY, "device A");
  if (!pl->hB && cudaMalloc(&pl->hB, bytes) != cudaSuccess) return fail(MF_ERR_OUT_OF_MEMORY, "device B");
  if (!pl->hC && cudaMalloc(&pl->hC, bytes) != cudaSuccess) return fail(MF_ERR_OUT_OF_MEMORY, "device C");
  const int ns = pipeline_slabs(*pl);
  // synchronous calls first finish every enqueued async call
  if (!async && (st = host_drain(pl)) != MF_OK) return st;
  if (ns <= 1) {
    // whole-matrix path (sharded, level-by-level, fused, batched or cuBLAS-leaf
    // plans): H2D, mf_dgemm, D2H.  Async calls alternate between two device
    // sets on three streams, so call k+1's copies in and call k-1's copy out
    // run under call k's compute; the compute stream orders the workspace.
    const int set = async ? (int)(pl->async_calls & 1) : 0;
    if (async) {
      if (!pl->hA2 && cudaMalloc(&pl->hA2, bytes) != cudaSuccess) return fail(MF_ERR_OUT_OF_MEMORY, "device A (2nd set)");
      if (!pl->hB2 && cudaMalloc(&pl->hB2, bytes) != cudaSuccess) return fail(MF_ERR_OUT_OF_MEMORY, "device B (2nd set)");
      if (!pl->hC2 && cudaMalloc(&pl->hC2, bytes) != cudaSuccess) return fail(MF_ERR_OUT_OF_MEMORY, "device C (2nd set)");
      for (cudaEvent_t* e : {&pl->set_free[0], &pl->set_free[1], &pl->ser_in[0], &pl->ser_in[1],
                             &pl->ser_done[0], &pl->ser_done[1]})
        if (!*e) MF_CUDA(cudaEventCreateWithFlags(e, cudaEventDisableTiming), "cudaEventCreate");
      for (cudaStream_t* q : {&pl->h2d, &pl->d2h, &pl->cs1})
        if (!*q) MF_CUDA(cudaStreamCreateWithFlags(q, cudaStreamNonBlocking), "stream");
    }
    double* const dA = set ? pl->hA2 : pl->hA;
    double* const dB = set ? pl->hB2 : pl->hB;
    double* const dC = set ? pl->hC2 : pl->hC;
    cudaStream_t cin = async ? pl->h2d : s, cc = async ? pl->cs1 : s, cout = async ? pl->d2h : s;
    // a set is refilled once its previous call's copy out (after its compute) is done
    if (async && pl->set_busy[set]) MF_CUDA(cudaStreamWaitEvent(cin, pl->set_free[set], 0), "wait");
    const int N = pl->shard_count;
    Comm* const xc = pl->comm;
    const bool slabs = xc && n % N == 0 && pl->opt.input_mode == MF_IN_REPLICATED &&
                       !getenv("MF_HOST_FULLCOPY");
    const int64_t rows = slabs ? n / N : n, r0 = slabs ? (int64_t)pl->shard_rank * rows : 0;
    // product-sharded ranks with replicated host inputs copy only their 1/N
    // row slab of A and B over their own PCIe link; the exchange all-gathers
    // the rest over NVLink (in place) -- host traffic per GPU falls by N.
    // MF_IN_ROOT: rank 0 alone copies A and B in; mf_dgemm broadcasts them
    // into the other ranks' device sets (slab by slab, under their K4).
    if (reads_inputs) {
      MF_CUDA(cudaMemcpy2DAsync(dA + r0 * n, n * 8, A + r0 * lda, lda * 8, n * 8, rows,
                                cudaMemcpyHostToDevice, cin), "H2D A");
      MF_CUDA(cudaMemcpy2DAsync(dB + r0 * n, n * 8, B + r0 * ldb, ldb * 8, n * 8, rows,
                                cudaMemcpyHostToDevice, cin), "H2D B");
    }
    if (async) {
      MF_CUDA(cudaEventRecord(pl->ser_in[set], cin), "event");
      MF_CUDA(cudaStreamWaitEvent(cc, pl->ser_in[set], 0), "wait");
    }
    if (slabs) {
      if ((st = xc->group_start()) != MF_OK) return st;
      if ((st = xc->allgather(dA + r0 * n, dA, (size_t)rows * n, cc)) != MF_OK ||
          (st = xc->allgather(dB + r0 * n, dB, (size_t)rows * n, cc)) != MF_OK) {
        xc->group_end();
        return st;
      }
      if ((st = xc->group_end()) != MF_OK) return st;
    }
    if (root_in && !reads_inputs) {
      pl->recvA = dA;  // receive rank 0's broadcast into this device set
      pl->recvB = dB;
      st = mf_dgemm(pl, alpha, nullptr, n, nullptr, n, dC, n, cc);
      pl->recvA = pl->recvB = nullptr;
    } else if (slabs) {
      mf_options saved = pl->opt;  // inputs are replicated now
      pl->opt.input_mode = MF_IN_REPLICATED;
      st = mf_dgemm(pl, alpha, dA, n, dB, n, dC, n, cc);
      pl->opt = saved;
    } else {
      st = mf_dgemm(pl, alpha, dA, n, dB, n, dC, n, cc);
    }
    if (st != MF_OK) return st;
    if (async) {
      MF_CUDA(cudaEventRecord(pl->ser_done[set], cc), "event");
      MF_CUDA(cudaStreamWaitEvent(cout, pl->ser_done[set], 0), "wait");
    }
    const int64_t c_rows =
        pl->comm && pl->opt.output_mode == MF_OUT_ROWSLAB ? n / pl->shard_count : n;
    // MF_OUT_ROOT: C is defined on rank 0 only -- the other ranks copy nothing back
    const bool want_c = !(pl->comm && pl->opt.output_mode == MF_OUT_ROOT && pl->shard_rank != 0);
    if (want_c)
      MF_CUDA(cudaMemcpy2DAsync(C, ldc * 8, dC, n * 8, n * 8, c_rows, cudaMemcpyDeviceToHost, cout), "D2H C");
    if (async) {
      MF_CUDA(cudaEventRecord(pl->set_free[set], cout), "event");
      pl->set_busy[set] = true;
      MF_CUDA(cudaStreamWaitEvent(s, pl->set_free[set], 0), "wait");  // the caller's stream ends after it
      ++pl->async_calls;
      return MF_OK;
    }
    MF_CUDA(cudaStreamSynchronize(s), "cudaStreamSynchronize");
    return MF_OK;
  }
  const int64_t m = pl->m;
  const int P = pl->P;
  const int nc = ns;  // square grid of regions
  // async calls alternate between two device sets so call k+1's inputs
  // stream in while call k computes
  const int set = async ? (int)(pl->async_calls & 1) : 0;
  if (async) {  // both sets on the first async call: no allocation inside a running stream
    if (!pl->hA2 && cudaMalloc(&pl->hA2, bytes) != cudaSuccess) return fail(MF_ERR_OUT_OF_MEMORY, "device A (2nd set)");
    if (!pl->hB2 && cudaMalloc(&pl->hB2, bytes) != cudaSuccess) return fail(MF_ERR_OUT_OF_MEMORY, "device B (2nd set)");
    if (!pl->hC2 && cudaMalloc(&pl->hC2, bytes) != cudaSuccess) return fail(MF_ERR_OUT_OF_MEMORY, "device C (2nd set)");
  }
  if (async) {
    for (cudaEvent_t* e : {&pl->set_free[0], &pl->set_free[1], &pl->compute_done})
      if (!*e) MF_CUDA(cudaEventCreateWithFlags(e, cudaEventDisableTiming), "cudaEventCreate");
    if (!pl->cs1) MF_CUDA(cudaStreamCreateWithFlags(&pl->cs1, cudaStreamNonBlocking), "stream");
  }
  double* const setA = set ? pl->hA2 : pl->hA;
  double* const setB = set ? pl->hB2 : pl->hB;
  double* const setC = set ? pl->hC2 : pl->hC;
  cudaStream_t const cs_main = async ? pl->cs1 : s;  // first compute stream
  if (!pl->h2d) MF_CUDA(cudaStreamCreateWithFlags(&pl->h2d, cudaStreamNonBlocking), "stream");
  if (!pl->d2h) MF_CUDA(cudaStreamCreateWithFlags(&pl->d2h, cudaStreamNonBlocking), "stream");
  if (!pl->s2) MF_CUDA(cudaStreamCreateWithFlags(&pl->s2, cudaStreamNonBlocking), "stream");
  if (!pl->mixs) {
    int lo = 0, hi = 0;
    MF_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi), "priority range");
    MF_CUDA(cudaStreamCreateWithPriority(&pl->mixs, cudaStreamNonBlocking, hi), "stream");
  }
  const size_t nev = 4 + 2 * (size_t)ns + 2 * (size_t)nc + (size_t)ns * nc;
  while (pl->pipe_events.size() < nev) {
    cudaEvent_t e;
    MF_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "cudaEventCreate");
    pl->pipe_events.push_back(e);
  }
  cudaEvent_t e_start = pl->pipe_events[0], e_done = pl->pipe_events[1], e_s2 = pl->pipe_events[2];
  cudaEvent_t* e_a = &pl->pipe_events[4];   // A slab i landed
  cudaEvent_t* e_b = e_a + ns;              // B slab j landed
  cudaEvent_t* e_pa = e_b + nc;             // K4(A_i) done
  cudaEvent_t* e_pb = e_pa + ns;            // K4(B_j) done
  cudaEvent_t* e_c = e_pb + nc;             // region done
  const double* dA = setA;
  const double* dB = setB;
  double* dC = setC;
  int region_no = 0;

  if (!async) {
    MF_CUDA(cudaEventRecord(e_start, s), "event");
    for (cudaStream_t st : {pl->h2d, pl->d2h, pl->mixs, pl->s2})
      MF_CUDA(cudaStreamWaitEvent(st, e_start, 0), "wait");
  } else {
    // inputs may overwrite this set once its previous user's D2H is done;
    // K4 rewrites the shared T/S workspace once the previous call's leaves ran
    if (pl->set_busy[set]) MF_CUDA(cudaStreamWaitEvent(pl->h2d, pl->set_free[set], 0), "wait");
    if (pl->compute_pending) MF_CUDA(cudaStreamWaitEvent(pl->mixs, pl->compute_done, 0), "wait");
  }
  // h2d: A_0, B_0, A_1, B_1, ...
  for (int k = 0; k < std::max(ns, nc); ++k) {
    if (k < ns) {
      const auto sr = tile_piece(m, k, ns);
      for (int br = 0; br < P; ++br) {
        const int64_t row = br * m + sr.first;
        MF_CUDA(cudaMemcpy2DAsync(setA + row * n, n * 8, A + row * lda, lda * 8, n * 8,
                                  sr.second - sr.first, cudaMemcpyHostToDevice, pl->h2d), "H2D A slab");
      }
      MF_CUDA(cudaEventRecord(e_a[k], pl->h2d), "event");
    }
    if (k < nc) {
      const auto sc = tile_piece(m, k, nc);
      for (int bc = 0; bc < P; ++bc)
        MF_CUDA(cudaMemcpy2DAsync(setB + bc * m + sc.first, n * 8, B + bc * m + sc.first, ldb * 8,
                                  (sc.second - sc.first) * 8, n, cudaMemcpyHostToDevice, pl->h2d),
                "H2D B slab");
      MF_CUDA(cudaEventRecord(e_b[k], pl->h2d), "event");
    }
  }
  // mixs: K4 per slab, as soon as it landed
  for (int k = 0; k < std::max(ns, nc); ++k) {
    if (k < ns) {
      MF_CUDA(cudaStreamWaitEvent(pl->mixs, e_a[k], 0), "wait");
      const auto sr = tile_piece(m, k, ns);
      Rows rows;
      rows.r0 = sr.first; rows.r1 = sr.second;
      if (pl->levels > 0)
        MF_CUDA(launch_premix(*pl, pl->mixA, dA, n, pl->T, pl->mixs, rows), "pre-add A (K4)");
      MF_CUDA(cudaEventRecord(e_pa[k], pl->mixs), "event");
    }
    if (k < nc) {
      MF_CUDA(cudaStreamWaitEvent(pl->mixs, e_b[k], 0), "wait");
      const auto sc = tile_piece(m, k, nc);
      Rows cols;
      cols.c0 = sc.first; cols.c1 = sc.second;
      if (pl->levels > 0)
        MF_CUDA(launch_premix(*pl, pl->mixB, dB, n, pl->S, pl->mixs, cols), "pre-add B (K4)");
      MF_CUDA(cudaEventRecord(e_pb[k], pl->mixs), "event");
    }
  }
  // regions in shells, alternating compute streams
  auto region = [&](int i, int j) -> mf_status {
    cudaStream_t cs = (region_no & 1) ? pl->s2 : cs_main;
    MF_CUDA(cudaStreamWaitEvent(cs, e_pa[i], 0), "wait");
    MF_CUDA(cudaStreamWaitEvent(cs, e_pb[j], 0), "wait");
    const auto sr = tile_piece(m, i, ns);
    const auto sc = tile_piece(m, j, nc);
    Rows rg;
    rg.r0 = sr.first; rg.r1 = sr.second; rg.c0 = sc.first; rg.c1 = sc.second;
    rg.overlapped = true;  // regions alternate over two compute streams
    if (pl->levels == 0) {
      if ((st = run_leaf(*pl, dA, n, dB, n, nullptr, nullptr, dC, n, 0, alpha, cs, rg)) != MF_OK) return st;
    } else {
      if ((st = run_leaf(*pl, dA, n, dB, n, pl->T, pl->S, pl->Pw, m, m * m, 1.0, cs, rg)) != MF_OK)
        return st;
      MF_CUDA(launch_postmix(*pl, pl->mixC, alpha, pl->Pw, dC, n, cs, rg), "post-add (K6)");
    }
    cudaEvent_t ev = e_c[region_no++];
    MF_CUDA(cudaEventRecord(ev, cs), "event");
    MF_CUDA(cudaStreamWaitEvent(pl->d2h, ev, 0), "wait");
    for (int br = 0; br < P; ++br)
      for (int bc = 0; bc < P; ++bc) {
        const int64_t row = br * m + rg.r0, col = bc * m + rg.c0;
        MF_CUDA(cudaMemcpy2DAsync(C + row * ldc + col, ldc * 8, dC + row * n + col, n * 8,
                                  (rg.c1 - rg.c0) * 8, rg.r1 - rg.r0, cudaMemcpyDeviceToHost,
                                  pl->d2h),
                "D2H C region");
      }
    return MF_OK;
  };
  for (int k = 0; k < std::max(ns, nc); ++k) {
    if (k < ns)
      for (int j = 0; j < std::min(k, nc); ++j)
        if ((st = region(k, j)) != MF_OK) return st;
    if (k < nc)
      for (int i = 0; i <= std::min(k, ns - 1); ++i)
        if ((st = region(i, k)) != MF_OK) return st;
  }
  if (async) {
    // compute done (both compute streams) -> the next call's K4 may start;
    // last D2H done -> this set is free; the caller's stream ends after both
    MF_CUDA(cudaEventRecord(e_s2, pl->s2), "event");
    MF_CUDA(cudaStreamWaitEvent(pl->cs1, e_s2, 0), "wait");
    MF_CUDA(cudaEventRecord(pl->compute_done, pl->cs1), "event");
    pl->compute_pending = true;
    MF_CUDA(cudaEventRecord(pl->set_free[set], pl->d2h), "event");
    pl->set_busy[set] = true;
    MF_CUDA(cudaStreamWaitEvent(s, pl->set_free[set], 0), "wait");
    ++pl->async_calls;
    return MF_OK;
  }
  MF_CUDA(cudaEventRecord(e_done, pl->d2h), "event");
  MF_CUDA(cudaEventRecord(e_s2, pl->s2), "event");
  MF_CUDA(cudaStreamWaitEvent(s, e_s2, 0), "wait");    // the call's stream ends after all work
  MF_CUDA(cudaStreamWaitEvent(s, e_done, 0), "wait");
  MF_CUDA(cudaEventSynchronize(e_done), "cudaEventSynchronize");
  return MF_OK;
}

// Diagnostic entry (include/mf.h): generate and compile the kernel of one
// coefficient table for an architecture, without a GPU -- the CPU tests use it
// to check the generator's output compiles.
mf_status mf_jit_compile_check(const double* coef, int32_t nout, int32_t nin,
                               int32_t in_P, int32_t out_P, const char* arch,
                               int32_t* vw_out, int64_t* cubin_bytes) {
  g_err.clear();
  if (!coef || nout <= 0 || nin <= 0 || in_P < 0 || out_P < 0 || !arch)
    return fail(MF_ERR_INVALID_ARG, "bad argument");
  MixTable t;
  t.nin = nin;
  t.nout = nout;
  t.coef.assign(coef, coef + (size_t)nout * nin);
  for (int o = 0; o < nout; ++o) t.out_map.push_back(o);
  const JitShape sh = jit_shape(t);
  if (vw_out) *vw_out = sh.vw;
  if (sh.vw == 0) return fail(MF_ERR_UNSUPPORTED, "table too large for a generated kernel");
  std::vector<char> cubin;
  std::string log;
  if (!jit_compile(jit_source(t, in_P, out_P, sh), arch, cubin, log))
    return fail(MF_ERR_UNSUPPORTED, "NVRTC: %.400s", log.c_str());
  if (cubin_bytes) *cubin_bytes = (int64_t)cubin.size();
  return MF_OK;
}

mf_status mf_premix(mf_plan_t pl, int32_t side, const double* X, int64_t ldx, double* out,
                    void* stream) {
  g_err.clear();
  if (!pl || !X || !out || (side != 0 && side != 1)) return fail(MF_ERR_INVALID_ARG, "bad argument");
  if (!pl->batches.empty()) return fail(MF_ERR_UNSUPPORTED, "component entry points need the full workspace");
  if (pl->opt.host_only) return fail(MF_ERR_INVALID_ARG, "host-only plan cannot compute");
  if (pl->levels == 0) return fail(MF_ERR_INVALID_ARG, "levels = 0 plan has no pre-additions");
  DeviceGuard guard(pl->device);
  MF_CUDA(launch_premix(*pl, side == 0 ? pl->mixA : pl->mixB, X, ldx, out,
                        static_cast<cudaStream_t>(stream)),
          "pre-add (K4)");
  return MF_OK;
}

mf_status mf_leaf(mf_plan_t pl, const double* A, int64_t lda, const double* B, int64_t ldb,
                  const double* T, const double* S, double* P, void* stream) {
  g_err.clear();
  if (!pl || !A || !B || !P) return fail(MF_ERR_INVALID_ARG, "bad argument");
  if (!pl->batches.empty()) return fail(MF_ERR_UNSUPPORTED, "component entry points need the full workspace");
  if (pl->opt.host_only) return fail(MF_ERR_INVALID_ARG, "host-only plan cannot compute");
  DeviceGuard guard(pl->device);
  return run_leaf(*pl, A, lda, B, ldb, T, S, P, pl->m, pl->m * pl->m, 1.0,
                  static_cast<cudaStream_t>(stream));
}

mf_status mf_postmix(mf_plan_t pl, double alpha, const double* P, double* C, int64_t ldc,
                     void* stream) {
  g_err.clear();
  if (!pl || !P || !C) return fail(MF_ERR_INVALID_ARG, "bad argument");
  if (!pl->batches.empty()) return fail(MF_ERR_UNSUPPORTED, "component entry points need the full workspace");
  if (pl->opt.host_only) return fail(MF_ERR_INVALID_ARG, "host-only plan cannot compute");
  if (pl->levels == 0) return fail(MF_ERR_INVALID_ARG, "levels = 0 plan has no post-addition");
  DeviceGuard guard(pl->device);
  MF_CUDA(launch_postmix(*pl, pl->mixC, alpha, P, C, ldc, static_cast<cudaStream_t>(stream)),
          "post-add (K6)");
  return MF_OK;
}

}  // extern "C"
