// mf_internal.h -- plan structure and kernel launchers shared by the libmf.so
// translation units (product path only; nothing here is shared with oracle/).
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <string>
#include <vector>

#include "../../include/mf.h"

namespace mf {

// error reporting (mf_api.cpp): sets the thread-local message of mf_last_error
mf_status fail(mf_status st, const char* fmt, ...);

// The exchange layer of the sharded path (mf_comm.cu): NCCL across processes,
// or N in-process loopback ranks (threads).  Handles returned through the ABI
// are Comm* (checked by magic).  Counts are in doubles.  Every rank issues the
// same collectives in the same order.
constexpr uint32_t kCommMagic = 0x4d46434du;  // "MFCM"
struct Comm {
  uint32_t magic = kCommMagic;
  int rank = 0, size = 1;
  virtual ~Comm() {}
  virtual const char* kind() const = 0;
  // in place: root's buf is the source, every other rank's buf receives it
  virtual mf_status bcast(void* buf, size_t count, int root, cudaStream_t s) = 0;
  // recv (root only) = sum over ranks of send; recv may equal send
  virtual mf_status reduce(const double* send, double* recv, size_t count, int root,
                           cudaStream_t s) = 0;
  virtual mf_status allreduce(const double* send, double* recv, size_t count, cudaStream_t s) = 0;
  // recv (recvcount) = sum over ranks of send[rank * recvcount ...]
  virtual mf_status reduce_scatter(const double* send, double* recv, size_t recvcount,
                                   cudaStream_t s) = 0;
  // recv[k * sendcount ...] = send of rank k (send may be recv + rank * sendcount)
  virtual mf_status allgather(const double* send, double* recv, size_t sendcount,
                              cudaStream_t s) = 0;
  virtual mf_status group_start() { return MF_OK; }
  virtual mf_status group_end() { return MF_OK; }
};
Comm* comm_from(void* handle);  // nullptr if handle is not a Comm of this library

// One collective of the exchange schedule (mf_api.cpp; mf_plan_exchange).
enum XKind : int32_t { XK_BCAST = 0, XK_REDUCE = 1, XK_ALLREDUCE = 2, XK_REDUCE_SCATTER = 3 };
enum XBuf : int32_t { XB_A = 0, XB_B = 1, XB_C = 2, XB_COUT = 3 };
struct XOp {
  int32_t kind, buf;        // XKind; the send buffer (XBuf)
  int64_t off, count;       // doubles (count: per rank for a reduce-scatter)
  int32_t root, recv_buf;   // root rank; the receive buffer
  int64_t recv_off;
  int32_t group, event;     // issued together; input slab event after the group (-1: none)
};

// Largest flattened split factor P = p^levels the mix kernels are built for
// (P^2 <= 81 blocks: p=9 one level, p=3 two levels, p=2 up to three levels).
constexpr int kMaxBlocks = 81;

// Operand source of a leaf product (mf_plan_products: a_src / b_src).
enum Src : int32_t { SRC_INPUT = 0, SRC_WORKSPACE = 1 };

// One leaf product P_q' = X_q * Y_q of the flattened triple.
struct Product {
  int32_t a_src, a_idx;  // A-block index (SRC_INPUT) or T slot (SRC_WORKSPACE)
  int32_t b_src, b_idx;  // B-block index or S slot
  int32_t sign;          // +-1 folded out of aliased operands
  int32_t shard;         // shard that computes it
};

// Product mask for the specialised K4/K6 (bit q = product q is computed by
// this plan's shard; up to 576 products).  Passed by value to the kernels.
struct ProdMask {
  uint64_t w[9];
  __host__ __device__ bool has(int q) const { return (w[q >> 6] >> (q & 63)) & 1ull; }
};

// Device-side routing entry of the leaf kernel (kept POD, 16 bytes).
struct LeafJob {
  int32_t a_coord;  // SRC_INPUT: (block_row << 16) | block_col; SRC_WORKSPACE: slot
  int32_t b_coord;
  int32_t flags;    // bit0: A from workspace, bit1: B from workspace
  int32_t out_idx;  // index of the output block in P (or 0 with direct C output)
};

// Fused post-addition (mf_options.fuse_postadd): product q's tiles are added
// into C blocks post[post_off[q] .. post_off[q+1]) with coef*alpha; terms of one
// product are sorted by coef so the epilogue restages its tile once per value.
// Ordered fold (fuse_postadd = 1): flags mark the product that writes C block
// i first (store, no load) and last (alpha applied) in ascending q; bits 8..
// hold the product's rank among block i's products (the flag value it waits for).
enum PostFlags : int32_t { POST_FIRST = 1, POST_LAST = 2 };
struct PostTerm {
  int32_t blk;    // (block_row << 16) | block_col of the C block
  int32_t flags;  // PostFlags (ordered fold only)
  double coef;    // W'[i][q] with the alias sign folded in
};

// Coefficient table of one mix kernel launch: nout outputs, each a
// combination of up to nin inputs, coef[o * nin + k] (0 = absent).
// Device form: MixRow[nrow] then MixTerm[nterm]; row o's terms are
// terms[first .. first+count) in ascending input order (the oracle's order).
enum MixKind : int32_t { MIX_POS = 0, MIX_NEG = 1, MIX_GEN = 2 };
struct MixRow {
  int32_t first, count;
  int32_t target;  // output block / slot id in the output view
  int32_t pad;
};
struct MixTerm {
  int32_t src;   // input block / slot id in the input view
  int32_t kind;  // MixKind
  double coef;   // used when kind == MIX_GEN
};

// Grouped form (the kernel used when it fits): outputs in groups of `gsize`
// (<= MIX_GMAX) that share inputs; a group lists the union of its outputs'
// inputs in ascending order, each entry carrying one coefficient per output
// (0 = absent), so a warp loads every input of its group once and updates all
// of the group's accumulators from registers.  Entry e of the device table is
// {int32 src, int32 pad, double coef[gsize]} (8 + 8*gsize bytes).
constexpr int MIX_GMAX = 4;
struct MixGroup {
  int32_t first, count;           // entries [first, first+count)
  int32_t target[MIX_GMAX];       // output block / slot per member, -1 = none
};

struct MixTable {
  int nin = 0, nout = 0;
  std::vector<double> coef;      // nout x nin
  std::vector<int32_t> out_map;  // output o -> slot / C block it writes
  int nrow = 0, nterm = 0;       // device table sizes
  void* d_table = nullptr;       // device MixRow + MixTerm table (owned by the plan),
                                 // then the grouped table at byte offset goff
  int gsize = 0, ngroup = 0;     // grouped form (gsize 0 = not built)
  size_t goff = 0, gbytes = 0;
  // kernel generated for this table at plan time (mf_jit.cpp; CUmodule /
  // CUfunction, owned by the plan), 0 = none
  void* jit_mod = nullptr;
  void* jit_fn = nullptr;
  int jit_vw = 0;
};

// mf_jit.cpp: K4/K6 generated per table (NVRTC) -- register shape, source,
// compile, load, launch
struct JitShape {
  int vw = 0;               // positions per thread (0 = does not fit)
  bool input_major = false; // accumulators held (true) or inputs held
};
JitShape jit_shape(const MixTable& t);
std::string jit_source(const MixTable& t, int in_P, int out_P, const JitShape& sh);
bool jit_compile(const std::string& src, const char* arch, std::vector<char>& cubin, std::string& log);
struct JitJob {
  MixTable* t;
  int in_P, out_P;  // partition factor of a block view, 0 = slot view
};
int jit_build_all(const std::vector<JitJob>& jobs);
void jit_free(MixTable& t);

// kinds of K4/K6 launches counted per plan (mf_plan_kernels)
enum MixKernelKind { MIXK_TABLE = 0, MIXK_FIXED = 1, MIXK_KRON = 2, MIXK_JIT = 3 };

struct Plan {
  int device = 0;
  // K4/K6 provenance: tables that asked for a generated kernel, kernels built,
  // and launches per MixKernelKind since the plan was made
  int jit_tables = 0, jit_built = 0;
  mutable int64_t mix_launches[4] = {0, 0, 0, 0};
  int p = 1, R = 1, levels = 0;
  int64_t n = 0;
  // flattened triple: P = p^levels, RL = R^levels; U/V/W are P^2 x RL row-major
  int P = 1;
  int64_t RL = 1, m = 0;
  std::vector<double> U, V, W;
  std::vector<Product> prods;
  int n_mat_a = 0, n_mat_b = 0;         // materialised T / S slots (whole triple)
  std::vector<int32_t> mat_a_col, mat_b_col;  // slot -> product column q
  mf_options opt{};
  int leaf = MF_LEAF_DMMA;
  int fixed_id = 0;  // 1..7: flattened K4/K6 (mf_fixed.cu); 8..: Kronecker-factored (mf_kron.cu)
  int shard_rank = 0, shard_count = 1;
  // shard-local view: the products this plan's rank computes whole,
  // and the leftover products (R^L mod N of them) of which every rank computes
  // the row slab part_rows -- exact balance at R^L / N products per rank
  std::vector<int32_t> my_prods;  // whole products q
  std::vector<int32_t> my_part;   // split products q (this rank: rows part_rows)
  int64_t part_r0 = 0, part_r1 = 0;
  // shard-local numbering: global slot / product -> local index (-1: not this
  // rank's), and the local counts the workspace is sized by
  std::vector<int32_t> loc_a, loc_b, loc_q;
  int n_loc_a = 0, n_loc_b = 0, n_loc_q = 0;
  MixTable mixA, mixB;            // pre-additions: A slots of whole products, all B slots used
  MixTable mixA2;                 // A slots of split products (rows part_rows only)
  MixTable mixC;                  // post-addition over the whole products (zero coef elsewhere)
  MixTable mixC2;                 // ... plus the split products (used on rows part_rows)
  int n_jobs_part = 0;            // leaf jobs of split products follow the whole ones in d_jobs
  ProdMask mask_whole{}, mask_part{}, mask_all{};  // for the specialised K4/K6
  // bounded workspace (mf_options.max_workspace): product batches with local
  // slot numbering; each has its own K4/K6 tables and leaf jobs (d_jobs + job0)
  struct Batch {
    MixTable mixA, mixB, mixC;
    int job0 = 0, n_jobs = 0;
    int n_a = 0, n_b = 0;  // local T / S slots
  };
  std::vector<Batch> batches;
  // device memory
  double* T = nullptr;   // n_mat_a x m x m
  double* S = nullptr;   // n_mat_b x m x m
  double* Pw = nullptr;  // RL x m x m (leaf outputs; not allocated when fused)
  bool fuse = false;     // mf_options.fuse_postadd != 0
  bool fuse_ordered = false;  // fuse_postadd == 1: deterministic ordered fold
  uint32_t* fuse_sync = nullptr;  // ordered fold: per-tile flags, ticket, done counter
  int64_t fuse_sync_len = 0;      // flags (tiles of the widest tiling)
  int32_t* d_post_off = nullptr;  // RL + 1
  PostTerm* d_post = nullptr;
  size_t ws_bytes = 0;
  LeafJob* d_jobs = nullptr;  // my_prods.size() jobs
  // small problems (mf_tiny.cu): the flattened U, V, W on the device
  double* d_tinyU = nullptr;
  double* d_tinyV = nullptr;
  double* d_tinyW = nullptr;
  std::vector<LeafJob> h_jobs;  // host copy (MF_LEAF_CUBLAS builds pointer arrays from it)
  void* cublas = nullptr;       // cublasHandle_t (MF_LEAF_CUBLAS), created on first use
  const double** d_ptrs = nullptr;  // device pointer arrays for cublasDgemmBatched
  size_t d_ptrs_cap = 0;
  double* Cfull = nullptr;      // MF_OUT_ROWSLAB: the full partial C before reduce-scatter
  // mf_options.graph: the step as an instantiated CUDA graph for one argument tuple
  struct GraphKey {
    const double *A = nullptr, *B = nullptr;
    double* C = nullptr;
    int64_t lda = 0, ldb = 0, ldc = 0;
    double alpha = 0.0;
    bool operator==(const GraphKey& o) const {
      return A == o.A && B == o.B && C == o.C && lda == o.lda && ldb == o.ldb && ldc == o.ldc &&
             alpha == o.alpha;
    }
  };
  GraphKey g_key, g_seen;       // key of g_exec; key of the last eager call
  bool g_has_seen = false;
  cudaGraphExec_t g_exec = nullptr;
  double* split_ws = nullptr;   // leaf split-K tail: partial tiles (grown on demand)
  int64_t split_ws_elems = 0;
  int* split_cnt = nullptr;     // ... and arrival counters (zeroed at allocation)
  int64_t split_cnt_len = 0;
  int n_jobs = 0;
  // host-buffer path (mf_dgemm_host): device copies of A, B, C
  double *hA = nullptr, *hB = nullptr, *hC = nullptr;
  // mf_dgemm_host_async: a second device set (calls alternate between the two),
  // the event that frees each set (its last D2H), the previous call's compute
  // completion, and the plan-owned first compute stream of async calls
  double *hA2 = nullptr, *hB2 = nullptr, *hC2 = nullptr;
  cudaEvent_t set_free[2] = {nullptr, nullptr};
  bool set_busy[2] = {false, false};
  cudaEvent_t compute_done = nullptr;
  cudaEvent_t ser_in[2] = {nullptr, nullptr};    // whole-matrix async path: inputs landed
  cudaEvent_t ser_done[2] = {nullptr, nullptr};  // ... and computed
  bool compute_pending = false;
  cudaStream_t cs1 = nullptr;
  int64_t async_calls = 0;
  // exchange (mf_options.comm): the communicator, MF_IN_ROOT
  // replicas of A and B on ranks that receive them, and -- set by the
  // host-buffer path for one call -- receive buffers used instead of them
  Comm* comm = nullptr;
  double *rA = nullptr, *rB = nullptr;
  double *recvA = nullptr, *recvB = nullptr;
  cudaEvent_t done = nullptr;
  // level-by-level recursion (mf_options.level_by_level): the plan of each
  // leaf product (levels - 1 levels at n / p); this plan is then one level
  Plan* child = nullptr;
  // host-buffer pipeline (mf_dgemm_host): copy streams and per-slab events
  cudaStream_t h2d = nullptr, d2h = nullptr, mixs = nullptr, s2 = nullptr;
  cudaStream_t comm_s = nullptr;  // exchange stream: input broadcasts, region reduces
  std::vector<cudaEvent_t> comm_events;  // region k computed (k < K), K4 done (K)
  std::vector<cudaEvent_t> in_events;    // MF_IN_ROOT: A slab k landed, B slab k landed, all
  std::vector<cudaEvent_t> pipe_events;
  // phase profiling (mf_options.profile): 6 events per mf_dgemm call
  std::vector<std::vector<cudaEvent_t>> prof_events;
  size_t prof_used = 0;   // event sets recorded (one per call, or per batch)
  int64_t prof_calls = 0; // mf_dgemm calls since the last reset
};

// Region [r0, r1) x [c0, c1) of every m x m block a launch covers (the whole
// block by default); the host-buffer pipeline runs the path piece by piece.
// Column bounds are multiples of 64 (or m) -- tile and vector aligned.
struct Rows {
  int64_t r0 = 0, r1 = -1;  // r1 < 0 => m
  int64_t c0 = 0, c1 = -1;  // c1 < 0 => m
  // the launch shares the GPU with concurrent launches on another stream (the
  // host pipeline's alternating regions): the leaf keeps 128-wide tiles, the
  // other stream fills its partial last wave
  bool overlapped = false;
  int64_t end(int64_t m) const { return r1 < 0 ? m : r1; }
  int64_t cend(int64_t m) const { return c1 < 0 ? m : c1; }
};

// ---- launchers (mf_mix.cu, mf_leaf.cu); return cudaError_t of the launch ----
cudaError_t launch_premix(const Plan& pl, const MixTable& t, const double* X, int64_t ldx,
                          double* out, cudaStream_t s, Rows rows = Rows());
cudaError_t launch_postmix(const Plan& pl, const MixTable& t, double alpha, const double* Pw,
                           double* C, int64_t ldc, cudaStream_t s, Rows rows = Rows(),
                           bool accumulate = false);

// mf_jit.cpp: launch a table's generated kernel; cudaErrorNotSupported when
// it has none or cannot serve these views (callers then use mf_mix.cu's)
cudaError_t jit_launch(const MixTable& t, const double* X, int64_t ldx, double* Y, int64_t ldy,
                       int64_t m, double alpha, Rows rows, int accumulate, cudaStream_t s);

struct LeafArgs {
  // operand views: matrices (4-D block view, SRC_INPUT) and workspaces (3-D)
  const double* A; int64_t lda;
  const double* B; int64_t ldb;
  const double* T; const double* S;
  int n_slots_a, n_slots_b;
  int P;          // blocks per side of the input partition
  int64_t m;      // leaf side
  double* out;    // output base: P workspace (ld m, block stride m*m) or C
  int64_t ldo;
  int64_t out_block_stride;  // elements between consecutive output blocks (0 => single)
  double alpha;
  const LeafJob* jobs; int n_jobs;
  Rows rows;      // output rows of each product computed (r0 multiple of 128)
  // fused post-addition: post != nullptr => job q's tile is added into C
  // (ldc) per post[post_off[out_idx] ..) instead of stored to out
  const int32_t* post_off = nullptr;
  const PostTerm* post = nullptr;
  // ordered fold (fuse_postadd = 1): products of one tile position update C
  // in job (= ascending q) order; flags[tiles] + ticket + done counter,
  // zero between launches (the kernel's last CTA resets them)
  uint32_t* fuse_sync = nullptr;
  int64_t fuse_sync_len = 0;
  // split-K tail workspace (plan-owned; sized from leaf_tiles): partial tiles
  // and per-tail-tile arrival counters (zero between launches)
  double* split_ws = nullptr;
  int64_t split_ws_elems = 0;
  int* split_cnt = nullptr;
  int64_t split_cnt_len = 0;
};
bool leaf_tma_supported(const LeafArgs& a);
// mf_tiny.cu: one cluster launch for a whole small level (n <= 64, R^L <= 64)
bool tiny_eligible(const Plan& pl);
cudaError_t launch_tiny(const Plan& pl, double alpha, const double* A, int64_t lda, const double* B,
                        int64_t ldb, double* C, int64_t ldc, cudaStream_t s);
// tile width and split-K tail chosen for a DMMA leaf launch (mf_leaf.cu)
struct LeafTiles {
  int bn = 128;
  int split = 1;         // k-range pieces per tail tile (1 = none)
  int64_t n_whole = 0;   // tiles computed whole (first blocks of the grid)
  int64_t n_tail = 0;    // tiles computed as `split` pieces each
  int64_t ws_elems = 0;  // doubles of partial-tile workspace needed
};
LeafTiles leaf_tiles(const LeafArgs& a);

// mf_fixed.cu: compile-time specialised K4/K6 for the catalog triples
int fixed_match(const Plan& pl);
bool fixed_vw4_ok(int64_t m, const void* a, int64_t lda, const void* b, int64_t ldb);
cudaError_t launch_premix_fixed(int id, int side, const double* X, int64_t ldx, int64_t m,
                                double* out, cudaStream_t s, Rows rows, const ProdMask& mask);
cudaError_t launch_postmix_fixed(int id, const double* Pw, int64_t m, double alpha, double* C,
                                 int64_t ldc, cudaStream_t s, Rows rows, const ProdMask& mask);
// mf_kron.cu: Kronecker-factored K4/K6 for deep powers (ids >= 8)
int kron_match(const Plan& pl);
cudaError_t launch_premix_kron(int id, int side, const double* X, int64_t ldx, int64_t m,
                               double* out, cudaStream_t s, Rows rows, const ProdMask& mask);
cudaError_t launch_postmix_kron(int id, const double* Pw, int64_t m, double alpha, double* C,
                                int64_t ldc, cudaStream_t s, Rows rows, const ProdMask& mask);
cudaError_t launch_leaf(const LeafArgs& a, int leaf_kind, cudaStream_t s);

}  // namespace mf
