/* mf.h -- C ABI of the B200-native Matrix Flow hot path (libmf.so).
 *
 * The method (arXiv 2312.12732, PAPER.md): C = alpha * A * B for square
 * n x n double-precision matrices, computed by
 * a bilinear factorization <U,V,W> -- the paper's a, b, c (PAPER.md
 * L196-220, Eq. "strassen"):
 *
 *     C_i = sum_q W[i][q] * P_q,   P_q = T_q * S_q,
 *     T_q = sum_k U[k][q] * A_k,   S_q = sum_l V[l][q] * B_l,
 *
 * over the p-way row-major block partition of A, B, C (PAPER.md L134-165,
 * L208-211), applied recursively `levels` times.  The
 * `levels` recursion is executed as ONE level of the Kronecker-flattened
 * triple U^(x)L, V^(x)L, W^(x)L, the bilinear map the
 * recursion computes.
 *
 * Conventions shared by every entry point:
 *  - Matrices are row-major fp64 with a leading dimension in ELEMENTS
 *    (ld >= n).  Device pointers unless a function says "host".
 *  - Coefficient arrays are HOST arrays of p*p x R doubles, row-major:
 *    U[k*R+q] = a_{k,q}, V[l*R+q] = b_{l,q}, W[i*R+q] = c_{i,q} with row i
 *    the C block in natural row-major order (PAPER.md prints c^t with rows
 *    C0, C2, C1, C3 -- L245-248; callers importing that layout must reorder).
 *  - Every function returns mf_status; no C++ exception crosses the ABI.
 *    On a non-OK status, mf_last_error() returns a thread-local message.
 *  - Work is stream-ordered and asynchronous on the given cudaStream_t
 *    (passed as void*, NULL = legacy default stream) unless stated.
 */
#ifndef MF_H
#define MF_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  MF_OK = 0,
  MF_ERR_INVALID_ARG = 1,   /* null/negative/overlapping/misaligned argument     */
  MF_ERR_INDIVISIBLE = 2,   /* n % p^levels != 0 (no padding: PAPER.md L487-488) */
  MF_ERR_BAD_TRIPLE = 3,    /* Brent equations violated or a dead product column */
  MF_ERR_OUT_OF_MEMORY = 4, /* device or host allocation failed                  */
  MF_ERR_CUDA = 5,          /* a CUDA runtime/driver call failed                 */
  MF_ERR_NCCL = 6,          /* an NCCL call failed                               */
  MF_ERR_UNSUPPORTED = 7    /* valid request outside what this build implements  */
} mf_status;

typedef struct mf_plan_st* mf_plan_t;

enum { MF_LEAF_DMMA = 0, MF_LEAF_SIMPLE = 1, MF_LEAF_CUBLAS = 2 };
enum { MF_IN_ROOT = 0, MF_IN_REPLICATED = 1 };
enum { MF_OUT_ROOT = 0, MF_OUT_ALL = 1, MF_OUT_ROWSLAB = 2 };

typedef struct {
  int32_t struct_size;  /* sizeof(mf_options); 0-initialised struct = defaults    */
  int32_t device;       /* CUDA device ordinal; -1 = current device (default)     */
  int32_t leaf;         /* MF_LEAF_DMMA (default): TMA + mma.sync f64 leaf GEMM;
                           MF_LEAF_SIMPLE: plain fp64 FMA leaf (test ablation);
                           MF_LEAF_CUBLAS: the R^L leaf products as
                           cublasDgemmBatched calls, one per operand-stride
                           group (ablation: same K4/K6, library leaf;
                           libcublas.so.12 is dlopen'ed, MF_ERR_CUDA if absent;
                           not with fuse_postadd)                              */
  int32_t shard_rank;   /* product sharding: this rank's index (default 0)        */
  int32_t shard_count;  /* number of shards; 0/1 = unsharded.  With comm == NULL
                           a sharded plan computes only its shard's PARTIAL C
                           (used to emulate rank r of N on one GPU).  With a
                           communicator, shard_rank / shard_count must equal its
                           rank / size (else MF_ERR_INVALID_ARG)              */
  void* comm;           /* communicator handle from mf_nccl_comm_create (NCCL,
                           one process per GPU) or mf_loop_comm_create (ranks
                           as threads of one process), or NULL = one rank     */
  int32_t input_mode;   /* MF_IN_REPLICATED (inputs valid on every rank) or
                           MF_IN_ROOT (only rank 0's A, B are read; the other
                           ranks may pass NULL and receive them by broadcasts
                           of row slabs, each slab's K4 starting as soon as it
                           landed; rank 0 sends in place from A and B when
                           lda == ldb == n, else from a packed copy)         */
  int32_t output_mode;  /* MF_OUT_ROOT (C summed onto rank 0), MF_OUT_ALL (C
                           summed onto every rank) or MF_OUT_ROWSLAB (rank r
                           receives rows [r*n/N, (r+1)*n/N) of the sum; its C
                           argument is that n/N x n slab, ldc == n; needs
                           n % N == 0; the full partial C lives in a
                           plan-owned buffer).  Only with comm; every mode
                           needs ldc == n                                     */
  int32_t profile;      /* 1: mf_dgemm records CUDA events around each phase on
                           the call's stream (read with mf_profile_read)          */
  int32_t host_only;    /* 1: plan the host logic only (Brent check, flattening,
                           classification, sharding) -- no device, no workspace;
                           mf_plan_info / mf_plan_products work, compute calls
                           return MF_ERR_INVALID_ARG                              */
  int32_t level_by_level; /* 0 (default): run `levels` as ONE level of the
                           Kronecker-flattened triple.  1: the paper's recursion
                            -- one level of <U,V,W> whose R leaf
                           products are each a (levels-1)-level product; same
                           bilinear map, more HBM passes (an ablation).  With 1,
                           mf_plan_info / mf_plan_products describe the top
                           level (R products, leaf_n = n / p)                    */
  int64_t max_workspace;  /* bytes; 0 (default) = unlimited.  If the T/S/P workspace
                           of all products would exceed it, products run in batches
                           that fit (the paper's OOM at n=24012,
                           P:L489-492): per batch K4 on its slots, K5, K6 adding
                           into C.  Unsharded flattened plans only              */
  int32_t fuse_postadd;   /* fold the post-additions into the leaf epilogue (SURVEY
                           §8a a4 / north_star (3): "optionally folded into the
                           leaf GEMM epilogue so each product is accumulated
                           straight into its C blocks"; no P workspace: saves
                           R^L (n/p^L)^2 doubles).  Needs levels >= 1,
                           flattened (not level_by_level), no batching, not
                           the cuBLAS leaf, else MF_ERR_UNSUPPORTED.
                           1 = ordered fold (SURVEY §8f NEXT-1 "deterministic
                           product-serial ordering"): the leaf tiles at one
                           position run in ascending q (a per-tile flag, tiles
                           scheduled in ticket order); each stores
                           W'[i][q]*P_q into C block i if q is the block's
                           first product, else adds it to C_i, and applies
                           alpha at the block's last product -- K6's
                           per-element order, so C is bitwise the unfused
                           result.  Unsharded plans only (MF_ERR_UNSUPPORTED
                           otherwise).
                           2 = bulk reductions: C is zeroed, then every leaf
                           tile adds alpha*W'[i][q]*P_q into its C blocks with
                           cp.reduce.async.bulk .add.f64; summation order
                           across products not fixed (not bitwise
                           reproducible; exact on integer data within 2^53).
                           Odd ldc or C not 16-byte aligned run the simple
                           leaf (f64 atomics for 2, one launch per product in
                           order for 1)                                      */
  int32_t graph;          /* 1: mf_dgemm replays a CUDA graph of its launches.  The
                           first call with a given (A, lda, B, ldb, C, ldc,
                           alpha) runs eagerly; the second captures the step
                           on the call's stream and instantiates it; later
                           calls with the same arguments launch the graph (one
                           host call instead of four launches: the n <= 4096
                           configs are host-issue bound).  Ignored on the
                           legacy default stream (NULL) and with profile,
                           comm, level_by_level or MF_LEAF_CUBLAS           */
  int32_t comm_regions;   /* sharded plans with comm: the leaf and post-addition
                           run in this many 128-aligned row regions, and each
                           region's rows of C are summed on the exchange stream
                           while the next region computes (SURVEY §8f NEXT-4:
                           "reduce C block-groups as products complete") --
                           reduce (MF_OUT_ROOT), all-reduce (MF_OUT_ALL) or a
                           reduce onto each owning rank (MF_OUT_ROWSLAB, a
                           region-wise reduce-scatter).  Also the number of
                           MF_IN_ROOT input slabs.  0 = default (8 when
                           shard_count > 1, else 1); 1 = one collective after
                           K6.  Without comm an explicit value > 1 still runs
                           the regions (the shard's partial C; for tests)    */
  int32_t recurse_levels; /* with level_by_level = 1: how many top levels run one
                           at a time (0 = levels - 1, the paper's full
                           recursion); the remaining levels run as ONE
                           flattened child plan, e.g. levels = 4,
                           recurse_levels = 1: one level of R products, each a
                           flattened 3-level product (R^3 leaves in one launch) */
} mf_options;

/* mf_plan -- validate and prepare <U,V,W> applied `levels` times at size n.
 * Host-side and untimed:
 *  1. checks p >= 1, R >= 1, levels >= 0, n >= 1 (MF_ERR_INVALID_ARG);
 *  2. checks the Brent equations exactly over all (p^2)^3 index triples
 *      and that no U/V column is zero (MF_ERR_BAD_TRIPLE;
 *     coefficients must be integers or dyadic rationals, else
 *     MF_ERR_UNSUPPORTED);
 *  3. checks n % p^levels == 0 (MF_ERR_INDIVISIBLE, message names n, p, L);
 *  4. Kronecker-flattens the triple `levels` times (SPEC.md L244 interleave,
 *     product index q = q_outer * R + q_inner);
 *  5. classifies operand columns: a column with a single +-1 entry aliases its
 *     A/B block (sign folded into W), others are materialised by the
 *     pre-addition kernel;
 *  6. allocates the device workspace (T, S, P blocks) and TMA descriptors.
 * levels == 0 plans a classical C = alpha*A*B on the leaf kernel (U,V,W may
 * then be NULL).  The plan owns its workspace; the caller owns A, B, C.
 * A plan is bound to one device.  *out is NULL on failure. */
mf_status mf_plan(mf_plan_t* out, int32_t p, int32_t R, const double* U, const double* V,
                  const double* W, int32_t levels, int64_t n, const mf_options* opt);

/* mf_dgemm -- C <- alpha * A * B through the planned algorithm: the problem
 * statement C = alpha A B (§3) computed as Eq. "strassen"
 * (L196-203): T_q, S_q pre-additions, the R^L products P_q, the
 * post-additions C_i (order of terms: DESIGN.md R7/R8).
 * A (n x n, lda), B (n x n, ldb): device, read-only.  C (n x n, ldc): device,
 * write-only (BLAS beta = 0: prior contents, even NaN, are ignored); C must
 * not overlap A or B (MF_ERR_INVALID_ARG).  Launches, in stream order:
 * pre-add A (K4), pre-add B (K4), the batched leaf DGEMM (K5), post-add
 * (K6) -- no host synchronisation.  Calls on one plan must be serialised by
 * the caller (they share the workspace).  Inputs must be finite: the fast
 * algorithm turns Inf-Inf into NaN where the classical product gives +-Inf.
 * With a sharded plan (shard_count > 1) and no NCCL communicator, C receives
 * this shard's PARTIAL sum (the W-combination over the shard's products). */
mf_status mf_dgemm(mf_plan_t plan, double alpha, const double* A, int64_t lda,
                   const double* B, int64_t ldb, double* C, int64_t ldc, void* stream);

/* mf_dgemm_host -- the same product with HOST A, B, C
 * (the end-to-end call; the paper's timings exclude transfers, L472-475; any host memory;
 * pinned memory is fastest).  Copies A and B to plan-owned device buffers,
 * runs mf_dgemm, copies C back; returns after C is complete on the host.
 * Single-GPU flattened plans pipeline the copies with the compute by row /
 * column slabs.  Sharded plans with a communicator and MF_IN_REPLICATED
 * inputs copy only their 1/N row slab of A and B and all-gather the rest over
 * NVLink (every rank must pass the full host A, B); with MF_IN_ROOT only rank
 * 0 reads (and must pass) host A and B, and the other ranks (A, B may be NULL)
 * receive them by the slab broadcasts of mf_dgemm; with MF_OUT_ROOT only rank
 * 0 copies C back, with MF_OUT_ROWSLAB each rank its slab. */
mf_status mf_dgemm_host(mf_plan_t plan, double alpha, const double* A, int64_t lda,
                        const double* B, int64_t ldb, double* C, int64_t ldc, void* stream);

/* mf_dgemm_host_async -- mf_dgemm_host without the final wait, for a stream of
 * products: consecutive calls alternate between two plan-owned device copies
 * of A, B, C, so call k+1's host->device copies run while call k computes and
 * call k's device->host copies run while call k+1 computes (the leaf/K6
 * workspace is shared, so computations stay in call order).  Results are
 * bitwise those of mf_dgemm_host.  A and B must stay unchanged and C unread
 * until mf_host_sync (or a synchronisation of `stream`, which waits for the
 * call's last copy) returns; pinned host memory is needed for the overlap.
 * Plans without the slab pipeline (sharded, NCCL, level-by-level, batched,
 * fused, non-DMMA leaf) stream whole matrices the same way (copy in, compute,
 * copy out on three streams); the fused plan's results equal the synchronous
 * call's to rounding (its bulk reductions add in a run-dependent order).  A
 * later synchronous call on the plan first waits for all enqueued async calls. */
mf_status mf_dgemm_host_async(mf_plan_t plan, double alpha, const double* A, int64_t lda,
                              const double* B, int64_t ldb, double* C, int64_t ldc, void* stream);

/* mf_host_sync -- wait until every mf_dgemm_host_async call enqueued on the
 * plan has finished (its C is on the host). */
mf_status mf_host_sync(mf_plan_t plan);

/* mf_destroy -- wait for the plan's outstanding work, free its workspace
 * (the T, S, P temporaries of PAPER.md L287-292), tables and streams.
 * NULL: no-op.  Always MF_OK. */
mf_status mf_destroy(mf_plan_t plan);

/* Thread-local message for the last non-OK status of this thread ("" if none);
 * failures are reported, not thrown (the CPU program's
 * convention, kept at the boundary).  The pointer stays valid until this
 * thread's next libmf call. */
const char* mf_last_error(void);

/* Plan facts: workspace bytes (the temporaries of PAPER.md L287-292), leaf
 * side m = n / p^levels, number of leaf products R^levels (the count law of
 * SPEC.md L395), materialised T / S counts (columns of U / V that are not a
 * single +-1 block, Eq. "strassen" L199-202).  Any pointer may be NULL.
 * (SURVEY §8(b) names three outputs; n_mat_a / n_mat_b are added.) */
mf_status mf_plan_info(mf_plan_t plan, size_t* workspace_bytes, int64_t* leaf_n,
                       int64_t* n_products, int32_t* n_mat_a, int32_t* n_mat_b);

/* Per-product routing of the flattened triple (Kronecker interleave of
 * PAPER.md L303-313 / SPEC.md L244), arrays of length n_products
 * (host, caller-allocated, any may be NULL): a_src[q] = 0 if P_q's left
 * operand aliases block a_idx[q] of A, 1 if it is materialised slot a_idx[q]
 * of the T workspace; b_src/b_idx likewise for B and S; sign[q] = +-1, the
 * sign folded out of aliased operands (P_q as produced by the leaf stage is
 * sign[q] times the P_q of Eq. "strassen"); shard[q] = the shard that computes
 * product q whole, or -1 for a product split by rows across all shards. */
mf_status mf_plan_products(mf_plan_t plan, int32_t* a_src, int32_t* a_idx, int32_t* b_src,
                           int32_t* b_idx, int32_t* sign, int32_t* shard);

/* Provenance of the plan's pre/post-addition kernels (K4/K6), for tests that
 * must know which implementation ran: *jit_tables = coefficient tables for
 * which mf_plan asked NVRTC for a generated kernel, *jit_built = how many it
 * built and loaded (fewer: NVRTC / driver API missing, or compilation failed;
 * those tables run the table-driven kernels); launches[4] = K4/K6 launches
 * since the plan was made by kind: [0] table-driven (mf_mix.cu), [1]
 * compiled-in specialised (mf_fixed.cu), [2] Kronecker-factored (mf_kron.cu),
 * [3] generated at plan time.  A level-by-level plan sums its child plans.
 * Any pointer may be NULL. */
mf_status mf_plan_kernels(mf_plan_t plan, int32_t* jit_tables, int32_t* jit_built,
                          int64_t* launches /* 4 */);

/* The exchange schedule of one mf_dgemm call of a sharded plan (SURVEY §8e, row
 * a6): the collectives this rank issues, in issue order, as mf_dgemm would with
 * a communicator (host-only plans included, so CPU tests can replay them with
 * another transport).  Op i: kind[i] = MF_X_BCAST / MF_X_REDUCE /
 * MF_X_ALLREDUCE / MF_X_REDUCE_SCATTER; buf / recv_buf = MF_XB_A, MF_XB_B
 * (the n x n inputs, ld n), MF_XB_C (the partial C, n x n, ld n) or MF_XB_COUT
 * (this rank's n/N x n output slab, MF_OUT_ROWSLAB); off / recv_off / count in
 * doubles (count per rank for a reduce-scatter); root rank; ops of one group
 * are issued as one NCCL group; phase 0 = the MF_IN_ROOT input broadcasts (B's
 * row slabs, then A's), phase 1 + k = the reduction of row region k (or of the
 * whole partial C, phase 1).  *n_ops = number of ops (arrays: cap entries,
 * any may be NULL); 0 for unsharded plans. */
enum { MF_X_BCAST = 0, MF_X_REDUCE = 1, MF_X_ALLREDUCE = 2, MF_X_REDUCE_SCATTER = 3 };
enum { MF_XB_A = 0, MF_XB_B = 1, MF_XB_C = 2, MF_XB_COUT = 3 };
mf_status mf_plan_exchange(mf_plan_t plan, int32_t* kind, int32_t* buf, int64_t* off, int64_t* count,
                           int32_t* root, int32_t* recv_buf, int64_t* recv_off, int32_t* group,
                           int32_t* phase, int64_t cap, int64_t* n_ops);

/* Product sharding: with shard_count = N, rank r computes
 * floor(R^L / N) whole products (a contiguous range) and, of each of the
 * R^L mod N leftover products (shard[q] = -1), the 128-aligned output row slab
 * [*r0, *r1) -- exact balance.  Leftovers go whole to ranks when m has fewer
 * than N tile rows (or for level-by-level plans); then *r0 = *r1 = 0. */
mf_status mf_plan_shard_rows(mf_plan_t plan, int64_t* r0, int64_t* r1);

/* Component entry points (the steps of mf_dgemm, exposed for step-by-step
 * parity tests against the oracle; stream-ordered, device pointers):
 *  mf_premix:  side 0: T slots from A, side 1: S slots from B.  out holds
 *              n_mat_{a,b} x m x m doubles; slot s = the s-th materialised
 *              column in ascending q (K4).
 *  mf_leaf:    P_q' = T_q * S_q for this plan's products (K5); A, B are the
 *              operands that alias, T, S the materialised slots (as mf_premix
 *              writes them), P holds n_products x m x m doubles.
 *  mf_postmix: C_i = alpha * sum_q (W[i][q]*sign[q]) * P_q' (K6), P as mf_leaf
 *              writes it. */
mf_status mf_premix(mf_plan_t plan, int32_t side, const double* X, int64_t ldx, double* out,
                    void* stream);
mf_status mf_leaf(mf_plan_t plan, const double* A, int64_t lda, const double* B, int64_t ldb,
                  const double* T, const double* S, double* P, void* stream);
mf_status mf_postmix(mf_plan_t plan, double alpha, const double* P, double* C, int64_t ldc,
                     void* stream);

/* Phase timing of a profile-enabled plan (mf_options.profile = 1): waits for
 * the recorded events and writes the summed device time in milliseconds of
 * each phase over the mf_dgemm calls since the last reset:
 *   ms[0] pre-add A (K4), ms[1] pre-add B (K4), ms[2] leaf products (K5),
 *   ms[3] post-add (K6), ms[4] NCCL exchange (0 on one GPU).
 * *calls = number of mf_dgemm calls summed; reset != 0 clears the sums. */
mf_status mf_profile_read(mf_plan_t plan, double* ms /* 5 */, int32_t* calls, int32_t reset);

/* Communicators of the product-sharded path.  The
 * paper's recursion makes the R^L leaf products independent ("each product can
 * be done recursively", Eq. "strassen" L196-202) and the
 * post-addition C_i = sum_q W[i][q] P_q is linear, so rank r computes the
 * products of shard r and the partial C sums of all ranks add up to C.  Each
 * rank passes its handle in mf_options.comm with shard_rank = rank and
 * shard_count = nranks; every rank then calls mf_dgemm (or mf_dgemm_host)
 * collectively with the same arguments, and the library broadcasts the inputs
 * (MF_IN_ROOT) and sums the partial C (mf_options.output_mode).
 *
 * NCCL (one process per GPU, NVLink / NVSwitch): the 128-byte unique id of
 * mf_nccl_unique_id is exchanged by the caller (e.g. torch.distributed); the
 * returned handle owns the ncclComm_t.  libnccl.so.2 is loaded at run time
 * (MF_ERR_NCCL if absent).
 *
 * Loopback (mf_loop_comm_create): nranks handles for ranks that are THREADS of
 * one process (on one device, or on devices with peer access).  Every
 * collective is a host rendezvous of the threads followed by stream-ordered
 * copies and a summation kernel (ascending rank order) that each receiving
 * rank enqueues on its own stream behind the senders' events; no kernel waits
 * on another rank's kernel.  It runs the multi-rank schedule where fewer GPUs
 * than ranks exist (tests).  A rank that stops calling collectives makes its
 * peers fail with MF_ERR_NCCL after 120 s.  nranks <= 16.
 *
 * mf_comm_destroy frees either kind (NULL: no-op); mf_nccl_comm_destroy is the
 * same call.  Destroy a handle only after the plans using it. */
enum { MF_COMM_NCCL = 0, MF_COMM_LOOPBACK = 1 };
mf_status mf_nccl_unique_id(void* id_out /* 128 bytes */);
mf_status mf_nccl_comm_create(void** comm_out, const void* id, int32_t rank, int32_t nranks);
mf_status mf_loop_comm_create(int32_t nranks, void** comms_out /* nranks handles */);
mf_status mf_comm_info(void* comm, int32_t* rank, int32_t* nranks, int32_t* kind);
mf_status mf_comm_destroy(void* comm);
mf_status mf_nccl_comm_destroy(void* comm);

/* Diagnostic: generate the fused-addition kernel mf_plan would build at run
 * time (NVRTC) for one coefficient table -- coef is nout x nin row-major
 * (coef[o*nin + k] = coefficient of input k in output o, 0 = absent; Eq.
 * "strassen") -- with inputs / outputs addressed as the
 * blocks of a P x P partition (in_P / out_P > 0) or as [slots][m][m] (0), and
 * compile it for `arch` (e.g. "sm_100a").  Needs no GPU.  *vw_out = positions
 * per thread chosen (0 = table too large for a generated kernel);
 * *cubin_bytes = size of the compiled code.  MF_ERR_UNSUPPORTED when NVRTC is
 * missing, the table does not fit, or compilation fails (message in
 * mf_last_error). */
mf_status mf_jit_compile_check(const double* coef, int32_t nout, int32_t nin, int32_t in_P,
                               int32_t out_P, const char* arch, int32_t* vw_out,
                               int64_t* cubin_bytes);

/* Kronecker composition of two triples ("4 as 2x2 and 49";
 * chains such as <6,6,6;161> = SW (x) Laderman, L275-293), for C callers that
 * plan a mixed chain: U, V, W (host, caller-allocated, (po*pi)^2 x (Ro*Ri)
 * doubles each) receive outer (x) inner with the row interleave of SPEC.md
 * L244 -- outer block b, inner block s -> row ((b/po)*pi + s/pi)*(po*pi) +
 * (b%po)*pi + s%pi -- and product q = q_outer*Ri + q_inner.  Plan the result
 * with levels = 1 (mf_plan runs the exact Brent check on it).  Host only. */
mf_status mf_triple_kron(int32_t po, int32_t Ro, const double* Uo, const double* Vo,
                         const double* Wo, int32_t pi, int32_t Ri, const double* Ui,
                         const double* Vi, const double* Wi, double* U, double* V, double* W);

/* Deviations from SURVEY.md §8(b)'s sketch of this ABI, and why:
 *  - mf_options has no `flatten` field; flattening is the default and
 *    `level_by_level = 1` selects the paper's recursion -- the
 *    inverse flag, so a zero-initialised struct gives the fast path.
 *  - mf_plan_info has two extra outputs (n_mat_a, n_mat_b).
 *  - `levels` repeats ONE triple; a mixed chain (SW (x) LD) is planned by
 *    composing it with mf_triple_kron and planning levels = 1.
 *  - added entry points: mf_dgemm_host / _async / mf_host_sync (host
 *    buffers), mf_plan_products / mf_plan_shard_rows / mf_plan_kernels
 *    / mf_plan_exchange (introspection for tests), mf_premix / mf_leaf / mf_postmix (step-by-step
 *    parity), mf_profile_read (phase timing), mf_loop_comm_create /
 *    mf_comm_info / mf_comm_destroy (communicators), mf_jit_compile_check
 *    (generator check without a GPU), mf_version. */

/* Library version, e.g. "mf 0.1.0 sm_100a". */
const char* mf_version(void);

#ifdef __cplusplus
}
#endif
#endif /* MF_H */
