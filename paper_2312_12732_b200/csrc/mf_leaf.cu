// mf_leaf.cu -- K5: the batched leaf products P_q' = X_q * Y_q of Eq.
// "strassen" ("There are seven products, each product can
// be done recursively"), here all R^L products of the flattened triple in ONE
// launch, fp64 on the B200 FP64 tensor path.
//
// B200 design:
//  * FP64 tensor math on sm_100a is the legacy warp-level mma.sync.m8n8k4.f64
//    (SASS DMMA.8x8x4); tcgen05 has no f64 kind.  Measured: 37.1 TF/s with
//    register-resident operands (tools/peaks_fp64.cu) = 64 FMA/clk/SM.
//  * Operands are staged into shared memory by TMA (cp.async.bulk.tensor)
//    with an mbarrier ring of STAGES slots.  8 MMA warps (2 per SM
//    sub-partition, so each may hold 255 registers); lane 0 of warp 0 issues
//    the TMA for slot kb+STAGES-1 once all warps released it (empty barrier).
//  * Operand views: an aliased operand is block (br, bc) of the caller's A/B,
//    addressed through a 4-D tensor map {col, block-col, row, block-row} so
//    TMA zero-fills past the block edge (ragged leaves never read a
//    neighbouring block); a materialised operand is a slot of the T/S
//    workspace (3-D map {col, row, slot}).
//  * CTA tile 128 x BNT (BNT = 128, or 64 for badly filled last waves), k 32
//    per ring stage (KSUB = 2 sub-blocks of 16; 3 stages in 192 KB), or k 48
//    (KSUB = 3, 2 stages) where m is a multiple of 48 or >= 8192.  A last
//    stage past the block edge multiplies only its sub-blocks that hold data;
//    that per-group guard also splits the DMMA stream into blocks ptxas
//    schedules without the DEPBAR scoreboard waits it used to insert (leaf
//    185.65 -> 183.92 ms at n=16384 SW^2, profiles/leaf_ksub_r01.json).  Each
//    MMA warp owns 64 x BNT/4 of C: 64 fp64 accumulators per thread at
//    BNT = 128.  Fragments are fetched with 128-bit LDS, which shared memory
//    serves per quarter-warp (8 lanes).
//      A is TMA-written with SWIZZLE_128B in rows of 16 doubles ([128 m][16 k]
//      per sub-block; physical 16-byte chunk = logical chunk ^ (row & 7)); lane
//      (r=L/4, kk=L%4) loads the k-pair chunk c(kk,g) of row r.  The
//      k-permutation k = 2c(kk,g) + s with c(.,0) = {0,3,5,6}, c(.,1) =
//      {1,2,4,7} takes one chunk of every pair {2j,2j+1}: conflict-free.
//      B is one unswizzled [32 k][BNT n] box per stage; lane (kk, nn=L/4)
//      loads B[2c(kk,g)+s][2nn..2nn+1] (4-way conflicted; the swizzled
//      alternatives measured slower, see below).  The n-permutation n = 2c + j
//      gives each thread 4 CONSECUTIVE output columns (one 256-bit store).
//  * Grid = products x tiles, 1 CTA/SM (256 threads, 192 KB ring); tiles of a
//    product are rasterised in groups of 8 tile-rows for L2 reuse.
//  * Split-K tail: when the tiles fill the SMs in few waves, the last
//    (partial) waves' tiles are cut into S k-ranges; each piece stores its
//    partial accumulators and the last piece to finish sums the S partials in
//    split order (deterministic) and runs the normal epilogue.
#include <cuda.h>

#include <atomic>
#include <cmath>
#include <cstdlib>
#include <mutex>

#include "mf_internal.h"

namespace mf {
namespace {

#ifdef MF_LEAF_TRACE
// Diagnostic build only (-DMF_LEAF_TRACE): per-CTA timestamps (globaltimer, ns)
// at entry, first data ready, end of the k loop and end of the epilogue, plus
// the SM id -- where a tile's time goes outside the DMMA stream.
constexpr int kTraceMax = 1 << 16;
__device__ unsigned long long g_leaf_trace[kTraceMax][5];
__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#define TRACE(i) \
  if (threadIdx.x == 0 && blockIdx.x < kTraceMax) g_leaf_trace[blockIdx.x][i] = gtime()
#else
#define TRACE(i)
#endif

constexpr int BM = 128, BN = 128, BK = 16;  // BN: the default (widest) tile; BK: one k sub-block
constexpr int MMA_WARPS = 8;   // one CTA per SM (the default shape)
constexpr int THREADS = MMA_WARPS * 32;
constexpr int A_SUB_BYTES = BM * BK * 8;  // one [128 m][16 k] swizzled A sub-tile
// A stage holds KSUB k sub-blocks (16 k each): A as KSUB swizzled sub-tiles,
// B as one [16*KSUB k][BNT n] box.  Deeper stages (KSUB = 2) halve the
// mbarrier waits per flop; the ring depth keeps ~190 KB of smem in flight per
// SM: one CTA of NW = 8 MMA warps with a 192 KB ring, or (NW = 4, 128 x 64
// tiles) two co-resident CTAs with 96 KB rings each.
template <int BNT, int KSUB> __host__ __device__ constexpr int a_bytes() { return KSUB * A_SUB_BYTES; }
template <int BNT, int KSUB> __host__ __device__ constexpr int stage_bytes() {
  return KSUB * A_SUB_BYTES + KSUB * BK * BNT * 8;
}
template <int BNT, int KSUB, int NW = 8> __host__ __device__ constexpr int n_stages() {
  return ((NW == 8 ? 192 : 96) * 1024) / stage_bytes<BNT, KSUB>() < 5
             ? ((NW == 8 ? 192 : 96) * 1024) / stage_bytes<BNT, KSUB>() : 5;
}
template <int BNT, int KSUB, int NW = 8> __host__ __device__ constexpr int smem_bytes() {
  return n_stages<BNT, KSUB, NW>() * stage_bytes<BNT, KSUB>() + 2 * n_stages<BNT, KSUB, NW>() * 8 + 1024;
}
constexpr int GROUP_M = 8;

// B staging: one unswizzled TMA box [16*KSUB k][BNT n] per stage.  Its LDS.128
// are 4-way bank conflicted; the conflict-free swizzled alternatives (8 boxes
// of [16 k][16 n], or one 5-D box with that layout) measured slower or equal
// (profiles/leaf_bmode_r01.json: TMA issues per stage, not smem banks, limit).

struct LeafParams {
  int64_t m;
  int group_m;  // tile-rows per rasterisation group
  int tm0, tn0;  // first tile row / column (region of the host-buffer pipeline)
  int tiles_m, tiles_n, kblocks;  // kblocks: stages of 16*KSUB k
  double* out;
  int64_t ldo, out_stride;
  double alpha;
  const LeafJob* jobs;
  const int32_t* post_off;  // fused post-addition (FUSE > 0): out = C, ldo = ldc
  const PostTerm* post;
  // ordered fold (FUSE == 2): flags[P*P][tiles_m * tiles_n] (per C block and
  // tile position: how many of the block's products have updated it), then
  // the ticket and done counters
  uint32_t* sync;
  int nP;
  // split-K tail: blocks >= n_whole are pieces (tile n_whole + (b - n_whole) / split,
  // k-range (b - n_whole) % split); partials in part_ws, arrivals in part_cnt
  int n_whole, split;
  double* part_ws;
  int* part_cnt;
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(bar), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  uint32_t done = 0;
  do {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done) : "r"(bar), "r"(parity) : "memory");
  } while (!done);
}

__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" :: "r"(bar) : "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(bar), "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void tma_load_3d(uint32_t dst, const CUtensorMap* map, uint32_t bar,
                                            int c0, int c1, int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4}], [%5];"
      :: "r"(dst), "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(bar)
      : "memory");
}

__device__ __forceinline__ void tma_load_4d(uint32_t dst, const CUtensorMap* map, uint32_t bar,
                                            int c0, int c1, int c2, int c3) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4, %5}], [%6];"
      :: "r"(dst), "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(c3),
         "r"(bar)
      : "memory");
}

__device__ __forceinline__ void lds128(uint32_t addr, double& x, double& y) {
  asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(x), "=d"(y) : "r"(addr));
}

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
      : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
}

__device__ __forceinline__ uint32_t ld_acquire(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void st_release(uint32_t* p, uint32_t v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" :: "l"(p), "r"(v) : "memory");
}

// Loads of C in the ordered fold: plain (weak) global loads after the flag's
// ld.acquire and a barrier -- the pattern the PTX memory model orders (the
// acquire is followed by CCTL.IVALL: no stale L1 line survives).  "memory":
// must not move above the barrier that follows the wait.  (Wrong tiles once
// blamed on these loads were the k loop's ring-release race; see the fence
// before mbar_arrive.)
__device__ __forceinline__ void ld_v2(const double* p, double& x, double& y) {
  asm volatile("ld.global.v2.f64 {%0, %1}, [%2];" : "=d"(x), "=d"(y) : "l"(p) : "memory");
}

__device__ __forceinline__ double ld_f64(const double* p) {
  double x;
  asm volatile("ld.global.f64 %0, [%1];" : "=d"(x) : "l"(p) : "memory");
  return x;
}

// BNT = CTA tile width (128, or 64 to cut wave quantisation on small batches):
// warps form a 2 x 4 grid of 64 x (BNT/4) warp tiles, NJ = BNT/64 16-column
// groups per warp.  FUSE: 0 = store P_q' (then K6), 1 = fused post-addition by
// bulk f64 reductions into C (order not fixed), 2 = ordered fold: the products
// of one tile position update C in job order (ascending q), store / add /
// alpha-last exactly as K6, so C is bitwise the unfused result.
// NW = MMA warps per CTA: 8 (2 x 4 warp grid, one CTA per SM) or 4 (2 x 2
// warp grid of 64 x 32 warp tiles at BNT = 64, two CTAs per SM: one CTA's
// prologue / epilogue runs beside the other's k loop).
template <int BNT, int KSUB, int FUSE, int NW = 8>
__global__ void __launch_bounds__(NW * 32, NW == 8 ? 1 : 2)
leaf_dmma_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmT,
                 const __grid_constant__ CUtensorMap tmB, const __grid_constant__ CUtensorMap tmS,
                 const LeafParams prm) {
  constexpr int MMA_WARPS = NW, THREADS = NW * 32, WARPS_N = NW / 2;
  constexpr int WN = BNT / WARPS_N, NJ = WN / 16;
  static_assert(NJ >= 1 && WN % 16 == 0, "warp tile width");
  constexpr int STAGES = n_stages<BNT, KSUB, NW>();
  constexpr int STAGE_BYTES = stage_bytes<BNT, KSUB>();
  constexpr int A_BYTES = a_bytes<BNT, KSUB>();
  constexpr int KS = BK * KSUB;  // k per stage
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  const uint32_t s_base = smem_u32(smem);
  const uint32_t full0 = s_base + STAGES * STAGE_BYTES;
  const uint32_t empty0 = full0 + STAGES * 8;

  // ---- block -> tile (whole, or one k-range piece of a tail tile) ----
  // ordered fold: tiles in ticket order, so the CTA a tile waits for (same
  // position, previous product) has started -- forward progress by induction
  int block = blockIdx.x;
  if constexpr (FUSE == 2) {
    __shared__ int s_ticket;
    if (threadIdx.x == 0)
      s_ticket = (int)atomicAdd(prm.sync + prm.nP * prm.nP * prm.tiles_m * prm.tiles_n, 1u);
    __syncthreads();
    block = s_ticket;
  }
  const bool piece = !FUSE && prm.split > 1 && block >= prm.n_whole;
  int tile = block, split_idx = 0, kb0 = 0, nk = prm.kblocks;
  if (piece) {
    const int pc = block - prm.n_whole;
    tile = prm.n_whole + pc / prm.split;
    split_idx = pc % prm.split;
    kb0 = split_idx * prm.kblocks / prm.split;
    nk = (split_idx + 1) * prm.kblocks / prm.split - kb0;
  }
  // ---- tile -> (product job, tm, tn), grouped rasterisation ----
  const int tiles_per_job = prm.tiles_m * prm.tiles_n;
  const int job_id = tile / tiles_per_job;
  const int t = tile - job_id * tiles_per_job;
  const int group_tiles = prm.group_m * prm.tiles_n;
  const int first_m = (t / group_tiles) * prm.group_m;
  const int gsz = min(prm.tiles_m - first_m, prm.group_m);
  const int tm = prm.tm0 + first_m + (t % group_tiles) % gsz;
  const int tn = prm.tn0 + (t % group_tiles) / gsz;
  const LeafJob job = prm.jobs[job_id];
  TRACE(0);
#ifdef MF_LEAF_TRACE
  if (threadIdx.x == 0 && blockIdx.x < kTraceMax) {
    unsigned smid;
    asm volatile("mov.u32 %0, %smid;" : "=r"(smid));
    g_leaf_trace[blockIdx.x][4] = smid;
  }
#endif

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(full0 + 8 * s, 1);
      mbar_init(empty0 + 8 * s, MMA_WARPS);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  // ---- TMA producer: warp 0 refills the slot freed one iteration earlier ----
  const bool a_ws = job.flags & 1, b_ws = job.flags & 2;
  const CUtensorMap* mapA = a_ws ? &tmT : &tmA;
  const CUtensorMap* mapB = b_ws ? &tmS : &tmB;
  const int a_br = job.a_coord >> 16, a_bc = job.a_coord & 0xffff;
  const int b_br = job.b_coord >> 16, b_bc = job.b_coord & 0xffff;
  auto issue = [&](int i) {  // i: stage of this block's k-range; k block kb0 + i
    const int s = i % STAGES, kb = kb0 + i;
    const uint32_t fb = full0 + 8 * s;
    mbar_expect_tx(fb, STAGE_BYTES);
    const uint32_t dA = s_base + s * STAGE_BYTES, dB = dA + A_BYTES;
#pragma unroll
    for (int j = 0; j < KSUB; ++j) {
      if (a_ws) tma_load_3d(dA + j * A_SUB_BYTES, mapA, fb, kb * KS + j * BK, tm * BM, job.a_coord);
      else      tma_load_4d(dA + j * A_SUB_BYTES, mapA, fb, kb * KS + j * BK, a_bc, tm * BM, a_br);
    }
    if (b_ws) tma_load_3d(dB, mapB, fb, tn * BNT, kb * KS, job.b_coord);
    else      tma_load_4d(dB, mapB, fb, tn * BNT, b_bc, kb * KS, b_br);
  };
  if (threadIdx.x == 0) {
    asm volatile("prefetch.tensormap [%0];" :: "l"(reinterpret_cast<uint64_t>(mapA)) : "memory");
    asm volatile("prefetch.tensormap [%0];" :: "l"(reinterpret_cast<uint64_t>(mapB)) : "memory");
    for (int i = 0; i < STAGES - 1 && i < nk; ++i) issue(i);
  }

  // ================= MMA warps =================
  const int wm = warp / WARPS_N;  // 0..1 -> 64-row half
  const int wn = warp % WARPS_N;  // WN-column slice
  const int lr = lane >> 2, lk = lane & 3;

  double acc[8][NJ][2][2];
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < NJ; ++j)
#pragma unroll
      for (int u = 0; u < 2; ++u) { acc[i][j][u][0] = 0.0; acc[i][j][u][1] = 0.0; }

  // per-lane shared-memory offsets (bytes) inside a stage; see the header
  // for the k-permutation c(kk, g) that makes every LDS.128 conflict-free.
  const uint32_t c0 = (0x6530u >> (4 * lk)) & 0xf;  // c(kk, 0) in {0,3,5,6}
  const uint32_t c1 = (0x7421u >> (4 * lk)) & 0xf;  // c(kk, 1) in {1,2,4,7}
  uint32_t offA[2], offB[2][2];
  offA[0] = (wm * 64 + lr) * 128 + ((c0 ^ lr) << 4);
  offA[1] = (wm * 64 + lr) * 128 + ((c1 ^ lr) << 4);
#pragma unroll
  for (int s2 = 0; s2 < 2; ++s2) {
    const uint32_t r0 = 2 * c0 + s2, r1 = 2 * c1 + s2;  // B rows (k) for g = 0, 1
    offB[0][s2] = r0 * (BNT * 8) + (wn * WN + 2 * lr) * 8;
    offB[1][s2] = r1 * (BNT * 8) + (wn * WN + 2 * lr) * 8;
  }

  // Fragment double buffering: group g+1's LDS are issued before group g's 64
  // DMMAs, so no k-group starts on an LDS-latency bubble.  A stage's slot is
  // released (mbarrier.arrive has release semantics: the LDS reads are
  // complete) as soon as its last fragment load has been issued.  Group g of
  // a stage = k sub-block g/2, half g%2 (8 k each).
  double fa0[8][2], fb0[NJ][2][2], fa1[8][2], fb1[NJ][2][2];
  auto load_frags = [&](uint32_t sA, uint32_t sB, int g, double (&fa)[8][2], double (&fb)[NJ][2][2]) {
    const uint32_t a = sA + (g >> 1) * A_SUB_BYTES + offA[g & 1];
    const uint32_t b = sB + (g >> 1) * (BK * BNT * 8) + 0;
#pragma unroll
    for (int mi = 0; mi < 8; ++mi) lds128(a + mi * 8 * 128, fa[mi][0], fa[mi][1]);
#pragma unroll
    for (int nj = 0; nj < NJ; ++nj)
#pragma unroll
      for (int s2 = 0; s2 < 2; ++s2)
        lds128(b + offB[g & 1][s2] + nj * 16 * 8, fb[nj][s2][0], fb[nj][s2][1]);
  };
  auto mma_group = [&](const double (&fa)[8][2], const double (&fb)[NJ][2][2]) {
#pragma unroll
    for (int s2 = 0; s2 < 2; ++s2)
#pragma unroll
      for (int mi = 0; mi < 8; ++mi)
#pragma unroll
        for (int nj = 0; nj < NJ; ++nj)
#pragma unroll
          for (int j = 0; j < 2; ++j)
            dmma(acc[mi][nj][j][0], acc[mi][nj][j][1], fa[mi][s2], fb[nj][s2][j]);
  };

  if (nk > 0) {
    mbar_wait(full0, 0);
    TRACE(1);
    load_frags(s_base, s_base + A_BYTES, 0, fa0, fb0);
  }
  // fragment groups of the last stage that hold data: when m is not a
  // multiple of the stage depth, the zero-filled k sub-blocks are not
  // multiplied (a sub-block's two groups interleave its 16 k through the
  // k-permutation, so the unit is the sub-block)
  const int last_groups = 2 * (int)min((int64_t)KSUB,
                                       (prm.m - (int64_t)(kb0 + nk - 1) * KS + BK - 1) / BK);
  for (int kb = 0; kb < nk; ++kb) {  // kb: stage index within this block's k-range
    // (128-wide tiles only: the 64-wide instantiation measured 2.9% slower
    // with the guard -- its zero-filled k is multiplied instead)
    const int ngv = BNT == 128 && kb == nk - 1 ? last_groups : 2 * KSUB;
    if (warp == 0) {
      const int kn = kb + STAGES - 1;  // refill the slot consumed at kb - 1
      if (kn < nk) {
        if (kb > 0) mbar_wait(empty0 + 8 * (kn % STAGES), ((kb - 1) / STAGES) & 1);
        if (lane == 0) issue(kn);
      }
    }
    const int s = kb % STAGES;
    const uint32_t sA = s_base + s * STAGE_BYTES, sB = sA + A_BYTES;
#pragma unroll
    for (int gg = 0; gg < 2 * KSUB; gg += 2) {
      load_frags(sA, sB, gg + 1, fa1, fb1);  // group gg+1 of this stage
      if (gg < ngv) mma_group(fa0, fb0);     // group gg
      if (gg + 2 < 2 * KSUB) {
        load_frags(sA, sB, gg + 2, fa0, fb0);
      } else {                               // last group: release, prefetch next stage
        // The slot is refilled by TMA (async proxy) once every warp has
        // arrived: its fragment loads (generic proxy) must have read the slot
        // first.  mbarrier.arrive's release does not order them against the
        // async proxy, and the SASS issued the arrive with the last LDS.128s
        // still in flight -- measured: a fragment of the next stage's data in
        // rows 64-127 of some tiles (ordered fold, two CTAs per SM, n >= 8192;
        // tools/ordered_dbg.py).  The proxy fence waits for them (MEMBAR.ALL.CTA
        // + FENCE.VIEW.ASYNC.S), after 64 DMMAs that cover their latency.
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
        if (lane == 0) mbar_arrive(empty0 + 8 * s);
        if (kb + 1 < nk) {
          const int s1 = (kb + 1) % STAGES;
          mbar_wait(full0 + 8 * s1, ((kb + 1) / STAGES) & 1);
          const uint32_t nA = s_base + s1 * STAGE_BYTES;
          load_frags(nA, nA + A_BYTES, 0, fa0, fb0);
        }
      }
      if (gg + 1 < ngv) mma_group(fa1, fb1); // group gg+1
    }
  }

  if constexpr (FUSE == 2) {
    // ---- ordered fold (north_star (3); SURVEY §8f NEXT-1 "deterministic
    // product-serial ordering"): for every C block i this product feeds, wait
    // until the block's previous products have updated this tile position,
    // then C_i = W'[i][q] * P (first product of block i) or C_i + W'[i][q] * P,
    // times alpha at the last product -- K6's per-element order exactly ----
    const int tiles = prm.tiles_m * prm.tiles_n;
    const int nflags = prm.nP * prm.nP * tiles;
    const int q = job.out_idx;
    const int t0 = prm.post_off[q], t1 = prm.post_off[q + 1];
    const double alpha = prm.alpha;
    // 256-bit stores need every C block's column offset (bc * m) 4-aligned too
    const bool vec_ok = ((prm.ldo & 3) == 0) && ((prm.m & 3) == 0) &&
                        ((reinterpret_cast<uintptr_t>(prm.out) & 31) == 0);
    for (int ti = t0; ti < t1; ++ti) {
      const PostTerm pt = prm.post[ti];
      const int br = pt.blk >> 16, bc = pt.blk & 0xffff;
      const int seq = pt.flags >> 8;  // products of block i before this one
      uint32_t* flag = prm.sync + (int64_t)(br * prm.nP + bc) * tiles + t;
      if (threadIdx.x == 0 && seq > 0)
        while (ld_acquire(flag) < (uint32_t)seq) __nanosleep(64);
      __syncthreads();
      const double w = pt.coef;
      const bool first = pt.flags & POST_FIRST;
      const bool scale = (pt.flags & POST_LAST) && alpha != 1.0;
      double* cb = prm.out + (int64_t)br * prm.m * prm.ldo + (int64_t)bc * prm.m;
      // the warp tile in HALVES row groups: each group's loads are all in
      // flight before its first add (128-wide tiles: two groups of 4 x 16
      // rows, 32 registers of C per thread -- a whole tile would spill)
      constexpr int HALVES = NJ == 2 ? 2 : 1, MH = 8 / HALVES;
#pragma unroll
      for (int h = 0; h < HALVES; ++h) {
        double old[MH][NJ][4];
        if (!first) {
#pragma unroll
          for (int mh = 0; mh < MH; ++mh) {
            const int mi = MH * h + mh;
            const int64_t row = (int64_t)tm * BM + wm * 64 + mi * 8 + lr;
#pragma unroll
            for (int nj = 0; nj < NJ; ++nj) {
              const int64_t col = (int64_t)tn * BNT + wn * WN + nj * 16 + 4 * lk;
              const double* src = cb + row * prm.ldo + col;
              if (row < prm.m && vec_ok && col + 3 < prm.m) {
                ld_v2(src, old[mh][nj][0], old[mh][nj][1]);
                ld_v2(src + 2, old[mh][nj][2], old[mh][nj][3]);
              } else {
#pragma unroll
                for (int u = 0; u < 4; ++u)
                  old[mh][nj][u] = (row < prm.m && col + u < prm.m) ? ld_f64(src + u) : 0.0;
              }
            }
          }
        }
#pragma unroll
        for (int mh = 0; mh < MH; ++mh) {
          const int mi = MH * h + mh;
          const int64_t row = (int64_t)tm * BM + wm * 64 + mi * 8 + lr;
          if (row >= prm.m) continue;
#pragma unroll
          for (int nj = 0; nj < NJ; ++nj) {
            const int64_t col = (int64_t)tn * BNT + wn * WN + nj * 16 + 4 * lk;
            double v[4] = {__dmul_rn(w, acc[mi][nj][0][0]), __dmul_rn(w, acc[mi][nj][1][0]),
                           __dmul_rn(w, acc[mi][nj][0][1]), __dmul_rn(w, acc[mi][nj][1][1])};
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              if (!first) v[u] = __dadd_rn(old[mh][nj][u], v[u]);
              if (scale) v[u] = __dmul_rn(alpha, v[u]);
            }
            double* dst = cb + row * prm.ldo + col;
            if (vec_ok && col + 3 < prm.m) {
              asm volatile("st.global.v4.f64 [%0], {%1,%2,%3,%4};"
                           :: "l"(dst), "d"(v[0]), "d"(v[1]), "d"(v[2]), "d"(v[3]) : "memory");
            } else {
#pragma unroll
              for (int u = 0; u < 4; ++u)
                if (col + u < prm.m) dst[u] = v[u];
            }
          }
        }
      }
      // publish: block i's tile is updated through this product
      __syncthreads();
      if (threadIdx.x == 0) {
        __threadfence();
        st_release(flag, (uint32_t)seq + 1);
      }
    }
    __shared__ int s_last;
    if (threadIdx.x == 0) s_last = atomicAdd(prm.sync + nflags + 1, 1u) == gridDim.x - 1;
    __syncthreads();
    if (s_last) {  // every CTA is done: zero the flags and counters for the next launch
      for (int i = threadIdx.x; i < nflags; i += THREADS) prm.sync[i] = 0;
      if (threadIdx.x == 0) { prm.sync[nflags] = 0; prm.sync[nflags + 1] = 0; }
    }
    return;
  } else if constexpr (FUSE == 1) {
    // ---- fused post-addition (north_star (3), "folded into the leaf GEMM
    // epilogue"): stage coef*alpha*acc in the drained ring, then threads
    // 0..127 each add one tile row into every C block product q feeds with a
    // bulk f64 reduction (performed at L2; no P round trip through HBM) ----
    constexpr int LDT = BNT + 2;  // +16 B per row: conflict-free v2 stores
    static_assert(BM * LDT * 8 <= STAGES * STAGE_BYTES, "fused tile must fit the ring");
    __syncthreads();  // every warp is past its last ring read; all TMA loads landed
    double* tile = reinterpret_cast<double*>(smem);
    const int q = job.out_idx;
    const int t0 = prm.post_off[q], t1 = prm.post_off[q + 1];
    const int64_t row0 = (int64_t)tm * BM, col0 = (int64_t)tn * BNT;
    const int rows_valid = (int)min((int64_t)BM, prm.m - row0);
    const int cols_valid = (int)min((int64_t)BNT, prm.m - col0);
    double staged = 0.0;
    for (int ti = t0; ti < t1; ++ti) {
      const PostTerm pt = prm.post[ti];
      const double c = pt.coef * prm.alpha;
      if (ti == t0 || c != staged) {
        if (ti > t0) {
          if (threadIdx.x < BM) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
          __syncthreads();
        }
#pragma unroll
        for (int mi = 0; mi < 8; ++mi) {
          const int r = wm * 64 + mi * 8 + lr;
#pragma unroll
          for (int nj = 0; nj < NJ; ++nj) {
            const int cc = wn * WN + nj * 16 + 4 * lk;
            double* d = tile + r * LDT + cc;
            const double v0 = c * acc[mi][nj][0][0], v1 = c * acc[mi][nj][1][0];
            const double v2 = c * acc[mi][nj][0][1], v3 = c * acc[mi][nj][1][1];
            asm volatile("st.shared.v2.f64 [%0], {%1, %2};" :: "r"(smem_u32(d)), "d"(v0), "d"(v1) : "memory");
            asm volatile("st.shared.v2.f64 [%0], {%1, %2};" :: "r"(smem_u32(d + 2)), "d"(v2), "d"(v3) : "memory");
          }
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncthreads();
        staged = c;
      }
      if ((int)threadIdx.x < rows_valid) {
        const int64_t br = pt.blk >> 16, bc = pt.blk & 0xffff;
        double* dst = prm.out + (br * prm.m + row0 + threadIdx.x) * prm.ldo + bc * prm.m + col0;
        asm volatile(
            "cp.reduce.async.bulk.global.shared::cta.bulk_group.add.f64 [%0], [%1], %2;"
            :: "l"(dst), "r"(smem_u32(tile + threadIdx.x * LDT)), "r"(cols_valid * 8) : "memory");
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      }
    }
    // smem must outlive the bulk reads; the grid's completion covers the adds
    // (waiting for their completion too measured the same: fused_postadd_r01.json)
    if (threadIdx.x < BM) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
    return;
  } else {
    if (piece) {
      // ---- split-K piece: publish the partial, the last arrival reduces ----
      constexpr int NACC = 8 * NJ * 4;
      const int tail = tile - prm.n_whole;
      double* ws = prm.part_ws + ((size_t)tail * prm.split + split_idx) * (NACC * THREADS);
#pragma unroll
      for (int mi = 0; mi < 8; ++mi)
#pragma unroll
        for (int nj = 0; nj < NJ; ++nj)
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const int e = (mi * NJ + nj) * 4 + u;
            __stcg(ws + e * THREADS + threadIdx.x, acc[mi][nj][u >> 1][u & 1]);
          }
      __threadfence();
      __syncthreads();
      __shared__ int s_last;
      if (threadIdx.x == 0) s_last = atomicAdd(prm.part_cnt + tail, 1) == prm.split - 1;
      __syncthreads();
      if (!s_last) return;
      __threadfence();
      const double* base = prm.part_ws + (size_t)tail * prm.split * (NACC * THREADS);
#pragma unroll
      for (int mi = 0; mi < 8; ++mi)
#pragma unroll
        for (int nj = 0; nj < NJ; ++nj)
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const int e = (mi * NJ + nj) * 4 + u;
            double v = __ldcg(base + e * THREADS + threadIdx.x);
            for (int sp = 1; sp < prm.split; ++sp)
              v += __ldcg(base + ((size_t)sp * NACC + e) * THREADS + threadIdx.x);
            acc[mi][nj][u >> 1][u & 1] = v;
          }
      if (threadIdx.x == 0) prm.part_cnt[tail] = 0;  // ready for the next launch
    }
    TRACE(2);
    // ---- epilogue: registers -> global (4 consecutive columns per thread) ----
    double* out = prm.out + (int64_t)job.out_idx * prm.out_stride;
    const double alpha = prm.alpha;
    const bool vec_ok = ((prm.ldo & 3) == 0) && ((reinterpret_cast<uintptr_t>(out) & 31) == 0);
#pragma unroll
    for (int mi = 0; mi < 8; ++mi) {
      const int64_t row = (int64_t)tm * BM + wm * 64 + mi * 8 + lr;
      if (row >= prm.m) continue;
#pragma unroll
      for (int nj = 0; nj < NJ; ++nj) {
        const int64_t col = (int64_t)tn * BNT + wn * WN + nj * 16 + 4 * lk;
        double v0 = acc[mi][nj][0][0], v1 = acc[mi][nj][1][0];
        double v2 = acc[mi][nj][0][1], v3 = acc[mi][nj][1][1];
        if (alpha != 1.0) {
          v0 = __dmul_rn(alpha, v0); v1 = __dmul_rn(alpha, v1);
          v2 = __dmul_rn(alpha, v2); v3 = __dmul_rn(alpha, v3);
        }
        double* dst = out + row * prm.ldo + col;
        if (vec_ok && col + 3 < prm.m) {
          asm volatile("st.global.v4.f64 [%0], {%1,%2,%3,%4};"
                       :: "l"(dst), "d"(v0), "d"(v1), "d"(v2), "d"(v3) : "memory");
        } else {
          if (col + 0 < prm.m) dst[0] = v0;
          if (col + 1 < prm.m) dst[1] = v1;
          if (col + 2 < prm.m) dst[2] = v2;
          if (col + 3 < prm.m) dst[3] = v3;
        }
      }
    }
    TRACE(3);
  }
}

// MF_LEAF_SIMPLE: one thread per output element, k ascending, fma.rn.f64.
// Any shape/alignment; an ablation and the fallback for views TMA cannot
// describe (odd m or odd leading dimension).
struct SimpleParams {
  const double *A, *B, *T, *S;
  int64_t lda, ldb, m, r0, r1, c0, c1;
  double* out;
  int64_t ldo, out_stride;
  double alpha;
  const LeafJob* jobs;
  const int32_t* post_off;  // fused post-addition: out = C, ldo = ldc
  const PostTerm* post;
  int ordered;  // ordered fold: one launch per job, in job order (stream-ordered)
};

__global__ void leaf_simple_kernel(const SimpleParams prm) {
  const LeafJob job = prm.jobs[blockIdx.z];
  const int64_t r = prm.r0 + (int64_t)blockIdx.y * 16 + threadIdx.y;
  const int64_t c = prm.c0 + (int64_t)blockIdx.x * 16 + threadIdx.x;
  if (r >= prm.r1 || c >= prm.c1) return;
  const int64_t mm = prm.m * prm.m;
  const double* X;
  int64_t ldx;
  if (job.flags & 1) { X = prm.T + job.a_coord * mm; ldx = prm.m; }
  else { X = prm.A + (job.a_coord >> 16) * prm.m * prm.lda + (job.a_coord & 0xffff) * prm.m; ldx = prm.lda; }
  const double* Y;
  int64_t ldy;
  if (job.flags & 2) { Y = prm.S + job.b_coord * mm; ldy = prm.m; }
  else { Y = prm.B + (job.b_coord >> 16) * prm.m * prm.ldb + (job.b_coord & 0xffff) * prm.m; ldy = prm.ldb; }
  double acc = 0.0;
  for (int64_t k = 0; k < prm.m; ++k) acc = fma(X[r * ldx + k], Y[k * ldy + c], acc);
  if (prm.post) {
    for (int t = prm.post_off[job.out_idx]; t < prm.post_off[job.out_idx + 1]; ++t) {
      const PostTerm pt = prm.post[t];
      const int64_t br = pt.blk >> 16, bc = pt.blk & 0xffff;
      double* dst = prm.out + (br * prm.m + r) * prm.ldo + bc * prm.m + c;
      if (prm.ordered) {  // K6's order: store first, add, alpha last
        double v = __dmul_rn(pt.coef, acc);
        if (!(pt.flags & POST_FIRST)) v = __dadd_rn(*dst, v);
        if ((pt.flags & POST_LAST) && prm.alpha != 1.0) v = __dmul_rn(prm.alpha, v);
        *dst = v;
      } else {
        atomicAdd(dst, pt.coef * prm.alpha * acc);
      }
    }
    return;
  }
  if (prm.alpha != 1.0) acc = __dmul_rn(prm.alpha, acc);
  prm.out[job.out_idx * prm.out_stride + r * prm.ldo + c] = acc;
}

// ---- tensor-map encoding through the driver entry point (no -lcuda) ----
using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                              const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                              const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                              CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeFn encode_fn() {
  static EncodeFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess && q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeFn>(p);
  });
  return fn;
}

// 4-D block view of an n x n row-major matrix: {col-in-block, block-col,
// row-in-block, block-row}; box {bc0, 1, bc2, 1}.
bool encode_block_view(CUtensorMap* map, const double* X, int64_t ld, int P, int64_t m,
                       uint32_t box0, uint32_t box2, CUtensorMapSwizzle sw) {
  cuuint64_t dims[4] = {(cuuint64_t)m, (cuuint64_t)P, (cuuint64_t)m, (cuuint64_t)P};
  cuuint64_t strides[3] = {(cuuint64_t)m * 8, (cuuint64_t)ld * 8, (cuuint64_t)m * ld * 8};
  cuuint32_t box[4] = {box0, 1, box2, 1};
  cuuint32_t es[4] = {1, 1, 1, 1};
  return encode_fn()(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, const_cast<double*>(X), dims, strides,
                     box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, sw,
                     CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// 3-D slot view of a workspace [slots][m][m]: {col, row, slot}.
bool encode_slot_view(CUtensorMap* map, const double* X, int slots, int64_t m, uint32_t box0,
                      uint32_t box1, CUtensorMapSwizzle sw) {
  cuuint64_t dims[3] = {(cuuint64_t)m, (cuuint64_t)m, (cuuint64_t)(slots > 0 ? slots : 1)};
  cuuint64_t strides[2] = {(cuuint64_t)m * 8, (cuuint64_t)m * m * 8};
  cuuint32_t box[3] = {box0, box1, 1};
  cuuint32_t es[3] = {1, 1, 1};
  return encode_fn()(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<double*>(X), dims, strides,
                     box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, sw,
                     CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

bool al16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

}  // namespace

#ifdef MF_LEAF_TRACE
extern "C" int mf_debug_leaf_trace(unsigned long long* out, int n) {
  n = n < kTraceMax ? n : kTraceMax;
  return (int)cudaMemcpyFromSymbol(out, g_leaf_trace, sizeof(unsigned long long) * 5 * n);
}
#endif

bool leaf_tma_supported(const LeafArgs& a) {
  // TMA: 16-byte aligned bases, strides multiple of 16 bytes (m, ld even).
  if (!encode_fn()) return false;
  if ((a.m & 1) || (a.lda & 1) || (a.ldb & 1)) return false;
  if (!al16(a.A) || !al16(a.B) || (a.T && !al16(a.T)) || (a.S && !al16(a.S))) return false;
  if (a.m > (int64_t)1 << 30 || a.P > 0xffff) return false;
  return true;
}

// Tile shape and split-K tail of one DMMA leaf launch.  Cost model in units of
// one 128x128 tile's time, waves of `sms` CTAs:
//  * BN = 128: ceil(tiles / sms);  BN = 64: ceil(tiles64 / sms) * 0.5 / 0.98
//    (2% per-tile penalty for the narrower tile);
//  * split-K (BN = 128): the first w full waves whole, the remaining tiles cut
//    into S k-ranges: w + ceil(tail * S / sms) * (1 / S + eps), eps = the
//    per-piece overhead (prologue + partial store/reload, ~4 us against a
//    0.13 us-per-k tile).
// E.g. 7 products of 2048^2 (config 2): 1792 tiles = 12.1 waves -> 12 whole
// waves + 16 tiles x 9 pieces (12.13) instead of 25 half-width waves (12.76);
// 49 products of 4096^2: 339 whole waves + the 4 leftover tiles as 16 pieces
// each (339.07 instead of 340).
// MF_LEAF_BN / MF_LEAF_SPLIT override.
LeafTiles leaf_tiles(const LeafArgs& a) {
  LeafTiles cfg;
  const int64_t r0 = a.rows.r0, r1 = a.rows.end(a.m), c0 = a.rows.c0, c1 = a.rows.cend(a.m);
  if (a.n_jobs == 0 || a.m == 0 || r1 <= r0 || c1 <= c0) return cfg;
  int sms = 148, dev = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t tm_tiles = (r1 - r0 + BM - 1) / BM;
  auto tiles = [&](int bn) { return tm_tiles * ((c1 - c0 + bn - 1) / bn) * a.n_jobs; };
  auto waves = [&](int64_t t) { return (double)((t + sms - 1) / sms); };
  const int64_t t128 = tiles(128);
  double best = waves(t128);
  cfg.bn = 128;
  if (!a.rows.overlapped && waves(tiles(64)) * 0.5 / 0.98 < best) {
    best = waves(tiles(64)) * 0.5 / 0.98;
    cfg.bn = 64;
  }
  const int kblocks = (int)((a.m + 31) / 32);
  // split only where the pieces cannot race another launch on the workspace:
  // full-width launches (the host pipeline's column regions run on two streams)
  const bool can_split = !a.post && c0 == 0 && c1 == a.m && kblocks >= 8;
  const double eps = std::max(0.01, 32.0 / (double)a.m);
  const int64_t full = t128 / sms;
  int max_split = 16;
  if (const char* e = getenv("MF_LEAF_SPLIT")) max_split = std::max(1, atoi(e));
  for (int64_t w = full; can_split && w >= std::max<int64_t>(0, full - 1); --w) {
    const int64_t tail = t128 - w * sms;
    if (tail <= 0) continue;
    for (int S = 2; S <= max_split && S <= kblocks / 4; ++S) {
      const double cost = (double)w + waves(tail * S) * (1.0 / S + eps);
      if (cost < best - 0.02) {  // worth at least 2% of one tile's time
        best = cost;
        cfg.bn = 128; cfg.split = S; cfg.n_whole = w * sms; cfg.n_tail = tail;
      }
    }
  }
  if (const char* e = getenv("MF_LEAF_BN")) {
    cfg.bn = atoi(e) == 64 ? 64 : 128;
    if (cfg.bn == 64) cfg.split = 1;
  }
  if (cfg.split > 1) cfg.ws_elems = cfg.n_tail * cfg.split * (int64_t)BM * 128;
  return cfg;
}

cudaError_t launch_leaf(const LeafArgs& a, int leaf_kind, cudaStream_t s) {
  const int64_t r0 = a.rows.r0, r1 = a.rows.end(a.m), c0 = a.rows.c0, c1 = a.rows.cend(a.m);
  if (a.n_jobs == 0 || a.m == 0 || r1 <= r0 || c1 <= c0) return cudaSuccess;
  // fused post-addition: bulk reductions need 16-byte aligned C rows (the
  // ordered fold stores from registers: any 8-byte aligned C)
  const bool ordered = a.post && a.fuse_sync;
  const bool fuse_ok = !a.post || ordered || (!(a.ldo & 1) && al16(a.out));
  if (leaf_kind == MF_LEAF_DMMA && leaf_tma_supported(a) && fuse_ok && r0 % BM == 0 &&
      c0 % BN == 0 && (c1 == a.m || c1 % BN == 0)) {
    const int64_t tm_tiles = (r1 - r0 + BM - 1) / BM;
    int dev = 0;
    cudaGetDevice(&dev);
    LeafTiles cfg = leaf_tiles(a);
    // the caller provides the split-K workspace (run_leaf sizes it from leaf_tiles)
    if (cfg.split > 1 && (!a.split_ws || a.split_ws_elems < cfg.ws_elems || a.split_cnt_len < cfg.n_tail))
      cfg.split = 1;
    // Two CTAs per SM (4 MMA warps, 128 x 64 tiles, 96 KB rings): one CTA's
    // epilogue runs beside the other's k loop.  The default for both folds,
    // whose epilogues it hides (SW^2 n=16384: bulk 188.3 ms vs unfused 187.8;
    // ordered 191.3 vs 194.0 ms on one CTA per SM; SW^3: ordered 182.9 vs
    // 193.3 ms; profiles/ordered_2cta_r02.jsonl), and for unfused leaves with
    // m <= 1536, where the per-tile prologue / epilogue is a larger share of a
    // tile's k loop: +0.4% (m = 1536) .. +9% (m = 512), SW^4 hybrid 158.2 ->
    // 157.2 ms -- when its 128 x 64 tiles fill at least one wave of two CTAs
    // per SM (smaller grids keep one CTA per SM and its split-K tail: n = 1024
    // SW^1, 224 tiles: 0.114 vs 0.118 ms); above m = 1536 one 128 x 128 CTA per
    // SM (m = 4096: 187.8 vs 189.9 ms; profiles/leaf2cta_m_r02.jsonl).
    // MF_LEAF_2CTA=1/0 forces it.
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int64_t tiles64 = tm_tiles * ((c1 - c0 + 63) / 64) * a.n_jobs;
    const char* e2 = getenv("MF_LEAF_2CTA");
    const bool two_cta = e2 ? atoi(e2) > 0 : (a.post != nullptr || (a.m <= 1536 && tiles64 >= 2 * sms));
    if (two_cta) { cfg.bn = 64; cfg.split = 1; }
    const int bn = cfg.bn;
    // k sub-blocks of 16 per pipeline stage: 2 (k = 32, 3-stage ring), or 3
    // (k = 48, 2 stages) where m is a multiple of 48 or large -- measured
    // +0.2% there, -0.3% at m = 4096 (profiles/leaf_ksub_r01.json)
    int ksub = (a.m % 48 == 0 || a.m >= 8192) && bn == 128 ? 3 : 2;
    if (const char* e = getenv("MF_LEAF_KSUB")) ksub = std::min(3, std::max(1, atoi(e)));
    if (ksub == 3 && bn != 128) ksub = 2;
    const bool fuse = a.post != nullptr;
    if (fuse) ksub = 2;  // the fused tile is staged in the KSUB=2 ring
    // the two-CTA shape has only the KSUB = 2 instantiation (KSUB = 1 with 4
    // stages measured 1.1% slower at n=16384 SW^2); set before the B box and
    // kblocks below are derived from ksub
    if (two_cta) ksub = 2;
    if (ordered &&
        (int64_t)a.P * a.P * ((r1 - r0 + BM - 1) / BM) * ((c1 - c0 + bn - 1) / bn) > a.fuse_sync_len)
      return cudaErrorInvalidValue;
    CUtensorMap mA, mT, mB, mS;
    const bool ok =
        encode_block_view(&mA, a.A, a.lda, a.P, a.m, BK, BM, CU_TENSOR_MAP_SWIZZLE_128B) &&
        encode_slot_view(&mT, a.T ? a.T : a.A, a.n_slots_a, a.m, BK, BM, CU_TENSOR_MAP_SWIZZLE_128B) &&
        encode_block_view(&mB, a.B, a.ldb, a.P, a.m, bn, BK * ksub, CU_TENSOR_MAP_SWIZZLE_NONE) &&
        encode_slot_view(&mS, a.S ? a.S : a.B, a.n_slots_b, a.m, bn, BK * ksub, CU_TENSOR_MAP_SWIZZLE_NONE);
    if (!ok) return cudaErrorInvalidValue;
    LeafParams prm;
    prm.m = a.m;
    prm.tm0 = (int)(r0 / BM);
    prm.tiles_m = (int)tm_tiles;
    prm.tn0 = (int)(c0 / bn);
    prm.tiles_n = (int)((c1 - c0 + bn - 1) / bn);
    prm.kblocks = (int)((a.m + BK * ksub - 1) / (BK * ksub));
    prm.out = a.out;
    prm.ldo = a.ldo;
    prm.out_stride = a.out_block_stride;
    prm.alpha = a.alpha;
    prm.jobs = a.jobs;
    prm.post_off = a.post_off;
    prm.post = a.post;
    prm.sync = a.fuse_sync;
    prm.nP = a.P;
    prm.split = cfg.split;
    prm.n_whole = cfg.split > 1 ? (int)cfg.n_whole : 0;
    prm.part_ws = a.split_ws;
    prm.part_cnt = a.split_cnt;
    prm.group_m = GROUP_M;
    if (const char* e = getenv("MF_LEAF_GROUPM")) prm.group_m = std::max(1, atoi(e));
    const int64_t grid = cfg.split > 1 ? cfg.n_whole + cfg.n_tail * cfg.split
                                       : (int64_t)prm.tiles_m * prm.tiles_n * a.n_jobs;
    if (grid > 0x7fffffff) return cudaErrorInvalidValue;
    // the >48 KB dynamic shared memory opt-in is per device: once per
    // (device, instantiation)
    static std::atomic<uint64_t> attr_set[12];
    const int inst = two_cta ? (ordered ? 10 : fuse ? 11 : 9)
                     : ordered ? (bn == 64 ? 8 : 7)
                     : fuse  ? (bn == 64 ? 5 : 4)
                             : (ksub == 3 ? 6 : (bn == 64 ? 2 : 0) + (ksub == 2 ? 1 : 0));
    const int threads = two_cta ? 128 : THREADS;
    const uint64_t dev_bit = 1ull << (dev & 63);
    auto launch = [&](auto kern, int smem) -> cudaError_t {
      if (!(attr_set[inst].load() & dev_bit)) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        if (e != cudaSuccess) return e;
        attr_set[inst].fetch_or(dev_bit);
      }
      kern<<<(unsigned)grid, threads, smem, s>>>(mA, mT, mB, mS, prm);
      return cudaSuccess;
    };
    cudaError_t e;
    switch (inst) {
      case 0: e = launch(leaf_dmma_kernel<128, 1, 0>, smem_bytes<128, 1>()); break;
      case 1: e = launch(leaf_dmma_kernel<128, 2, 0>, smem_bytes<128, 2>()); break;
      case 2: e = launch(leaf_dmma_kernel<64, 1, 0>, smem_bytes<64, 1>()); break;
      case 3: e = launch(leaf_dmma_kernel<64, 2, 0>, smem_bytes<64, 2>()); break;
      case 4: e = launch(leaf_dmma_kernel<128, 2, 1>, smem_bytes<128, 2>()); break;
      case 6: e = launch(leaf_dmma_kernel<128, 3, 0>, smem_bytes<128, 3>()); break;
      case 7: e = launch(leaf_dmma_kernel<128, 2, 2>, smem_bytes<128, 2>()); break;
      case 8: e = launch(leaf_dmma_kernel<64, 2, 2>, smem_bytes<64, 2>()); break;
      case 9: e = launch(leaf_dmma_kernel<64, 2, 0, 4>, smem_bytes<64, 2, 4>()); break;
      case 10: e = launch(leaf_dmma_kernel<64, 2, 2, 4>, smem_bytes<64, 2, 4>()); break;
      case 11: e = launch(leaf_dmma_kernel<64, 2, 1, 4>, smem_bytes<64, 2, 4>()); break;
      default: e = launch(leaf_dmma_kernel<64, 2, 1>, smem_bytes<64, 2>()); break;
    }
    if (e != cudaSuccess) return e;
    return cudaGetLastError();
  }
  SimpleParams prm{a.A, a.B, a.T, a.S, a.lda, a.ldb, a.m, r0, r1, c0, c1, a.out, a.ldo,
                   a.out_block_stride, a.alpha, a.jobs, a.post_off, a.post, ordered ? 1 : 0};
  if (ordered) {  // one launch per product, in order (the stream serialises them)
    dim3 grid((unsigned)((c1 - c0 + 15) / 16), (unsigned)((r1 - r0 + 15) / 16), 1);
    for (int j = 0; j < a.n_jobs; ++j) {
      prm.jobs = a.jobs + j;
      leaf_simple_kernel<<<grid, dim3(16, 16), 0, s>>>(prm);
    }
    return cudaGetLastError();
  }
  dim3 grid((unsigned)((c1 - c0 + 15) / 16), (unsigned)((r1 - r0 + 15) / 16), (unsigned)a.n_jobs);
  leaf_simple_kernel<<<grid, dim3(16, 16), 0, s>>>(prm);
  return cudaGetLastError();
}

}  // namespace mf
