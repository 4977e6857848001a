// Batched early-stopping column-pivoted Householder QR of interface panels:
// the sparsification step.  Restates, per panel,
//   _rrqr_core      /root/reference/pkg/src/spdkit/dense.py:117-183
//   rrqr_sparsify   dense.py:186-222
//   make_sparsification + EliminationState.sparsify
//                   schemes.py:272-318, factorize.py:175-196
//
// One launch processes one WAVE of interfaces (no two of them are
// neighbours, so they are independent).  Every panel gets a GROUP of CTAs
// that together run the pivoted QR with one group barrier per elimination
// step; the launch is cooperative so all groups are co-resident.  The
// panel's columns are split in contiguous ranges over the group's CTAs and
// never move: pivoting is bookkeeping (perm / pos arrays), exactly the
// reference's swap order, so ties resolve to the smallest CURRENT position
// like np.argmax on the swapped norms.  Per step, a CTA updates its own
// columns with the Householder reflector (one warp per column: dot, rank-1
// update, row-k entry, exact tail norm), downdates the running norms with
// the reference's 0.01 refresh rule, and proposes its local argmax; the
// reflector is rebuilt redundantly in every CTA from the winning column,
// and Q (= H_0 H_1 ...) is updated row-parallel.
//
// Deciding values (eta, r11, stop test, coarse test) follow the reference
// formulas; only summation order differs, so ranks match except within
// ~1e-15 relative of a threshold (the events record the margins).
#include <cooperative_groups.h>
#include <cstdio>
#include <type_traits>

#include "common.cuh"
#include "../../include/spand_b200.h"


namespace {
constexpr int kT = 256;
constexpr int kWarps = kT / 32;
// v (the reflector) lives in shared memory: up to 24576 rows (192 KB; a
// wave holding such a panel runs one CTA per SM -- spand_rrqr_capacity)
constexpr int kMaxM = 24576;

// panel row (16 int64):
//  0 p        1 nbr_begin  2 nbr_end   3 W (double*, temp, >= m*n)
//  4 Q (double*, m*m, compact ld = m)  5 aux (double*)  6 iaux (int32*)
//  7 group_begin  8 group_size  9 counters (uint32[2]: arrivals, release)  10 event slot
//  11 ncap (column capacity of aux arrays)  12 mcap
//  13 near-kernel workspace (nearkernel.cu; 0: none)
//  14 clustered launches: the per-CTA list copies (int32, 4 G (ncap / (G / cs) + 2);
//     0: inside the int-list region)  15 unused
// nbr row (4 int64): {w, block ptr, orientation, 0}
//  orientation 0: block (p, w) stored with rows of p (ld = m0[p])
//  orientation 1: block (w, p) stored with rows of w (ld = m0[w])
// event row (12 int64): {p, m, n, k_stop, k_c, rank_f2, n_fine,
//  bits(eta_stop), bits(r11), 0, 0, 0}

constexpr int kCR = 4;   // candidate record stride (doubles): contiguous, coalesced scans
constexpr int kLDS = 68;       // frozen-column DMMA tiles (conflict-free fragments)
// dynamic shared memory floor: write-back staging (8 warps x 16 x 33) and
// the frozen-GEMM epilogue tile (64 x 65)
constexpr size_t kMinSmem = (size_t)4 * 16 * kLDS * sizeof(double);   // 2 stages x (A, B)
// cold-column maintenance layout in the dynamic shared memory (doubles):
// scratch (2 stages x kPBK rows of the A (64) and V (32) operands, and the
// 64 x 65 update tile) | T [32][33] | Y/Z [64][33] | R rows [64][33] | tails [64]
constexpr int kPBK = 32;         // rows per stage of the cold-column product
// columns per sweep of the blocked reflector updates (cold maintenance, Q
// formation): kMT DMMA m-tiles of 8.  The reflector block V_b is streamed once
// per sweep, so wider sweeps halve its traffic for CTAs with > 16 columns.
#ifndef SPAND_COLD_MT
#define SPAND_COLD_MT 2
#endif
constexpr int kMT = SPAND_COLD_MT, kSweep = 8 * kMT;
static_assert(kMT == 2 || kMT == 4, "sweep width 16 or 32 columns");
constexpr int kScr0 = 2 * kPBK * (kLDS + 36), kScr1 = 8 * kSweep * 32;   // stages | per-warp partials
constexpr int kCScr = 0, kCT = kScr0 > kScr1 ? kScr0 : kScr1, kCZ = kCT + 32 * 33,
              kCR2 = kCZ + 64 * 33, kCTail = kCR2 + 64 * 33, kColdEnd = kCTail + 64;
constexpr size_t kColdSmem = (size_t)kColdEnd * sizeof(double);
#ifndef SPAND_ROW_UNROLL
#define SPAND_ROW_UNROLL 1
#endif
constexpr int kRowUnroll = SPAND_ROW_UNROLL;   // row loops of the DMMA block updates
#ifndef SPAND_ROW_BATCH
#define SPAND_ROW_BATCH 1
#endif
constexpr int kRowBatch = SPAND_ROW_BATCH;     // 8-row slabs loaded ahead per iteration
#ifndef SPAND_BLK
#define SPAND_BLK 32
#endif
constexpr int kBlk = SPAND_BLK;  // reflectors per cold-column block update (<= 32)
#ifndef SPAND_BLK0
#define SPAND_BLK0 8
#endif
// hot iff running norm^2 >= rho * pivot norm^2; rho grows with the panel
// height (cheaper blocked cold updates vs. per-step column work; measured on
// C4-L15 with rho in {0.1 .. 0.9}: best 0.35 below 700 rows, 0.5 below 1200,
// 0.65 below 2000, 0.75 above)
__device__ __forceinline__ double hot_rho(int m) {
#ifdef SPAND_HOT_RHO
  return SPAND_HOT_RHO;
#else
#ifndef SPAND_RHO_A
#define SPAND_RHO_A 0.35
#define SPAND_RHO_B 0.5
#define SPAND_RHO_C 0.65
#define SPAND_RHO_D 0.75
#endif
  return m < 700 ? SPAND_RHO_A : (m < 1200 ? SPAND_RHO_B : (m < 2000 ? SPAND_RHO_C : SPAND_RHO_D));
#endif
}
static_assert(kColdSmem >= 128 * 65 * sizeof(double), "epilogue tile");
// frozen-column GEMM (qt_a): kFS cp.async stages of kFK rows of A (64 + 4
// padded) and B (128 + 4 padded); the classic kernel runs one CTA per SM, so
// its launches ask for kLaunchSmem of dynamic shared memory
constexpr int kFK = 32, kFS = 3;
constexpr size_t kFrozenSmem = (size_t)kFS * kFK * (68 + 132) * sizeof(double);
constexpr size_t kLaunchSmem = kFrozenSmem > kColdSmem ? kFrozenSmem : kColdSmem;
static_assert(kLaunchSmem >= 128 * 65 * sizeof(double), "frozen GEMM epilogue");
static_assert(kMinSmem >= (size_t)kWarps * 16 * 33 * sizeof(double), "gather tiles");
static_assert(kColdSmem >= kMinSmem, "cold layout covers the other phases");
// clustered loop layout in the dynamic shared memory (doubles): exchange
// partials [2][kXB] | sums [kXB] | pivot rows [kXS] | scratch 4096 | T, Z [32][33]
constexpr int kXB = 1056, kXS = 512, kHC = 512;
// partials [2][kXB] | sums [kXB] | pivot rows [kXS] | cp.async stages
// [2][V, X][32][33] | Z, T [32][33] | hot state: cur, ref [kHC] + 4 int [kHC]
constexpr int kClEnd = 3 * kXB + kXS + 4 * 32 * 33 + 2 * 32 * 33 + 2 * kHC + 2 * kHC;
constexpr size_t kClSmem = (size_t)kClEnd * sizeof(double);
static_assert((kClSmem > kFrozenSmem ? kClSmem : kFrozenSmem) >= kColdSmem,
              "clustered launches cover the post-loop phases");
// the clustered kernel shares the post-loop phases, so its launches must also
// cover the frozen-column GEMM's staging buffers
constexpr size_t kClLaunchSmem = kClSmem > kFrozenSmem ? kClSmem : kFrozenSmem;

// largest group whose frozen-column product is dealt tile by tile over the
// whole group (larger groups keep the per-CTA lists)
constexpr int kMaxG = 320;
struct Sh {
  double red[kWarps];
  double bval[kWarps];
  int64_t bpos[kWarps];
  int64_t bpc[kWarps];
  double bfm[kWarps];
  double bcm[kWarps];
  int bq[kWarps];
  int bcol[kWarps];
  int nfrz;
  int nact;
  int ncold;
  double coldmax;
  int nhot, nhot3;
  double red8[kWarps][8];   // multi-value block reductions of the column pass
  double tot8[8];
  double xk[2][4];          // row k of the column-pass batch (by batch parity)
  int nfrz_tmp;             // k_c search
  unsigned long long fmax;   // bits of the max norm^2 of my frozen columns (>= 0)
  int nb_start[1025];  // column start of each neighbour (panels with <= 1024)
  int wsum[kWarps];
  int wsum2[2 * kWarps];
  double ccur[32], cref[32];   // clustered cold maintenance: running norms before the exchanges
  int nhot_cl, ncold_cl;      // clustered loop: list lengths (identical in the cluster)
  unsigned long long mcl;     // clustered reclassification: max running norm^2 (bits)
  double* cbase[128];  // frozen GEMM epilogue: column base in the pool
  int64_t cstride[128];
  int fcol[128];
  int fpre[kMaxG + 1];  // frozen GEMM: prefix sums of the group's frozen-column counts
};

__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void st_release(unsigned* p, unsigned v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;\n" ::"l"(p), "r"(v) : "memory");
}

// Group barrier: ctr[0] counts arrivals, the last CTA of generation `gen`
// publishes gen in ctr[1] (release); the others poll ctr[1] (acquire), so
// the polled word changes once per barrier instead of once per arrival.
// `tgt` accumulates the arrivals expected so far: every CTA arrives at a
// group barrier (G), only cluster leaders at the clustered loop's step
// barrier (cluster_step_barrier, G / CS), on the same two words.
__device__ __forceinline__ void barrier_arrive_wait(unsigned* ctr, unsigned add, bool arrive,
                                                    unsigned& gen, unsigned& tgt, int tag,
                                                    int64_t* flag) {
  __threadfence();
  ++gen;
  tgt += add;
  bool done = false;
  if (arrive) done = atomicAdd(ctr, 1u) + 1u == tgt;
  if (done) {
    st_release(ctr + 1, gen);
  } else {
    const long long t0 = clock64();
    while (ld_acquire(ctr + 1) < gen) {
      // watchdog: a group that never completes a barrier is a bug; report
      // and fall through (~2 s) instead of hanging the device
      if (clock64() - t0 > 4000000000ll) {
        printf("[spand rrqr] barrier timeout block %d tag %d gen %u ctr %u tgt %u\n",
               (int)blockIdx.x, tag, gen, ld_acquire(ctr), tgt);
        if (flag) atomicExch(reinterpret_cast<unsigned long long*>(flag), 1ull);
        break;
      }
    }
  }
  __threadfence();
}

__device__ __forceinline__ void group_barrier(unsigned* ctr, int G, unsigned& gen, unsigned& tgt,
                                              int tag = -1, int64_t* flag = nullptr) {
  __syncthreads();
  if (G > 1) {
    if (threadIdx.x == 0) barrier_arrive_wait(ctr, (unsigned)G, true, gen, tgt, tag, flag);
    __syncthreads();
  }
}

// ---- thread-block clusters (the clustered elimination loop)
__device__ __forceinline__ unsigned cluster_size_() {
  unsigned r;
  asm volatile("mov.u32 %0, %%cluster_nctarank;\n" : "=r"(r));
  return r;
}
__device__ __forceinline__ __attribute__((unused)) unsigned cluster_rank_() {
  unsigned r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;\n" : "=r"(r));
  return r;
}
// every thread of every CTA of the cluster; release/acquire at cluster scope
__device__ __forceinline__ void cluster_sync_() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n"
               "barrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}
// shared::cluster load of the word at local shared address a in CTA r; no
// compiler memory clobber (the loads of one exchange overlap; ordering comes
// from the cluster barrier before them and the __syncthreads after)
__device__ __forceinline__ double ld_dsmem_nc(unsigned a, unsigned r) {
  unsigned ra;
  double v;
  asm volatile(
      "mapa.shared::cluster.u32 %1, %2, %3;\n"
      "ld.shared::cluster.f64 %0, [%1];\n"
      : "=d"(v), "=&r"(ra)
      : "r"(a), "r"(r));
  return v;
}
// the clustered loop's step barrier: every CTA's global writes fenced, a
// cluster barrier, then one arrival per cluster on the group counter; all
// CTAs poll the release word
__device__ __forceinline__ void cluster_step_barrier(unsigned* ctr, int NC, bool leader,
                                                     unsigned& gen, unsigned& tgt, int tag,
                                                     int64_t* flag) {
  if (threadIdx.x == 0) __threadfence();
  cluster_sync_();
  if (threadIdx.x == 0) barrier_arrive_wait(ctr, (unsigned)NC, leader, gen, tgt, tag, flag);
  __syncthreads();
}

// block-wide stable compaction of up to kT flagged items per call: item
// `val` of thread tid is kept in category cat (1 or 2; 0 drops it) and
// written to out1 / out2 at base1 / base2 + its rank among the kept items of
// the same category in thread order.  Returns both counts in c1 / c2 (every
// thread).  `wsum` needs 2 * kWarps ints.
__device__ __forceinline__ void stable_split(int cat, int val, int32_t* out1, int base1,
                                             int32_t* out2, int base2, int* wsum, int& c1,
                                             int& c2) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const unsigned b1 = __ballot_sync(0xffffffffu, cat == 1);
  const unsigned b2 = __ballot_sync(0xffffffffu, cat == 2);
  const unsigned lt = (1u << lane) - 1u;
  if (lane == 0) {
    wsum[warp] = __popc(b1);
    wsum[kWarps + warp] = __popc(b2);
  }
  __syncthreads();
  int o1 = 0, o2 = 0, t1 = 0, t2 = 0;
#pragma unroll
  for (int w = 0; w < kWarps; ++w) {
    if (w < warp) {
      o1 += wsum[w];
      o2 += wsum[kWarps + w];
    }
    t1 += wsum[w];
    t2 += wsum[kWarps + w];
  }
  if (cat == 1) out1[base1 + o1 + __popc(b1 & lt)] = val;
  else if (cat == 2) out2[base2 + o2 + __popc(b2 & lt)] = val;
  c1 = t1;
  c2 = t2;
  __syncthreads();
}

// better(a, b): larger value wins, ties -> smaller position
__device__ __forceinline__ bool better(double va, int64_t pa, double vb, int64_t pb) {
  return va > vb || (va == vb && pa < pb);
}

__device__ __forceinline__ void cp_async8(double* smem, const double* gmem, bool pred) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  const int sz = pred ? 8 : 0;
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(sa), "l"(gmem), "r"(sz));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::); }
__device__ __forceinline__ void cp_wait_all() { asm volatile("cp.async.wait_group 0;\n" ::); }
__device__ __forceinline__ void cp_wait_1() { asm volatile("cp.async.wait_group 1;\n" ::); }

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
#ifdef SPAND_DMMA_VOLATILE
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
#else
  // not volatile: the scheduler may hoist the next fragments' loads above it
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
#endif
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

// N (<= 8) block-wide sums at once, fixed order, result in every thread
template <int N>
__device__ __forceinline__ void block_reduce_n(double (&v)[N], Sh& sh) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int q = 0; q < N; ++q) v[q] = warp_sum(v[q]);
  if (lane == 0) {
#pragma unroll
    for (int q = 0; q < N; ++q) sh.red8[warp][q] = v[q];
  }
  __syncthreads();
  if (threadIdx.x < N) {
    double t = 0.0;
#pragma unroll
    for (int w = 0; w < kWarps; ++w) t += sh.red8[w][threadIdx.x];
    sh.tot8[threadIdx.x] = t;
  }
  __syncthreads();
#pragma unroll
  for (int q = 0; q < N; ++q) v[q] = sh.tot8[q];
}

struct ColCtx {
  double* W;
  int m, k, len;
  double tau;
  const double* v;        // reflector (shared memory), rows k..m-1
  double* cur;
  double* ref;
  const int32_t* pos;
  const int32_t* list;    // this step's active columns, interleaved slots
  int rank, G;
  unsigned long long* refresh_ctr;
  int jpos;               // this step's swap: position k now belongs to jpos
  // current position of column c: the owner may not have applied this
  // step's swap yet when another CTA processes c, so apply it here
  __device__ int64_t posof(int c) const {
    const int p = pos[c];
    return p == k ? jpos : p;
  }
};

// Householder update of B active columns at a time by the whole CTA: every
// thread holds E rows of each column in registers (one read, one write per
// step), dot products and tail norms are reduced CTA-wide.  Thread b < B
// then applies the reference's norm downdate / refresh rule (dense.py:
// 168-178) to column b and keeps the best candidate it has seen.
template <int B, int E>
__device__ void colpass_batch(const ColCtx& X, int a0, int nb, Sh& sh, double& bv,
                              int64_t& bp, int& bc) {
  const int tid = threadIdx.x;
  int cs[B];
  double x[B][E];
#pragma unroll
  for (int b = 0; b < B; ++b) cs[b] = b < nb ? X.list[X.rank + X.G * (a0 + b)] : -1;
#pragma unroll
  for (int b = 0; b < B; ++b) {
    const double* col = X.W + (int64_t)(cs[b] < 0 ? 0 : cs[b]) * X.m + X.k;
#pragma unroll
    for (int e = 0; e < E; ++e) {
      const int i = tid + kT * e;
      x[b][e] = (cs[b] >= 0 && i < X.len) ? col[i] : 0.0;
    }
  }
  // running norms of the batch (broadcast loads; only thread b writes them,
  // after the reductions) and row k of each column (thread 0 holds it)
  double cur0[B], ref0[B];
#pragma unroll
  for (int b = 0; b < B; ++b) {
    cur0[b] = cs[b] >= 0 ? X.cur[cs[b]] : 0.0;
    ref0[b] = cs[b] >= 0 ? X.ref[cs[b]] : 0.0;
  }
  // (double-buffered by batch parity: the previous batch may still read its
  // copy when no second reduction separates the batches)
  double* xk = sh.xk[(a0 / B) & 1];
  if (tid == 0) {
#pragma unroll
    for (int b = 0; b < B; ++b) xk[b] = x[b][0];
  }
  double d[B];
#pragma unroll
  for (int b = 0; b < B; ++b) {
    d[b] = 0.0;
#pragma unroll
    for (int e = 0; e < E; ++e) {
      const int i = tid + kT * e;
      if (i < X.len) d[b] += X.v[i] * x[b][e];
    }
  }
  block_reduce_n<B>(d, sh);
  // row-k entry r_k = x_k - tau d v_k in every thread: the norm downdate
  // needs the exact tail only when the refresh rule fires (dense.py:172-178)
  double rkv[B];
  bool need = false;
#pragma unroll
  for (int b = 0; b < B; ++b) {
    rkv[b] = xk[b] - X.tau * d[b] * X.v[0];
    double cn = cur0[b] - rkv[b] * rkv[b];
    if (cn < 0.0) cn = 0.0;
    need |= (b < nb) && (cn < 0.01 * ref0[b]);
  }
  double t[B];
#pragma unroll
  for (int b = 0; b < B; ++b) {
    const double w = X.tau * d[b];
    double* col = X.W + (int64_t)(cs[b] < 0 ? 0 : cs[b]) * X.m + X.k;
    double tail = 0.0;
#pragma unroll
    for (int e = 0; e < E; ++e) {
      const int i = tid + kT * e;
      if (cs[b] >= 0 && i < X.len) {
        const double y = x[b][e] - w * X.v[i];
        col[i] = y;
        if (i != 0) tail += y * y;
      }
    }
    t[b] = tail;
  }
  if (need) block_reduce_n<B>(t, sh);
#pragma unroll
  for (int b = 0; b < B; ++b) {
    if (tid == b && b < nb) {
      const int c = cs[b];
      const double rk = rkv[b], tail = t[b];
      double cn = cur0[b] - rk * rk;
      if (cn < 0.0) cn = 0.0;
      if (cn < 0.01 * ref0[b]) {
        // exact tail norm of the updated column (dense.py:172-178)
        cn = tail;
        X.ref[c] = tail;
        atomicAdd(X.refresh_ctr, 1ull);
      }
      X.cur[c] = cn;
      const int64_t ps = X.posof(c);
      if (better(cn, ps, bv, bp)) {
        bv = cn;
        bp = ps;
        bc = c;
      }
    }
  }
}

// short / medium columns (len <= 32 R): a warp per column, U columns in flight per
// warp, warp reductions only; lane u applies the norm logic of column u and
// keeps its best candidate (reduced per warp afterwards)
template <int U, int R>
__device__ void colpass_warp(const ColCtx& X, int nact, double& bv, int64_t& bp, int& bc) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int a0 = warp * U; a0 < nact; a0 += kWarps * U) {
    int cs[U];
    double x[U][R];
#pragma unroll
    for (int u = 0; u < U; ++u) cs[u] = a0 + u < nact ? X.list[X.rank + X.G * (a0 + u)] : -1;
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const double* col = X.W + (int64_t)(cs[u] < 0 ? 0 : cs[u]) * X.m + X.k;
#pragma unroll
      for (int e = 0; e < R; ++e) {
        const int i = lane + 32 * e;
        x[u][e] = (cs[u] >= 0 && i < X.len) ? col[i] : 0.0;
      }
    }
    double d[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      double a = 0.0;
#pragma unroll
      for (int e = 0; e < R; ++e) {
        const int i = lane + 32 * e;
        if (i < X.len) a += X.v[i] * x[u][e];
      }
      d[u] = warp_sum(a);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const double w = X.tau * d[u];
      double* col = X.W + (int64_t)(cs[u] < 0 ? 0 : cs[u]) * X.m + X.k;
      double tail = 0.0, rk = 0.0;
#pragma unroll
      for (int e = 0; e < R; ++e) {
        const int i = lane + 32 * e;
        if (cs[u] >= 0 && i < X.len) {
          const double y = x[u][e] - w * X.v[i];
          col[i] = y;
          if (i == 0) rk = y;
          else tail += y * y;
        }
      }
      tail = warp_sum(tail);
      rk = __shfl_sync(0xffffffffu, rk, 0);
      if (lane == u && cs[u] >= 0) {
        const int c = cs[u];
        double cn = X.cur[c] - rk * rk;
        if (cn < 0.0) cn = 0.0;
        if (cn < 0.01 * X.ref[c]) {
          cn = tail;
          X.ref[c] = tail;
          atomicAdd(X.refresh_ctr, 1ull);
        }
        X.cur[c] = cn;
        const int64_t ps = X.posof(c);
        if (better(cn, ps, bv, bp)) {
          bv = cn;
          bp = ps;
          bc = c;
        }
      }
    }
  }
}

// columns longer than 16 rows per thread: chunked, the update re-reads
__device__ void colpass_long(const ColCtx& X, int a0, Sh& sh, double& bv, int64_t& bp, int& bc) {
  const int tid = threadIdx.x;
  const int c = X.list[X.rank + X.G * a0];
  double* col = X.W + (int64_t)c * X.m + X.k;
  double d[1] = {0.0};
  for (int i = tid; i < X.len; i += kT) d[0] += X.v[i] * col[i];
  block_reduce_n<1>(d, sh);
  const double w = X.tau * d[0];
  double t[2] = {0.0, 0.0};
  for (int i = tid; i < X.len; i += kT) {
    const double y = col[i] - w * X.v[i];
    col[i] = y;
    if (i == 0) t[1] = y;
    else t[0] += y * y;
  }
  block_reduce_n<2>(t, sh);
  if (tid == 0) {
    double cn = X.cur[c] - t[1] * t[1];
    if (cn < 0.0) cn = 0.0;
    if (cn < 0.01 * X.ref[c]) {
      cn = t[0];
      X.ref[c] = t[0];
      atomicAdd(X.refresh_ctr, 1ull);
    }
    X.cur[c] = cn;
    const int64_t ps = X.posof(c);
    if (better(cn, ps, bv, bp)) {
      bv = cn;
      bp = ps;
      bc = c;
    }
  }
}

template <int B, int E>
__device__ void qform_batched(double* Q, const double* V, const double* taus, int m, int kst,
                              int rank, int G, Sh& sh) {
  const int tid = threadIdx.x;
  for (int u0 = 0; rank + G * u0 < m; u0 += B) {
    int cs[B];
    int cmax = 0;
#pragma unroll
    for (int b = 0; b < B; ++b) {
      const int c = rank + G * (u0 + b);
      cs[b] = c < m ? c : -1;
      if (c < m) cmax = c;
    }
    double x[B][E];
#pragma unroll
    for (int b = 0; b < B; ++b)
#pragma unroll
      for (int e = 0; e < E; ++e) x[b][e] = (tid + kT * e == cs[b]) ? 1.0 : 0.0;
    for (int t = min(kst - 1, cmax); t >= 0; --t) {
      const double tt = __ldcg(taus + t);
      if (tt == 0.0) continue;
      double v[E];
#pragma unroll
      for (int e = 0; e < E; ++e) {
        const int i = tid + kT * e;
        v[e] = (i >= t && i < m) ? __ldcg(V + (int64_t)t * m + i) : 0.0;
      }
      double d[B];
#pragma unroll
      for (int b = 0; b < B; ++b) {
        d[b] = 0.0;
#pragma unroll
        for (int e = 0; e < E; ++e) d[b] += v[e] * x[b][e];
      }
      block_reduce_n<B>(d, sh);
#pragma unroll
      for (int b = 0; b < B; ++b) {
        const double f = tt * d[b];
#pragma unroll
        for (int e = 0; e < E; ++e) x[b][e] -= f * v[e];
      }
    }
#pragma unroll
    for (int b = 0; b < B; ++b) {
      if (cs[b] < 0) continue;
      double* col = Q + (int64_t)cs[b] * m;
#pragma unroll
      for (int e = 0; e < E; ++e) {
        const int i = tid + kT * e;
        if (i < m) col[i] = x[b][e];
      }
    }
  }
}

#ifndef SPAND_CL_MINB1
#define SPAND_CL_MINB1 2
#endif
#ifndef SPAND_MINB_CLASSIC
#define SPAND_MINB_CLASSIC 1
#endif
#define SPAND_CL_MINB (kCl ? SPAND_CL_MINB1 : SPAND_MINB_CLASSIC)
template <bool kCl, int kSch>
__global__ void __launch_bounds__(kT, SPAND_CL_MINB)
rrqr_wave_kernel(int npanel, const int64_t* __restrict__ panels, const int64_t* __restrict__ nbrs,
                 int32_t* __restrict__ m0, int32_t* __restrict__ off, double eps, int scheme_flags,
                 int64_t* __restrict__ events) {
  // scheme_flags: scheme (0 first, 1 second-full, 2 superfine) | 4: keep every
  // fine row of Q^T W in the dead slots (local-error diagnostics,
  // schemes.py:297-306), not only the correction rows
  // the scheme is a template parameter (superfine-only code is compiled out
  // of the other schemes' kernels: fewer registers); scheme_flags & 3 == kSch
  constexpr int scheme = kSch;
  const bool keep_fine = (scheme_flags & 4) != 0;
  extern __shared__ double vsh[];
  __shared__ Sh sh;
  // gather / write-back staging aliases the reflector buffer (disjoint phases)
  double (*tile)[16][33] = reinterpret_cast<double (*)[16][33]>(vsh);
  // ---- locate my panel and rank in its group
  int lo = 0, hi = npanel - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (panels[16 * (int64_t)mid + 7] <= blockIdx.x) lo = mid;
    else hi = mid - 1;
  }
  const int64_t* P = panels + 16 * (int64_t)lo;
  const int G = (int)P[8];
  const int rank = (int)blockIdx.x - (int)P[7];
  if (rank >= G) return;
  const int p = (int)P[0];
  const int nb0 = (int)P[1], nb1 = (int)P[2];
  double* W = reinterpret_cast<double*>(P[3]);
  double* Q = reinterpret_cast<double*>(P[4]);
  double* aux = reinterpret_cast<double*>(P[5]);
  int32_t* iaux = reinterpret_cast<int32_t*>(P[6]);
  unsigned* ctr = reinterpret_cast<unsigned*>(P[9]);
  const int64_t slot = P[10];
  const int64_t ncap = P[11], mcap = P[12];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  unsigned gen = 0, tgt = 0;

  const int offp = off[p];
  const int ldp = m0[p];
  // near-kernel extension (nearkernel.cu): the last nkr live rows hold the
  // near-kernel directions U^T W and stay coarse; only the first m rows are
  // factored.  nkr = 0 (no workspace) is the reference path.
  const int nkr = P[13] ? (int)reinterpret_cast<const double*>(P[13])[0] : 0;
  const int m = ldp - offp - nkr;
  // column layout over neighbours (live columns at kernel start): block
  // prefix scan of the live widths
  constexpr int kMaxNb = 1024;
  const int nnb = nb1 - nb0;
  int n = 0;
  for (int base = 0; base < nnb; base += kT) {
    const int j = base + tid;
    int len = 0;
    if (j < nnb) {
      const int w = (int)nbrs[4 * (int64_t)(nb0 + j)];
      len = m0[w] - off[w];
    }
    int x = len;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) sh.wsum[warp] = x;
    __syncthreads();
    if (warp == 0) {
      int y = lane < kWarps ? sh.wsum[lane] : 0;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int z = __shfl_up_sync(0xffffffffu, y, o);
        if (lane >= o) y += z;
      }
      if (lane < kWarps) sh.wsum[lane] = y;
    }
    __syncthreads();
    if (j < nnb && j < kMaxNb) sh.nb_start[j] = n + (warp ? sh.wsum[warp - 1] : 0) + x - len;
    n += sh.wsum[kWarps - 1];
    __syncthreads();
  }
  if (tid == 0) {
    if (nnb <= kMaxNb) sh.nb_start[nnb] = n;
    sh.nfrz = 0;
    sh.nact = 0;
    sh.ncold = 0;
    sh.coldmax = -1.0;
    sh.fmax = 0ull;
  }
  __syncthreads();

  double* cur = aux;
  double* ref = aux + ncap;
  double* piv = aux + 2 * ncap;
  double* betas = aux + 2 * ncap + mcap;                       // mcap
  double* taus = betas + mcap;                                 // mcap
  double* cand = taus + mcap;                                  // 2 G kCR, by step parity
  double* Gbuf = cand + (int64_t)2 * G * kCR;                  // 32 x 32: V_b^T V_b of the block
  double* V = W + (int64_t)mcap * ncap;                        // m x kmax reflectors
  int32_t* flist = reinterpret_cast<int32_t*>(V + (int64_t)mcap * mcap);  // frozen columns
  int32_t* perm = iaux;
  int32_t* pos = iaux + ncap;
  int32_t* done = iaux + 2 * ncap;   // 0 active, 1 pivoted, 2 frozen
  // superfine only: columns whose coarse rows (R rows < k_c) the first-order
  // run of the same panel -- which stops at k_c -- forms as Q_c^T a (it froze
  // them, or they were cold when it stopped); formed the same way here, so
  // the trailing matrix is bit for bit the same in every scheme
  int32_t* fofl = flist + 24 * ncap;
  // 1: frozen at step 0 of the classic loop, before any reflector touched
  // the column: W still holds the original data (no restore needed)
  int32_t* untouched = flist + 28 * ncap;

  const int c0 = (int)(((int64_t)n * rank) / G), c1 = (int)(((int64_t)n * (rank + 1)) / G);
  const int q0 = (int)(((int64_t)m * rank) / G), q1 = (int)(((int64_t)m * (rank + 1)) / G);
  const int kmax = m < n ? m : n;

  // neighbour of column c: binary search of the column starts (the last
  // neighbour starting at or before c; zero-width neighbours are skipped)
  auto nbr_of = [&](int c, int& j, int& cc) {
    int jj = 0, start = 0;
    if (nnb <= kMaxNb) {
      int lo2 = 0, hi2 = nnb - 1;
      while (lo2 < hi2) {
        const int mid = (lo2 + hi2 + 1) >> 1;
        if (sh.nb_start[mid] <= c) lo2 = mid;
        else hi2 = mid - 1;
      }
      jj = lo2;
      start = sh.nb_start[jj];
    } else {
      int s = 0;
      for (jj = 0; jj < nnb; ++jj) {
        const int w = (int)nbrs[4 * (int64_t)(nb0 + jj)];
        const int len = m0[w] - off[w];
        if (c < s + len) break;
        s += len;
      }
      start = s;
    }
    j = jj;
    cc = c - start;
  };
  // element (i, c) of the ORIGINAL panel lives in the pool block until the
  // final write-back: base + i * stride
  auto pool_col = [&](int c, double*& base, int64_t& stride) {
    int j, cc;
    nbr_of(c, j, cc);
    const int64_t* nr = nbrs + 4 * (int64_t)(nb0 + j);
    const int w = (int)nr[0];
    double* blk = reinterpret_cast<double*>(nr[1]);
    if (nr[2] == 0) {
      base = blk + (int64_t)offp + (int64_t)(off[w] + cc) * ldp;
      stride = 1;
    } else {
      base = blk + (int64_t)(off[w] + cc) + (int64_t)offp * m0[w];
      stride = m0[w];
    }
  };

  // ---- gather my columns of the panel into W (ld = m), 32x32 tiles per warp
  {
    const int ntc = (c1 - c0 + 15) / 16, ntr = (m + 31) / 32;
    for (int tix = warp; tix < ntc * ntr; tix += kWarps) {
      const int tc = c0 + (tix / ntr) * 16, tr = (tix % ntr) * 32;
      for (int q = 0; q < 16; ++q) {
        const int c = tc + q;
        double val = 0.0;
        if (c < c1) {
          int j, cc;
          nbr_of(c, j, cc);
          const int64_t* nr = nbrs + 4 * (int64_t)(nb0 + j);
          const int w = (int)nr[0];
          const double* blk = reinterpret_cast<const double*>(nr[1]);
          const int i = tr + lane;
          if (i < m) {
            if (nr[2] == 0) val = blk[(int64_t)(offp + i) + (int64_t)(off[w] + cc) * ldp];
            else val = blk[(int64_t)(off[w] + cc) + (int64_t)(offp + i) * m0[w]];
          }
        }
        tile[warp][q][lane] = val;
      }
      __syncwarp();
      for (int q = 0; q < 16; ++q) {
        const int c = tc + q, i = tr + lane;
        if (c < c1 && i < m) W[(int64_t)i + (int64_t)c * m] = tile[warp][q][lane];
      }
      __syncwarp();
    }
  }
  __syncthreads();
  // ---- initial norms, positions, local argmax
  double bv = -1.0;
  int64_t bp = 0x7fffffffffffLL;
  int bc = -1;
  for (int c = c0 + warp; c < c1; c += kWarps) {
    const double* col = W + (int64_t)c * m;
    double s = 0.0;
    for (int i = lane; i < m; i += 32) s += col[i] * col[i];
    s = warp_sum(s);
    if (lane == 0) {
      cur[c] = s;
      ref[c] = s;
      pos[c] = c;
      perm[c] = c;   // position -> column (the clustered loop keeps it current)
      done[c] = 0;
      fofl[c] = 0;
      if (!kCl) untouched[c] = 0;   // (the clustered loop's lists may use that region)
      if (better(s, c, bv, bp)) {
        bv = s;
        bp = c;
        bc = c;
      }
    }
  }
  // candidate record: {value, (pos << 32 | col), max norm^2 of my frozen columns}
  auto publish = [&](double v, int64_t ps, int c, int parity) {
    if (lane == 0) {
      sh.bval[warp] = v;
      sh.bpos[warp] = ps;
      sh.bcol[warp] = c;
    }
    __syncthreads();
    if (tid == 0) {
      double vv = sh.bval[0];
      int64_t pp = sh.bpos[0];
      int cc = sh.bcol[0];
      for (int q = 1; q < kWarps; ++q)
        if (better(sh.bval[q], sh.bpos[q], vv, pp)) {
          vv = sh.bval[q];
          pp = sh.bpos[q];
          cc = sh.bcol[q];
        }
      double* rec = cand + (int64_t)(parity * G + rank) * kCR;
      rec[0] = vv;
      reinterpret_cast<int64_t*>(rec)[1] = (pp << 32) | (int64_t)(uint32_t)cc;
      rec[2] = __longlong_as_double((long long)sh.fmax);
      rec[3] = sh.coldmax;
    }
    __syncthreads();
  };
  publish(bv, bp, bc, 0);
  group_barrier(ctr, G, gen, tgt, -1, events + 12 * slot + 9);

  // ---- elimination (unblocked Householder steps on the ACTIVE columns).
  // Inside the loop column c belongs to CTA c % G (interleaved): the
  // columns that stay active longest are those of the most strongly coupled
  // neighbours, which are contiguous, so a contiguous split would leave a
  // few CTAs with all the work.
  // A column whose running norm^2 is below a quarter of (stop_tol r11)^2 can
  // never be a pivot again (running norms only decrease, and within the
  // reference's 0.01 refresh rule they track the exact tail norm to ~1e-11
  // relative): it is FROZEN -- no more per-step work -- and its final column
  // Q^T a is produced at the end by one tensor-core product with Q.
  const double stop_tol = (scheme == 2) ? eps * eps : eps;
  double r11 = 0.0, eta_last = 0.0;
  double thr2 = 0.0;   // 0.25 (stop_tol r11)^2
  double thr2_fo = 0.0;   // the first-order scheme's freeze threshold 0.25 (eps r11)^2
  bool fo_track = scheme == 2;   // until k_c: mirror the first-order freezes
  int k = 0;
#ifdef SPAND_RRQR_PHASES
  long long ph_t[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  long long ph_last = clock64(), nact_sum = 0, hot_sum = 0, hot3_sum = 0;
  if (tid == 0) sh.nhot = sh.nhot3 = 0;
  int ph_cur = 7;
#define PH(x) do { long long _n = clock64(); ph_t[ph_cur] += _n - ph_last; ph_last = _n; ph_cur = (x); } while (0)
  // cold maintenance sub-phases: 0 T build, 1 Y, 2 reduce + Z, 3 X, 4 tails + replay, 5 reclassify, 6 maintenance barrier
  long long cm_t[8] = {0, 0, 0, 0, 0, 0, 0, 0}, cm_last = 0, cm_calls = 0, cm_cols = 0;
#define CM0() do { cm_last = clock64(); } while (0)
#define CM(x) do { long long _n = clock64(); cm_t[(x)] += _n - cm_last; cm_last = _n; } while (0)
#else
#define PH(x) do {} while (0)
#define CM0() do {} while (0)
#define CM(x) do {} while (0)
#endif
  // ---- hot / cold columns.  Only columns whose running norm^2 is within
  // kHotRho of the current pivot value are updated every step (HOT); the
  // others (COLD) cannot be the next pivots and are brought up to date every
  // kBlk steps with the blocked reflectors Q_b^T X = X - V T^T V^T X (two
  // tensor-core products), their running norms replayed step by step with the
  // reference's downdate / refresh rule (exact tail norms are suffix sums of
  // the updated column).  Each step checks that no cold column's (stale,
  // larger) norm reaches the pivot value; if one does, the block ends early
  // and every cold column becomes hot.
  // int lists in the F region (interleaved slots rank + G u; regions 4 ncap
  // apart since rebalanced per-CTA counts may exceed a CTA's own share)
  int32_t* hotA = flist + 4 * ncap;
  int32_t* hotB = flist + 8 * ncap;
  int32_t* coldA = flist + 12 * ncap;
  int32_t* coldB = flist + 16 * ncap;
  int32_t* coldl = coldA;
  auto cold_maint = [&](int ka, int kb) {
    const int nb = kb - ka;
    const int nc = sh.ncold;
    if (nb <= 0 || nc == 0) return;
    double (*TT)[33] = reinterpret_cast<double (*)[33]>(vsh + kCT);
    double (*ZT)[33] = reinterpret_cast<double (*)[33]>(vsh + kCZ);
    double (*RK)[33] = reinterpret_cast<double (*)[33]>(vsh + kCR2);
    double* TAIL = vsh + kCTail;
    CM0();
#ifdef SPAND_RRQR_PHASES
    ++cm_calls;
    cm_cols += nc;
#endif
    // per-warp partials (fixed-order reductions): [warp][16][32] for Y^T,
    // [warp][16] for the tails
    double (*RED)[kSweep][32] = reinterpret_cast<double (*)[kSweep][32]>(vsh + kCScr);
    double (*RED2)[kSweep] = reinterpret_cast<double (*)[kSweep]>(vsh + kCScr);
    // T of Q_b = H_ka ... H_{kb-1} = I - V T V^T (dlarft, forward columnwise)
    // from the Gram columns gathered during the block's steps
    __syncthreads();
    for (int e = tid; e < 32 * 32; e += kT) {
      const int c = e >> 5, q = e & 31;
      ZT[c][q] = (c < q && q < nb) ? __ldcg(Gbuf + c * 32 + q) : 0.0;
    }
    __syncthreads();
    if (warp == 0) {
      for (int jj = 0; jj < nb; ++jj) {
        const double tj = __ldcg(taus + ka + jj);
        double v = 0.0;
        if (lane < jj) {
          for (int c = lane; c < jj; ++c) v += TT[lane][c] * ZT[c][jj];
          v *= -tj;
        }
        __syncwarp();
        if (lane < jj) TT[lane][jj] = v;
        else if (lane == jj) TT[jj][jj] = tj;
        else TT[lane][jj] = 0.0;
        __syncwarp();
      }
    }
    __syncthreads();
    CM(0);
    // rows ka..m-1 split over the 8 warps (4-row aligned chunks): every warp
    // streams its own rows of the cold columns and of V through DMMA
    // fragments straight from L2 -- no block barriers inside the row loops
    const int L = m - ka;
    const int chunk = ((L + 4 * kWarps - 1) / (4 * kWarps)) * 4;
    const int rb = ka + warp * chunk, re = min(m, rb + chunk);
    const int l4 = lane & 3, l8 = lane >> 2;
    for (int ct = 0; ct < nc; ct += kSweep) {
      const int ncl = min(kSweep, nc - ct);
      if (tid < kSweep) sh.fcol[tid] = tid < ncl ? coldl[rank + G * (ct + tid)] : -1;
      __syncthreads();
      // ---- Y^T[c][q] = sum_{i >= ka} X_c[i] V[i, ka + q]: M = columns (2 x 8),
      // N = reflectors (4 x 8), K = rows
      {
        double acc[kMT][4][2];
#pragma unroll
        for (int a = 0; a < kMT; ++a)
#pragma unroll
          for (int b = 0; b < 4; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;
        const double* xa[kMT];
        bool oka[kMT];
#pragma unroll
        for (int mi = 0; mi < kMT; ++mi) {
          const int c = sh.fcol[mi * 8 + l8];
          oka[mi] = c >= 0;
          xa[mi] = W + (int64_t)(c >= 0 ? c : 0) * m;
        }
        // kRowBatch 8-row slabs per iteration, all their loads issued before
        // the first DMMA (same accumulation order).  Measured on C4-L15:
        // 1 slab 871 ms, 2 slabs 872 ms, 4 slabs 944 ms (spills) -- the loop is
        // bound by the 8-sector fragment loads and the DMMA issue rate, not
        // by the latency of one load round trip
        #pragma unroll kRowUnroll
        for (int r = rb; r < re; r += 8 * kRowBatch) {
          double af[2 * kRowBatch][kMT], bf[2 * kRowBatch][4];
#pragma unroll
          for (int s = 0; s < 2 * kRowBatch; ++s) {
            const int i = r + 4 * s + l4;
            const bool okr = i < re;
#pragma unroll
            for (int mi = 0; mi < kMT; ++mi) af[s][mi] = (okr && oka[mi]) ? __ldcg(xa[mi] + i) : 0.0;
#pragma unroll
            for (int ni = 0; ni < 4; ++ni) {
              const int q = ni * 8 + l8;
              bf[s][ni] = (okr && q < nb && i >= ka + q) ? __ldcg(V + (int64_t)(ka + q) * m + i)
                                                         : 0.0;
            }
          }
#pragma unroll
          for (int s = 0; s < 2 * kRowBatch; ++s)
#pragma unroll
            for (int mi = 0; mi < kMT; ++mi)
#pragma unroll
              for (int ni = 0; ni < 4; ++ni)
                dmma(acc[mi][ni][0], acc[mi][ni][1], af[s][mi], bf[s][ni]);
        }
        // C[row = column l8 (+8 mi)][col = reflector 2 l4 + h (+8 ni)]
#pragma unroll
        for (int mi = 0; mi < kMT; ++mi)
#pragma unroll
          for (int ni = 0; ni < 4; ++ni)
#pragma unroll
            for (int h = 0; h < 2; ++h) RED[warp][mi * 8 + l8][ni * 8 + 2 * l4 + h] = acc[mi][ni][h];
      }
      __syncthreads();
      CM(1);
      for (int e = tid; e < kSweep * 32; e += kT) {
        const int c = e >> 5, q = e & 31;
        double s = 0.0;
#pragma unroll
        for (int w2 = 0; w2 < kWarps; ++w2) s += RED[w2][c][q];
        ZT[c][q] = s;
      }
      __syncthreads();
      // ---- Z^T = Y^T T
      double zv[kMT];
#pragma unroll
      for (int u = 0; u < kMT; ++u) {
        const int e = tid + kT * u;
        const int c = e >> 5, q = e & 31;
        double z = 0.0;
        if (c < ncl && q < nb)
          for (int pp = 0; pp <= q; ++pp) z += ZT[c][pp] * TT[pp][q];
        zv[u] = z;
      }
      __syncthreads();
#pragma unroll
      for (int u = 0; u < kMT; ++u) {
        const int e = tid + kT * u;
        ZT[e >> 5][e & 31] = zv[u];
      }
      __syncthreads();
      CM(2);
      // ---- X -= V Z: M = rows (8-row tiles of the warp's chunk), N = columns
      // (2 x 8), K = reflectors; rows ka..kb-1 captured, squares below summed
      {
        double tail[kMT][2] = {};
        double bz[8][kMT];
#pragma unroll
        for (int kq = 0; kq < 8; ++kq)
#pragma unroll
          for (int ni = 0; ni < kMT; ++ni) bz[kq][ni] = ZT[ni * 8 + l8][kq * 4 + l4];
        double* xc[kMT][2];
        bool okc[kMT][2];
#pragma unroll
        for (int ni = 0; ni < kMT; ++ni)
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int c = sh.fcol[ni * 8 + 2 * l4 + h];
            okc[ni][h] = c >= 0;
            xc[ni][h] = W + (int64_t)(c >= 0 ? c : 0) * m;
          }
        const int nkq = (nb + 3) >> 2;
        #pragma unroll kRowUnroll
        for (int r0 = rb; r0 < re; r0 += 8 * kRowBatch) {
          // kRowBatch 8-row slabs: every load first (see the Y loop)
          double af[kRowBatch][8], xo[kRowBatch][kMT][2];
#pragma unroll
          for (int u = 0; u < kRowBatch; ++u) {
            const int i = r0 + 8 * u + l8;   // this lane's A row and C row
#pragma unroll
            for (int kq = 0; kq < 8; ++kq) {
              const int q = kq * 4 + l4;
              af[u][kq] = (kq < nkq && i < re && q < nb && i >= ka + q)
                              ? __ldcg(V + (int64_t)(ka + q) * m + i)
                              : 0.0;
            }
#pragma unroll
            for (int ni = 0; ni < kMT; ++ni)
#pragma unroll
              for (int h = 0; h < 2; ++h)
                xo[u][ni][h] = (i < re && okc[ni][h]) ? xc[ni][h][i] : 0.0;
          }
#pragma unroll
          for (int u = 0; u < kRowBatch; ++u) {
            const int i = r0 + 8 * u + l8;
            double acc[kMT][2] = {};
#pragma unroll
            for (int kq = 0; kq < 8; ++kq)
#pragma unroll
              for (int ni = 0; ni < kMT; ++ni) dmma(acc[ni][0], acc[ni][1], af[u][kq], bz[kq][ni]);
            if (i < re) {
#pragma unroll
              for (int ni = 0; ni < kMT; ++ni)
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                  if (!okc[ni][h]) continue;
                  const double xv = xo[u][ni][h] - acc[ni][h];
                  xc[ni][h][i] = xv;
                  if (i < kb) RK[ni * 8 + 2 * l4 + h][i - ka] = xv;
                  else tail[ni][h] += xv * xv;
                }
            }
          }
        }
        // lanes sharing l4 hold the same columns: reduce over l8
#pragma unroll
        for (int ni = 0; ni < kMT; ++ni)
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            double t = tail[ni][h];
            t += __shfl_xor_sync(0xffffffffu, t, 4);
            t += __shfl_xor_sync(0xffffffffu, t, 8);
            t += __shfl_xor_sync(0xffffffffu, t, 16);
            tail[ni][h] = t;
          }
        __syncthreads();   // RED (aliased by RED2) fully consumed
        CM(3);
        if (l8 == 0) {
#pragma unroll
          for (int ni = 0; ni < kMT; ++ni)
#pragma unroll
            for (int h = 0; h < 2; ++h) RED2[warp][ni * 8 + 2 * l4 + h] = tail[ni][h];
        }
      }
      __syncthreads();
      if (tid < kSweep) {
        double s = 0.0;
#pragma unroll
        for (int w2 = 0; w2 < kWarps; ++w2) s += RED2[w2][tid];
        TAIL[tid] = s;
      }
      __syncthreads();
      // replay the running norms of the block's steps (dense.py:168-178):
      // the exact tail at step t is the suffix norm of the updated column
      if (tid < ncl) {
        const int c = sh.fcol[tid];
        double suf = TAIL[tid];
        for (int t = kb - 1; t >= ka; --t) {
          ZT[tid][t - ka] = suf;
          suf += RK[tid][t - ka] * RK[tid][t - ka];
        }
        double cn = cur[c], rf = ref[c];
        for (int t = ka; t < kb; ++t) {
          const double rk = RK[tid][t - ka];
          double d = cn - rk * rk;
          if (d < 0.0) d = 0.0;
          if (d < 0.01 * rf) {
            d = ZT[tid][t - ka];
            rf = d;
            atomicAdd(reinterpret_cast<unsigned long long*>(events + 12 * slot + 10), 1ull);
          }
          cn = d;
        }
        cur[c] = cn;
        ref[c] = rf;
      }
      __syncthreads();
      CM(4);
    }
  };
  // ---- blocked Q formation (large panels): Q = Q_0 Q_1 ... with
  // Q_b = H_ka ... H_{kb-1} = I - V_b T_b V_b^T over 32-reflector blocks.
  // T_b (dlarft, forward columnwise) is built by CTA b % G from the Gram
  // matrix of V_b and shared through global memory; then every CTA applies
  // the blocks from the last to the first to its own columns
  // X = Q[:, rank + G u] (initially e_c) as X -= V_b (T_b (V_b^T X)), rows
  // split over the warps with DMMA fragments streamed from L2 (same scheme
  // as cold_maint).  Blocks with ka > max(c) leave e_c unchanged.
  auto qform_blocked = [&](int kst) {
    double* Tbuf = V + (int64_t)mcap * mcap + 32 * (ncap + mcap);
    double (*TT)[33] = reinterpret_cast<double (*)[33]>(vsh + kCT);
    double (*ZT)[33] = reinterpret_cast<double (*)[33]>(vsh + kCZ);
    double (*RED)[kSweep][32] = reinterpret_cast<double (*)[kSweep][32]>(vsh + kCScr);
    const int nblk = (kst + 31) / 32;
    const int l4 = lane & 3, l8 = lane >> 2;
    // (1) T of my blocks
    for (int b = rank; b < nblk; b += G) {
      const int ka = 32 * b, nb = min(32, kst - ka);
      // Gram V_b^T V_b over rows ka..m-1: 4 x 4 tiles of 8, rows split over warps
      const int L = m - ka;
      const int chunk = ((L + 4 * kWarps - 1) / (4 * kWarps)) * 4;
      const int rb = ka + warp * chunk, re = min(m, rb + chunk);
      double acc[4][4][2];
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int c = 0; c < 4; ++c) acc[a][c][0] = acc[a][c][1] = 0.0;
      #pragma unroll kRowUnroll
      for (int r = rb; r < re; r += 4) {
        const int i = r + l4;
        double f[4];
#pragma unroll
        for (int t = 0; t < 4; ++t) {
          const int q = t * 8 + l8;
          f[t] = (i < re && q < nb && i >= ka + q) ? __ldcg(V + (int64_t)(ka + q) * m + i) : 0.0;
        }
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
          for (int c = 0; c < 4; ++c) dmma(acc[a][c][0], acc[a][c][1], f[a], f[c]);
      }
      __syncthreads();
      // partials of the 32 x 32 Gram: 4 slots [4][32][32] in the scratch
      // region; warps w and w + 4 share slot w (fixed order)
      double* R2 = vsh + kCScr;
      if (warp < 4) {
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
          for (int c = 0; c < 4; ++c)
#pragma unroll
            for (int h = 0; h < 2; ++h)
              R2[warp * 1024 + (a * 8 + l8) * 32 + c * 8 + 2 * l4 + h] = acc[a][c][h];
      }
      __syncthreads();
      if (warp >= 4) {
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
          for (int c = 0; c < 4; ++c)
#pragma unroll
            for (int h = 0; h < 2; ++h)
              R2[(warp - 4) * 1024 + (a * 8 + l8) * 32 + c * 8 + 2 * l4 + h] += acc[a][c][h];
      }
      __syncthreads();
      for (int e = tid; e < 32 * 32; e += kT) {
        const int c = e >> 5, q = e & 31;
        const double s = (R2[e] + R2[1024 + e]) + (R2[2048 + e] + R2[3072 + e]);
        ZT[c][q] = (c < q && q < nb) ? s : 0.0;
      }
      __syncthreads();
      if (warp == 0) {
        for (int jj = 0; jj < nb; ++jj) {
          const double tj = __ldcg(taus + ka + jj);
          double v = 0.0;
          if (lane < jj) {
            for (int c = lane; c < jj; ++c) v += TT[lane][c] * ZT[c][jj];
            v *= -tj;
          }
          __syncwarp();
          if (lane < jj) TT[lane][jj] = v;
          else if (lane == jj) TT[jj][jj] = tj;
          else TT[lane][jj] = 0.0;
          __syncwarp();
        }
      }
      __syncthreads();
      for (int e = tid; e < 32 * 32; e += kT) {
        const int p = e >> 5, q = e & 31;
        Tbuf[(int64_t)b * 1024 + e] = (p < nb && q < nb) ? TT[p][q] : 0.0;
      }
      __syncthreads();
    }
    // my columns start as e_c
    for (int u = 0; rank + G * u < m; ++u) {
      double* col = Q + (int64_t)(rank + G * u) * m;
      const int c = rank + G * u;
      for (int i = tid; i < m; i += kT) col[i] = (i == c) ? 1.0 : 0.0;
    }
    group_barrier(ctr, G, gen, tgt, 300000, events + 12 * slot + 9);   // every T_b published
    const int nown = (m - rank + G - 1) / G;
    for (int u0 = 0; u0 < nown; u0 += kSweep) {
      const int ncl = min(kSweep, nown - u0);
      const int cmax = rank + G * (u0 + ncl - 1);
      __syncthreads();
      if (tid < kSweep) sh.fcol[tid] = tid < ncl ? rank + G * (u0 + tid) : -1;
      __syncthreads();
      for (int b = min(nblk - 1, cmax / 32); b >= 0; --b) {
        const int ka = 32 * b, nb = min(32, kst - ka);
        for (int e = tid; e < 32 * 32; e += kT) TT[e >> 5][e & 31] = __ldcg(Tbuf + (int64_t)b * 1024 + e);
        const int L = m - ka;
        const int chunk = ((L + 4 * kWarps - 1) / (4 * kWarps)) * 4;
        const int rb = ka + warp * chunk, re = min(m, rb + chunk);
        // Y^T = X^T V_b
        {
          double acc[kMT][4][2];
#pragma unroll
          for (int a = 0; a < kMT; ++a)
#pragma unroll
            for (int c = 0; c < 4; ++c) acc[a][c][0] = acc[a][c][1] = 0.0;
          const double* xa[kMT];
          bool oka[kMT];
#pragma unroll
          for (int mi = 0; mi < kMT; ++mi) {
            const int c = sh.fcol[mi * 8 + l8];
            oka[mi] = c >= 0;
            xa[mi] = Q + (int64_t)(c >= 0 ? c : 0) * m;
          }
          #pragma unroll kRowUnroll
          for (int r = rb; r < re; r += 8 * kRowBatch) {
            double af[2 * kRowBatch][kMT], bf[2 * kRowBatch][4];
#pragma unroll
            for (int s = 0; s < 2 * kRowBatch; ++s) {
              const int i = r + 4 * s + l4;
              const bool okr = i < re;
#pragma unroll
              for (int mi = 0; mi < kMT; ++mi) af[s][mi] = (okr && oka[mi]) ? __ldcg(xa[mi] + i) : 0.0;
#pragma unroll
              for (int ni = 0; ni < 4; ++ni) {
                const int q = ni * 8 + l8;
                bf[s][ni] = (okr && q < nb && i >= ka + q) ? __ldcg(V + (int64_t)(ka + q) * m + i)
                                                           : 0.0;
              }
            }
#pragma unroll
            for (int s = 0; s < 2 * kRowBatch; ++s)
#pragma unroll
              for (int mi = 0; mi < kMT; ++mi)
#pragma unroll
                for (int ni = 0; ni < 4; ++ni)
                  dmma(acc[mi][ni][0], acc[mi][ni][1], af[s][mi], bf[s][ni]);
          }
#pragma unroll
          for (int mi = 0; mi < kMT; ++mi)
#pragma unroll
            for (int ni = 0; ni < 4; ++ni)
#pragma unroll
              for (int h = 0; h < 2; ++h) RED[warp][mi * 8 + l8][ni * 8 + 2 * l4 + h] = acc[mi][ni][h];
        }
        __syncthreads();
        // Z^T[c][q] = sum_{p >= q} Y^T[c][p] T[q][p]  (Z = T Y)
        double zv[kMT];
#pragma unroll
        for (int u = 0; u < kMT; ++u) {
          const int e = tid + kT * u;
          const int c = e >> 5, q = e & 31;
          double z = 0.0;
          if (c < ncl && q < nb)
            for (int p = q; p < nb; ++p) {
              double y = 0.0;
#pragma unroll
              for (int w2 = 0; w2 < kWarps; ++w2) y += RED[w2][c][p];
              z += y * TT[q][p];
            }
          zv[u] = z;
        }
        __syncthreads();
#pragma unroll
        for (int u = 0; u < kMT; ++u) {
          const int e = tid + kT * u;
          ZT[e >> 5][e & 31] = zv[u];
        }
        __syncthreads();
        // X -= V_b Z
        {
          double bz[8][kMT];
#pragma unroll
          for (int kq = 0; kq < 8; ++kq)
#pragma unroll
            for (int ni = 0; ni < kMT; ++ni) bz[kq][ni] = ZT[ni * 8 + l8][kq * 4 + l4];
          double* xc[kMT][2];
          bool okc[kMT][2];
#pragma unroll
          for (int ni = 0; ni < kMT; ++ni)
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              const int c = sh.fcol[ni * 8 + 2 * l4 + h];
              okc[ni][h] = c >= 0;
              xc[ni][h] = Q + (int64_t)(c >= 0 ? c : 0) * m;
            }
          const int nkq = (nb + 3) >> 2;
          #pragma unroll kRowUnroll
          for (int r0 = rb; r0 < re; r0 += 8 * kRowBatch) {
            double af[kRowBatch][8], xo[kRowBatch][kMT][2];
#pragma unroll
            for (int u = 0; u < kRowBatch; ++u) {
              const int i = r0 + 8 * u + l8;
#pragma unroll
              for (int kq = 0; kq < 8; ++kq) {
                const int q = kq * 4 + l4;
                af[u][kq] = (kq < nkq && i < re && q < nb && i >= ka + q)
                                ? __ldcg(V + (int64_t)(ka + q) * m + i)
                                : 0.0;
              }
#pragma unroll
              for (int ni = 0; ni < kMT; ++ni)
#pragma unroll
                for (int h = 0; h < 2; ++h)
                  xo[u][ni][h] = (i < re && okc[ni][h]) ? xc[ni][h][i] : 0.0;
            }
#pragma unroll
            for (int u = 0; u < kRowBatch; ++u) {
              const int i = r0 + 8 * u + l8;
              double acc[kMT][2] = {};
#pragma unroll
              for (int kq = 0; kq < 8; ++kq)
#pragma unroll
                for (int ni = 0; ni < kMT; ++ni) dmma(acc[ni][0], acc[ni][1], af[u][kq], bz[kq][ni]);
              if (i < re) {
#pragma unroll
                for (int ni = 0; ni < kMT; ++ni)
#pragma unroll
                  for (int h = 0; h < 2; ++h)
                    if (okc[ni][h]) xc[ni][h][i] = xo[u][ni][h] - acc[ni][h];
              }
            }
          }
        }
        __syncthreads();
      }
    }
  };
  int k0 = 0, maint = 0, cpar = 0;
  double last_wv = 0.0;
  if constexpr (kCl) {
    const int CS = (int)cluster_size_();
    // ================= clustered elimination loop =================
    // The group is NC = G / CS thread-block clusters of CS CTAs.  Column c
    // belongs to cluster c % NC; within a cluster the ROWS are split: CTA s
    // owns the 32-row chunks q = s (mod CS), so every CTA of the cluster
    // works on all of the cluster's columns, over its own rows.  Per step:
    // one candidate record and one group-counter arrival per cluster; the
    // pivot column's norm and the hot columns' dot products are summed over
    // the cluster through distributed shared memory (fixed rank order), so
    // every CTA of the cluster -- and every cluster, for the pivot
    // quantities -- computes bit-identical values.  The hot columns' state
    // (running norms, position, first-order flag) lives in shared memory,
    // identical copies in the cluster's CTAs; cold columns live in global
    // memory and are brought up to date every kBlk steps by a cp.async-fed
    // DMMA stream over the CTA's rows.  Step 0 keeps every column cold: the
    // first maintenance (k = 1) applies reflector 0 and classifies.
    const int NC = G / CS, cr = rank / CS, s = rank % CS;
    const bool leader = s == 0;
    int64_t* wflag = events + 12 * slot + 9;
    unsigned long long* rctr = reinterpret_cast<unsigned long long*>(events + 12 * slot + 10);
    double* xb = vsh;                    // [2][kXB] my partials (read by the peers)
    double* Sx = xb + 2 * kXB;           // [kXB] the cluster sums
    double* xs = Sx + kXB;               // pivot column on my rows [kXS]
    double* stg = xs + kXS;              // [2 stages][V, X][32][33]
    double (*ZT)[33] = reinterpret_cast<double (*)[33]>(stg + 4 * 32 * 33);
    double (*TT)[33] = reinterpret_cast<double (*)[33]>(stg + 5 * 32 * 33);
    double* hcur = stg + 6 * 32 * 33;    // hot state [kHC] x 6
    double* href = hcur + kHC;
    int* hc = reinterpret_cast<int*>(href + kHC);
    int* hpos = hc + kHC;
    int* hfo = hpos + kHC;
    int* hk = hfo + kHC;
    int xpar = 0;
#ifdef SPAND_RRQR_PHASES
    long long mt_[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    long long mt_last = 0;
#define MT(x) do { long long _n = clock64(); if ((x) > 0) mt_[(x)] += _n - mt_last; mt_last = _n; } while (0)
#else
#define MT(x) do {} while (0)
#endif
    // Sx[0..L) = sum over the cluster's CTAs (rank order) of xb[xpar][0..L)
    auto exchange = [&](int L) {
      cluster_sync_();
      const double* mine = xb + xpar * kXB;
      for (int i = tid; i < L; i += kT) {
        // all remote loads in flight at once, then summed in rank order
        double v[8];
        const unsigned a = (unsigned)__cvta_generic_to_shared(mine + i);
#pragma unroll
        for (int r = 0; r < 8; ++r) v[r] = r < CS ? ld_dsmem_nc(a, (unsigned)r) : 0.0;
        double t = v[0];
#pragma unroll
        for (int r = 1; r < 8; ++r)
          if (r < CS) t += v[r];
        Sx[i] = t;
      }
      __syncthreads();
      xpar ^= 1;
    };
    // per-CTA copies of the cluster's cold list (ping-pong 0 / 1)
    const int lcap = (int)(ncap / NC) + 2;
    int32_t* lbase = P[14] ? reinterpret_cast<int32_t*>(P[14]) : flist + 26 * ncap;
    auto clist = [&](int which) { return lbase + ((int64_t)which * G + rank) * lcap; };
    int csel = 0, nh = 0, ncd = 0;
    // my 32-row chunks intersecting [kk, m): qf, qf + CS, ... (nq of them)
    auto own_rows = [&](int kk, int& qf, int& nq) {
      const int qlo = kk >> 5, qhi = (m - 1) >> 5;
      qf = qlo + (s - qlo % CS + CS) % CS;
      nq = (m > kk && qf <= qhi) ? (qhi - qf) / CS + 1 : 0;
    };
    // candidate of the cluster (identical in its CTAs), the leader writes it
    auto publish_cl = [&](double v, int64_t ps, int c, int parity) {
      if (lane == 0) {
        sh.bval[warp] = v;
        sh.bpos[warp] = ps;
        sh.bcol[warp] = c;
      }
      __syncthreads();
      if (tid == 0 && leader) {
        double vv = sh.bval[0];
        int64_t pp = sh.bpos[0];
        int cc = sh.bcol[0];
        for (int q = 1; q < kWarps; ++q)
          if (better(sh.bval[q], sh.bpos[q], vv, pp)) {
            vv = sh.bval[q];
            pp = sh.bpos[q];
            cc = sh.bcol[q];
          }
        double* rec = cand + (int64_t)(parity * G + cr) * kCR;
        rec[0] = vv;
        reinterpret_cast<int64_t*>(rec)[1] = (pp << 32) | (int64_t)(uint32_t)cc;
        rec[2] = __longlong_as_double((long long)sh.fmax);
        rec[3] = sh.coldmax;
      }
      __syncthreads();
    };
    auto warp_best = [&](double& v, int64_t& ps, int& c) {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const double v2 = __shfl_xor_sync(0xffffffffu, v, o);
        const int64_t p2 = __shfl_xor_sync(0xffffffffu, ps, o);
        const int c2 = __shfl_xor_sync(0xffffffffu, c, o);
        if (better(v2, p2, v, ps)) {
          v = v2;
          ps = p2;
          c = c2;
        }
      }
    };
    // freeze tests (the classic loop's consider()): a cold (global state)
    // column, a hot (shared state) entry
    auto freeze_glob = [&](int c, double cc) -> bool {
      if (fo_track && cc < thr2_fo) fofl[c] = 1;
      return cc < thr2 && (fo_track || scheme != 2 || __ldcg(fofl + c) != 0);
    };
    auto freeze_hot = [&](int u) -> bool {
      const double cc = hcur[u];
      if (fo_track && cc < thr2_fo && !hfo[u]) {
        hfo[u] = 1;
        fofl[hc[u]] = 1;
      }
      return cc < thr2 && (fo_track || scheme != 2 || hfo[u] != 0);
    };
    // ---- cold columns brought up to date with the block's reflectors
    // ka..kb-1 over my rows: Q_b^T X = X - V T^T (V^T X), the row sums
    // completed through the cluster; running norms replayed with the
    // reference's downdate / refresh rule (dense.py:168-178)
    auto cold_maint_cl = [&](int ka, int kb) {
      const int nb = kb - ka;
      const int nc = ncd;
      if (nb <= 0 || nc == 0) return;
      const int32_t* lst = clist(csel);
      int qf, nq;
      own_rows(ka, qf, nq);
      const int l4 = lane & 3, l8 = lane >> 2;
      MT(0);
      // (1) Gram V_b^T V_b over my rows (8-row units split over the warps) -> T
      {
        const int U = 4 * nq;
        const int u0 = (warp * U) / kWarps, u1 = ((warp + 1) * U) / kWarps;
        double acc[4][4][2];
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
          for (int c = 0; c < 4; ++c) acc[a][c][0] = acc[a][c][1] = 0.0;
        for (int u = u0; u < u1; ++u) {
          const int rb = ((qf + CS * (u >> 2)) << 5) + ((u & 3) << 3);
#pragma unroll
          for (int ss = 0; ss < 2; ++ss) {
            const int i = rb + 4 * ss + l4;
            double f[4];
#pragma unroll
            for (int t = 0; t < 4; ++t) {
              const int q = t * 8 + l8;
              f[t] = (i < m && q < nb && i >= ka + q) ? __ldcg(V + (int64_t)(ka + q) * m + i) : 0.0;
            }
#pragma unroll
            for (int a = 0; a < 4; ++a)
#pragma unroll
              for (int c = 0; c < 4; ++c) dmma(acc[a][c][0], acc[a][c][1], f[a], f[c]);
          }
        }
        double* R2 = stg;   // [4][32][32] (the stages are idle here)
        __syncthreads();
        if (warp < 4) {
#pragma unroll
          for (int a = 0; a < 4; ++a)
#pragma unroll
            for (int c = 0; c < 4; ++c)
#pragma unroll
              for (int h = 0; h < 2; ++h)
                R2[warp * 1024 + (a * 8 + l8) * 32 + c * 8 + 2 * l4 + h] = acc[a][c][h];
        }
        __syncthreads();
        if (warp >= 4) {
#pragma unroll
          for (int a = 0; a < 4; ++a)
#pragma unroll
            for (int c = 0; c < 4; ++c)
#pragma unroll
              for (int h = 0; h < 2; ++h)
                R2[(warp - 4) * 1024 + (a * 8 + l8) * 32 + c * 8 + 2 * l4 + h] += acc[a][c][h];
        }
        __syncthreads();
        double* P = xb + xpar * kXB;
        for (int e = tid; e < 1024; e += kT) P[e] = (R2[e] + R2[1024 + e]) + (R2[2048 + e] + R2[3072 + e]);
        MT(1);
        exchange(1024);
        MT(2);
        for (int e = tid; e < 32 * 32; e += kT) {
          const int c = e >> 5, q = e & 31;
          ZT[c][q] = (c < q && q < nb) ? Sx[e] : 0.0;
        }
        __syncthreads();
        if (warp == 0) {
          for (int jj = 0; jj < nb; ++jj) {
            const double tj = __ldcg(taus + ka + jj);
            double v = 0.0;
            if (lane < jj) {
              for (int c = lane; c < jj; ++c) v += TT[lane][c] * ZT[c][jj];
              v *= -tj;
            }
            __syncwarp();
            if (lane < jj) TT[lane][jj] = v;
            else if (lane == jj) TT[jj][jj] = tj;
            else TT[lane][jj] = 0.0;
            __syncwarp();
          }
        }
        __syncthreads();
      }
      // (2) 32-column chunks: Y = X^T V_b, Z = Y T, X -= V_b Z^T, streamed over
      // my 32-row chunks through two cp.async stages of (V_b rows, X rows)
      const int mt = warp & 3, nh2 = warp >> 2;
      auto load_stage = [&](int b, int t) {
        double* Vs = stg + b * 2 * 32 * 33;   // [q][33]
        double* Xs = Vs + 32 * 33;            // [c][33]
        const int r0 = (qf + CS * t) << 5;
#pragma unroll
        for (int it = 0; it < 4; ++it) {
          const int e = tid + it * kT;
          const int q = e >> 5, r = e & 31, i = r0 + r;
          const bool okv = q < nb && i >= ka + q && i < m;
          cp_async8(Vs + q * 33 + r, okv ? V + (int64_t)(ka + q) * m + i : V, okv);
          const int c = sh.fcol[q];
          const bool okx = c >= 0 && i >= ka && i < m;
          cp_async8(Xs + q * 33 + r, okx ? W + (int64_t)c * m + i : W, okx);
        }
        cp_commit();
      };
      for (int ct = 0; ct < nc; ct += 32) {
        const int ncl = min(32, nc - ct);
        __syncthreads();
        if (tid < 32) {
          const int c = tid < ncl ? lst[ct + tid] : -1;
          sh.fcol[tid] = c;
          sh.ccur[tid] = c >= 0 ? __ldcg(cur + c) : 0.0;
          sh.cref[tid] = c >= 0 ? __ldcg(ref + c) : 0.0;
        }
        __syncthreads();
        MT(1);
        // ---- Y^T: warp (mt, nh2) -> columns mt*8.., reflectors nh2*16..
        {
          double acc[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
          if (nq > 0) load_stage(0, 0);
          for (int t = 0; t < nq; ++t) {
            if (t + 1 < nq) {
              load_stage((t + 1) & 1, t + 1);
              cp_wait_1();
            } else {
              cp_wait_all();
            }
            __syncthreads();
            const double* Vs = stg + (t & 1) * 2 * 32 * 33;
            const double* Xs = Vs + 32 * 33;
#pragma unroll
            for (int kq = 0; kq < 8; ++kq) {
              const int r = kq * 4 + l4;
              const double af = Xs[(mt * 8 + l8) * 33 + r];
#pragma unroll
              for (int ni = 0; ni < 2; ++ni)
                dmma(acc[ni][0], acc[ni][1], af, Vs[(nh2 * 16 + ni * 8 + l8) * 33 + r]);
            }
            __syncthreads();
          }
          double* P = xb + xpar * kXB;
#pragma unroll
          for (int ni = 0; ni < 2; ++ni)
#pragma unroll
            for (int h = 0; h < 2; ++h)
              P[(mt * 8 + l8) * 32 + nh2 * 16 + ni * 8 + 2 * l4 + h] = acc[ni][h];
        }
        MT(3);
        exchange(32 * 32);
        MT(2);
        // ---- Z^T = Y^T T
        for (int e = tid; e < 32 * 32; e += kT) {
          const int c = e >> 5, q = e & 31;
          double z = 0.0;
          if (c < ncl && q < nb)
            for (int pp = 0; pp <= q; ++pp) z += Sx[c * 32 + pp] * TT[pp][q];
          ZT[c][q] = z;
        }
        double* P2 = xb + xpar * kXB;
        for (int e = tid; e < 32 * 33; e += kT) P2[e] = 0.0;
        __syncthreads();
        // ---- X -= V_b Z^T: warp -> columns mt*8.. (B = Z^T), row tiles nh2, nh2 + 2 of each chunk
        {
          double bz[8];
#pragma unroll
          for (int kq = 0; kq < 8; ++kq) bz[kq] = ZT[mt * 8 + l8][kq * 4 + l4];
          int cc2[2];
#pragma unroll
          for (int h = 0; h < 2; ++h) cc2[h] = sh.fcol[mt * 8 + 2 * l4 + h];
          double tl[2] = {0.0, 0.0};
          if (nq > 0) load_stage(0, 0);
          for (int t = 0; t < nq; ++t) {
            if (t + 1 < nq) {
              load_stage((t + 1) & 1, t + 1);
              cp_wait_1();
            } else {
              cp_wait_all();
            }
            __syncthreads();
            const double* Vs = stg + (t & 1) * 2 * 32 * 33;
            const double* Xs = Vs + 32 * 33;
            const int r0 = (qf + CS * t) << 5;
#pragma unroll
            for (int uu = 0; uu < 2; ++uu) {
              const int rl = (nh2 + 2 * uu) * 8 + l8;
              double acc2[2] = {0.0, 0.0};
#pragma unroll
              for (int kq = 0; kq < 8; ++kq) dmma(acc2[0], acc2[1], Vs[(kq * 4 + l4) * 33 + rl], bz[kq]);
              const int i = r0 + rl;
              if (i >= ka && i < m) {
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                  const int c = cc2[h];
                  if (c < 0) continue;
                  const int cl = mt * 8 + 2 * l4 + h;
                  const double xv = Xs[cl * 33 + rl] - acc2[h];
                  W[(int64_t)c * m + i] = xv;
                  if (i < kb) P2[cl * 32 + (i - ka)] = xv;
                  else tl[h] += xv * xv;
                }
              }
            }
            __syncthreads();
          }
          // lanes sharing l4 hold the same columns: reduce over l8, then the
          // two row halves (warps w, w + 4) in fixed order
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            double t = tl[h];
            t += __shfl_xor_sync(0xffffffffu, t, 4);
            t += __shfl_xor_sync(0xffffffffu, t, 8);
            t += __shfl_xor_sync(0xffffffffu, t, 16);
            tl[h] = t;
          }
          if (l8 == 0) {
#pragma unroll
            for (int h = 0; h < 2; ++h) Sx[nh2 * 32 + mt * 8 + 2 * l4 + h] = tl[h];
          }
        }
        __syncthreads();
        MT(4);
        if (tid < 32) P2[1024 + tid] = Sx[tid] + Sx[32 + tid];
        exchange(32 * 33);
        MT(2);
        // replay the block's steps (identical in every CTA of the cluster)
        if (tid < ncl) {
          const int c = sh.fcol[tid];
          double suf = Sx[1024 + tid];
          for (int t = kb - 1; t >= ka; --t) {
            ZT[tid][t - ka] = suf;
            const double rk = Sx[tid * 32 + (t - ka)];
            suf += rk * rk;
          }
          double cn = sh.ccur[tid], rf = sh.cref[tid];
          for (int t = ka; t < kb; ++t) {
            const double rk = Sx[tid * 32 + (t - ka)];
            double d = cn - rk * rk;
            if (d < 0.0) d = 0.0;
            if (d < 0.01 * rf) {
              d = ZT[tid][t - ka];
              rf = d;
              if (leader) atomicAdd(rctr, 1ull);
            }
            cn = d;
          }
          cur[c] = cn;
          ref[c] = rf;
        }
        __syncthreads();
        MT(5);
      }
    };
#ifdef SPAND_RRQR_PHASES
    long long cl_hotsteps = 0, cl_rounds = 0, cl_maint = 0, cl_flush = 0, cl_cold = 0;
#endif
    int blk_len = 1;   // step 0 keeps every column cold; the first block is one step
    int flushes = 0;
    while (k < kmax) {
      PH(0);
      if (maint) {
        PH(6);
#ifdef SPAND_RRQR_PHASES
        ++cl_maint;
        cl_flush += maint == 2;
        cl_cold += ncd;
#endif
        cold_maint_cl(k0, k);
        MT(0);
        // ---- reclassify hot (shared) ++ cold (global) -> hot (shared) + cold (global)
        const int32_t* cin = clist(csel);
        int32_t* cout = clist(csel ^ 1);
        const int tot = nh + ncd;
        if (tid == 0) sh.mcl = 0ull;
        __syncthreads();
        for (int u = tid; u < tot; u += kT) {
          double cc;
          bool fz;
          if (u < nh) {
            cc = hcur[u];
            fz = freeze_hot(u);
          } else {
            const int c = cin[u - nh];
            cc = __ldcg(cur + c);
            fz = freeze_glob(c, cc);
          }
          if (!fz) atomicMax(&sh.mcl, (unsigned long long)__double_as_longlong(cc));
        }
        __syncthreads();
        const double mcl = __longlong_as_double((long long)sh.mcl);
        // hot iff within rho of min(last pivot value, the cluster's max):
        // the cluster's largest column is always hot, so no cold column can
        // reach the next pivot value right after a classification
        double tau_hot = hot_rho(m) * (maint == 2 ? mcl : fmin(last_wv, mcl));
        if (tot > kHC) {
          // the hot state holds kHC entries: raise the threshold toward the max
          for (int it = 0; it < 60; ++it) {
            if (tid == 0) sh.nact = 0;
            __syncthreads();
            int cnt = 0;
            for (int u = tid; u < tot; u += kT) {
              const double cc = u < nh ? hcur[u] : __ldcg(cur + cin[u - nh]);
              const bool fz = u < nh ? freeze_hot(u) : freeze_glob(cin[u - nh], cc);
              cnt += (!fz && cc >= tau_hot);
            }
            atomicAdd(&sh.nact, cnt);
            __syncthreads();
            const int tot_hot = sh.nact;
            __syncthreads();
            if (tot_hot <= kHC || tau_hot >= mcl) break;
            tau_hot = fmin(mcl, 0.5 * (tau_hot + mcl));
          }
        }
        if (tid == 0) sh.coldmax = 0.0;
        __syncthreads();
        int nh2 = 0, nc2 = 0;
        for (int b0 = 0; b0 < tot; b0 += kT) {
          const int u = b0 + tid;
          int cat = 0, c = -1, ps = 0, fo = 0;
          double cc = 0.0, rf = 0.0;
          if (u < tot) {
            if (u < nh) {
              c = hc[u];
              cc = hcur[u];
              rf = href[u];
              ps = hpos[u];
              fo = hfo[u];
              cat = freeze_hot(u) ? 0 : (cc >= tau_hot ? 1 : 2);
            } else {
              c = cin[u - nh];
              cc = __ldcg(cur + c);
              cat = freeze_glob(c, cc) ? 0 : (cc >= tau_hot ? 1 : 2);
              if (cat == 1) {
                rf = __ldcg(ref + c);
                ps = __ldcg(pos + c);
                fo = __ldcg(fofl + c);
              }
            }
            if (cat == 0) {
              done[c] = 2;
              atomicMax(&sh.fmax, (unsigned long long)__double_as_longlong(cc));
            }
          }
          // hot ranks first (capped at kHC; the excess stays cold), then cold
          const unsigned b1 = __ballot_sync(0xffffffffu, cat == 1);
          if (lane == 0) sh.wsum2[warp] = __popc(b1);
          __syncthreads();
          int o1 = 0, t1 = 0;
#pragma unroll
          for (int w = 0; w < kWarps; ++w) {
            if (w < warp) o1 += sh.wsum2[w];
            t1 += sh.wsum2[w];
          }
          const int hpos1 = nh2 + o1 + __popc(b1 & ((1u << lane) - 1u));
          if (cat == 1 && hpos1 >= kHC) cat = 2;
          const unsigned b2 = __ballot_sync(0xffffffffu, cat == 2);
          __syncthreads();
          if (lane == 0) sh.wsum2[kWarps + warp] = __popc(b2);
          __syncthreads();
          int o2 = 0, t2 = 0;
#pragma unroll
          for (int w = 0; w < kWarps; ++w) {
            if (w < warp) o2 += sh.wsum2[kWarps + w];
            t2 += sh.wsum2[kWarps + w];
          }
          if (cat == 1) {
            hc[hpos1] = c;
            hcur[hpos1] = cc;
            href[hpos1] = rf;
            hpos[hpos1] = ps;
            hfo[hpos1] = fo;
          } else if (cat == 2) {
            cout[nc2 + o2 + __popc(b2 & ((1u << lane) - 1u))] = c;
            if (u < nh) {   // hot -> cold: its state goes back to global memory
              cur[c] = cc;
              ref[c] = rf;
            }
            atomicMax(reinterpret_cast<unsigned long long*>(&sh.coldmax),
                      (unsigned long long)__double_as_longlong(cc));
          }
          nh2 = min(kHC, nh2 + t1);
          nc2 += t2;
          __syncthreads();
        }
        if (nc2 == 0 && tid == 0) sh.coldmax = -1.0;
        nh = nh2;
        ncd = nc2;
        csel ^= 1;
        k0 = k;
        blk_len = kBlk;
        double bvm = -1.0;
        int64_t bpm = 0x7fffffffffffLL;
        int bcm = -1;
        __syncthreads();
        for (int u = tid; u < nh; u += kT) {
          if (better(hcur[u], hpos[u], bvm, bpm)) {
            bvm = hcur[u];
            bpm = hpos[u];
            bcm = hc[u];
          }
        }
        warp_best(bvm, bpm, bcm);
        __syncthreads();
        publish_cl(bvm, bpm, bcm, cpar ^ 1);
        MT(6);
        cpar ^= 1;
        maint = 0;
        cluster_step_barrier(ctr, NC, leader, gen, tgt, -2, wflag);
        PH(0);
      }
      // ---- winning column over the records (as the classic loop)
      const int nrec = k == 0 ? G : NC;   // the prologue published one record per CTA
      double wv = -1.0, wf = -1.0, wc = -1.0;
      int64_t wp = 0x7fffffffffffLL, wpc = 0;
      int wq = 0x7fffffff;
      const int par = cpar;
      for (int q = tid; q < nrec; q += kT) {
        const double* rec = cand + (int64_t)(par * G + q) * kCR;
        const double v = __ldcg(rec);
        const int64_t pc = __ldcg(reinterpret_cast<const long long*>(rec) + 1);
        const double fm = __ldcg(rec + 2);
        if (fm > wf) wf = fm;
        const double cm = __ldcg(rec + 3);
        if (cm > wc) wc = cm;
        const int64_t ps = pc >> 32;
        if (better(v, ps, wv, wp) || (v == wv && ps == wp && q < wq)) {
          wv = v;
          wp = ps;
          wpc = pc;
          wq = q;
        }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const double v2 = __shfl_xor_sync(0xffffffffu, wv, o);
        const int64_t p2 = __shfl_xor_sync(0xffffffffu, wp, o);
        const int64_t c2 = __shfl_xor_sync(0xffffffffu, wpc, o);
        const int q2 = __shfl_xor_sync(0xffffffffu, wq, o);
        const double f2 = __shfl_xor_sync(0xffffffffu, wf, o);
        if (f2 > wf) wf = f2;
        const double c3 = __shfl_xor_sync(0xffffffffu, wc, o);
        if (c3 > wc) wc = c3;
        if (better(v2, p2, wv, wp) || (v2 == wv && p2 == wp && q2 < wq)) {
          wv = v2;
          wp = p2;
          wpc = c2;
          wq = q2;
        }
      }
      if (lane == 0) {
        sh.bval[warp] = wv;
        sh.bpos[warp] = wp;
        sh.bpc[warp] = wpc;
        sh.bq[warp] = wq;
        sh.bfm[warp] = wf;
        sh.bcm[warp] = wc;
      }
      __syncthreads();
      wv = sh.bval[0];
      wp = sh.bpos[0];
      wpc = sh.bpc[0];
      wq = sh.bq[0];
      wf = sh.bfm[0];
      wc = sh.bcm[0];
      for (int w2 = 1; w2 < kWarps; ++w2) {
        const double v2 = sh.bval[w2];
        const int64_t p2 = sh.bpos[w2];
        const int q2 = sh.bq[w2];
        if (sh.bfm[w2] > wf) wf = sh.bfm[w2];
        if (sh.bcm[w2] > wc) wc = sh.bcm[w2];
        if (better(v2, p2, wv, wp) || (v2 == wv && p2 == wp && q2 < wq)) {
          wv = v2;
          wp = p2;
          wpc = sh.bpc[w2];
          wq = q2;
        }
      }
      __syncthreads();
      if (k > 0 && wc >= 0.0 && wc >= wv) {
        // a cold column's (stale, upper-bound) norm reaches the pivot value
        maint = 2;
        if (++flushes > 4) __trap();   // classification cannot converge (kHC ties)
        continue;
      }
      flushes = 0;
      if (wv < 0.0) {
        eta_last = sqrt(wf > 0.0 ? wf : 0.0);
        break;
      }
      const int jpos = (int)wp;
      const int j = (int)(uint32_t)(wpc & 0xffffffffLL);
      PH(1);
      // ---- my rows of the pivot column (cp.async, zero-filled), x0 owner
      int qf, nq;
      own_rows(k, qf, nq);
      const bool own_k = ((k >> 5) % CS) == s;
      {
        const double* colj = W + (int64_t)j * m;
        for (int e = tid; e < nq * 32; e += kT) {
          const int i = ((qf + CS * (e >> 5)) << 5) + (e & 31);
          const bool ok = i >= k && i < m;
          cp_async8(xs + e, ok ? colj + i : colj, ok);
        }
        cp_commit();
      }
      // the hot entry at position k moves to jpos (reference swap order)
      for (int u = tid; u < nh; u += kT)
        if (hpos[u] == k) hpos[u] = jpos;
      // ---- pivot quantities (identical everywhere): eta, beta, tau
      double eta = 0.0, beta = 0.0, tau = 0.0, v0 = 0.0;
      auto take_eta = [&](double s2, double x0) -> bool {
        eta = sqrt(s2);
        eta_last = eta;
        if (k == 0) {
          r11 = eta;
          if (r11 == 0.0) return true;
          thr2 = 0.25 * (stop_tol * r11) * (stop_tol * r11);
          thr2_fo = 0.25 * (eps * r11) * (eps * r11);
        }
        if (fo_track && eta < eps * r11) {
          // k_c reached: the first-order run stops here and finishes its
          // cold columns as Q^T a (identical decisions in every CTA)
          fo_track = false;
          const int32_t* cl2 = clist(csel);
          for (int u = tid; u < ncd; u += kT) fofl[cl2[u]] = 1;
          __syncthreads();
        }
        if (eta < stop_tol * r11) return true;
        if (eta > 0.0) {
          beta = x0 >= 0.0 ? -eta : eta;
          v0 = x0 - beta;
          tau = 2.0 / (s2 - x0 * x0 + v0 * v0);
        }
        return false;
      };
      // my partial |x|^2 (CTA sum in fixed order) and x0
      auto x_partials = [&]() {
        cp_wait_all();
        __syncthreads();
        double sx = 0.0;
        for (int e = tid; e < nq * 32; e += kT) sx += xs[e] * xs[e];
        sx = warp_sum(sx);
        if (lane == 0) sh.red[warp] = sx;
        __syncthreads();
        if (tid == 0) {
          double t = 0.0;
#pragma unroll
          for (int w2 = 0; w2 < kWarps; ++w2) t += sh.red[w2];
          double* P = xb + xpar * kXB;
          P[0] = t;
          P[1] = own_k ? xs[k & 31] : 0.0;
        }
      };
      // V column k on my rows, position bookkeeping (rank 0 keeps pos /
      // perm current: nobody else reads them inside the loop), pivot data
      auto after_eta = [&]() {
        for (int e = tid; e < nq * 32; e += kT) {
          const int i = ((qf + CS * (e >> 5)) << 5) + (e & 31);
          if (i >= k && i < m) V[(int64_t)k * m + i] = eta > 0.0 ? (i == k ? v0 : xs[e]) : 0.0;
        }
        if (rank == 0 && tid == 0) {
          piv[k] = eta;
          taus[k] = tau;
          betas[k] = beta;
          const int ck = __ldcg(perm + k);   // the column at position k
          pos[ck] = jpos;
          perm[jpos] = ck;
          pos[j] = k;
          perm[k] = j;
          done[j] = 1;
        }
      };
      if (k == 0) {
        // ---- step 0: no hot columns; every other column starts cold (or
        // frozen: the classic loop's consider() at k = 0)
        x_partials();
        exchange(2);
        if (take_eta(Sx[0], Sx[1])) break;
        after_eta();
        int32_t* c0l = clist(csel);
        const int nin = n > cr ? (n - cr + NC - 1) / NC : 0;
        int nc2 = 0;
        if (tid == 0) sh.coldmax = 0.0;
        __syncthreads();
        for (int b0 = 0; b0 < nin; b0 += kT) {
          const int u = b0 + tid;
          int cat = 0, c = -1;
          if (u < nin) {
            c = cr + NC * u;
            if (c != j) {
              const double cc = __ldcg(cur + c);
              if (freeze_glob(c, cc)) {
                done[c] = 2;
                atomicMax(&sh.fmax, (unsigned long long)__double_as_longlong(cc));
              } else {
                cat = 2;
                atomicMax(reinterpret_cast<unsigned long long*>(&sh.coldmax),
                          (unsigned long long)__double_as_longlong(cc));
              }
            }
          }
          int a1, a2;
          stable_split(cat, c, c0l, 0, c0l, nc2, sh.wsum2, a1, a2);
          nc2 += a2;
        }
        if (nc2 == 0 && tid == 0) sh.coldmax = -1.0;
        ncd = nc2;
        nh = 0;
        __syncthreads();
        publish_cl(-1.0, 0x7fffffffffffLL, -1, cpar ^ 1);
        cpar ^= 1;
        last_wv = wv;
        ++k;
        if (k - k0 >= blk_len) maint = 1;
        cluster_step_barrier(ctr, NC, leader, gen, tgt, k, wflag);
        continue;
      }
      double bv1 = -1.0;
      int64_t bp1 = 0x7fffffffffffLL;
      int bc1 = -1;
      bool stop = false, eta_done = false;
      PH(3);
      // one round: UW hot entries per warp, E of my 32-row chunks in registers
      auto hot_round = [&](auto Et, auto Ut, int r0) {
        constexpr int E = decltype(Et)::value, UW = decltype(Ut)::value;
        int us[UW];
        double a[UW][E];
#pragma unroll
        for (int t = 0; t < UW; ++t) {
          const int u = r0 + warp + kWarps * t;
          us[t] = u < nh ? u : -1;
        }
#pragma unroll
        for (int t = 0; t < UW; ++t) {
          const double* col = W + (int64_t)(us[t] >= 0 ? hc[us[t]] : 0) * m;
#pragma unroll
          for (int e = 0; e < E; ++e) {
            const int i = ((qf + CS * e) << 5) + lane;
            a[t][e] = (us[t] >= 0 && e < nq && i >= k && i < m) ? col[i] : 0.0;
          }
        }
        if (!eta_done) x_partials();
        double* P = xb + xpar * kXB;
#pragma unroll
        for (int t = 0; t < UW; ++t) {
          double d = 0.0;
#pragma unroll
          for (int e = 0; e < E; ++e)
            if (e < nq) d += xs[e * 32 + lane] * a[t][e];
          d = warp_sum(d);
          const double akv = __shfl_sync(0xffffffffu, a[t][0], k & 31);
          if (lane == 0) {
            P[2 + 2 * (warp + kWarps * t)] = d;
            P[3 + 2 * (warp + kWarps * t)] = own_k ? akv : 0.0;
          }
        }
        PH(2);
        exchange(2 + 2 * kWarps * UW);
        PH(3);
        if (!eta_done) {
          eta_done = true;
          if (take_eta(Sx[0], Sx[1])) {
            stop = true;
            return;
          }
          after_eta();
          // this step's filter (the classic loop's consider(), after the stop
          // tests): keep flags for every hot entry; frozen ones marked now
          for (int u = tid; u < nh; u += kT) {
            const int c = hc[u];
            bool keep = false;
            if (c != j) {
              if (freeze_hot(u)) {
                done[c] = 2;
                atomicMax(&sh.fmax, (unsigned long long)__double_as_longlong(hcur[u]));
              } else {
                keep = true;
              }
            }
            hk[u] = keep;
          }
          __syncthreads();
        }
        double tl[UW], cn[UW];
        bool need = false;
#pragma unroll
        for (int t = 0; t < UW; ++t) {
          tl[t] = 0.0;
          cn[t] = 0.0;
          if (us[t] < 0 || !hk[us[t]]) continue;
          const int i2 = 2 + 2 * (warp + kWarps * t);
          const double ak = Sx[i2 + 1];
          const double w = tau * (Sx[i2] - beta * ak);
          const double rk = ak - w * v0;
          double* col = W + (int64_t)hc[us[t]] * m;
          double tail = 0.0;
#pragma unroll
          for (int e = 0; e < E; ++e) {
            const int i = ((qf + CS * e) << 5) + lane;
            if (e < nq && i >= k && i < m) {
              const double y = a[t][e] - w * (i == k ? v0 : xs[e * 32 + lane]);
              col[i] = y;
              if (i > k) tail += y * y;
            }
          }
          tl[t] = warp_sum(tail);
          double c2 = hcur[us[t]] - rk * rk;
          if (c2 < 0.0) c2 = 0.0;
          cn[t] = c2;
          need |= c2 < 0.01 * href[us[t]];
        }
        // (identical in every CTA of the cluster)
        if (__syncthreads_or(need)) {
          double* P3 = xb + xpar * kXB;
          if (lane == 0) {
#pragma unroll
            for (int t = 0; t < UW; ++t) P3[warp + kWarps * t] = tl[t];
          }
          exchange(kWarps * UW);
#pragma unroll
          for (int t = 0; t < UW; ++t) tl[t] = Sx[warp + kWarps * t];
        }
#pragma unroll
        for (int t = 0; t < UW; ++t) {
          if (us[t] < 0 || !hk[us[t]]) continue;
          const int u = us[t];
          double c2 = cn[t];
          if (c2 < 0.01 * href[u]) {
            // exact tail norm of the updated column (dense.py:172-178)
            c2 = tl[t];
            if (lane == 0) {
              href[u] = c2;
              if (leader) atomicAdd(rctr, 1ull);
            }
          }
          if (lane == 0) {
            hcur[u] = c2;
            if (better(c2, hpos[u], bv1, bp1)) {
              bv1 = c2;
              bp1 = hpos[u];
              bc1 = hc[u];
            }
          }
        }
      };
      // the round shape must be the same in every CTA of the cluster (one
      // exchange per round): it follows the largest chunk count
      const int nqx = m > k ? ((m - 1) / 32 - k / 32) / CS + 1 : 0;
      for (int r0 = 0; r0 == 0 || r0 < nh;) {
        if (nqx <= 4) {
          hot_round(std::integral_constant<int, 4>{}, std::integral_constant<int, 4>{}, r0);
          r0 += kWarps * 4;
        } else if (nqx <= 8) {
          hot_round(std::integral_constant<int, 8>{}, std::integral_constant<int, 4>{}, r0);
          r0 += kWarps * 4;
        } else {
          hot_round(std::integral_constant<int, kXS / 32>{}, std::integral_constant<int, 2>{}, r0);
          r0 += kWarps * 2;
        }
        if (stop) break;
      }
      if (stop) break;
      PH(4);
#ifdef SPAND_RRQR_PHASES
      cl_hotsteps += nh;
      cl_rounds += (nh + 15) / 16;
#endif
      // compact the hot state in place (stable: kept entries keep their order)
      {
        int nk = 0;
        __syncthreads();
        for (int b0 = 0; b0 < nh; b0 += kT) {
          const int u = b0 + tid;
          const bool keep = u < nh && hk[u];
          int c = 0, ps = 0, fo = 0;
          double cc = 0.0, rf = 0.0;
          if (keep) {
            c = hc[u];
            ps = hpos[u];
            fo = hfo[u];
            cc = hcur[u];
            rf = href[u];
          }
          const unsigned b1 = __ballot_sync(0xffffffffu, keep);
          if (lane == 0) sh.wsum2[warp] = __popc(b1);
          __syncthreads();
          int o1 = 0, t1 = 0;
#pragma unroll
          for (int w = 0; w < kWarps; ++w) {
            if (w < warp) o1 += sh.wsum2[w];
            t1 += sh.wsum2[w];
          }
          if (keep) {
            const int d = nk + o1 + __popc(b1 & ((1u << lane) - 1u));
            hc[d] = c;
            hpos[d] = ps;
            hfo[d] = fo;
            hcur[d] = cc;
            href[d] = rf;
          }
          nk += t1;
          __syncthreads();
        }
        nh = nk;
      }
      warp_best(bv1, bp1, bc1);
      __syncthreads();
      publish_cl(bv1, bp1, bc1, cpar ^ 1);
      cpar ^= 1;
      last_wv = wv;
      ++k;
      if (k - k0 >= blk_len) maint = 1;
      PH(5);
      cluster_step_barrier(ctr, NC, leader, gen, tgt, k, wflag);
    }
#ifdef SPAND_RRQR_PHASES
    if (tid == 0 && m >= SPAND_PHASE_MMIN && (rank == 0 || rank == G / 2))
      printf("[rrqr cl] p %d m %d n %d G %d rank %d k %d hot-col-steps %lld rounds(16) %lld maint %lld flush %lld cold-cols %lld | maint kcyc: gram %lld xch %lld Ypass %lld Zupd %lld replay %lld reclass %lld\n",
             p, m, n, G, rank, k, cl_hotsteps, cl_rounds, cl_maint, cl_flush, cl_cold, mt_[1] / 1000, mt_[2] / 1000, mt_[3] / 1000, mt_[4] / 1000, mt_[5] / 1000, mt_[6] / 1000);
#endif
    const bool k_c_seen_cl = scheme == 2 && !fo_track;
    if (scheme == 2 && ncd > 0 && k_c_seen_cl) cold_maint_cl(k0, k);
    __syncthreads();
    {
      const int32_t* cl2 = clist(csel);
      for (int u = tid; u < ncd; u += kT) {
        const int c = cl2[u];
        if (scheme != 2 || !k_c_seen_cl || __ldcg(fofl + c)) done[c] = 2;
      }
    }
    if (tid == 0) sh.ncold = 0;
    __syncthreads();
  } else {
  while (k < kmax) {
    PH(0);
    if (maint) {
      PH(6);
      // bring the cold columns up to date (reflectors k0..k-1), then either
      // reclassify (block end) or make every column hot (a cold column could
      // have won), and republish this CTA's candidate
      int32_t* hot_in = (k & 1) ? hotA : hotB;
      int32_t* tmpl = flist + 20 * ncap;
      cold_maint(k0, k);
      CM0();
      const int nh = sh.nact, ncd = sh.ncold;
      __syncthreads();
      if (tid == 0) {
        sh.nact = 0;
        sh.ncold = 0;
        sh.coldmax = 0.0;   // bits of a non-negative max (atomicMax below)
      }
      __syncthreads();
      int32_t* cold_out = (coldl == coldA) ? coldB : coldA;
      const double tau_hot = (maint == 2) ? -1.0 : hot_rho(m) * last_wv;
      for (int u = tid; u < nh + ncd; u += kT) {
        const int c = u < nh ? hot_in[rank + G * u] : coldl[rank + G * (u - nh)];
        if (done[c]) continue;
        if (fo_track && cur[c] < thr2_fo) fofl[c] = 1;
        if (cur[c] < thr2 && (fo_track || scheme != 2 || fofl[c])) {
          done[c] = 2;
          atomicMax(&sh.fmax, (unsigned long long)__double_as_longlong(cur[c]));
          continue;
        }
        if (cur[c] >= tau_hot) {
          tmpl[rank + G * atomicAdd(&sh.nact, 1)] = c;
        } else {
          cold_out[rank + G * atomicAdd(&sh.ncold, 1)] = c;
          atomicMax(reinterpret_cast<unsigned long long*>(&sh.coldmax),
                    (unsigned long long)__double_as_longlong(cur[c]));
        }
      }
      __syncthreads();
      if (sh.ncold == 0 && tid == 0) sh.coldmax = -1.0;
      int nh2 = sh.nact;
      // (columns stay with their owner CTA.  Re-dealing hot / cold columns
      // evenly over the group here keeps the pivots bit for bit and shortens
      // the root panel by ~6 %, but its extra barrier and L1-bypassing loads
      // cost the other panels more: 1108 -> 1136 ms over C4-L15, commit
      // 5ae96c5 has it as SPAND_REBALANCE)
      for (int u = tid; u < nh2; u += kT) hot_in[rank + G * u] = tmpl[rank + G * u];
      coldl = cold_out;
      k0 = k;
      maint = 0;
      bv = -1.0;
      bp = 0x7fffffffffffLL;
      bc = -1;
      __syncthreads();
      for (int u = tid; u < nh2; u += kT) {
        const int c = hot_in[rank + G * u];
        const double cv = cur[c];
        const int64_t ps = pos[c];
        if (better(cv, ps, bv, bp)) {
          bv = cv;
          bp = ps;
          bc = c;
        }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const double v2 = __shfl_xor_sync(0xffffffffu, bv, o);
        const int64_t p2 = __shfl_xor_sync(0xffffffffu, bp, o);
        const int c2 = __shfl_xor_sync(0xffffffffu, bc, o);
        if (better(v2, p2, bv, bp)) {
          bv = v2;
          bp = p2;
          bc = c2;
        }
      }
      __syncthreads();
      publish(bv, bp, bc, cpar ^ 1);
      cpar ^= 1;
      CM(5);
      group_barrier(ctr, G, gen, tgt, -2, events + 12 * slot + 9);
      CM(6);
      PH(0);
    }
    // ---- winning column: max value, smallest current position (ties in
    // both: lowest record, as a sequential scan).  Records are scanned in
    // parallel and reduced over the CTA.
    double wv = -1.0, wf = -1.0, wc = -1.0;
    int64_t wp = 0x7fffffffffffLL, wpc = 0;
    int wq = 0x7fffffff;
    const int par = cpar;
    for (int q = tid; q < G; q += kT) {
      const double* rec = cand + (int64_t)(par * G + q) * kCR;
      const double v = __ldcg(rec);
      const int64_t pc = __ldcg(reinterpret_cast<const long long*>(rec) + 1);
      const double fm = __ldcg(rec + 2);
      if (fm > wf) wf = fm;
      const double cm = __ldcg(rec + 3);
      if (cm > wc) wc = cm;
      const int64_t ps = pc >> 32;
      if (better(v, ps, wv, wp) || (v == wv && ps == wp && q < wq)) {
        wv = v;
        wp = ps;
        wpc = pc;
        wq = q;
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double v2 = __shfl_xor_sync(0xffffffffu, wv, o);
      const int64_t p2 = __shfl_xor_sync(0xffffffffu, wp, o);
      const int64_t c2 = __shfl_xor_sync(0xffffffffu, wpc, o);
      const int q2 = __shfl_xor_sync(0xffffffffu, wq, o);
      const double f2 = __shfl_xor_sync(0xffffffffu, wf, o);
      if (f2 > wf) wf = f2;
      const double c3 = __shfl_xor_sync(0xffffffffu, wc, o);
      if (c3 > wc) wc = c3;
      if (better(v2, p2, wv, wp) || (v2 == wv && p2 == wp && q2 < wq)) {
        wv = v2;
        wp = p2;
        wpc = c2;
        wq = q2;
      }
    }
    if (lane == 0) {
      sh.bval[warp] = wv;
      sh.bpos[warp] = wp;
      sh.bpc[warp] = wpc;
      sh.bq[warp] = wq;
      sh.bfm[warp] = wf;
      sh.bcm[warp] = wc;
    }
    __syncthreads();
    wv = sh.bval[0];
    wp = sh.bpos[0];
    wpc = sh.bpc[0];
    wq = sh.bq[0];
    wf = sh.bfm[0];
    wc = sh.bcm[0];
    for (int w2 = 1; w2 < kWarps; ++w2) {
      const double v2 = sh.bval[w2];
      const int64_t p2 = sh.bpos[w2];
      const int q2 = sh.bq[w2];
      if (sh.bfm[w2] > wf) wf = sh.bfm[w2];
      if (sh.bcm[w2] > wc) wc = sh.bcm[w2];
      if (better(v2, p2, wv, wp) || (v2 == wv && p2 == wp && q2 < wq)) {
        wv = v2;
        wp = p2;
        wpc = sh.bpc[w2];
        wq = q2;
      }
    }
    __syncthreads();
    if (wc >= 0.0 && wc >= wv) {
      // a cold column's (upper-bound) norm reaches the pivot value
      maint = 2;
      continue;
    }
    if (wv < 0.0) {
      // every remaining column is frozen: the reference's next pivot is one
      // of them and its eta (< stop_tol r11 / 2) stops the elimination
      eta_last = sqrt(wf > 0.0 ? wf : 0.0);
      break;
    }
    const int jpos = (int)wp;
    const int j = (int)(uint32_t)(wpc & 0xffffffffLL);
    PH(1);
    // pivot column rows k..m-1 (current: every active column is updated
    // in place each step)
    const int len = m - k;
    const double* colj = W + (int64_t)j * m + k;
    double s = 0.0;
    for (int i = tid; i < len; i += kT) {
      const double x = __ldcg(colj + i);
      vsh[i] = x;
      s += x * x;
    }
    const double s2 = block_sum<kT>(s, sh.red);
    const double eta = sqrt(s2);
    eta_last = eta;
    if (k == 0) {
      r11 = eta;
      if (r11 == 0.0) break;
      thr2 = 0.25 * (stop_tol * r11) * (stop_tol * r11);
      thr2_fo = 0.25 * (eps * r11) * (eps * r11);
    }
    if (fo_track && eta < eps * r11) {
      // k_c reached: the first-order run stops here and finishes its cold
      // columns as Q^T a (identical decisions so far in every CTA)
      fo_track = false;
      for (int u = tid; u < sh.ncold; u += kT) fofl[coldl[rank + G * u]] = 1;
      __syncthreads();
    }
    if (eta < stop_tol * r11) break;
    // ---- swap bookkeeping (reference: r[:, [k, j]], perm[[k, j]] ...): the
    // column at position k moves to j's old position; owners update their
    // own columns' positions (no shared permutation array)
    const bool own_j = (j % G) == rank;   // loop ownership is interleaved
    if (own_j && tid == 0) {
      pos[j] = k;
      done[j] = 1;
    }
    if (rank == 0 && tid == 0) piv[k] = eta;
    __syncthreads();
    for (int c = rank + G * tid; c < n; c += G * kT)
      if (c != j && done[c] != 1 && pos[c] == k) pos[c] = jpos;
    PH(2);
    // ---- reflector v = x - beta e1, beta = -sign(x0) eta (dense.py:155-159)
    double beta = 0.0, tau = 0.0;
    if (eta > 0.0) {
      const double x0 = vsh[0];
      beta = x0 >= 0.0 ? -eta : eta;
      // v.v = |x|^2 - x0^2 + (x0 - beta)^2: no second reduction
      const double v0 = x0 - beta;
      tau = 2.0 / (s2 - x0 * x0 + v0 * v0);
      __syncthreads();
      if (tid == 0) vsh[0] = v0;
      __syncthreads();
    } else {
      __syncthreads();
      for (int i = tid; i < len; i += kT) vsh[i] = 0.0;
    }
    __syncthreads();
    if (rank == 0) {
      for (int i = tid; i < len; i += kT) V[(int64_t)k * m + k + i] = vsh[i];
      if (tid == 0) {
        taus[k] = tau;
        betas[k] = beta;
      }
    }
    // ---- Gram column of the block's reflectors for the cold update:
    // G[q][jb] = V[:, k0 + q] . v_k (q < jb), dots q = rank (mod G).  One dot:
    // the whole CTA; several (small groups): a warp per dot, no block barriers
    {
      const int jb = k - k0;
      const int nd = rank < jb ? (jb - 1 - rank) / G + 1 : 0;
      if (nd == 1) {
        const double* vq = V + (int64_t)(k0 + rank) * m + k;
        double d = 0.0;
        for (int i = tid; i < len; i += kT) d += __ldcg(vq + i) * vsh[i];
        d = block_sum<kT>(d, sh.red);
        if (tid == 0) Gbuf[rank * 32 + jb] = d;
      } else if (nd > 1) {
        for (int u = warp; u < nd; u += kWarps) {
          const int q = rank + G * u;
          const double* vq = V + (int64_t)(k0 + q) * m + k;
          double d = 0.0;
          for (int i = lane; i < len; i += 32) d += __ldcg(vq + i) * vsh[i];
          d = warp_sum(d);
          if (lane == 0) Gbuf[q * 32 + jb] = d;
        }
      }
    }
    // ---- owned active columns: a -= tau (v.a) v, row-k entry, norm
    // downdate with the reference's refresh rule (dense.py:160-178), freeze
    PH(3);
    bv = -1.0;
    bp = 0x7fffffffffffLL;
    bc = -1;
    // (a) this step's active columns: filter the previous step's list (the
    // set only shrinks; lists ping-pong between the perm array, written only
    // after the loop, and a spare region); freeze columns below the threshold
    int32_t* list_out = (k & 1) ? hotB : hotA;
    const int32_t* list_in = (k & 1) ? hotA : hotB;
    __syncthreads();
    const int nprev = sh.nact;
    __syncthreads();
    if (tid == 0) sh.nact = 0;
    __syncthreads();
    auto consider = [&](int c) {
      if (c == j || done[c]) return;
      if (fo_track && cur[c] < thr2_fo) fofl[c] = 1;
      // (superfine after k_c: a column the first-order run left active keeps
      // its in-loop coarse rows, so it is never frozen)
      if (cur[c] < thr2 && (fo_track || scheme != 2 || fofl[c])) {
        done[c] = 2;
        if (k == 0) untouched[c] = 1;
        atomicMax(&sh.fmax, (unsigned long long)__double_as_longlong(cur[c]));
      } else {
        list_out[rank + G * atomicAdd(&sh.nact, 1)] = c;
#ifdef SPAND_RRQR_PHASES
        if (cur[c] >= 0.25 * wv) atomicAdd(&sh.nhot, 1);
        if (cur[c] >= 0.09 * wv) atomicAdd(&sh.nhot3, 1);
#endif
      }
    };
    if (k == 0) {
      for (int c = rank + G * tid; c < n; c += G * kT) consider(c);
    } else {
      for (int u = tid; u < nprev; u += kT) consider(list_in[rank + G * u]);
    }
    __syncthreads();
    const int nact = sh.nact;
#ifdef SPAND_RRQR_PHASES
    if (tid == 0) {
      nact_sum += nact;
      hot_sum += sh.nhot;
      hot3_sum += sh.nhot3;
      sh.nhot = sh.nhot3 = 0;
    }
#endif
    // (b) Householder updates: warp per column for short columns, CTA-wide
    // batches for long ones
    {
      ColCtx X{W, m, k, len, tau, vsh, cur, ref, pos, list_out, rank, G,
               reinterpret_cast<unsigned long long*>(events + 12 * slot + 10), jpos};
      if (len <= 256) {
        colpass_warp<4, 8>(X, nact, bv, bp, bc);
      } else if (len <= 512) {
        colpass_warp<2, 16>(X, nact, bv, bp, bc);
      } else if (len <= 1024) {
        colpass_warp<1, 32>(X, nact, bv, bp, bc);
      } else if (len <= 8 * kT) {
        for (int a0 = 0; a0 < nact; a0 += 4)
          colpass_batch<4, 8>(X, a0, min(4, nact - a0), sh, bv, bp, bc);
      } else if (len <= 16 * kT) {
        for (int a0 = 0; a0 < nact; a0 += 2)
          colpass_batch<2, 16>(X, a0, min(2, nact - a0), sh, bv, bp, bc);
      } else {
        for (int a0 = 0; a0 < nact; ++a0) colpass_long(X, a0, sh, bv, bp, bc);
      }
    }
    // candidates live in lanes of every warp: reduce to lane 0
    {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const double v2 = __shfl_xor_sync(0xffffffffu, bv, o);
        const int64_t p2 = __shfl_xor_sync(0xffffffffu, bp, o);
        const int c2 = __shfl_xor_sync(0xffffffffu, bc, o);
        if (better(v2, p2, bv, bp)) {
          bv = v2;
          bp = p2;
          bc = c2;
        }
      }
    }
    __syncthreads();
    PH(4);
    publish(bv, bp, bc, cpar ^ 1);
    cpar ^= 1;
    last_wv = wv;
    ++k;
    // the first block is SPAND_BLK0 steps (every active column is hot until
    // the first classification; C4-L15 swept over 1 / 4 / 8 / 32: 8 best, -2 %)
    if (k - k0 >= (k0 == 0 ? SPAND_BLK0 : kBlk)) maint = 1;
    PH(5);
    group_barrier(ctr, G, gen, tgt, k, events + 12 * slot + 9);
  }
  }   // classic loop
  const int k_stop = k;
  const bool k_c_seen_sf = scheme == 2 && !fo_track;
  // remaining cold columns finish like frozen ones (Q^T a from the original)
  // -- except, in the superfine scheme, those the first-order run kept
  // active up to k_c: they are brought up to date (their rows < k_c are the
  // in-loop values of every scheme) and written back like active columns
  if (scheme == 2 && sh.ncold > 0 && k_c_seen_sf) cold_maint(k0, k);
  __syncthreads();
  for (int u = tid; u < sh.ncold; u += kT) {
    const int c = coldl[rank + G * u];
    if (scheme != 2 || !k_c_seen_sf || fofl[c]) done[c] = 2;
  }
  // frozen list of my own columns (static ownership c % G)
  group_barrier(ctr, G, gen, tgt, -5, events + 12 * slot + 9);
  if (tid == 0) sh.nfrz = 0;
  __syncthreads();
  for (int c = rank + G * tid; c < n; c += G * kT)
    if (__ldcg(done + c) == 2) flist[rank + G * atomicAdd(&sh.nfrz, 1)] = c;
  __syncthreads();
#ifdef SPAND_RRQR_PHASES
  PH(7);
  long long tl = clock64(), tq = 0, trs = 0, tg = 0, twb = 0;
#define TL(var) do { long long _n = clock64(); var += _n - tl; tl = _n; } while (0)
#else
#define TL(var) do {} while (0)
#endif
  // every CTA must be done reading this step's pivot column (the loop may
  // have stopped on it) before owners patch their columns
  group_barrier(ctr, G, gen, tgt, 100000 + k, events + 12 * slot + 9);
  // pivoted columns: R(t, t) = beta, zeros below (dense.py:161-162)
  for (int c = c0 + warp; c < c1; c += kWarps) {
    const int t = pos[c];
    if (done[c] == 1) {
      double* col = W + (int64_t)c * m;
      const double bt = __ldcg(betas + t);
      if (__ldcg(taus + t) != 0.0)
        for (int i = t + lane; i < m; i += 32) col[i] = (i == t) ? bt : 0.0;
      __syncwarp();
    }
    if (lane == 0) perm[t] = c;
  }
  __syncthreads();
  TL(twb);   // (patch: counted with the write-back)
  // ---- Q = H_0 H_1 ... H_{k_stop-1}, accumulated backwards (dorg2r order).
  // Column c of Q is H_0 ... H_{k-1} e_c, and H_t leaves e_c alone for t > c.
  // Columns are interleaved over the group (c = rank + G u) for balance;
  // each CTA keeps 4 columns in registers and streams the reflectors.
#ifndef SPAND_QB_MMIN
#define SPAND_QB_MMIN 64
#endif
  // k_c: first pivot below eps * r11 (dense.py:181-182)
  // (parallel first-index search: a sequential scan of k_stop dependent
  // L2 loads cost ~1.5 ms on the largest panels)
  if (tid == 0) sh.nfrz_tmp = k_stop;
  __syncthreads();
  for (int t = tid; t < k_stop; t += kT)
    if (__ldcg(piv + t) < eps * r11) {
      atomicMin(&sh.nfrz_tmp, t);
      break;
    }
  __syncthreads();
  const int k_c = sh.nfrz_tmp;
  // the formation method depends on k_c, not k_stop, so the coarse columns
  // of Q -- and the coarse rows Q_c^T a below -- are bit for bit the same in
  // every scheme (k_c is scheme-independent; k_stop is not): the trailing
  // matrix is then identical across schemes (test_factorize.py:104-113)
  if (k_c >= 64 && m >= SPAND_QB_MMIN) qform_blocked(k_stop);
  else if (m <= 8 * kT) qform_batched<4, 8>(Q, V, taus, m, k_stop, rank, G, sh);
  else if (m <= 16 * kT) qform_batched<2, 16>(Q, V, taus, m, k_stop, rank, G, sh);
  else {
    for (int64_t e = tid; e < (int64_t)(q1 - q0) * m; e += kT) {
      const int i = (int)(e % m), c = q0 + (int)(e / m);
      Q[(int64_t)i + (int64_t)c * m] = (i == c) ? 1.0 : 0.0;
    }
    for (int t = k_stop - 1; t >= 0; --t) {
      const double tt = __ldcg(taus + t);
      if (tt == 0.0) continue;
      if (q1 <= t) continue;
      const int len = m - t;
      __syncthreads();
      for (int i = tid; i < len; i += kT) vsh[i] = __ldcg(V + (int64_t)t + i + (int64_t)t * m);
      __syncthreads();
      for (int c = max(q0, t) + warp; c < q1; c += kWarps) {
        double* col = Q + (int64_t)c * m + t;
        double d = 0.0;
        for (int i = lane; i < len; i += 32) d += vsh[i] * col[i];
        d = warp_sum(d) * tt;
        for (int i = lane; i < len; i += 32) col[i] -= d * vsh[i];
      }
    }
  }
  __syncthreads();
  TL(tq);
  const int n_fine = m - k_c;
  int n_corr = 0;  // rows of e_tilde kept in the dead slots
  if (scheme == 1 || keep_fine) n_corr = n_fine;
  else if (scheme == 2) n_corr = k_stop - k_c;
  // ---- frozen columns: R rows t < k_c + n_corr of Q^T a (a = original
  // column, restored in W) on the tensor cores (DMMA), written straight to
  // the pool in the write-back slot order: slot = t < k_c ? n_fine + t : t - k_c
  const int nf = sh.nfrz;
  // frozen columns: restore the ORIGINAL data (still in the pool blocks; a
  // column frozen after step 0 was already updated in W) with the coalesced
  // tile gather, for my contiguous column range
  {
    const int ntc = (c1 - c0 + 15) / 16, ntr = (m + 31) / 32;
    for (int tix = warp; tix < ntc * ntr; tix += kWarps) {
      const int tc = c0 + (tix / ntr) * 16, tr = (tix % ntr) * 32;
      bool any = false;
      for (int q = 0; q < 16; ++q)
        any |= (tc + q < c1) && done[tc + q] == 2 && (kCl || !__ldcg(untouched + tc + q));
      if (!any) continue;
      for (int q = 0; q < 16; ++q) {
        const int c = tc + q;
        double val = 0.0;
        if (c < c1 && done[c] == 2 && (kCl || !__ldcg(untouched + c))) {
          int j, cc;
          nbr_of(c, j, cc);
          const int64_t* nr = nbrs + 4 * (int64_t)(nb0 + j);
          const int w = (int)nr[0];
          const double* blk = reinterpret_cast<const double*>(nr[1]);
          const int i = tr + lane;
          if (i < m) {
            if (nr[2] == 0) val = blk[(int64_t)(offp + i) + (int64_t)(off[w] + cc) * ldp];
            else val = blk[(int64_t)(off[w] + cc) + (int64_t)(offp + i) * m0[w]];
          }
        }
        tile[warp][q][lane] = val;
      }
      __syncwarp();
      for (int q = 0; q < 16; ++q) {
        const int c = tc + q, i = tr + lane;
        if (c < c1 && i < m && done[c] == 2 && (kCl || !__ldcg(untouched + c)))
          W[(int64_t)i + (int64_t)c * m] = tile[warp][q][lane];
      }
      __syncwarp();
    }
  }
  // frozen-column counts of every CTA (the candidate records are free now:
  // nobody reads them after the loop's last barrier)
  int32_t* fcnt_g = reinterpret_cast<int32_t*>(cand);
  if (tid == 0) fcnt_g[rank] = nf;
  group_barrier(ctr, G, gen, tgt, 200000, events + 12 * slot + 9);   // Q and W complete
  const bool deal = G <= kMaxG;
  if (deal) {
    for (int r = tid; r < G; r += kT) sh.fpre[r + 1] = __ldcg(fcnt_g + r);
    __syncthreads();
    if (tid == 0) {
      sh.fpre[0] = 0;
      for (int r = 0; r < G; ++r) sh.fpre[r + 1] += sh.fpre[r];
    }
    __syncthreads();
  }
  TL(trs);
  // R rows t < T of Q^T a for a list of columns (a = ORIGINAL column) on
  // the tensor cores (DMMA).  to_w = false: frozen columns, a restored in W,
  // rows written straight to the pool in the write-back slot order (slot =
  // t < k_c ? n_fine + t : t - k_c).  to_w = true: a read from the pool (not
  // yet written back), rows written into W (replacing the in-loop values).
  // Element (t, c) accumulates over the rows in the same order in both
  // modes, whatever T and the column's tile.
  //
  // dealt = true (frozen columns): the group's frozen lists are taken as one
  // list (rank-major) cut into 128-column tiles, and the (column tile, row
  // tile) items are dealt round-robin over the whole group.  Every CTA gets
  // the same number of items (+-1) whatever its own frozen count, and the
  // group works on ~G / (T / 64) column tiles at a time, so their columns
  // (3 MB each for the root panel) stay in L2 while Q is swept: with per-CTA
  // lists the G column tiles in flight (470 MB) missed L2 on every sweep.
  auto qt_a = [&](const int32_t* lst, const int cnt, const int T, const bool to_w,
                  const bool dealt) {
    // CTA tile 64 rows (of Q^T) x 128 columns, warp tile 32 x 32 (16 DMMAs
    // per k-step: one CTA per SM, 255 registers); two cp.async stages of A
    // (Q^T rows) and B (original columns).  The K order per element is that
    // of the previous 64 x 64 tiling (bit-identical results).
    constexpr int kLB = 132;
    double (*As)[kFK][kLDS] = reinterpret_cast<double (*)[kFK][kLDS]>(vsh);                 // [kFS][kFK][kLDS]
    double (*Bs)[kFK][kLB] = reinterpret_cast<double (*)[kFK][kLB]>(vsh + kFS * kFK * kLDS);  // [kFS][kFK][kLB]
    double (*Cs)[65] = reinterpret_cast<double (*)[65]>(vsh);                  // [128][65] (epilogue)
    const int wm = warp >> 2, wn = warp & 3;
    const int total = dealt ? sh.fpre[G] : cnt;
    const int nrt = (T + 63) / 64;
    const int64_t nitem = (int64_t)((total + 127) / 128) * nrt;
    int loaded = -1;
    for (int64_t it = dealt ? rank : 0; it < nitem; it += dealt ? G : 1) {
      const int cti = (int)(it / nrt);
      const int ct = cti * 128, rt = (int)(it % nrt) * 64;
      if (cti != loaded) {
        loaded = cti;
        __syncthreads();
        if (tid < 128) {
          if (ct + tid < total) {
            double* base;
            int64_t stride;
            int c;
            if (dealt) {
              // owner of the tile's column: last r with fpre[r] <= index
              const int g = ct + tid;
              int lo2 = 0, hi2 = G - 1;
              while (lo2 < hi2) {
                const int mid = (lo2 + hi2 + 1) >> 1;
                if (sh.fpre[mid] <= g) lo2 = mid;
                else hi2 = mid - 1;
              }
              c = __ldcg(lst + lo2 + (int64_t)G * (g - sh.fpre[lo2]));
            } else {
              c = lst[rank + G * (ct + tid)];
            }
            pool_col(c, base, stride);
            sh.cbase[tid] = base;
            sh.cstride[tid] = stride;
            sh.fcol[tid] = c;
          } else {
            sh.fcol[tid] = -1;
          }
        }
        __syncthreads();
      }
      {
        double acc[4][4][2];
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
          for (int b = 0; b < 4; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;
        // one eighth of a stage's copies (1 of the 8 A and 2 of the 16 B copies
        // of each thread): the next stage is issued in pieces between the
        // k-steps of the current one, so the tensor pipe does not idle behind
        // a block of address arithmetic at every stage boundary
        static_assert((kFK * 64) / kT == 8 && (kFK * 128) / kT == 16 && kFK / 4 == 8,
                      "stage copies split over the 8 k-steps");
        auto load_part = [&](int st, int i0, int part) {
          {
            const int e = tid + part * kT;
            const int kk = e % kFK, cl = e / kFK;
            const int i = i0 + kk;
            const bool oka = i < m && rt + cl < T;
            cp_async8(&As[st][kk][cl], oka ? Q + (int64_t)i + (int64_t)(rt + cl) * m : Q, oka);
          }
#pragma unroll
          for (int r = 2 * part; r < 2 * part + 2; ++r) {
            const int e = tid + r * kT;
            const int kk = e % kFK, cl = e / kFK;
            const int i = i0 + kk;
            const int fc = sh.fcol[cl];
            const bool okb = i < m && fc >= 0;
            const double* bsrc =
                !okb ? W : (to_w ? sh.cbase[cl] + (int64_t)i * sh.cstride[cl]
                                 : W + (int64_t)i + (int64_t)fc * m);
            cp_async8(&Bs[st][kk][cl], bsrc, okb);
          }
        };
        auto load_stage = [&](int st, int i0) {
#pragma unroll
          for (int part = 0; part < 8; ++part) load_part(st, i0, part);
          cp_commit();
        };
        __syncthreads();
        // kFS-stage pipeline: stages s + 1 .. s + kFS - 1 in flight while s computes
        const int nstep = (m + kFK - 1) / kFK;
#pragma unroll
        for (int q = 0; q < kFS - 1; ++q) {
          if (q < nstep) load_stage(q, q * kFK);
          else cp_commit();
        }
        for (int s2 = 0; s2 < nstep; ++s2) {
          asm volatile("cp.async.wait_group %0;\n" ::"n"(kFS - 2));
          __syncthreads();
          const int nx = s2 + kFS - 1;
          const bool more = nx < nstep;
          const int st = s2 % kFS;
#pragma unroll
          for (int kq = 0; kq < kFK / 4; ++kq) {
            if (more) load_part(nx % kFS, nx * kFK, kq);
            if (kq == kFK / 4 - 1) cp_commit();
            const int kr = kq * 4 + (lane & 3);
            double af[4], bf[4];
#pragma unroll
            for (int mi = 0; mi < 4; ++mi) af[mi] = As[st][kr][wm * 32 + mi * 8 + (lane >> 2)];
#pragma unroll
            for (int ni = 0; ni < 4; ++ni) bf[ni] = Bs[st][kr][wn * 32 + ni * 8 + (lane >> 2)];
#pragma unroll
            for (int mi = 0; mi < 4; ++mi)
#pragma unroll
              for (int ni = 0; ni < 4; ++ni) dmma(acc[mi][ni][0], acc[mi][ni][1], af[mi], bf[ni]);
          }
        }
        cp_wait_all();
        __syncthreads();
#pragma unroll
        for (int mi = 0; mi < 4; ++mi)
#pragma unroll
          for (int ni = 0; ni < 4; ++ni)
#pragma unroll
            for (int h = 0; h < 2; ++h)
              Cs[wn * 32 + ni * 8 + (lane & 3) * 2 + h][wm * 32 + mi * 8 + (lane >> 2)] =
                  acc[mi][ni][h];
        __syncthreads();
        for (int e = tid; e < 64 * 128; e += kT) {
          const int r = e & 63, cl = e >> 6;
          const int t = rt + r;
          if (t < T && ct + cl < total) {
            if (to_w) {
              W[(int64_t)t + (int64_t)sh.fcol[cl] * m] = Cs[cl][r];
            } else {
              const int sl = t < k_c ? n_fine + t : t - k_c;
              sh.cbase[cl][(int64_t)sl * sh.cstride[cl]] = Cs[cl][r];
            }
          }
        }
      }
    }
  };
  if (deal) {
    if (sh.fpre[G] > 0) qt_a(flist, 0, k_c + n_corr, false, true);
  } else if (nf > 0) {
    qt_a(flist, nf, k_c + n_corr, false, false);
  }
  // superfine: the columns the first-order run would have formed as Q^T a
  // (fofl) but that stayed active here get their R rows < k_c the same way,
  // from the original column (rows >= k_c keep their in-loop values)
  if (scheme == 2) {
    int32_t* l2 = flist + 4 * ncap;   // the loop's hot lists are free now
    if (tid == 0) sh.nact = 0;
    __syncthreads();
    for (int c = rank + G * tid; c < n; c += G * kT)
      if (__ldcg(fofl + c) && __ldcg(done + c) != 2) l2[rank + G * atomicAdd(&sh.nact, 1)] = c;
    __syncthreads();
    const int n2 = sh.nact;
    if (n2 > 0 && k_c > 0) qt_a(l2, n2, k_c, true, false);
    // the write-back below covers contiguous column ranges, the product
    // above the interleaved ownership
    group_barrier(ctr, G, gen, tgt, 300000, events + 12 * slot + 9);
  }
  TL(tg);
  // ---- write back (non-frozen columns): new slot s < n_fine <- R row
  //      k_c + s (only s < n_corr are read later); slot n_fine + t <- R row t
  __syncthreads();
  {
    const int ntc = (c1 - c0 + 15) / 16, ntr = (m + 31) / 32;
    for (int tix = warp; tix < ntc * ntr; tix += kWarps) {
      const int tc = c0 + (tix / ntr) * 16, tr = (tix % ntr) * 32;
      for (int q = 0; q < 16; ++q) {
        const int c = tc + q, sl = tr + lane;
        double val = 0.0;
        if (c < c1 && sl < m) {
          const int row = sl < n_fine ? k_c + sl : sl - n_fine;
          val = W[(int64_t)row + (int64_t)c * m];
        }
        tile[warp][q][lane] = val;
      }
      __syncwarp();
      for (int q = 0; q < 16; ++q) {
        const int c = tc + q;
        if (c >= c1 || done[c] == 2) continue;
        int j, cc;
        nbr_of(c, j, cc);
        const int64_t* nr = nbrs + 4 * (int64_t)(nb0 + j);
        const int w = (int)nr[0];
        double* blk = reinterpret_cast<double*>(nr[1]);
        const int sl = tr + lane;
        if (sl < m && (sl >= n_fine || sl < n_corr)) {
          if (nr[2] == 0) blk[(int64_t)(offp + sl) + (int64_t)(off[w] + cc) * ldp] = tile[warp][q][lane];
          else blk[(int64_t)(off[w] + cc) + (int64_t)(offp + sl) * m0[w]] = tile[warp][q][lane];
        }
      }
      __syncwarp();
    }
  }
  if (tid == 0 && nf > 0)
    atomicAdd(reinterpret_cast<unsigned long long*>(events + 12 * slot + 11), (unsigned long long)nf);
  TL(twb);
#ifdef SPAND_RRQR_PHASES
  if (lane == 0 && warp == 0 && m >= SPAND_PHASE_MMIN && (rank == 0 || rank == G / 2))
    printf("[rrqr maint] p %d m %d rank %d calls %lld cols %lld | kcycles: T %lld Y %lld Z %lld X %lld replay %lld reclass %lld barrier %lld\n",
           p, m, rank, cm_calls, cm_cols, cm_t[0] / 1000, cm_t[1] / 1000, cm_t[2] / 1000, cm_t[3] / 1000,
           cm_t[4] / 1000, cm_t[5] / 1000, cm_t[6] / 1000);
  if (lane == 0 && warp == 0 && m >= SPAND_PHASE_MMIN && (rank == 0 || rank == G / 2))
    printf("[rrqr phases] p %d m %d n %d G %d rank %d k %d nf %d act-steps %lld hot %lld hot3 %lld | kcycles: cand %lld maint %lld pivcol %lld refl %lld colpass %lld publish %lld barrier %lld | Q %lld restore %lld frozen-gemm %lld writeback %lld\n",
           p, m, n, G, rank, k_stop, nf, nact_sum, hot_sum, hot3_sum, ph_t[0] / 1000, ph_t[6] / 1000, ph_t[1] / 1000, ph_t[2] / 1000,
           ph_t[3] / 1000, ph_t[4] / 1000, ph_t[5] / 1000, tq / 1000, trs / 1000, tg / 1000,
           twb / 1000);
#endif
  if (rank == 0 && tid == 0) {
    int64_t* ev = events + 12 * slot;
    ev[0] = p;
    ev[1] = m + nkr;
    ev[2] = n;
    ev[3] = k_stop + nkr;
    ev[4] = k_c + nkr;
    ev[5] = (scheme == 2) ? k_stop - k_c : 0;
    ev[6] = n_fine;
    ev[7] = __double_as_longlong(eta_last);
    ev[8] = __double_as_longlong(r11);
  }
  // every CTA of the group must finish reading off[p] before it moves
  group_barrier(ctr, G, gen, tgt, -1, events + 12 * slot + 9);
  if (rank == 0 && tid == 0) off[p] = offp + n_fine;
}
}  // namespace

extern "C" {

int spand_rrqr_cta_count(void) {
  int dev = 0, sms = 0, per = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return -1;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  // capacity for panels up to 4224 rows (the tile staging size); taller
  // panels need more shared memory and are launched with smaller groups
  const size_t smem = kLaunchSmem;
  cudaFuncSetAttribute(rrqr_wave_kernel<false, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)(kMaxM * sizeof(double) > kColdSmem ? kMaxM * sizeof(double) : kColdSmem));
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, rrqr_wave_kernel<false, 1>, kT, smem) != cudaSuccess)
    return -1;
  return per * sms;
}

int spand_rrqr_capacity(int vmax) {
  // the occupancy only depends on the dynamic shared memory size; cache it
  // per (device, size) -- the planner asks once per sparsification wave
  static int cached_dev = -1, cached_per = -1;
  static size_t cached_smem = 0;
  int dev = 0, sms = 0, per = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return -1;
  {
    size_t smem0 = kLaunchSmem;
    if ((size_t)vmax * sizeof(double) > smem0) smem0 = (size_t)vmax * sizeof(double);
    if (dev == cached_dev && smem0 == cached_smem && cached_per > 0) {
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
      return cached_per * sms;
    }
  }
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  size_t smem = kLaunchSmem;
  if ((size_t)vmax * sizeof(double) > smem) smem = (size_t)vmax * sizeof(double);
  cudaFuncSetAttribute(rrqr_wave_kernel<false, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)(kMaxM * sizeof(double) > kColdSmem ? kMaxM * sizeof(double) : kColdSmem));
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, rrqr_wave_kernel<false, 1>, kT, smem) != cudaSuccess)
    return -1;
  cached_dev = dev;
  cached_smem = smem;
  cached_per = per;
  return per * sms;
}

int spand_rrqr_wave(int npanel, int grid, int vmax, const int64_t* panels, const int64_t* nbrs,
                    int32_t* m0, int32_t* off, double eps, int scheme, int64_t* events,
                    void* stream) {
  if (npanel < 0 || grid < 0 || vmax < 0 || vmax > kMaxM) return -1;
  if (npanel == 0 || grid == 0) return 0;
  const size_t tile_bytes = kLaunchSmem;
  size_t smem = (size_t)(vmax > 0 ? vmax : 1) * sizeof(double);
  if (smem < tile_bytes) smem = tile_bytes;
  cudaError_t e = cudaFuncSetAttribute(
      rrqr_wave_kernel<false, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
      (int)(kMaxM * sizeof(double) > kColdSmem ? kMaxM * sizeof(double) : kColdSmem));
  if (e != cudaSuccess) return (int)e;
  void* args[] = {&npanel, &panels, &nbrs, &m0, &off, &eps, &scheme, &events};
  const int sch = scheme & 3;
  void* fn = sch == 0 ? (void*)rrqr_wave_kernel<false, 0>
                      : (sch == 1 ? (void*)rrqr_wave_kernel<false, 1> : (void*)rrqr_wave_kernel<false, 2>);
  e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)(kMaxM * sizeof(double) > kColdSmem ? kMaxM * sizeof(double) : kColdSmem));
  if (e != cudaSuccess) return (int)e;
  e = cudaLaunchCooperativeKernel(fn, dim3(grid), dim3(kT), args, smem, (cudaStream_t)stream);
  if (e != cudaSuccess) return (int)e;
  return 0;
}

// Clustered variant (one launch per wave of large panels): thread-block
// clusters of cs CTAs; every panel's group is a multiple of cs CTAs starting
// at a multiple of cs.  The elimination loop then splits each cluster's
// columns by rows over its CTAs (see the kernel).  Co-residency of the
// whole grid is guaranteed by the cooperative attribute.
static cudaLaunchConfig_t cluster_cfg(int grid, int cs, size_t smem, cudaStream_t st,
                                      cudaLaunchAttribute* at) {
  cudaLaunchConfig_t cfg = {};
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = (unsigned)cs;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  at[1].id = cudaLaunchAttributeCooperative;
  at[1].val.cooperative = 1;
  cfg.gridDim = dim3((unsigned)grid);
  cfg.blockDim = dim3(kT);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cfg.attrs = at;
  cfg.numAttrs = 2;
  return cfg;
}

int spand_rrqr_cluster_capacity(int vmax, int cs) {
  if (cs < 2 || cs > 8 || (cs & (cs - 1))) return -1;
  size_t smem = kClLaunchSmem;
  if ((size_t)vmax * sizeof(double) > smem) smem = (size_t)vmax * sizeof(double);
  if (cudaFuncSetAttribute(rrqr_wave_kernel<true, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)(kMaxM * sizeof(double) > kColdSmem ? kMaxM * sizeof(double)
                                                                    : kColdSmem)) != cudaSuccess)
    return -1;
  cudaLaunchAttribute at[2];
  cudaLaunchConfig_t cfg = cluster_cfg(cs * 8, cs, smem, 0, at);
  int ncl = 0;
  if (cudaOccupancyMaxActiveClusters(&ncl, (void*)rrqr_wave_kernel<true, 1>, &cfg) != cudaSuccess) return -1;
  return ncl * cs;
}

int spand_rrqr_max_rows_clustered(int cs) { return kXS * cs; }

int spand_rrqr_wave_clustered(int npanel, int grid, int vmax, int cs, const int64_t* panels,
                              const int64_t* nbrs, int32_t* m0, int32_t* off, double eps,
                              int scheme, int64_t* events, void* stream) {
  if (npanel < 0 || grid < 0 || vmax < 0 || vmax > kXS * cs) return -1;
  if (cs < 2 || cs > 8 || (cs & (cs - 1)) || grid % cs) return -1;
  if (npanel == 0 || grid == 0) return 0;
  size_t smem = (size_t)(vmax > 0 ? vmax : 1) * sizeof(double);
  if (smem < kClLaunchSmem) smem = kClLaunchSmem;
  cudaError_t e = cudaFuncSetAttribute(
      rrqr_wave_kernel<true, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
      (int)(kMaxM * sizeof(double) > kColdSmem ? kMaxM * sizeof(double) : kColdSmem));
  if (e != cudaSuccess) return (int)e;
  cudaLaunchAttribute at[2];
  cudaLaunchConfig_t cfg = cluster_cfg(grid, cs, smem, (cudaStream_t)stream, at);
  const int sch = scheme & 3;
  auto fn = sch == 0 ? rrqr_wave_kernel<true, 0> : (sch == 1 ? rrqr_wave_kernel<true, 1> : rrqr_wave_kernel<true, 2>);
  e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)(kMaxM * sizeof(double) > kColdSmem ? kMaxM * sizeof(double) : kColdSmem));
  if (e != cudaSuccess) return (int)e;
  e = cudaLaunchKernelEx(&cfg, fn, npanel, panels, nbrs, m0, off, eps, scheme, events);
  if (e != cudaSuccess) return (int)e;
  return 0;
}

}  // extern "C"
