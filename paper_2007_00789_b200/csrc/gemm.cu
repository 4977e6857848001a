// Grouped FP64 GEMM on the DMMA tensor pipe (mma.sync.m8n8k4 f64 ->
// SASS DMMA.8x8x4 on sm_100a).  Serves the Schur-complement / fill-in update
// A_ww -= A_ws A_ss^-1 A_sw (schemes.py:220 + factorize.py:150-161, fused
// over every same-level interior that touches a target block: K-concatenated
// segments, one read-modify-write of C), the TRSMs of schemes.py:217,235
// (as products with explicit triangular inverses) and the trailing updates
// of the blocked factorizations.
//
// CTA tile BM x BN, 4 warps of WM x WN, K staged 16 at a time through a
// 2-deep cp.async shared-memory pipeline; live sizes come from the device
// geometry so tiles past a block's live extent exit at once.  Tile shapes
// (tri >> 4): 0 64x64 (the default), 1 64x16, 2 32x32, 3 16x16, 4 16x64,
// 5 64x32, 6 32x64 --
// the leaf levels' targets are a few rows or columns wide, and a 64x64 tile
// on a 6-column target spends 90 % of its tensor work on padding.
#include <type_traits>

#include "common.cuh"
#include "../../include/spand_b200.h"

namespace {
constexpr int BK = 16;
constexpr int kThreads = 128;

__device__ __forceinline__ void cp_async8(double* smem, const double* gmem, bool pred) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  const int sz = pred ? 8 : 0;
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(gmem), "r"(sz));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::); }
__device__ __forceinline__ void cp_wait_all() { asm volatile("cp.async.wait_group 0;\n" ::); }

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

struct SegIter {
  int seg, seg_end, k0;
};

// four CTAs per SM (<= 128 registers, no spills: 124 for the 64x64 tile,
// which takes 154 unconstrained = three CTAs per SM; GEMM 171 -> 163 ms)
#ifndef SPAND_GEMM_MINB
#define SPAND_GEMM_MINB 4
#endif
template <int BM, int BN, int WM, int WN>
__global__ void __launch_bounds__(kThreads, SPAND_GEMM_MINB)
gemm_grouped_kernel(const int64_t* __restrict__ tiles, const int64_t* __restrict__ targets,
                    const int64_t* __restrict__ segs, const int32_t* __restrict__ m0,
                    const int32_t* __restrict__ off, double alpha, double beta, int bT,
                    int lower_only, int tri, const int64_t* __restrict__ btab, int compact,
                    const unsigned char* __restrict__ kmask, const int64_t* __restrict__ kmoff) {
  static_assert((BM / WM) * (BN / WN) == kThreads / 32, "4 warps per tile");
  constexpr int FM = WM / 8, FN = WN / 8;              // 8x8 fragments per warp
  constexpr int LDA = BM + 4, LDB = BN + 4;            // padding: conflict-free frags
  __shared__ __align__(16) double As[2][BK][LDA];
  __shared__ __align__(16) double Bs[2][BK][LDB];
  // packed tile: target << 32 | (i0 / BM) << 16 | (j0 / BN)
  const int64_t tr = tiles[blockIdx.x];
  const int64_t t = tr >> 32;
  const int i0 = (int)((tr >> 16) & 0xffff) * BM, j0 = (int)(tr & 0xffff) * BN;
  if (lower_only && j0 >= i0 + BM) return;
  const int64_t* trow = targets + 8 * t;
  const Opnd C = load_opnd(trow, m0, off);
  if (i0 >= C.rows || j0 >= C.cols) return;
  const int sb = (int)trow[7], se = (int)targets[8 * (t + 1) + 7];

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp / (BN / WN), wn = warp % (BN / WN);
  double acc[FM][FN][2];
#pragma unroll
  for (int a = 0; a < FM; ++a)
#pragma unroll
    for (int b = 0; b < FN; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;

  // segment operands: 14 int64 {A, B operand rows}, or (compact) one int64
  // {A block << 32 | B block} into the block table (rows {ptr, rc, cc})
  auto seg_opnds = [&](int s, Opnd& a, Opnd& b) {
    if (!compact) {
      a = load_opnd(segs + 14 * (int64_t)s, m0, off);
      b = load_opnd(segs + 14 * (int64_t)s + 7, m0, off);
    } else {
      const int64_t e = segs[s];
      const int64_t* ra = btab + 3 * (e >> 32);
      const int64_t* rb = btab + 3 * (e & 0xffffffffLL);
      const int64_t da[7] = {ra[0], ra[1], ra[2], 0, 0, -1, -1};
      const int64_t db[7] = {rb[0], rb[1], rb[2], 0, 0, -1, -1};
      a = load_opnd(da, m0, off);
      b = load_opnd(db, m0, off);
    }
  };
  // chunk iterator over (segment, k0).  Triangular operands (explicit
  // inverses, zero above the diagonal) bound each segment's K range:
  // tri & 1: A lower -> k < i0 + BM; tri & 2: B lower, C = A B^T -> k < j0 + BN;
  // tri & 4: B lower, C = A B -> k >= j0.  The skipped products are exact zeros.
  auto krange = [&](const Opnd& a, const Opnd& b, int& klo, int& khi) {
    khi = a.cols;
    const int kb = bT ? b.cols : b.rows;
    if (kb < khi) khi = kb;
    if ((tri & 1) && i0 + BM < khi) khi = i0 + BM;
    if ((tri & 2) && j0 + BN < khi) khi = j0 + BN;
    klo = (tri & 4) ? j0 : 0;
  };
  // K-chunk mask of the target's (single) segment: byte c is nonzero when
  // rows 16 c .. 16 c + 15 of B hold a nonzero (kmask_kernel below).  Chunks
  // of zero rows are not even loaded: an unscaled interface block couples a
  // separator to a neighbour through a few of its rows only.
  const unsigned char* mk = (kmask && !compact) ? kmask + kmoff[t] : nullptr;
  // bT = 1 (panel TRSM C = A L^-T, A = the panel (w, s) of an eliminated
  // interior): the bytes flag 16-row chunks of A instead.  A tile whose rows
  // of A are all zero has nothing to load: it writes its zeros and leaves
  // (on the leaf levels most 64-row tiles of a panel are such).
  bool a_rows_zero = false;
  if (mk && bT) {
    const int c1 = ((i0 + BM < C.rows ? i0 + BM : C.rows) + 15) >> 4;
    bool any = false;
    for (int c = i0 >> 4; c < c1; ++c) any |= mk[c] != 0;
    a_rows_zero = !any;
    mk = nullptr;
  }
  auto next_k = [&](int k, int kend) {
    if (mk)
      while (k < kend && !mk[k >> 4]) k += BK;
    return k;
  };
  // Compact (Schur) segments with flags: kmoff[s] = {A panel's flag offset <<
  // 32 | B panel's} into the row-chunk flags of the level's panels.  A tile of
  // a separator block is touched by few of the interiors whose segments its
  // target lists (root x root: ~2000 segments, a few dozen per tile), so the
  // segments are tested 128 at a time, one per thread, and only those whose A
  // rows (the tile's i range) and B rows (its j range) both hold a nonzero
  // are opened, in their original order (same sums, bit for bit).
  const bool seglist = compact && kmask != nullptr;
  __shared__ int slist[kThreads];
  __shared__ int wcnt[kThreads / 32];
  int sbase = sb, scount = 0, spos = 0;
  const int ca0 = i0 >> 4, ca1 = ((i0 + BM < C.rows ? i0 + BM : C.rows) + 15) >> 4;
  const int cb0 = j0 >> 4, cb1 = ((j0 + BN < C.cols ? j0 + BN : C.cols) + 15) >> 4;
  auto seg_pass = [&](int s) {
    const int64_t fo = kmoff[s];
    const unsigned char* fa = kmask + (fo >> 32);
    const unsigned char* fb = kmask + (fo & 0xffffffffLL);
    bool a = false, b = false;
    for (int c = ca0; c < ca1; ++c) a |= fa[c] != 0;
    if (!a) return false;
    for (int c = cb0; c < cb1; ++c) b |= fb[c] != 0;
    return b;
  };
  // the segment after `cur` (block-uniform calls only: the list refill
  // synchronises the CTA)
  auto following = [&](int cur) -> int {
    if (!seglist) return cur + 1;
    while (true) {
      if (spos < scount) return slist[spos++];
      if (sbase >= se) return se;
      const int s = sbase + tid;
      const bool pass = s < se && seg_pass(s);
      const unsigned bal = __ballot_sync(0xffffffffu, pass);
      if (lane == 0) wcnt[warp] = __popc(bal);
      __syncthreads();
      int before = 0, total = 0;
#pragma unroll
      for (int w = 0; w < kThreads / 32; ++w) {
        if (w < warp) before += wcnt[w];
        total += wcnt[w];
      }
      if (pass) slist[before + __popc(bal & ((1u << lane) - 1u))] = s;
      __syncthreads();
      sbase += kThreads;
      scount = total;
      spos = 0;
    }
  };
  int seg = seglist ? following(sb) : sb, k0 = 0;
  Opnd A, B;
  int K = 0;
  auto open_seg = [&](int s) {
    seg_opnds(s, A, B);
    krange(A, B, k0, K);
    k0 = next_k(k0, K);
  };
  if (a_rows_zero) seg = se;
  // skip empty segments
  while (seg < se) {
    open_seg(seg);
    if (K > k0) break;
    seg = following(seg);
  }
  auto load_stage = [&](int st, const Opnd& a, const Opnd& b, int kbase, int kmax) {
#pragma unroll
    for (int r = 0; r < (BM * BK) / kThreads; ++r) {
      const int e = tid + r * kThreads;
      const int m = e % BM, k = e / BM;
      const int gm = i0 + m, gk = kbase + k;
      const bool ok = gm < a.rows && gk < kmax;
      cp_async8(&As[st][k][m], ok ? a.p + gm + (int64_t)gk * a.ld : a.p, ok);
    }
    if (bT) {
#pragma unroll
      for (int r = 0; r < (BN * BK) / kThreads; ++r) {
        const int e = tid + r * kThreads;
        const int nn = e % BN, k = e / BN;
        const int gn = j0 + nn, gk = kbase + k;
        const bool ok = gn < b.rows && gk < kmax;
        cp_async8(&Bs[st][k][nn], ok ? b.p + gn + (int64_t)gk * b.ld : b.p, ok);
      }
    } else {
#pragma unroll
      for (int r = 0; r < (BN * BK) / kThreads; ++r) {
        const int e = tid + r * kThreads;
        const int k = e % BK, nn = e / BK;
        const int gn = j0 + nn, gk = kbase + k;
        const bool ok = gn < b.cols && gk < kmax;
        cp_async8(&Bs[st][k][nn], ok ? b.p + gk + (int64_t)gn * b.ld : b.p, ok);
      }
    }
    cp_commit();
  };

  if (seg < se) {
    int st = 0;
    int dense_run = 0, unchecked = 0;   // zero-slice test policy (warp-uniform)
    load_stage(0, A, B, k0, K);
    while (true) {
      // advance iterator to the next chunk and prefetch it
      Opnd An = A, Bn = B;
      int Kn = K, segn = seg, kn = next_k(k0 + BK, K);
      bool have_next = true;
      if (kn >= Kn) {
        segn = following(segn);
        while (segn < se) {
          seg_opnds(segn, An, Bn);
          krange(An, Bn, kn, Kn);
          kn = next_k(kn, Kn);
          if (Kn > kn) break;
          segn = following(segn);
        }
        have_next = segn < se;
      }
      cp_wait_all();
      __syncthreads();
      if (have_next) load_stage(st ^ 1, An, Bn, kn, Kn);
      // The operands are block-sparse by rows: an eliminated interior
      // touches a few dofs of each separator, so most 4-deep k-slices of a
      // panel's rows (Schur update) or of an unscaled interface block
      // (Z^-1 B) are exact zeros over a warp's 32 rows / columns.  A slice
      // whose A or B fragments are all zero adds +-0 to every accumulator
      // (they start at +0, so the bits do not change): its DMMAs are skipped.
      // The test splits the unrolled k-loop (no fragment prefetch across
      // slices), which costs ~15 % on dense operands, so a warp that skipped
      // nothing in two consecutive stages runs the next 16 stages unchecked.
      auto stage = [&](auto checked) {
        constexpr bool kCheck = decltype(checked)::value;
        bool skipped = false;
#pragma unroll
        for (int kk = 0; kk < BK / 4; ++kk) {
          double af[FM], bf[FN];
          const int kr = kk * 4 + (lane & 3);
          bool nzb = false;
#pragma unroll
          for (int ni = 0; ni < FN; ++ni) {
            bf[ni] = Bs[st][kr][wn * WN + ni * 8 + (lane >> 2)];
            if (kCheck) nzb |= bf[ni] != 0.0;
          }
          if (kCheck && !__any_sync(0xffffffffu, nzb)) {
            skipped = true;
            continue;
          }
          bool nza = false;
#pragma unroll
          for (int mi = 0; mi < FM; ++mi) {
            af[mi] = As[st][kr][wm * WM + mi * 8 + (lane >> 2)];
            if (kCheck) nza |= af[mi] != 0.0;
          }
          if (kCheck && !__any_sync(0xffffffffu, nza)) {
            skipped = true;
            continue;
          }
#pragma unroll
          for (int mi = 0; mi < FM; ++mi)
#pragma unroll
            for (int ni = 0; ni < FN; ++ni) dmma(acc[mi][ni][0], acc[mi][ni][1], af[mi], bf[ni]);
        }
        return skipped;
      };
#ifdef SPAND_GEMM_NOSKIP
      stage(std::false_type{});
#else
      if (unchecked > 0) {
        --unchecked;
        stage(std::false_type{});
      } else if (stage(std::true_type{})) {
        dense_run = 0;
      } else if (++dense_run >= 2) {
        dense_run = 0;
        unchecked = 16;
      }
#endif
      __syncthreads();
      if (!have_next) break;
      st ^= 1;
      A = An;
      B = Bn;
      K = Kn;
      seg = segn;
      k0 = kn;
    }
  }
  // epilogue: C = beta C + alpha acc
#pragma unroll
  for (int mi = 0; mi < FM; ++mi) {
    const int r = i0 + wm * WM + mi * 8 + (lane >> 2);
    if (r >= C.rows) continue;
#pragma unroll
    for (int ni = 0; ni < FN; ++ni) {
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int c = j0 + wn * WN + ni * 8 + (lane & 3) * 2 + h;
        if (c >= C.cols) continue;
        double* pc = C.p + r + (int64_t)c * C.ld;
        const double v = alpha * acc[mi][ni][h];
        *pc = (beta == 0.0) ? v : beta * (*pc) + v;
      }
    }
  }
}
// Row-chunk masks of a masked GEMM launch: B = the A (which = 0) or B
// (which = 1) operand of the target's first segment (14-int64 segment
// rows); kmask[kmoff[t] + c] = any nonzero in rows 16 c .. 16 c + 15 of it.  Work unit = (target, 128-row slab): one
// row per thread (coalesced column reads, 8 independent loads in flight), a
// chunk is 16 consecutive lanes.  Slabs of a target are dealt over
// gridDim.y CTAs (the blocks between two top separators have ~10^7 entries).
constexpr int kMaskY = 8;
__global__ void __launch_bounds__(kThreads)
kmask_kernel(const int64_t* __restrict__ targets, const int64_t* __restrict__ segs,
             const int32_t* __restrict__ m0, const int32_t* __restrict__ off,
             unsigned char* __restrict__ kmask, const int64_t* __restrict__ kmoff, int which) {
  const int64_t t = blockIdx.x;
  const int64_t s = targets[8 * t + 7];
  const Opnd B = load_opnd(segs + 14 * s + (which ? 7 : 0), m0, off);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nch = (B.rows + 15) >> 4;
  unsigned char* out = kmask + kmoff[t];
  for (int r0 = kThreads * blockIdx.y; r0 < B.rows; r0 += kThreads * gridDim.y) {
    const int r = r0 + tid;
    bool nz = false;
    if (r < B.rows) {
      const double* rp = B.p + r;
      int col = 0;
      for (; col + 8 <= B.cols; col += 8) {
        double v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) v[u] = __ldg(rp + (int64_t)(col + u) * B.ld);
#pragma unroll
        for (int u = 0; u < 8; ++u) nz |= v[u] != 0.0;
      }
      for (; col < B.cols; ++col) nz |= __ldg(rp + (int64_t)col * B.ld) != 0.0;
    }
    const unsigned bal = __ballot_sync(0xffffffffu, nz);
    if (lane == 0) {
      const int c = (r0 >> 4) + 2 * warp;
      if (c < nch) out[c] = (bal & 0xffffu) ? 1 : 0;
      if (c + 1 < nch) out[c + 1] = (bal >> 16) ? 1 : 0;
    }
  }
}
}  // namespace

extern "C" int spand_gemm_kmask(int ntarget, const int64_t* targets, const int64_t* segs,
                                const int32_t* m0, const int32_t* off, unsigned char* kmask,
                                const int64_t* kmoff, int which, void* stream) {
  if (ntarget < 0) return -1;
  if (ntarget == 0) return 0;
  kmask_kernel<<<dim3(ntarget, kMaskY), kThreads, 0, as_stream(stream)>>>(targets, segs, m0, off,
                                                                          kmask, kmoff, which);
  SPAND_CHECK_LAUNCH();
  return 0;
}

extern "C" int spand_gemm_grouped(int ntile, const int64_t* tiles, const int64_t* targets,
                                  const int64_t* segs, const int32_t* m0, const int32_t* off,
                                  double alpha, double beta, int bT, int lower_only,
                                  int tri, const int64_t* btab, int compact, void* stream) {
  return spand_gemm_grouped_masked(ntile, tiles, targets, segs, m0, off, alpha, beta, bT,
                                   lower_only, tri, btab, compact, nullptr, nullptr, stream);
}

extern "C" int spand_gemm_grouped_masked(int ntile, const int64_t* tiles, const int64_t* targets,
                                  const int64_t* segs, const int32_t* m0, const int32_t* off,
                                  double alpha, double beta, int bT, int lower_only,
                                  int tri, const int64_t* btab, int compact,
                                  const unsigned char* kmask, const int64_t* kmoff,
                                  void* stream) {
  if (ntile < 0) return -1;
  // masks describe 16-row chunks of B (bT = 0: K chunks) or of A (bT = 1: a
  // tile's own rows), with 14-int64 segment rows
  // (compact = 1: per-segment flag offsets of the A and B panels)
  if (kmask && !kmoff) return -1;
  if (ntile == 0) return 0;
  const int shape = (tri >> 4) & 7;
  tri &= 7;
  cudaStream_t st = as_stream(stream);
#define SPAND_GEMM_LAUNCH(BM_, BN_, WM_, WN_)                                             \
  gemm_grouped_kernel<BM_, BN_, WM_, WN_><<<ntile, kThreads, 0, st>>>(                    \
      tiles, targets, segs, m0, off, alpha, beta, bT, lower_only, tri, btab, compact, kmask, kmoff)
  switch (shape) {
    case 0: SPAND_GEMM_LAUNCH(64, 64, 32, 32); break;
    case 1: SPAND_GEMM_LAUNCH(64, 16, 16, 16); break;
    case 2: SPAND_GEMM_LAUNCH(32, 32, 16, 16); break;
    case 3: SPAND_GEMM_LAUNCH(16, 16, 8, 8); break;
    case 4: SPAND_GEMM_LAUNCH(16, 64, 16, 16); break;
    case 5: SPAND_GEMM_LAUNCH(64, 32, 32, 16); break;
    case 6: SPAND_GEMM_LAUNCH(32, 64, 16, 32); break;
    default: return -1;
  }
#undef SPAND_GEMM_LAUNCH
  SPAND_CHECK_LAUNCH();
  return 0;
}
