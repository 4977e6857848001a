// Batched FP64 Cholesky, triangular inverse and copies on live windows
// (replace LAPACK dpotrf / dtrtri calls of dense.py:45-93 as used by
// schemes.py:199-236 and factorize.py:131-220).  One CTA per matrix; sizes
// are read from the device geometry so a whole level is one launch with no
// host round trip.  The diagonal 32x32 tiles are factored in shared memory
// with warp-level reductions; the rest is blocked left-looking updates.
#include "common.cuh"
#include "../../include/spand_b200.h"

namespace {
constexpr int kT = 256;
constexpr int NB = 32;

// Left-looking blocked Cholesky of one live window (in place, lower).
__global__ void __launch_bounds__(kT)
potrf_kernel(const int64_t* __restrict__ ops, const int32_t* __restrict__ m0,
             const int32_t* __restrict__ off, int32_t* __restrict__ info, int piv_off,
             int first_only) {
  // one buffer: the general path's Bk / D tiles, or a whole block of <= 64
  __shared__ double raw[64 * 65];
  double (*Bk)[65] = reinterpret_cast<double (*)[65]>(raw);                // [NB][65]: rows jb..jb+NB of columns kb..kb+64
  double (*D)[NB + 1] = reinterpret_cast<double (*)[NB + 1]>(raw + NB * 65);  // [NB][NB + 1]: diagonal tile
  __shared__ int bad;
  const int64_t* row = ops + 8 * (int64_t)blockIdx.x;
  const Opnd A = load_opnd(row, m0, off);
  const int n = A.rows < A.cols ? A.rows : A.cols;
  const int ld = A.ld;
  double* a = A.p;
  if (threadIdx.x == 0) bad = 0;
  __syncthreads();
  if (n <= 64) {
    // Blocks of <= 64 (leaf interiors, the diagonal steps of the blocked
    // factorization): the lower triangle is staged in shared memory and
    // factored right-looking by the whole CTA -- per column: sqrt, scale,
    // rank-1 update of the trailing triangle (element (i, c) accumulates its
    // updates in column order).  One coalesced read and one write of the
    // block instead of the left-looking passes over global memory.
    double (*S)[65] = reinterpret_cast<double (*)[65]>(raw);
    for (int e = threadIdx.x; e < n * n; e += kT) {
      const int r = e % n, c = e / n;
      S[r][c] = (c <= r) ? a[r + (int64_t)c * ld] : 0.0;
    }
    __syncthreads();
    for (int j = 0; j < n; ++j) {
      const double d = S[j][j];
      if (!(d > 0.0)) {  // also catches NaN (uniform: every thread reads the same d)
        if (threadIdx.x == 0) bad = j + 1;
        break;
      }
      const double rd = sqrt(d);
      __syncthreads();
      if (threadIdx.x == 0) S[j][j] = rd;
      for (int i = j + 1 + threadIdx.x; i < n; i += kT) S[i][j] /= rd;
      __syncthreads();
      // trailing lower triangle: rows i > j, columns j < c <= i
      const int tl = n - j - 1;
      for (int e = threadIdx.x; e < tl * tl; e += kT) {
        const int i = j + 1 + e % tl, c = j + 1 + e / tl;
        if (c <= i) S[i][c] -= S[i][j] * S[c][j];
      }
      __syncthreads();
    }
    __syncthreads();
    if (!bad) {
      for (int e = threadIdx.x; e < n * n; e += kT) {
        const int r = e % n, c = e / n;
        a[r + (int64_t)c * ld] = S[r][c];   // zeros above the diagonal (dense.py:53)
      }
    }
    if (threadIdx.x == 0) {
      int32_t* slot = info + row[7];
      if (!first_only) *slot = bad ? bad + piv_off : 0;
      else if (bad && *slot == 0) *slot = bad + piv_off;
    }
    return;
  }
  for (int jb = 0; jb < n; jb += NB) {
    const int nbk = min(NB, n - jb);
    // ---- panel update A[jb:, jb:jb+nbk] -= A[jb:, :jb] * A[jb:jb+nbk, :jb]^T
    // each thread owns rows i = jb + tid + kT*r, 32 accumulators per row
    for (int rb = jb; rb < n; rb += kT) {
      const int i = rb + threadIdx.x;
      double acc[NB];
#pragma unroll
      for (int j = 0; j < NB; ++j) acc[j] = 0.0;
      for (int kb = 0; kb < jb; kb += 64) {
        const int kc = min(64, jb - kb);
        __syncthreads();
        for (int e = threadIdx.x; e < NB * 64; e += kT) {
          const int j = e / 64, k = e % 64;
          Bk[j][k] = (j < nbk && k < kc) ? a[(jb + j) + (int64_t)(kb + k) * ld] : 0.0;
        }
        __syncthreads();
        if (i < n) {
          for (int k = 0; k < kc; ++k) {
            const double aik = a[i + (int64_t)(kb + k) * ld];
#pragma unroll
            for (int j = 0; j < NB; ++j) acc[j] += aik * Bk[j][k];
          }
        }
      }
      if (i < n) {
#pragma unroll
        for (int j = 0; j < NB; ++j)
          if (j < nbk) a[i + (int64_t)(jb + j) * ld] -= acc[j];
      }
    }
    __syncthreads();
    // ---- factor the diagonal tile in shared memory
    for (int e = threadIdx.x; e < NB * NB; e += kT) {
      const int r = e / NB, c = e % NB;
      D[r][c] = (r < nbk && c < nbk && c <= r) ? a[(jb + r) + (int64_t)(jb + c) * ld] : 0.0;
    }
    __syncthreads();
    if (threadIdx.x < 32) {
      const int l = threadIdx.x;
      for (int j = 0; j < nbk; ++j) {
        double d = D[j][j];
        if (!(d > 0.0)) {  // also catches NaN
          if (l == 0 && bad == 0) bad = jb + j + 1;
          break;
        }
        d = sqrt(d);
        __syncwarp();
        if (l == 0) D[j][j] = d;
        if (l > j && l < nbk) D[l][j] /= d;
        __syncwarp();
        // rank-1 update of the trailing tile (lower part), lane = row
        if (l > j && l < nbk)
          for (int c = j + 1; c <= l; ++c) D[l][c] -= D[l][j] * D[c][j];
        __syncwarp();
      }
    }
    __syncthreads();
    if (bad) break;
    for (int e = threadIdx.x; e < NB * NB; e += kT) {
      const int r = e / NB, c = e % NB;
      if (r < nbk && c < nbk && c <= r) a[(jb + r) + (int64_t)(jb + c) * ld] = D[r][c];
    }
    // ---- rows below: x = row * L_d^{-T}  (forward substitution per row)
    for (int i = jb + nbk + threadIdx.x; i < n; i += kT) {
      double x[NB];
#pragma unroll
      for (int j = 0; j < NB; ++j) x[j] = (j < nbk) ? a[i + (int64_t)(jb + j) * ld] : 0.0;
#pragma unroll
      for (int j = 0; j < NB; ++j) {
        if (j < nbk) {
          double s = x[j];
#pragma unroll
          for (int k = 0; k < j; ++k) s -= x[k] * D[j][k];
          x[j] = s / D[j][j];
        }
      }
#pragma unroll
      for (int j = 0; j < NB; ++j)
        if (j < nbk) a[i + (int64_t)(jb + j) * ld] = x[j];
    }
    __syncthreads();
  }
  // zero the strict upper triangle (LAPACK dpotrf with clean=1, dense.py:53)
  if (!bad) {
    for (int64_t e = threadIdx.x; e < (int64_t)n * n; e += kT) {
      const int r = (int)(e % n), c = (int)(e / n);
      if (r < c) a[r + (int64_t)c * ld] = 0.0;
    }
  }
  if (threadIdx.x == 0) {
    int32_t* slot = info + row[7];
    if (!first_only) *slot = bad ? bad + piv_off : 0;
    else if (bad && *slot == 0) *slot = bad + piv_off;
  }
}

// Lower-triangular inverse, one thread per column (forward substitution),
// x kept in the output column (L1 resident).
__global__ void __launch_bounds__(kT)
trtri_kernel(const int64_t* __restrict__ ops, const int32_t* __restrict__ m0,
             const int32_t* __restrict__ off) {
  const Opnd L = load_opnd(ops + 14 * (int64_t)blockIdx.x, m0, off);
  const Opnd X = load_opnd(ops + 14 * (int64_t)blockIdx.x + 7, m0, off);
  const int n = L.rows;
  for (int j = threadIdx.x; j < n; j += kT) {
    double* x = X.p + (int64_t)j * X.ld;
    for (int i = 0; i < j; ++i) x[i] = 0.0;
    x[j] = 1.0 / L.p[j + (int64_t)j * L.ld];
    for (int i = j + 1; i < n; ++i) {
      double s = 0.0;
      for (int k = j; k < i; ++k) s += L.p[i + (int64_t)k * L.ld] * x[k];
      x[i] = -s / L.p[i + (int64_t)i * L.ld];
    }
  }
}

__global__ void __launch_bounds__(kT)
copy_kernel(const int64_t* __restrict__ ops, const int32_t* __restrict__ m0,
            const int32_t* __restrict__ off) {
  const int64_t* d = ops + 15 * (int64_t)blockIdx.x;
  const int mode = (int)d[14];
  const Opnd D = load_opnd(d + 7, m0, off);
  Opnd S = D;
  if (mode != 2) S = load_opnd(d, m0, off);
  const int rows = D.rows, cols = D.cols;
  const int64_t total = (int64_t)rows * cols;
  for (int64_t e = (int64_t)blockIdx.y * kT + threadIdx.x; e < total; e += (int64_t)gridDim.y * kT) {
    const int r = (int)(e % rows), c = (int)(e / rows);
    double v;
    if (mode == 2) v = (r == c) ? 1.0 : 0.0;
    else if (mode == 1 && r < c) v = 0.0;
    else v = (r < S.rows && c < S.cols) ? S.p[r + (int64_t)c * S.ld] : 0.0;
    D.p[r + (int64_t)c * D.ld] = v;
  }
}
}  // namespace

extern "C" {

int spand_potrf_batched(int ntask, const int64_t* ops, const int32_t* m0, const int32_t* off,
                        int32_t* info, int piv_off, int first_only, void* stream) {
  if (ntask < 0) return -1;
  if (ntask == 0) return 0;
  potrf_kernel<<<ntask, kT, 0, as_stream(stream)>>>(ops, m0, off, info, piv_off, first_only);
  SPAND_CHECK_LAUNCH();
  return 0;
}

int spand_trtri_batched(int ntask, const int64_t* ops, const int32_t* m0, const int32_t* off,
                        void* stream) {
  if (ntask < 0) return -1;
  if (ntask == 0) return 0;
  trtri_kernel<<<ntask, kT, 0, as_stream(stream)>>>(ops, m0, off);
  SPAND_CHECK_LAUNCH();
  return 0;
}

int spand_copy_batched(int ntask, const int64_t* ops, const int32_t* m0, const int32_t* off,
                       void* stream) {
  if (ntask < 0) return -1;
  if (ntask == 0) return 0;
  // few tasks = the large blocks of the top levels (up to 3104^2 entries):
  // enough CTAs per task to fill the device (16 each left a 77 MB copy on 16 SMs)
  int gy = 16;
  if (ntask < 74) gy = (1184 + ntask - 1) / ntask;
  dim3 grid(ntask, gy);
  copy_kernel<<<grid, kT, 0, as_stream(stream)>>>(ops, m0, off);
  SPAND_CHECK_LAUNCH();
  return 0;
}

}  // extern "C"

// ---------------------------------------------------------------------------
// Final dense block (factorize.py:198-220) and payload nonzero counts
// (schemes.py:114-117,142-144,168-170,194-196).
namespace {
// cl rows: {cluster id}; block rows (4 int64): {ci index in cl, cj index in cl, ptr, 0}
__global__ void __launch_bounds__(kT)
assemble_kernel(int ncl, const int64_t* __restrict__ cl, const int64_t* __restrict__ blocks,
                const int32_t* __restrict__ m0, const int32_t* __restrict__ off, int fid,
                double* __restrict__ dst) {
  const int cap = m0[fid];
  const int64_t* br = blocks + 4 * (int64_t)blockIdx.x;
  const int a = (int)br[0], b = (int)br[1];
  const double* src = reinterpret_cast<const double*>(br[2]);
  int total = 0, pa = 0, pb = 0;
  for (int t = 0; t < ncl; ++t) {
    const int c = (int)cl[t];
    if (t == a) pa = total;
    if (t == b) pb = total;
    total += m0[c] - off[c];
  }
  const int base = cap - total;
  const int ca = (int)cl[a], cb = (int)cl[b];
  const int ra = m0[ca] - off[ca], rb = m0[cb] - off[cb];
  const int lda = m0[ca];
  for (int64_t e = threadIdx.x; e < (int64_t)ra * rb; e += kT) {
    const int r = (int)(e % ra), c = (int)(e / ra);
    const double v = src[(int64_t)(off[ca] + r) + (int64_t)(off[cb] + c) * lda];
    dst[(int64_t)(base + pa + r) + (int64_t)(base + pb + c) * cap] = v;
    if (a != b) dst[(int64_t)(base + pb + c) + (int64_t)(base + pa + r) * cap] = v;
  }
}

__global__ void set_off_kernel(int ncl, const int64_t* __restrict__ cl, const int32_t* __restrict__ m0,
                               int32_t* __restrict__ off, int fid) {
  int total = 0;
  for (int t = 0; t < ncl; ++t) {
    const int c = (int)cl[t];
    total += m0[c] - off[c];
  }
  off[fid] = m0[fid] - total;
}

// view rows (4 int64): {ptr, ld, rows, cols}; out[i] = nonzero count
__global__ void __launch_bounds__(kT)
count_kernel(const int64_t* __restrict__ views, unsigned long long* __restrict__ out) {
  const int64_t* v = views + 4 * (int64_t)blockIdx.x;
  const double* p = reinterpret_cast<const double*>(v[0]);
  const int64_t ld = v[1], rows = v[2], cols = v[3];
  unsigned long long c = 0;
  for (int64_t e = (int64_t)blockIdx.y * kT + threadIdx.x; e < rows * cols; e += (int64_t)gridDim.y * kT) {
    const int64_t r = e % rows, q = e / rows;
    c += p[r + q * ld] != 0.0;
  }
  for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
  if ((threadIdx.x & 31) == 0 && c) atomicAdd(out + blockIdx.x, c);
}

// Balanced variant: views are split into pieces of <= kCountPiece elements
// (whole columns; pstart[v] = first piece of view v, exclusive prefix sum of
// ceil(cols / max(1, kCountPiece / rows))), one CTA per piece, one total.
constexpr int kCountPiece = 65536;
__global__ void __launch_bounds__(kT)
count_pieces_kernel(const int64_t* __restrict__ views, const int64_t* __restrict__ pstart,
                    int nview, const double* pool, const double* fac,
                    unsigned long long* __restrict__ total) {
  const int64_t pc = blockIdx.x;
  int lo = 0, hi = nview - 1;
  while (lo < hi) {   // last view whose first piece is <= pc
    const int mid = (lo + hi + 1) >> 1;
    if (pstart[mid] <= pc) lo = mid;
    else hi = mid - 1;
  }
  const int64_t* v = views + 4 * (int64_t)lo;
  const int64_t ld = v[1], rows = v[2], cols = v[3];
  const int64_t cpp = rows >= kCountPiece ? 1 : kCountPiece / rows;
  const int64_t c0 = (pc - pstart[lo]) * cpp, c1 = min(cols, c0 + cpp);
  // view offset: bit 62 selects the factor buffer (collector convention)
  const int64_t o = v[0] & ((int64_t(1) << 62) - 1);
  const double* p = (((v[0] >> 62) & 1) ? fac : pool) + o + c0 * ld;
  unsigned long long c = 0;
  if (rows >= 64) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int64_t q = warp; q < c1 - c0; q += kT / 32)
      for (int64_t r = lane; r < rows; r += 32) c += p[r + q * ld] != 0.0;
  } else {
    const int rr = (int)rows, ne = (int)((c1 - c0) * rows);
    for (int e = threadIdx.x; e < ne; e += kT) c += p[e % rr + (int64_t)(e / rr) * ld] != 0.0;
  }
  for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
  __shared__ unsigned long long part[kT / 32];
  if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = c;
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long t = 0;
    for (int w = 0; w < kT / 32; ++w) t += part[w];
    if (t) atomicAdd(total, t);
  }
}
}  // namespace

extern "C" {

int spand_count_nonzero_pieces(int nview, const int64_t* views, const int64_t* pstart,
                               int64_t npiece, const double* pool, const double* fac,
                               unsigned long long* total, void* stream) {
  if (nview < 0 || npiece < 0 || npiece >= (int64_t(1) << 31)) return -1;
  if (nview == 0 || npiece == 0) return 0;
  count_pieces_kernel<<<(unsigned)npiece, kT, 0, as_stream(stream)>>>(views, pstart, nview, pool,
                                                                      fac, total);
  SPAND_CHECK_LAUNCH();
  return 0;
}

int spand_assemble_final(int ncl, const int64_t* cl, int64_t nblk, const int64_t* blocks,
                         const int32_t* m0, int32_t* off, int32_t final_id, double* dst,
                         void* stream) {
  if (ncl < 0 || nblk < 0) return -1;
  if (ncl == 0) return 0;
  // off[final_id] = m0[final_id] - (sum of live sizes): the live parts are
  // packed at the bottom-right of the m0[final_id]^2 buffer
  set_off_kernel<<<1, 1, 0, as_stream(stream)>>>(ncl, cl, m0, off, final_id);
  if (nblk > 0)
    assemble_kernel<<<(unsigned)nblk, kT, 0, as_stream(stream)>>>(ncl, cl, blocks, m0, off,
                                                                  final_id, dst);
  SPAND_CHECK_LAUNCH();
  return 0;
}

int spand_count_nonzero(int nview, const int64_t* views, unsigned long long* out, void* stream) {
  if (nview < 0) return -1;
  if (nview == 0) return 0;
  dim3 grid(nview, 4);
  count_kernel<<<grid, kT, 0, as_stream(stream)>>>(views, out);
  SPAND_CHECK_LAUNCH();
  return 0;
}

}  // extern "C"

// ---------------------------------------------------------------------------
// Inverse of <= 64 x 64 lower-triangular diagonal tiles in shared memory; the
// off-diagonal blocks of L^-1 are then assembled by recursive doubling with
// the DMMA GEMM ([A 0; B C]^-1 = [A^-1 0; -C^-1 B A^-1, C^-1]), so a whole
// level's triangular inverses (dense.py:85-93) are O(log n) batched launches.
namespace {
__global__ void __launch_bounds__(kT)
trtri_tile_kernel(const int64_t* __restrict__ ops, const int32_t* __restrict__ m0,
                  const int32_t* __restrict__ off) {
  extern __shared__ double tri_sm[];
  double (*Ls)[65] = reinterpret_cast<double (*)[65]>(tri_sm);
  double (*Xs)[65] = reinterpret_cast<double (*)[65]>(tri_sm + 64 * 65);
  const Opnd L = load_opnd(ops + 14 * (int64_t)blockIdx.x, m0, off);
  const Opnd X = load_opnd(ops + 14 * (int64_t)blockIdx.x + 7, m0, off);
  const int n = min(L.rows, L.cols);
  if (n <= 0) return;
  for (int e = threadIdx.x; e < 64 * 64; e += kT) {
    const int r = e % 64, c = e / 64;
    Ls[r][c] = (r < n && c <= r) ? L.p[r + (int64_t)c * L.ld] : 0.0;
    Xs[r][c] = 0.0;
  }
  __syncthreads();
  // column j of X solves L x = e_j by forward substitution; four lanes per
  // column split each row's dot product (terms k = j + p, j + p + 4, ...) and
  // add their partials in a fixed order.  The row loop is warp-uniform (a
  // warp holds 8 columns): rows above a column's diagonal are predicated off.
  {
    const int j = threadIdx.x >> 2, p = threadIdx.x & 3;
    if (p == 0 && j < n) Xs[j][j] = 1.0 / Ls[j][j];
    __syncwarp();
    for (int i = 1; i < n; ++i) {
      double sum = 0.0;
      if (j < i)
        for (int k = j + p; k < i; k += 4) sum += Ls[i][k] * Xs[k][j];
      const double s1 = sum + __shfl_xor_sync(0xffffffffu, sum, 1);
      const double s2 = s1 + __shfl_xor_sync(0xffffffffu, s1, 2);
      if (p == 0 && j < i) Xs[i][j] = -s2 / Ls[i][i];
      __syncwarp();
    }
  }
  __syncthreads();
  const int nr = min(X.rows, 64), nc = min(X.cols, 64);
  for (int e = threadIdx.x; e < nr * nc; e += kT) {
    const int r = e % nr, c = e / nr;
    X.p[r + (int64_t)c * X.ld] = (r < n && c < n) ? Xs[r][c] : 0.0;
  }
}
}  // namespace

extern "C" int spand_trtri_tiles(int ntask, const int64_t* ops, const int32_t* m0,
                                 const int32_t* off, void* stream) {
  if (ntask < 0) return -1;
  if (ntask == 0) return 0;
  const int smem = 2 * 64 * 65 * (int)sizeof(double);
  cudaFuncSetAttribute(trtri_tile_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  trtri_tile_kernel<<<ntask, kT, smem, as_stream(stream)>>>(ops, m0, off);
  SPAND_CHECK_LAUNCH();
  return 0;
}

// ---------------------------------------------------------------------------
// Trailing-matrix fingerprint (reference EliminationState.digest,
// factorize.py:222-229): per block alive at a level end, an order-free hash
// of its live window -- the sum over entries of splitmix64(bits(v) ^
// position) mod 2^64, integer atomics, so the result does not depend on the
// thread schedule.  Diagonal blocks hash their lower triangle only (the
// stored triangle; the reference's diagonal blocks are symmetric).  Piece
// rows (6 int64): {block ptr, i, j, first column, columns, record ptr};
// records (5 int64): {i, j, live rows, live cols, hash}.
namespace {
__device__ __forceinline__ unsigned long long mix64(unsigned long long x) {
  x += 0x9e3779b97f4a7c15ull;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
  return x ^ (x >> 31);
}

__global__ void __launch_bounds__(kT)
digest_kernel(const int64_t* __restrict__ rows, const int32_t* __restrict__ m0,
              const int32_t* __restrict__ off) {
  const int64_t* d = rows + 6 * (int64_t)blockIdx.x;
  const double* blk = reinterpret_cast<const double*>(d[0]);
  const int i = (int)d[1], j = (int)d[2];
  const int c0 = (int)d[3], nc = (int)d[4];
  unsigned long long* rec = reinterpret_cast<unsigned long long*>(d[5]);
  const int ld = m0[i];
  const int ri = off[i], cj = off[j];
  const int lr = m0[i] - ri, lc = m0[j] - cj;
  if (c0 == 0 && threadIdx.x == 0) {
    rec[0] = (unsigned long long)i;
    rec[1] = (unsigned long long)j;
    rec[2] = (unsigned long long)(lr > 0 ? lr : 0);
    rec[3] = (unsigned long long)(lc > 0 ? lc : 0);
  }
  const int cb = max(c0, cj), ce = min(c0 + nc, m0[j]);
  unsigned long long h = 0;
  if (lr > 0 && cb < ce) {
    const int64_t total = (int64_t)lr * (ce - cb);
    for (int64_t e = threadIdx.x; e < total; e += kT) {
      const int r = (int)(e % lr), c = cb + (int)(e / lr) - cj;
      if (i == j && r < c) continue;
      const double v = blk[(int64_t)(ri + r) + (int64_t)(cj + c) * ld];
      const unsigned long long pos = ((unsigned long long)r << 32) | (unsigned)c;
      h += mix64((unsigned long long)__double_as_longlong(v) ^ mix64(pos));
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) h += __shfl_xor_sync(0xffffffffu, h, o);
  __shared__ unsigned long long part[kT / 32];
  if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = h;
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long t = 0;
    for (int w = 0; w < kT / 32; ++w) t += part[w];
    if (t) atomicAdd(rec + 4, t);
  }
}
}  // namespace

extern "C" int spand_digest_pieces(int npiece, const int64_t* rows, const int32_t* m0,
                                   const int32_t* off, void* stream) {
  if (npiece < 0) return -1;
  if (npiece == 0) return 0;
  digest_kernel<<<npiece, kT, 0, as_stream(stream)>>>(rows, m0, off);
  SPAND_CHECK_LAUNCH();
  return 0;
}
