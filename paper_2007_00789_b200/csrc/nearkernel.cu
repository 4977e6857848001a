// Near-kernel preservation inside the sparsification (EXTENSION; not in the
// reference -- SURVEY.md §8a-11, PAPER.md:2005 names it as compatible future
// work, SPEC.md:350 lists it as a non-goal of spdkit).  The CPU restatement
// and its derivation live in oracle/spand_oracle.py (nk_basis,
// sparsify_panel_nk); with no vectors nothing here is launched and the
// factorization is the reference path.
//
// The vectors v (n x k) are carried through the factorization's congruences
// in the cluster-contiguous numbering: u = B^-T v restricted to the live
// slots.  Eliminations and error corrections leave live entries unchanged;
// a Scaling maps u_p <- Z_p^T u_p (spand_nk_rescale); a sparsification of p
//   1. factors u_p = H [R_u; 0] with a column-pivoted Householder QR (rank r,
//      spand_nk_basis), and sets u_p <- [0 (m - r); R_u] (rotated order);
//   2. replaces the panel W by the ROTATED reflection [U_perp^T W; U^T W]
//      (spand_nk_deflate), so the RRQR (rrqr.cu, which reads r and factors
//      only the first m - r rows) leaves the last r slots -- U^T W, the rows
//      of the near-kernel directions -- as kept coarse rows;
//   3. builds the orthogonal factor [U_perp q2_c, U, U_perp q2_f] (stored
//      coarse-first, rotated by k_c + r like the plain Q) from the RRQR's q2
//      (spand_nk_qform).
// rrqr.cu adds r to the event's k_stop / k_c / m, so the host collector
// (collect.cpp) sees an ordinary Orthogonal op with k_c2 + r coarse columns.
#include "common.cuh"
#include "../../include/spand_b200.h"

namespace {

constexpr int kNT = 256;
constexpr int kMaxK = 16;
// workspace per panel (doubles): [0] r, [1] live m at sparsification start,
// [2] m0[p] (ld of V and X), [3, 3 + kMaxK) taus, then V (mcap x k, reflector t in column t, rows t..),
// then X (mcap x k, the working copy of u_p)
constexpr int kWsHead = 3 + kMaxK;

// nk row (10 int64): {p, ws, q2, Qfin, nb0, nb1, colbeg, qbeg, slot, ustart}
//   q2: where the RRQR wrote its orthogonal factor (compact, ld = m - r)
//   Qfin: the Orthogonal op's storage (compact, ld = m)
//   colbeg / qbeg: first CTA of the panel in the deflate / qform grids
//   (capacity-sized: sum of m0[w] over the neighbours, m0[p])
// nbrs rows are the RRQR's (4 int64): {w, block ptr, orientation, 0}

__device__ __forceinline__ int find_row(const int64_t* rows, int nrow, int field, int64_t b) {
  int lo = 0, hi = nrow - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (rows[10 * (int64_t)mid + field] <= b) lo = mid;
    else hi = mid - 1;
  }
  return lo;
}

// u_p <- L_p^T u_p for the live window of each rescaled interface.
// row (3 int64): {p, L ptr (ld m0[p], original-size block), ustart}; grid =
// ntask * k (one CTA per interface and vector).
__global__ void __launch_bounds__(kNT) nk_rescale_kernel(const int64_t* __restrict__ rows,
                                                         const int32_t* __restrict__ m0,
                                                         const int32_t* __restrict__ off,
                                                         double* __restrict__ U, int64_t ldu,
                                                         int k) {
  extern __shared__ double us[];
  const int task = blockIdx.x / k, v = blockIdx.x % k;
  const int64_t* R = rows + 3 * (int64_t)task;
  const int p = (int)R[0];
  const int o = off[p], ld = m0[p], m = ld - o;
  if (m <= 0) return;
  const double* L = reinterpret_cast<const double*>(R[1]) + (int64_t)o + (int64_t)o * ld;
  double* u = U + (int64_t)v * ldu + R[2] + o;
  for (int i = threadIdx.x; i < m; i += kNT) us[i] = u[i];
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  // y_i = sum_{j >= i} L[j, i] u_j : column i of L is contiguous
  for (int i = warp; i < m; i += kNT / 32) {
    const double* col = L + (int64_t)i * ld;
    double s = 0.0;
    for (int j = i + lane; j < m; j += 32) s += col[j] * us[j];
    s = warp_sum(s);
    if (lane == 0) u[i] = s;
  }
}

// Column-pivoted Householder QR of u_p (one CTA per panel).
__global__ void __launch_bounds__(kNT) nk_basis_kernel(const int64_t* __restrict__ rows,
                                                       const int64_t* __restrict__ nbrs,
                                                       const int32_t* __restrict__ m0,
                                                       const int32_t* __restrict__ off,
                                                       double* __restrict__ U, int64_t ldu, int k,
                                                       double rtol) {
  __shared__ double red[kNT / 32];
  __shared__ int ncols;
  const int64_t* R = rows + 10 * (int64_t)blockIdx.x;
  const int p = (int)R[0];
  double* ws = reinterpret_cast<double*>(R[1]);
  const int nb0 = (int)R[4], nb1 = (int)R[5];
  const int o = off[p], mc = m0[p], m = mc - o;
  double* taus = ws + 3;
  double* V = ws + kWsHead;
  double* X = V + (int64_t)mc * k;
  const int tid = threadIdx.x;
  if (tid == 0) ncols = 0;
  __syncthreads();
  {
    int s = 0;
    for (int j = nb0 + tid; j < nb1; j += kNT) {
      const int w = (int)nbrs[4 * (int64_t)j];
      s += m0[w] - off[w];
    }
    if (s) atomicAdd(&ncols, s);
  }
  __syncthreads();
  if (tid == 0) {
    ws[1] = (double)m;
    ws[2] = (double)mc;
  }
  // no neighbour columns (or no rows): nothing is dropped, reference path
  if (ncols == 0 || m <= 0) {
    if (tid == 0) ws[0] = 0.0;
    return;
  }
  double* u = U + R[9] + o;
  for (int j = 0; j < k; ++j)
    for (int i = tid; i < m; i += kNT) X[i + (int64_t)j * mc] = u[i + (int64_t)j * ldu];
  __syncthreads();
  double nrm0 = 0.0;
  for (int j = 0; j < k; ++j) {
    double s = 0.0;
    for (int i = tid; i < m; i += kNT) {
      const double x = X[i + (int64_t)j * mc];
      s += x * x;
    }
    s = block_sum<kNT>(s, red);
    nrm0 = fmax(nrm0, s);
  }
  nrm0 = sqrt(nrm0);
  unsigned used = 0u;
  int r = 0;
  const int tmax = m < k ? m : k;
  for (int t = 0; t < tmax; ++t) {
    double best = -1.0;
    int c = -1;
    for (int j = 0; j < k; ++j) {
      double s = 0.0;
      for (int i = t + tid; i < m; i += kNT) {
        const double x = X[i + (int64_t)j * mc];
        s += x * x;
      }
      s = block_sum<kNT>(s, red);
      if (!((used >> j) & 1u) && s > best) {
        best = s;
        c = j;
      }
    }
    const double eta = sqrt(best);
    if (nrm0 == 0.0 || eta <= rtol * nrm0) break;
    const double x0 = X[t + (int64_t)c * mc];
    const double beta = x0 >= 0.0 ? -eta : eta;
    double* v = V + (int64_t)t * mc;
    for (int i = t + tid; i < m; i += kNT) v[i] = X[i + (int64_t)c * mc] - (i == t ? beta : 0.0);
    __syncthreads();
    double vv = 0.0;
    for (int i = t + tid; i < m; i += kNT) vv += v[i] * v[i];
    vv = block_sum<kNT>(vv, red);
    const double tau = 2.0 / vv;
    for (int j = 0; j < k; ++j) {
      double* x = X + (int64_t)j * mc;
      double d = 0.0;
      for (int i = t + tid; i < m; i += kNT) d += v[i] * x[i];
      d = block_sum<kNT>(d, red) * tau;
      for (int i = t + tid; i < m; i += kNT) x[i] -= d * v[i];
      __syncthreads();
    }
    if (tid == 0) taus[t] = tau;
    used |= 1u << c;
    r = t + 1;
  }
  if (tid == 0) ws[0] = (double)r;
  if (r == 0) return;
  // new coordinates in the rotated slot order: 0 on the first m - r slots,
  // R_u = (H^T u_p)[:r] on the last r
  for (int j = 0; j < k; ++j)
    for (int i = tid; i < m; i += kNT)
      u[i + (int64_t)j * ldu] = i < m - r ? 0.0 : X[(i - (m - r)) + (int64_t)j * mc];
}

// W <- rotate(H^T W) column by column (one CTA per capacity column).
__global__ void __launch_bounds__(128) nk_deflate_kernel(int npanel, const int64_t* __restrict__ rows,
                                                         const int64_t* __restrict__ nbrs,
                                                         const int32_t* __restrict__ m0,
                                                         const int32_t* __restrict__ off) {
  extern __shared__ double col[];
  __shared__ double red[4];
  const int pi = find_row(rows, npanel, 6, blockIdx.x);
  const int64_t* R = rows + 10 * (int64_t)pi;
  const double* ws = reinterpret_cast<const double*>(R[1]);
  const int r = (int)ws[0];
  if (r == 0) return;
  const int p = (int)R[0];
  const int nb0 = (int)R[4], nb1 = (int)R[5];
  int64_t c = (int64_t)blockIdx.x - R[6];
  int j = nb0;
  for (; j < nb1; ++j) {
    const int w = (int)nbrs[4 * (int64_t)j];
    if (c < m0[w]) break;
    c -= m0[w];
  }
  if (j >= nb1) return;
  const int64_t* nr = nbrs + 4 * (int64_t)j;
  const int w = (int)nr[0];
  if (c >= m0[w] - off[w]) return;   // capacity beyond the live columns
  const int offp = off[p], ldp = m0[p];
  const int m = (int)ws[1];
  double* blk = reinterpret_cast<double*>(nr[1]);
  double* base;
  int64_t stride;
  if (nr[2] == 0) {
    base = blk + (int64_t)offp + (int64_t)(off[w] + c) * ldp;
    stride = 1;
  } else {
    base = blk + (int64_t)(off[w] + c) + (int64_t)offp * m0[w];
    stride = m0[w];
  }
  const int tid = threadIdx.x;
  for (int i = tid; i < m; i += 128) col[i] = base[(int64_t)i * stride];
  __syncthreads();
  const double* V = ws + kWsHead;
  const double* taus = ws + 3;
  for (int t = 0; t < r; ++t) {
    const double* v = V + (int64_t)t * ldp;
    double d = 0.0;
    for (int i = t + tid; i < m; i += 128) d += v[i] * col[i];
    d = block_sum<128>(d, red) * taus[t];
    for (int i = t + tid; i < m; i += 128) col[i] -= d * v[i];
    __syncthreads();
  }
  for (int s = tid; s < m; s += 128) {
    const int i = s < m - r ? s + r : s - (m - r);
    base[(int64_t)s * stride] = col[i];
  }
}

// Qfin column j (one CTA per capacity column of m0[p]):
//   j < kc2: H [0_r; q2[:, j]];  kc2 <= j < kc2 + r: H e_{j - kc2};
//   j >= kc2 + r: H [0_r; q2[:, j - r]]
// r == 0: plain copy of the RRQR's factor (q2 is then m x m).
__global__ void __launch_bounds__(128) nk_qform_kernel(int npanel, const int64_t* __restrict__ rows,
                                                       const int64_t* __restrict__ events) {
  extern __shared__ double e[];
  __shared__ double red[4];
  const int pi = find_row(rows, npanel, 7, blockIdx.x);
  const int64_t* R = rows + 10 * (int64_t)pi;
  const double* ws = reinterpret_cast<const double*>(R[1]);
  const double* q2 = reinterpret_cast<const double*>(R[2]);
  double* Q = reinterpret_cast<double*>(R[3]);
  const int r = (int)ws[0], m = (int)ws[1], mc = (int)ws[2];
  const int j = (int)((int64_t)blockIdx.x - R[7]);
  if (j >= m) return;
  const int tid = threadIdx.x;
  const int me = m - r;
  if (r == 0) {
    for (int i = tid; i < m; i += 128) Q[i + (int64_t)j * m] = q2[i + (int64_t)j * m];
    return;
  }
  const int kc2 = (int)events[12 * R[8] + 4] - r;
  int src = -1, unit = -1;
  if (j < kc2) src = j;
  else if (j < kc2 + r) unit = j - kc2;
  else src = j - r;
  for (int i = tid; i < m; i += 128) {
    double x;
    if (i < r) x = (i == unit) ? 1.0 : 0.0;
    else x = src >= 0 ? q2[(i - r) + (int64_t)src * me] : 0.0;
    e[i] = x;
  }
  __syncthreads();
  const double* V = ws + kWsHead;
  const double* taus = ws + 3;
  for (int t = r - 1; t >= 0; --t) {
    const double* v = V + (int64_t)t * mc;
    double d = 0.0;
    for (int i = t + tid; i < m; i += 128) d += v[i] * e[i];
    d = block_sum<128>(d, red) * taus[t];
    for (int i = t + tid; i < m; i += 128) e[i] -= d * v[i];
    __syncthreads();
  }
  for (int i = tid; i < m; i += 128) Q[i + (int64_t)j * m] = e[i];
}

}  // namespace

extern "C" {

int spand_nk_rescale(int ntask, const int64_t* rows, const int32_t* m0, const int32_t* off,
                     double* U, int64_t ldu, int k, int vmax, void* stream) {
  if (ntask < 0 || k < 0 || k > kMaxK || vmax < 0 || vmax > 6144) return -1;
  if (ntask == 0 || k == 0) return 0;
  const size_t smem = (size_t)(vmax > 0 ? vmax : 1) * sizeof(double);
  nk_rescale_kernel<<<ntask * k, kNT, smem, as_stream(stream)>>>(rows, m0, off, U, ldu, k);
  SPAND_CHECK_LAUNCH();
  return 0;
}

int spand_nk_basis(int npanel, const int64_t* rows, const int64_t* nbrs, const int32_t* m0,
                   const int32_t* off, double* U, int64_t ldu, int k, double rtol, void* stream) {
  if (npanel < 0 || k < 0 || k > kMaxK) return -1;
  if (npanel == 0) return 0;
  nk_basis_kernel<<<npanel, kNT, 0, as_stream(stream)>>>(rows, nbrs, m0, off, U, ldu, k, rtol);
  SPAND_CHECK_LAUNCH();
  return 0;
}

int spand_nk_deflate(int npanel, int64_t ncols, const int64_t* rows, const int64_t* nbrs,
                     const int32_t* m0, const int32_t* off, int vmax, void* stream) {
  if (npanel < 0 || ncols < 0 || vmax < 0 || vmax > 6144) return -1;
  if (npanel == 0 || ncols == 0) return 0;
  const size_t smem = (size_t)(vmax > 0 ? vmax : 1) * sizeof(double);
  nk_deflate_kernel<<<(unsigned)ncols, 128, smem, as_stream(stream)>>>(npanel, rows, nbrs, m0, off);
  SPAND_CHECK_LAUNCH();
  return 0;
}

int spand_nk_qform(int npanel, int64_t ncols, const int64_t* rows, const int64_t* events, int vmax,
                   void* stream) {
  if (npanel < 0 || ncols < 0 || vmax < 0 || vmax > 6144) return -1;
  if (npanel == 0 || ncols == 0) return 0;
  const size_t smem = (size_t)(vmax > 0 ? vmax : 1) * sizeof(double);
  nk_qform_kernel<<<(unsigned)ncols, 128, smem, as_stream(stream)>>>(npanel, rows, events);
  SPAND_CHECK_LAUNCH();
  return 0;
}

}  // extern "C"
