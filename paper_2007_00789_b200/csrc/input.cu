// Input side on the device: the BASELINE finite-volume
// generator and the Jacobi prescale, written straight into device CSR.
//
// fv: -div(a grad u) on a 2D/3D cell grid with a piecewise-constant
// coefficient (one value per block of `block` cells per axis), harmonic
// faces, Dirichlet faces adding the cell's own coefficient -- the package's
// host generator sparse.diffusion_fv / log_uniform_block_field (the
// reference's boundary convention, sparse.py:278-282), reproduced bit for
// bit: every face weight is 2 a_lo a_hi / (a_lo + a_hi) evaluated in the
// same order, and the diagonal accumulates its terms in the host's order
// (per axis: upper face, lower face, first boundary, last boundary).
// Columns of a row ascend (lower neighbours by decreasing stride, the
// diagonal, upper neighbours by increasing stride).
//
// jacobi: A' = D^-1/2 A D^-1/2, b' = D^-1/2 b with s = 1 / sqrt(diag) and
// a'_ij = a_ij (s_i s_j) (reference sparse.py:290-308): the product of the
// two scales is formed first, so (i, j) and (j, i) round alike.
#include "common.cuh"
#include "../../include/spand_b200.h"

namespace {
constexpr int kT = 256;

struct Grid {
  int nd;
  int64_t d[3], s[3];
  int block;
  int64_t nb[3];
};

__device__ __forceinline__ double coef(const Grid& g, const double* bv, const int64_t* x) {
  int64_t q = 0;
  for (int ax = 0; ax < g.nd; ++ax) q = q * g.nb[ax] + x[ax] / g.block;
  return bv[q];
}

__device__ __forceinline__ double harmonic(double a1, double a2) {
  return 2.0 * a1 * a2 / (a1 + a2);
}

__device__ __forceinline__ void coords(const Grid& g, int64_t r, int64_t* x) {
  for (int ax = g.nd - 1; ax >= 0; --ax) {
    x[ax] = r % g.d[ax];
    r /= g.d[ax];
  }
}

__global__ void __launch_bounds__(kT) fv_count_kernel(Grid g, int64_t n, int64_t* cnt) {
  const int64_t r = (int64_t)blockIdx.x * kT + threadIdx.x;
  if (r >= n) return;
  int64_t x[3];
  coords(g, r, x);
  int64_t c = 1;
  for (int ax = 0; ax < g.nd; ++ax) c += (x[ax] > 0) + (x[ax] + 1 < g.d[ax]);
  cnt[r] = c;
}

__global__ void __launch_bounds__(kT)
fv_fill_kernel(Grid g, int64_t n, const double* __restrict__ bv,
               const int64_t* __restrict__ rp, int64_t* __restrict__ ci,
               double* __restrict__ va) {
  const int64_t r = (int64_t)blockIdx.x * kT + threadIdx.x;
  if (r >= n) return;
  int64_t x[3];
  coords(g, r, x);
  const double ar = coef(g, bv, x);
  double wl[3], wu[3];
  double diag = 0.0;
  for (int ax = 0; ax < g.nd; ++ax) {
    wl[ax] = wu[ax] = 0.0;
    int64_t y[3] = {x[0], x[1], x[2]};
    if (x[ax] + 1 < g.d[ax]) {   // this cell is the lower one of a face
      y[ax] = x[ax] + 1;
      wu[ax] = harmonic(ar, coef(g, bv, y));
      diag += wu[ax];
    }
    if (x[ax] > 0) {             // this cell is the upper one of a face
      y[ax] = x[ax] - 1;
      wl[ax] = harmonic(coef(g, bv, y), ar);
      diag += wl[ax];
    }
    if (x[ax] == 0) diag += ar;
    if (x[ax] == g.d[ax] - 1) diag += ar;
  }
  int64_t e = rp[r];
  for (int ax = 0; ax < g.nd; ++ax)   // lower neighbours, largest stride first
    if (x[ax] > 0) {
      ci[e] = r - g.s[ax];
      va[e++] = -wl[ax];
    }
  ci[e] = r;
  va[e++] = diag;
  for (int ax = g.nd - 1; ax >= 0; --ax)   // upper neighbours, smallest stride first
    if (x[ax] + 1 < g.d[ax]) {
      ci[e] = r + g.s[ax];
      va[e++] = -wu[ax];
    }
}

__global__ void __launch_bounds__(kT)
jacobi_scale_kernel(int64_t n, const int64_t* __restrict__ rp, const int64_t* __restrict__ ci,
                    double* __restrict__ va, const double* __restrict__ s) {
  const int64_t r = (int64_t)blockIdx.x * kT + threadIdx.x;
  if (r >= n) return;
  const double sr = s[r];
  for (int64_t e = rp[r]; e < rp[r + 1]; ++e) va[e] = va[e] * (sr * s[ci[e]]);
}

__global__ void __launch_bounds__(kT)
jacobi_diag_kernel(int64_t n, const int64_t* __restrict__ rp, const int64_t* __restrict__ ci,
                   const double* __restrict__ va, double* __restrict__ diag,
                   double* __restrict__ s, double* __restrict__ b, int* __restrict__ bad) {
  const int64_t r = (int64_t)blockIdx.x * kT + threadIdx.x;
  if (r >= n) return;
  double d = 0.0;
  for (int64_t e = rp[r]; e < rp[r + 1]; ++e)
    if (ci[e] == r) d = va[e];
  diag[r] = d;
  if (!(d > 0.0)) atomicExch(bad, 1);
  const double sr = 1.0 / sqrt(d);
  s[r] = sr;
  if (b) b[r] = b[r] * sr;
}
}  // namespace

extern "C" {

// row counts of the grid's CSR (cnt[n]); the caller forms row_ptr
int spand_fv_counts(int nd, const int64_t* dims, int64_t* cnt, void* stream) {
  if (nd < 2 || nd > 3) return -1;
  Grid g{};
  g.nd = nd;
  int64_t n = 1;
  for (int ax = 0; ax < nd; ++ax) {
    g.d[ax] = dims[ax];
    n *= dims[ax];
  }
  if (n <= 0) return 0;
  fv_count_kernel<<<(unsigned)((n + kT - 1) / kT), kT, 0, as_stream(stream)>>>(g, n, cnt);
  SPAND_CHECK_LAUNCH();
  return 0;
}

// fill col_idx / values given row_ptr (n + 1); bv: block values in C order
// over ceil-free block counts dims[ax] / block
int spand_fv_fill(int nd, const int64_t* dims, int block, const double* bv, const int64_t* rp,
                  int64_t* ci, double* va, void* stream) {
  if (nd < 2 || nd > 3 || block < 1) return -1;
  Grid g{};
  g.nd = nd;
  g.block = block;
  int64_t n = 1;
  for (int ax = 0; ax < nd; ++ax) {
    g.d[ax] = dims[ax];
    g.nb[ax] = dims[ax] / block;
    if (g.nb[ax] * block != dims[ax]) return -2;
    n *= dims[ax];
  }
  int64_t st = 1;
  for (int ax = nd - 1; ax >= 0; --ax) {
    g.s[ax] = st;
    st *= g.d[ax];
  }
  if (n <= 0) return 0;
  fv_fill_kernel<<<(unsigned)((n + kT - 1) / kT), kT, 0, as_stream(stream)>>>(g, n, bv, rp, ci,
                                                                            va);
  SPAND_CHECK_LAUNCH();
  return 0;
}

// in place: diag[n] <- diagonal, s[n] <- 1 / sqrt(diag), b[n] <- b s (b may
// be null), values <- values (s_i s_j); *bad (zeroed by the caller) is set
// when a diagonal entry is not positive (the outputs are then meaningless)
int spand_jacobi_prescale(int64_t n, const int64_t* rp, const int64_t* ci, double* va,
                          double* diag, double* s, double* b, int* bad, void* stream) {
  if (n < 0) return -1;
  if (n == 0) return 0;
  const unsigned grid = (unsigned)((n + kT - 1) / kT);
  jacobi_diag_kernel<<<grid, kT, 0, as_stream(stream)>>>(n, rp, ci, va, diag, s, b, bad);
  jacobi_scale_kernel<<<grid, kT, 0, as_stream(stream)>>>(n, rp, ci, va, s);
  SPAND_CHECK_LAUNCH();
  return 0;
}

}  // extern "C"
