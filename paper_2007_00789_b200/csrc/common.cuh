// Shared helpers for the spand_b200 sm_100a kernels.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#define SPAND_CHECK_LAUNCH()                                   \
  do {                                                         \
    cudaError_t _e = cudaGetLastError();                       \
    if (_e != cudaSuccess) return (int)_e;                     \
  } while (0)

static inline cudaStream_t as_stream(void* s) { return (cudaStream_t)s; }

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// block-wide sum, result broadcast to all threads (fixed reduction order)
template <int NT>
__device__ __forceinline__ double block_sum(double v, double* sh) {
  v = warp_sum(v);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) sh[w] = v;
  __syncthreads();
  double t = 0.0;
  if (w == 0) {
    t = (l < NT / 32) ? sh[l] : 0.0;
    t = warp_sum(t);
    if (l == 0) sh[0] = t;
  }
  __syncthreads();
  t = sh[0];
  __syncthreads();
  return t;
}

// Operand descriptor (7 x int64): {ptr, rc, cc, rskip, cskip, rcount, ccount}
struct Opnd {
  double* p;  // pointer to element (row0, col0)
  int ld;
  int rows, cols;
};

__device__ __forceinline__ Opnd load_opnd(const int64_t* d, const int32_t* m0,
                                          const int32_t* off) {
  Opnd o;
  const int rc = (int)d[1], cc = (int)d[2];
  const int rs = (int)d[3], cs = (int)d[4];
  const int rcount = (int)d[5], ccount = (int)d[6];
  const int ld = m0[rc];
  const int r0 = off[rc] + rs, c0 = off[cc] + cs;
  int rows = m0[rc] - r0, cols = m0[cc] - c0;
  if (rows < 0) rows = 0;
  if (cols < 0) cols = 0;
  if (rcount >= 0 && rows > rcount) rows = rcount;
  if (ccount >= 0 && cols > ccount) cols = ccount;
  o.ld = ld;
  o.rows = rows;
  o.cols = cols;
  o.p = reinterpret_cast<double*>(d[0]) + (int64_t)r0 + (int64_t)c0 * ld;
  return o;
}
