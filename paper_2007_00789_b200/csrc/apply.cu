// Preconditioner apply: batched dense GEMV tiles + ordered scatter.
// Replaces the per-operator NumPy GEMVs and fancy-index gathers/scatters of
// schemes.py:102-112,136-140,162-166,188-192 (apply_inv / apply_inv_t).
// HBM-bound: every payload entry is read once per pass, coalesced along the
// column-major storage; vectors are staged in shared memory.
#include <cstdio>

#include "common.cuh"
#include "../../include/spand_b200.h"

namespace {
constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr int kTileOut = 64;
constexpr int kTileK = 2048;

struct Task {
  const double* M;
  int64_t ld;
  int rows, cols, trans, rot, in_kind;
  const void* in;
};

__device__ __forceinline__ Task load_task(const int64_t* t) {
  Task k;
  k.M = reinterpret_cast<const double*>(t[0]);
  k.ld = t[1];
  k.rows = (int)t[2];
  k.cols = (int)t[3];
  k.trans = (int)t[4];
  k.rot = (int)t[5];
  k.in_kind = (int)t[6];
  k.in = reinterpret_cast<const void*>(t[7]);
  return k;
}

__device__ __forceinline__ int phys_col(int j, int rot, int cols) {
  int c = j + rot;
  return c >= cols ? c - cols : c;
}

__global__ void __launch_bounds__(kThreads)
gemv_tiles_kernel(const int64_t* __restrict__ tiles, const int64_t* __restrict__ tasks,
                  const double* __restrict__ x, int64_t ldx, double* __restrict__ scratch,
                  int64_t ldscr, int nvec) {
  __shared__ double vin[kTileK];
  __shared__ double part[kWarps][kTileOut];
  const int64_t* tr = tiles + 8 * (int64_t)blockIdx.x;
  const Task T = load_task(tasks + 8 * tr[0]);
  const int ob = (int)tr[1], oc = (int)tr[2], kb = (int)tr[3], kc = (int)tr[4];
  double* out = scratch + tr[5];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int v = 0; v < nvec; ++v) {
    const double* xv = x + v * ldx;
    __syncthreads();
    for (int k = threadIdx.x; k < kc; k += kThreads) {
      const int kk = kb + k;
      vin[k] = T.in_kind == 0 ? xv[reinterpret_cast<const int32_t*>(T.in)[kk]]
                              : reinterpret_cast<const double*>(T.in)[kk + v * ldx];
    }
    __syncthreads();
    if (T.trans == 0) {
      // y[r] = sum_c M[r, c] in[c]; warp w takes columns w, w+8, ...;
      // lane takes rows ob+lane and ob+lane+32 (coalesced down a column)
      double a0 = 0.0, a1 = 0.0;
      const int r0 = ob + lane, r1 = ob + lane + 32;
      const bool ok0 = lane < oc, ok1 = lane + 32 < oc;
      int c = w;
      for (; c + 3 * kWarps < kc; c += 4 * kWarps) {
        double m0v[4], m1v[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const double* col = T.M + (int64_t)phys_col(kb + c + u * kWarps, T.rot, T.cols) * T.ld;
          m0v[u] = ok0 ? __ldg(col + r0) : 0.0;
          m1v[u] = ok1 ? __ldg(col + r1) : 0.0;
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const double xi = vin[c + u * kWarps];
          a0 += m0v[u] * xi;
          a1 += m1v[u] * xi;
        }
      }
      for (; c < kc; c += kWarps) {
        const double* col = T.M + (int64_t)phys_col(kb + c, T.rot, T.cols) * T.ld;
        const double xi = vin[c];
        if (ok0) a0 += __ldg(col + r0) * xi;
        if (ok1) a1 += __ldg(col + r1) * xi;
      }
      part[w][lane] = a0;
      part[w][lane + 32] = a1;
    } else {
      // y[j] = sum_r M[r, j] in[r]
      // warp w owns columns w, w + 8, ... (narrow tiles still use every warp)
      for (int jj = 0; jj < kTileOut / kWarps; jj += 2) {
        const int j = w + kWarps * jj, j1 = w + kWarps * (jj + 1);
        if (j >= oc) break;
        double a = 0.0, b = 0.0;
        const bool okj = true, okj1 = j1 < oc;
        const double* col = T.M + (int64_t)phys_col(ob + j, T.rot, T.cols) * T.ld + kb;
        const double* col1 = T.M + (int64_t)phys_col(okj1 ? ob + j1 : ob, T.rot, T.cols) * T.ld + kb;
        int r = lane;
        for (; r + 96 < kc; r += 128) {
          double p[4], q[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            p[u] = okj ? __ldg(col + r + 32 * u) : 0.0;
            q[u] = okj1 ? __ldg(col1 + r + 32 * u) : 0.0;
          }
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            a += p[u] * vin[r + 32 * u];
            b += q[u] * vin[r + 32 * u];
          }
        }
        for (; r < kc; r += 32) {
          if (okj) a += __ldg(col + r) * vin[r];
          if (okj1) b += __ldg(col1 + r) * vin[r];
        }
        a = warp_sum(a);
        b = warp_sum(b);
        if (lane == 0) {
          part[0][j] = a;
          if (okj1) part[0][j1] = b;
        }
      }
    }
    __syncthreads();
    if (threadIdx.x < oc) {
      double s;
      if (T.trans == 0) {
        s = 0.0;
#pragma unroll
        for (int i = 0; i < kWarps; ++i) s += part[i][threadIdx.x];
      } else {
        s = part[0][threadIdx.x];
      }
      out[threadIdx.x + v * ldscr] = s;
    }
  }
}

// Warp-granular GEMV work items (the apply's hot kernel).  An item (task,
// ob, oc, kb, kc, out_off) is a tile (packed in 2 int64, see below), but
// it is processed by ONE warp and sized by the host to ~16-32 KB of payload:
//   trans 0 (y = M x, outputs are rows): oc <= 128 rows, lane holds rows
//     ob + lane + 32 q (q < 4), columns streamed two at a time;
//   trans 1 (y = M^T x, outputs are columns): oc <= 4 columns, lanes stride
//     the kc rows of all oc columns at once (one input load per row, two
//     row steps in flight).
// A grid of persistent warps walks the items (warp g takes g, g + W, ...),
// so thousands of tiny operators share CTAs and big ones are split evenly.
// <= 64 registers: 4 CTAs (32 warps) per SM.
constexpr int kItemRows = 128;   // trans 0: max rows per item
constexpr int kItemCols = 4;     // trans 1: max columns per item

template <bool kCoherent = false>
__device__ __forceinline__ double load_in(const Task& T, const double* xv, int64_t ldx, int v,
                                          int kk) {
  // kCoherent: x changes while the kernel runs (dataflow apply): L2 loads
  if (kCoherent)   // plain loads: valid after the dependency acquire (L1 invalidated)
    return T.in_kind == 0 ? xv[reinterpret_cast<const int32_t*>(T.in)[kk]]
                          : reinterpret_cast<const double*>(T.in)[kk + v * ldx];
  return T.in_kind == 0 ? xv[reinterpret_cast<const int32_t*>(T.in)[kk]]
                        : __ldg(reinterpret_cast<const double*>(T.in) + kk + v * ldx);
}

// NV right-hand sides per launch (x and scratch column-major with leading
// dimensions ldx / ldscr): every payload element is loaded once and used
// for all NV vectors (multi-RHS apply, reference factorize.py:262-267).
// one work item by one warp (see gemv_items_kernel)
template <int NV, bool kCoherent>
__device__ __forceinline__ void gemv_item(int it, const int64_t* __restrict__ items,
                                          const int64_t* __restrict__ tasks, const double* x,
                                          int64_t ldx, double* scratch, int64_t ldscr, int v0) {
  const int lane = threadIdx.x & 31;
  {
    // packed item (2 x int64): {task << 32 | ob << 12 | oc, out_off << 28 | kb << 11 | kc}
    const int64_t w0 = __ldg(items + 2 * (int64_t)it), w1 = __ldg(items + 2 * (int64_t)it + 1);
    const int64_t t0 = w0 >> 32;
    const int ob = (int)((w0 >> 12) & 0xfffff), oc = (int)(w0 & 0xfff);
    const int kb = (int)((w1 >> 11) & 0x1ffff), kc = (int)(w1 & 0x7ff);
    const int64_t oo = w1 >> 28;
    const Task T = load_task(tasks + 8 * t0);
    if (T.trans == 0) {
      double acc[NV][4];
#pragma unroll
      for (int v = 0; v < NV; ++v)
#pragma unroll
        for (int q = 0; q < 4; ++q) acc[v][q] = 0.0;
      int c = 0;
      for (; c + 1 < kc; c += 2) {
        double x0[NV], x1[NV];
#pragma unroll
        for (int v = 0; v < NV; ++v) {
          x0[v] = load_in<kCoherent>(T, x + (v0 + v) * ldx, ldx, v0 + v, kb + c);
          x1[v] = load_in<kCoherent>(T, x + (v0 + v) * ldx, ldx, v0 + v, kb + c + 1);
        }
        const double* c0 = T.M + (int64_t)phys_col(kb + c, T.rot, T.cols) * T.ld + ob;
        const double* c1 = T.M + (int64_t)phys_col(kb + c + 1, T.rot, T.cols) * T.ld + ob;
        double m0v[4], m1v[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int r = lane + 32 * q;
          m0v[q] = r < oc ? __ldg(c0 + r) : 0.0;
          m1v[q] = r < oc ? __ldg(c1 + r) : 0.0;
        }
#pragma unroll
        for (int v = 0; v < NV; ++v)
#pragma unroll
          for (int q = 0; q < 4; ++q) acc[v][q] += m0v[q] * x0[v] + m1v[q] * x1[v];
      }
      if (c < kc) {
        const double* c0 = T.M + (int64_t)phys_col(kb + c, T.rot, T.cols) * T.ld + ob;
        double m0v[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int r = lane + 32 * q;
          m0v[q] = r < oc ? __ldg(c0 + r) : 0.0;
        }
#pragma unroll
        for (int v = 0; v < NV; ++v) {
          const double x0 = load_in<kCoherent>(T, x + (v0 + v) * ldx, ldx, v0 + v, kb + c);
#pragma unroll
          for (int q = 0; q < 4; ++q) acc[v][q] += m0v[q] * x0;
        }
      }
#pragma unroll
      for (int v = 0; v < NV; ++v)
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int r = lane + 32 * q;
          if (r < oc) scratch[oo + (v0 + v) * ldscr + r] = acc[v][q];
        }
    } else {
      double acc[NV][kItemCols];
      const double* col[kItemCols];
#pragma unroll
      for (int j = 0; j < kItemCols; ++j) {
#pragma unroll
        for (int v = 0; v < NV; ++v) acc[v][j] = 0.0;
        col[j] = T.M + (int64_t)phys_col(ob + (j < oc ? j : 0), T.rot, T.cols) * T.ld + kb;
      }
      int r = lane;
      for (; r + 32 < kc; r += 64) {
        double in2[NV][2], p[2][kItemCols];
#pragma unroll
        for (int v = 0; v < NV; ++v)
#pragma unroll
          for (int u = 0; u < 2; ++u) in2[v][u] = load_in<kCoherent>(T, x + (v0 + v) * ldx, ldx, v0 + v, kb + r + 32 * u);
#pragma unroll
        for (int u = 0; u < 2; ++u)
#pragma unroll
          for (int j = 0; j < kItemCols; ++j) p[u][j] = j < oc ? __ldg(col[j] + r + 32 * u) : 0.0;
#pragma unroll
        for (int v = 0; v < NV; ++v)
#pragma unroll
          for (int u = 0; u < 2; ++u)
#pragma unroll
            for (int j = 0; j < kItemCols; ++j) acc[v][j] += p[u][j] * in2[v][u];
      }
      for (; r < kc; r += 32) {
        double p[kItemCols];
#pragma unroll
        for (int j = 0; j < kItemCols; ++j) p[j] = j < oc ? __ldg(col[j] + r) : 0.0;
#pragma unroll
        for (int v = 0; v < NV; ++v) {
          const double i0 = load_in<kCoherent>(T, x + (v0 + v) * ldx, ldx, v0 + v, kb + r);
#pragma unroll
          for (int j = 0; j < kItemCols; ++j) acc[v][j] += p[j] * i0;
        }
      }
#pragma unroll
      for (int v = 0; v < NV; ++v) {
#pragma unroll
        for (int j = 0; j < kItemCols; ++j) acc[v][j] = warp_sum(acc[v][j]);
        if (lane < oc) {
          double s = acc[v][0];
#pragma unroll
          for (int j = 1; j < kItemCols; ++j)
            if (lane == j) s = acc[v][j];
          scratch[oo + (v0 + v) * ldscr + lane] = s;
        }
      }
    }
  }
}

template <int NV>
__global__ void __launch_bounds__(kThreads, NV == 1 ? 4 : 2)
gemv_items_kernel(int nitem, const int64_t* __restrict__ items, const int64_t* __restrict__ tasks,
                  const double* __restrict__ x, int64_t ldx, double* __restrict__ scratch,
                  int64_t ldscr, int v0) {
  const int W = gridDim.x * kWarps;
  for (int it = blockIdx.x * kWarps + (threadIdx.x >> 5); it < nitem; it += W)
    gemv_item<NV, false>(it, items, tasks, x, ldx, scratch, ldscr, v0);
}

__global__ void __launch_bounds__(kThreads)
scatter_kernel(int nout, const int64_t* __restrict__ dst, const int64_t* __restrict__ mode,
               const int64_t* __restrict__ ptr, const int64_t* __restrict__ src,
               double* __restrict__ x, int64_t ldx, const double* __restrict__ scratch,
               int64_t ldscr, int nvec) {
  const int e = blockIdx.x * kThreads + threadIdx.x;
  if (e >= nout) return;
  const int64_t b = ptr[e], f = ptr[e + 1];
  const int64_t d = dst[e];
  const int md = (int)mode[e];
  for (int v = 0; v < nvec; ++v) {
    double s = 0.0;
    for (int64_t t = b; t < f; ++t) s += scratch[src[t] + v * ldscr];
    double* xd = x + d + v * ldx;
    if (md == 0) *xd = s;
    else *xd -= s;
  }
}

// Run-structured ordered accumulation: chunk row (8 int64)
// {dst, len, mode, cb, ce, eoff, idx, splits}; element i < len of the chunk is
// x[d] with d = dst + eoff + i (idx == 0) or ((int32*)idx)[eoff + i]; the value is
// the sum of scratch[contrib[c] + eoff + i] over c in [cb, ce).  The
// contributions come in four summation groups (splits: 16-bit offsets of
// groups 1-3 from cb), each summed strictly in order by its own thread group,
// the group sums combined in a fixed order: an image that drops exact-zero
// parts gives the same bits (collect.cpp compile_phase).
__device__ __forceinline__ void group_range(int64_t cb, int64_t ce, int64_t splits, int g,
                                            int64_t& gb, int64_t& ge) {
  const int64_t s1 = cb + (splits & 0xffff), s2 = cb + ((splits >> 16) & 0xffff),
                s3 = cb + ((splits >> 32) & 0xffff);
  gb = g == 0 ? cb : (g == 1 ? s1 : (g == 2 ? s2 : s3));
  ge = g == 0 ? s1 : (g == 1 ? s2 : (g == 2 ? s3 : ce));
}

__device__ __forceinline__ void runs_chunk(const int64_t* __restrict__ ch,
                                           const int64_t* __restrict__ contrib, double* x,
                                           int64_t ldx, const double* scratch, int64_t ldscr,
                                           int nvec, int v0, double* part);

__global__ void __launch_bounds__(kThreads)
runs_kernel(const int64_t* __restrict__ chunks, const int64_t* __restrict__ contrib,
            double* __restrict__ x, int64_t ldx, const double* __restrict__ scratch,
            int64_t ldscr, int nvec) {
  __shared__ double part[kThreads];
  runs_chunk(chunks + 8 * (int64_t)blockIdx.x, contrib, x, ldx, scratch, ldscr, nvec, 0, part);
}

// one chunk by one CTA (vectors v0 .. v0 + nvec - 1)
__device__ __forceinline__ void runs_chunk(const int64_t* __restrict__ ch,
                                           const int64_t* __restrict__ contrib, double* x,
                                           int64_t ldx, const double* scratch, int64_t ldscr,
                                           int nvec, int v0, double* part) {
  const int len = (int)ch[1];
  const int i = threadIdx.x & 63, g = threadIdx.x >> 6;
  const int64_t dst = ch[0], cb = ch[3], ce = ch[4], eoff = ch[5], idx = ch[6];
  const int md = (int)ch[2];
  int64_t gb, ge;
  group_range(cb, ce, ch[7], g, gb, ge);
  for (int v = v0; v < v0 + nvec; ++v) {
    double s = 0.0;
    if (i < len) {
      const double* sv = scratch + eoff + i + (int64_t)v * ldscr;
      int64_t c = gb;
      for (; c + 3 < ge; c += 4) {
        const double v0 = sv[__ldg(contrib + c)], v1 = sv[__ldg(contrib + c + 1)],
                     v2 = sv[__ldg(contrib + c + 2)], v3 = sv[__ldg(contrib + c + 3)];
        s += v0;
        s += v1;
        s += v2;
        s += v3;
      }
      for (; c < ge; ++c) s += sv[__ldg(contrib + c)];
    }
    __syncthreads();
    part[threadIdx.x] = s;
    __syncthreads();
    if (threadIdx.x < len) {
      const double t = (part[i] + part[i + 64]) + (part[i + 128] + part[i + 192]);
      const int64_t d = idx ? (int64_t)reinterpret_cast<const int32_t*>(idx)[eoff + i] : dst + eoff + i;
      double* xd = x + d + (int64_t)v * ldx;
      if (md == 0) *xd = t;
      else *xd -= t;
    }
  }
}

// sum of one output of a chunk (runs_kernel layout) by one thread (the
// dataflow kernel's warp path)
__device__ __forceinline__ double chunk_sum(const double* sv, const int64_t* __restrict__ contrib,
                                            int64_t cb, int64_t ce, int64_t splits) {
  double p[4];   // the four summation groups, as runs_kernel
#pragma unroll
  for (int g = 0; g < 4; ++g) {
    int64_t gb, ge;
    group_range(cb, ce, splits, g, gb, ge);
    double s = 0.0;
    for (int64_t c = gb; c < ge; ++c) s += __ldcg(sv + __ldg(contrib + c));
    p[g] = s;
  }
  return (p[0] + p[1]) + (p[2] + p[3]);
}

// ---- persistent pass: one cooperative launch runs every phase of a pass
// (items, grid barrier, accumulation chunks, grid barrier) instead of two
// launches per phase (~690 per apply_m).  Grid barrier: arrival counter +
// release word, as the RRQR group barrier.
__device__ __forceinline__ void pass_barrier(unsigned* bar, unsigned& gen) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    ++gen;
    if (atomicAdd(bar, 1u) + 1u == gen * gridDim.x) {
      asm volatile("st.release.gpu.global.u32 [%0], %1;\n" ::"l"(bar + 1), "r"(gen) : "memory");
    } else {
      unsigned v;
      do {
        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];\n" : "=r"(v) : "l"(bar + 1) : "memory");
      } while (v < gen);
    }
    __threadfence();
  }
  __syncthreads();
}

template <int NV>
__global__ void __launch_bounds__(kThreads, NV == 1 ? 4 : 2)
pass_kernel(int nphase, const int64_t* __restrict__ ph, const int64_t* __restrict__ image,
            double* x, int64_t ldx, double* scratch, int64_t ldscr, unsigned* bar, int v0) {
  __shared__ double part[kThreads];
  unsigned gen = 0;
  const int warp = threadIdx.x >> 5;
  const int W = gridDim.x * kWarps;
  for (int q = 0; q < nphase; ++q) {
    const int64_t* r = ph + 10 * (int64_t)q;
    const int64_t* tasks = image + r[0];
    const int64_t* items = image + r[2];
    const int nitem = (int)r[3];
    for (int it = blockIdx.x * kWarps + warp; it < nitem; it += W)
      gemv_item<NV, true>(it, items, tasks, x, ldx, scratch, ldscr, v0);
    pass_barrier(bar, gen);
    const int64_t* chunks = image + r[4];
    const int64_t* contrib = image + r[6];
    const int nch = (int)r[5];
    for (int c = blockIdx.x; c < nch; c += gridDim.x)
      runs_chunk(chunks + 8 * (int64_t)c, contrib, x, ldx, scratch, ldscr, NV, v0, part);
    pass_barrier(bar, gen);
  }
}

// ---- dataflow apply: the whole apply_m (forward + backward) in one launch.
// Persistent warps take units (work items, accumulation chunks) in phase
// order from a global counter, kDisp at a time, wait for their dependency
// counters (host schedule, collect.cpp build_dataflow) and bump their own
// when done: no grid-wide barrier between the ~690 phases, independent
// subtrees of the nested dissection overlap.  Sums keep a fixed order
// (deterministic).  Dependencies only point to earlier units, so warps
// holding earlier units always make progress (no deadlock); a warp flushes
// its pending signals before it waits.
__device__ __forceinline__ unsigned long long ld_acq_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];\n" : "=l"(v) : "l"(p) : "memory");
  return v;
}

// one accumulation chunk (runs_kernel layout, <= 64 outputs) by one warp
template <int NV>
__device__ __forceinline__ void chunk_warp(const int64_t* __restrict__ ch,
                                           const int64_t* __restrict__ contrib, double* x,
                                           int64_t ldx, const double* scratch, int64_t ldscr,
                                           int v0) {
  const int lane = threadIdx.x & 31;
  const int64_t dst = __ldg(ch), eoff = __ldg(ch + 5), cb = __ldg(ch + 3), ce = __ldg(ch + 4);
  const int64_t sp = __ldg(ch + 7);
  const int len = (int)__ldg(ch + 1), md = (int)__ldg(ch + 2);
  const int32_t* idx = reinterpret_cast<const int32_t*>(__ldg(ch + 6));
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int i = lane + 32 * h;
    if (i >= len) continue;
    const int64_t e = eoff + i;
    const int64_t d = idx ? (int64_t)idx[e] : dst + e;
#pragma unroll
    for (int v = 0; v < NV; ++v) {
      const double t = chunk_sum(scratch + e + (int64_t)(v0 + v) * ldscr, contrib, cb, ce, sp);
      double* xd = x + d + (int64_t)(v0 + v) * ldx;
      *xd = md == 0 ? t : __ldcg(xd) - t;
    }
  }
}

constexpr int kDisp = 1;   // units per dispatch

template <int NV>
__global__ void __launch_bounds__(kThreads, NV == 1 ? 4 : 2)
dataflow_kernel(int64_t nunit, const int64_t* __restrict__ units, const int64_t* __restrict__ deps,
                unsigned long long* ctrs, const int64_t* __restrict__ ph,
                const int64_t* __restrict__ image, double* x, int64_t ldx, double* scratch,
                int64_t ldscr, int v0) {
  const int lane = threadIdx.x & 31;
  // pending signals (lane 0): consecutive units bumping the same counters
  int64_t pc0 = -1, pc1 = -1;
  unsigned long long pn0 = 0, pn1 = 0;
  auto flush = [&]() {
    __syncwarp();
    if (lane == 0 && (pn0 || pn1)) {
      __threadfence();
      if (pn0) atomicAdd(ctrs + pc0, pn0);
      if (pn1) atomicAdd(ctrs + pc1, pn1);
    }
    pn0 = pn1 = 0;
    pc0 = pc1 = -1;
  };
#ifdef SPAND_DF_STATS
  long long st_wait = 0, st_item = 0, st_chunk = 0, st_disp = 0, st_flush = 0, n_item = 0, n_chunk = 0;
  long long t_ = clock64();
#define DFT(var) do { long long _n = clock64(); var += _n - t_; t_ = _n; } while (0)
#else
#define DFT(var) do {} while (0)
#endif
  for (;;) {
    long long u0 = 0;
    DFT(st_flush);
    if (lane == 0) u0 = (long long)atomicAdd(ctrs, (unsigned long long)kDisp);
    u0 = __shfl_sync(0xffffffffu, u0, 0);
    DFT(st_disp);
    if (u0 >= nunit) break;
    const long long u1 = min((long long)nunit, u0 + kDisp);
    for (long long u = u0; u < u1; ++u) {
      const int64_t* U = units + 8 * u;
      const int64_t g = __ldg(U), kind = __ldg(U + 1), li = __ldg(U + 2);
      const int64_t doff = __ldg(U + 3), dn = __ldg(U + 4), inc0 = __ldg(U + 5), inc1 = __ldg(U + 6);
      if (dn > 0) {
        flush();
        // every lane acquires (the loads of one address coalesce)
        for (int64_t d = 0; d < dn; ++d) {
          const int64_t c = __ldg(deps + 2 * (doff + d));
          const unsigned long long tg = (unsigned long long)__ldg(deps + 2 * (doff + d) + 1);
          unsigned ns = 32;
          while (ld_acq_u64(ctrs + c) < tg) {
            __nanosleep(ns);
            if (ns < 1024) ns <<= 1;
          }
        }
      }
      DFT(st_wait);
      const int64_t* P = ph + 8 * g;
      double* scr = scratch + __ldg(P + 4);
      if (kind == 0) {
        gemv_item<NV, true>((int)li, image + __ldg(P + 1), image + __ldg(P), x, ldx, scr, ldscr, v0);
        DFT(st_item);
#ifdef SPAND_DF_STATS
        ++n_item;
#endif
      } else {
        chunk_warp<NV>(image + __ldg(P + 2) + 8 * li, image + __ldg(P + 3), x, ldx, scr, ldscr, v0);
        DFT(st_chunk);
#ifdef SPAND_DF_STATS
        ++n_chunk;
#endif
      }
      // signal at once: dependents are on the critical path
      pc0 = inc0;
      pn0 = 1;
      if (inc1 >= 0) {
        pc1 = inc1;
        pn1 = 1;
      }
      flush();
    }
  }
  flush();
#ifdef SPAND_DF_STATS
  if (lane == 0) {
    unsigned long long* S = ctrs + 1;   // debug: stats after the counters (caller sizes)
    (void)S;
    printf("[df] blk %d warp %d wait %lld item %lld chunk %lld disp %lld flush %lld items %lld chunks %lld\n",
           (int)blockIdx.x, (int)(threadIdx.x >> 5), st_wait / 1000, st_item / 1000, st_chunk / 1000,
           st_disp / 1000, st_flush / 1000, n_item, n_chunk);
  }
#endif
}

// Nonzero-row bits of column-major panels (rows {address, ld, rows, cols,
// first word}): bit i of the panel's words is set iff row i has a nonzero.
// One CTA per panel, a warp per 32-row word (coalesced down each column).
__global__ void __launch_bounds__(kThreads)
row_bits_kernel(const int64_t* __restrict__ panels, uint32_t* __restrict__ bits) {
  const int64_t* r = panels + 5 * (int64_t)blockIdx.x;
  const double* M = reinterpret_cast<const double*>(r[0]);
  const int64_t ld = r[1];
  const int rows = (int)r[2], cols = (int)r[3];
  const int64_t w0 = r[4];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int wd = warp; wd * 32 < rows; wd += kWarps) {
    const int i = wd * 32 + lane;
    bool nz = false;
    if (i < rows)
      for (int j = 0; j < cols && !nz; ++j) nz = __ldg(M + i + (int64_t)j * ld) != 0.0;
    const unsigned b = __ballot_sync(0xffffffffu, nz);
    if (lane == 0) bits[w0 + wd] = b;
  }
}
}  // namespace

extern "C" {

// a whole forward or backward pass as one cooperative launch per group of
// <= 4 vectors; ph: the phase table on the DEVICE (10 int64 per phase, image
// offsets); bar: 2 uint32 of zeroed scratch (reset here)
int spand_apply_pass_persistent(int nphase, const int64_t* ph, const int64_t* image, double* x,
                                int64_t ldx, double* scratch, int64_t ldscr, int nvec,
                                unsigned* bar, void* stream) {
  if (nphase < 0 || nvec < 1) return -1;
  if (nphase == 0) return 0;
  static int sms = 0, occ1 = 0, occ2 = 0, occ4 = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ1, pass_kernel<1>, kThreads, 0);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ2, pass_kernel<2>, kThreads, 0);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ4, pass_kernel<4>, kThreads, 0);
  }
  cudaStream_t st = as_stream(stream);
  for (int v0 = 0; v0 < nvec;) {
    const int left = nvec - v0;
    cudaError_t e = cudaMemsetAsync(bar, 0, 2 * sizeof(unsigned), st);
    if (e != cudaSuccess) return (int)e;
    int nv = left >= 4 ? 4 : (left >= 2 ? 2 : 1);
    int grid = sms * (nv == 4 ? occ4 : (nv == 2 ? occ2 : occ1));
    void* args[] = {&nphase, (void*)&ph, (void*)&image, &x, &ldx, &scratch, &ldscr, &bar, &v0};
    if (nv == 4) e = cudaLaunchCooperativeKernel((void*)pass_kernel<4>, grid, kThreads, args, 0, st);
    else if (nv == 2) e = cudaLaunchCooperativeKernel((void*)pass_kernel<2>, grid, kThreads, args, 0, st);
    else e = cudaLaunchCooperativeKernel((void*)pass_kernel<1>, grid, kThreads, args, 0, st);
    if (e != cudaSuccess) return (int)e;
    v0 += nv;
  }
  return 0;
}

int spand_apply_dataflow(int64_t nunit, const int64_t* units, const int64_t* deps, int64_t nctr,
                         unsigned long long* ctrs, const int64_t* phases, const int64_t* image,
                         double* x, int64_t ldx, double* scratch, int64_t ldscr, int nvec,
                         void* stream) {
  if (nunit < 0 || nctr < 1 || nvec < 1) return -1;
  if (nunit == 0) return 0;
  static int sms = 0, occ1 = 0, occ2 = 0, occ4 = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ1, dataflow_kernel<1>, kThreads, 0);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ2, dataflow_kernel<2>, kThreads, 0);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ4, dataflow_kernel<4>, kThreads, 0);
  }
  cudaStream_t st = as_stream(stream);
  for (int v0 = 0; v0 < nvec;) {
    const int left = nvec - v0;
    cudaError_t e = cudaMemsetAsync(ctrs, 0, (size_t)nctr * sizeof(unsigned long long), st);
    if (e != cudaSuccess) return (int)e;
    if (left >= 4) {
      dataflow_kernel<4><<<sms * occ4, kThreads, 0, st>>>(nunit, units, deps, ctrs, phases, image,
                                                         x, ldx, scratch, ldscr, v0);
      v0 += 4;
    } else if (left >= 2) {
      dataflow_kernel<2><<<sms * occ2, kThreads, 0, st>>>(nunit, units, deps, ctrs, phases, image,
                                                         x, ldx, scratch, ldscr, v0);
      v0 += 2;
    } else {
      dataflow_kernel<1><<<sms * occ1, kThreads, 0, st>>>(nunit, units, deps, ctrs, phases, image,
                                                         x, ldx, scratch, ldscr, v0);
      v0 += 1;
    }
    SPAND_CHECK_LAUNCH();
  }
  return 0;
}

int spand_row_bits(int npanel, const int64_t* panels, uint32_t* bits, void* stream) {
  if (npanel < 0) return -1;
  if (npanel == 0) return 0;
  row_bits_kernel<<<npanel, kThreads, 0, as_stream(stream)>>>(panels, bits);
  SPAND_CHECK_LAUNCH();
  return 0;
}

int spand_apply_runs(int nchunk, const int64_t* chunks, const int64_t* contrib, double* x,
                     int64_t ldx, const double* scratch, int64_t ldscr, int nvec, void* stream) {
  if (nchunk < 0 || nvec < 1) return -1;
  if (nchunk == 0) return 0;
  runs_kernel<<<nchunk, kThreads, 0, as_stream(stream)>>>(chunks, contrib, x, ldx, scratch,
                                                          ldscr, nvec);
  SPAND_CHECK_LAUNCH();
  return 0;
}

int spand_gemv_tiles(int ntiles, const int64_t* tiles, const int64_t* tasks, const double* x,
                     int64_t ldx, double* scratch, int64_t ldscr, int nvec, void* stream) {
  if (ntiles < 0 || nvec < 1) return -1;
  if (ntiles == 0) return 0;
  gemv_tiles_kernel<<<ntiles, kThreads, 0, as_stream(stream)>>>(tiles, tasks, x, ldx, scratch,
                                                                ldscr, nvec);
  SPAND_CHECK_LAUNCH();
  return 0;
}

int spand_gemv_items(int nitem, int grid, const int64_t* items, const int64_t* tasks,
                     const double* x, int64_t ldx, double* scratch, int64_t ldscr, int nvec,
                     void* stream) {
  if (nitem < 0 || grid < 0 || nvec < 1) return -1;
  if (nitem == 0) return 0;
  if (grid == 0) grid = (nitem + kWarps - 1) / kWarps;
  // vectors in groups of 4 (then 2, 1), payload read once per group
  // (task rows address vector 0; the kernel offsets by (v0 + v) * ldx)
  for (int v0 = 0; v0 < nvec;) {
    const int left = nvec - v0;
    if (left >= 4) {
      gemv_items_kernel<4><<<grid, kThreads, 0, as_stream(stream)>>>(nitem, items, tasks, x, ldx,
                                                                    scratch, ldscr, v0);
      v0 += 4;
    } else if (left >= 2) {
      gemv_items_kernel<2><<<grid, kThreads, 0, as_stream(stream)>>>(nitem, items, tasks, x, ldx,
                                                                    scratch, ldscr, v0);
      v0 += 2;
    } else {
      gemv_items_kernel<1><<<grid, kThreads, 0, as_stream(stream)>>>(nitem, items, tasks, x, ldx,
                                                                    scratch, ldscr, v0);
      v0 += 1;
    }
    SPAND_CHECK_LAUNCH();
  }
  return 0;
}

// one whole pass (forward or backward) of a structured plan from its phase
// table: the per-phase gemv + runs launches are issued here, not from Python
int spand_apply_pass(int nphase, const int64_t* ph, const int64_t* image, double* x, int64_t ldx,
                     double* scratch, int64_t ldscr, int nvec, void* stream) {
  if (nphase < 0 || nvec < 1) return -1;
  for (int q = 0; q < nphase; ++q) {
    const int64_t* r = ph + 10 * (int64_t)q;
    // {tasks, ntask, items, nitem, chunks, nchunk, contrib, grid, -, -} (image offsets)
    const int st1 = spand_gemv_items((int)r[3], (int)r[7], image + r[2], image + r[0], x, ldx,
                                     scratch, ldscr, nvec, stream);
    if (st1 != 0) return st1;
    const int st2 = spand_apply_runs((int)r[5], image + r[4], image + r[6], x, ldx, scratch,
                                     ldscr, nvec, stream);
    if (st2 != 0) return st2;
  }
  return 0;
}

int spand_apply_scatter(int nout, const int64_t* dst, const int64_t* mode, const int64_t* ptr,
                        const int64_t* src, double* x, int64_t ldx, const double* scratch,
                        int64_t ldscr, int nvec, void* stream) {
  if (nout < 0 || nvec < 1) return -1;
  if (nout == 0) return 0;
  scatter_kernel<<<(nout + kThreads - 1) / kThreads, kThreads, 0, as_stream(stream)>>>(
      nout, dst, mode, ptr, src, x, ldx, scratch, ldscr, nvec);
  SPAND_CHECK_LAUNCH();
  return 0;
}

}  // extern "C"
