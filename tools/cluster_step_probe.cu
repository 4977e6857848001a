// Latency floor of one RRQR elimination step with the cluster layout
// (tools/, not product code): G CTAs in clusters of CS, 256 threads, 2 per
// SM.  Per step:
//   cluster leader publishes one 32-byte record; cluster barrier; the leader
//   arrives on the group counter (NC = G / CS arrivals); every CTA polls the
//   release flag (mode 0) or the leader polls and a cluster barrier releases
//   the others (mode 1); every CTA scans the NC records, reads its 1/CS row
//   slice of an m-row pivot column from L2, reduces its norm, and the CS
//   partial vectors (L doubles) are summed through DSMEM after a second
//   cluster barrier.
// Output: ns per step per (CS, mode).  Build:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/cluster_step_probe tools/cluster_step_probe.cu
#include <cooperative_groups.h>
#include <cstdio>
#include <cstdlib>

namespace cg = cooperative_groups;

__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(unsigned* p, unsigned v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;\n" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void cl_arrive() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n" ::: "memory");
}
__device__ __forceinline__ void cl_wait() {
  asm volatile("barrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}

constexpr int L = 64;

__global__ void __launch_bounds__(256, 2) probe(int steps, int m, int mode, unsigned* ctr, double* rec,
                                                const double* col, double* out) {
  __shared__ double red[8];
  __shared__ double best;
  __shared__ double part[2][L];
  cg::cluster_group cl = cg::this_cluster();
  const int CS = (int)cl.num_blocks(), s = (int)cl.block_rank();
  const int G = gridDim.x, NC = G / CS, ci = blockIdx.x / CS, tid = threadIdx.x;
  unsigned gen = 0;
  double acc = 0.0;
  for (int k = 0; k < steps; ++k) {
    if (s == 0 && tid == 0) {
      double* r = rec + 4 * ((k & 1) * NC + ci);
      r[0] = (double)(ci ^ k);
      r[1] = (double)k;
    }
    __syncthreads();
    if (tid == 0) __threadfence();
    cl_arrive();
    cl_wait();
    if (tid == 0) {
      ++gen;
      if (s == 0) {
        if (atomicAdd(ctr, 1u) + 1u == gen * (unsigned)NC) st_release(ctr + 1, gen);
        else if (mode == 0 || true) while (ld_acquire(ctr + 1) < gen) {}
      } else if (mode == 0) {
        while (ld_acquire(ctr + 1) < gen) {}
      }
      __threadfence();
    }
    if (mode == 1) {
      cl_arrive();
      cl_wait();
    }
    __syncthreads();
    // candidate scan over NC records
    double v = -1.0;
    for (int q = tid; q < NC; q += 256) v = fmax(v, __ldcg(rec + 4 * ((k & 1) * NC + q)));
    for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
    if ((tid & 31) == 0) red[tid >> 5] = v;
    __syncthreads();
    if (tid == 0) {
      double b = red[0];
      for (int w = 1; w < 8; ++w) b = fmax(b, red[w]);
      best = b;
    }
    __syncthreads();
    // my row slice (32-row chunks q = s mod CS) of the pivot column
    const double* c = col + (size_t)((int)best % 64) * m;
    double sacc = 0.0;
    const int nch = (m + 31) / 32;
    for (int q = s + CS * (tid >> 5); q < nch; q += CS * 8) {
      const int i = q * 32 + (tid & 31);
      if (i < m) {
        const double x = __ldcg(c + i);
        sacc += x * x;
      }
    }
    for (int o = 16; o > 0; o >>= 1) sacc += __shfl_xor_sync(0xffffffffu, sacc, o);
    if ((tid & 31) == 0) red[tid >> 5] = sacc;
    __syncthreads();
    if (tid < L) {
      double t = 0.0;
      for (int w = 0; w < 8; ++w) t += red[w];
      part[k & 1][tid] = t + tid;
    }
    // DSMEM pull exchange of L partials
    cl_arrive();
    cl_wait();
    if (tid < L) {
      double t = 0.0;
      for (int r = 0; r < CS; ++r) t += cl.map_shared_rank(&part[k & 1][0], r)[tid];
      if (tid == 0) acc += t;
    }
    __syncthreads();
  }
  if (tid == 0) out[blockIdx.x] = acc;
}

int main(int argc, char** argv) {
  const int m = argc > 1 ? atoi(argv[1]) : 3104;
  unsigned* ctr;
  double *rec, *col, *out;
  cudaMalloc(&ctr, 8);
  cudaMalloc(&rec, 8 * 4 * 2 * 4096);
  cudaMalloc(&col, 8 * (size_t)m * 64);
  cudaMalloc(&out, 8 * 4096);
  cudaMemset(col, 0, 8 * (size_t)m * 64);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int CS : {1, 2, 4, 8}) {
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = CS;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    at[1].id = cudaLaunchAttributeCooperative;
    at[1].val.cooperative = 1;
    cfg.blockDim = dim3(256);
    cfg.dynamicSmemBytes = 96 * 1024;
    cfg.attrs = at;
    cfg.numAttrs = 2;
    cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024);
    int ncl = 0;
    cfg.gridDim = dim3(CS * 8);
    cudaError_t oe = cudaOccupancyMaxActiveClusters(&ncl, (void*)probe, &cfg);
    printf("{\"CS\": %d, \"max_active_clusters\": %d, \"occ_err\": \"%s\"}\n", CS, ncl,
           cudaGetErrorString(oe));
    for (int G : {296, 288, 256, 148}) {
      if (G % CS) continue;
      if (ncl > 0 && G / CS > ncl) continue;
      for (int mode = 0; mode < 2; ++mode) {
        int steps = 2000;
        for (int rep = 0; rep < 2; ++rep) {
          cudaMemset(ctr, 0, 8);
          cfg.gridDim = dim3(G);
          int mm = m, md = mode;
          cudaEventRecord(e0);
          cudaError_t le = cudaLaunchKernelEx(&cfg, probe, steps, mm, md, ctr, rec, (const double*)col, out);
          cudaEventRecord(e1);
          cudaError_t se = cudaEventSynchronize(e1);
          float ms = 0;
          cudaEventElapsedTime(&ms, e0, e1);
          if (le != cudaSuccess || se != cudaSuccess) {
            printf("{\"CS\": %d, \"G\": %d, \"error\": \"%s / %s\"}\n", CS, G, cudaGetErrorString(le),
                   cudaGetErrorString(se));
            return 1;
          }
          if (rep) printf("{\"CS\": %d, \"G\": %d, \"mode\": %d, \"m\": %d, \"ns_per_step\": %.1f}\n", CS, G, mode, m, 1e6 * ms / steps);
        }
      }
    }
  }
  return 0;
}
