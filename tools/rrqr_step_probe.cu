// Latency floor of one RRQR elimination step (tools/, not product code):
// a cooperative grid of G CTAs (256 threads, 2 per SM) repeats the step's
// unavoidable synchronisation skeleton with no column work --
//   publish a 32-byte candidate record, group barrier (arrival counter +
//   release flag, as rrqr.cu), every CTA scans the G records, reads an
//   m-row pivot column from L2 and reduces its norm over the CTA.
// Output: ns per step.  Build: nvcc -gencode arch=compute_100a,code=sm_100a
//   -O3 -o tools/rrqr_step_probe tools/rrqr_step_probe.cu
#include <cooperative_groups.h>
#include <cstdio>
#include <cstdlib>

__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(unsigned* p, unsigned v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;\n" ::"l"(p), "r"(v) : "memory");
}

__global__ void __launch_bounds__(256, 2) probe(int steps, int m, unsigned* ctr, double* rec,
                                                const double* col, double* out) {
  __shared__ double red[8];
  __shared__ double best;
  const int G = gridDim.x, tid = threadIdx.x;
  unsigned gen = 0;
  double acc = 0.0;
  for (int k = 0; k < steps; ++k) {
    if (tid == 0) {
      double* r = rec + 4 * ((k & 1) * G + blockIdx.x);
      r[0] = (double)(blockIdx.x ^ k);
      r[1] = (double)k;
    }
    __syncthreads();
    if (tid == 0) {
      __threadfence();
      ++gen;
      if (atomicAdd(ctr, 1u) + 1u == gen * (unsigned)G) st_release(ctr + 1, gen);
      else while (ld_acquire(ctr + 1) < gen) {}
      __threadfence();
    }
    __syncthreads();
    // candidate scan
    double v = -1.0;
    for (int q = tid; q < G; q += 256) v = fmax(v, __ldcg(rec + 4 * ((k & 1) * G + q)));
    for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
    if ((tid & 31) == 0) red[tid >> 5] = v;
    __syncthreads();
    if (tid == 0) {
      double b = red[0];
      for (int w = 1; w < 8; ++w) b = fmax(b, red[w]);
      best = b;
    }
    __syncthreads();
    // pivot column (m rows) from L2 and its norm
    const double* c = col + (size_t)((int)best % 64) * m;
    double s = 0.0;
    for (int i = tid; i < m; i += 256) s += __ldcg(c + i) * __ldcg(c + i);
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if ((tid & 31) == 0) red[tid >> 5] = s;
    __syncthreads();
    if (tid == 0) {
      double t = 0.0;
      for (int w = 0; w < 8; ++w) t += red[w];
      acc += t;
    }
    __syncthreads();
  }
  if (tid == 0) out[blockIdx.x] = acc;
}

int main(int argc, char** argv) {
  const int m = argc > 1 ? atoi(argv[1]) : 3104;
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
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
  for (int G : {148, 296}) {
    if (G > 2 * sms) continue;
    int steps = 2000;
    for (int rep = 0; rep < 2; ++rep) {
      cudaMemset(ctr, 0, 8);
      void* args[] = {&steps, (void*)&m, &ctr, &rec, &col, &out};
      int mm = m;
      args[1] = &mm;
      cudaEventRecord(e0);
      cudaLaunchCooperativeKernel((void*)probe, dim3(G), dim3(256), args, 0, 0);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms = 0;
      cudaEventElapsedTime(&ms, e0, e1);
      if (rep) printf("{\"G\": %d, \"m\": %d, \"ns_per_step\": %.1f}\n", G, m, 1e6 * ms / steps);
    }
  }
  return 0;
}
