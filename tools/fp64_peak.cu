// FP64 roofline probe for B200 (sm_100a): sustained DFMA and DMMA (mma.sync f64)
// throughput, used as the FP64 denominator of the Schur-update roofline
// (MEASURED_PEAKS.json carries no FP64 figure).  Build:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/fp64_peak tools/fp64_peak.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void dfma_loop(double* out, int iters) {
  double a0 = threadIdx.x * 1e-7, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3;
  double a4 = a0 + 4, a5 = a0 + 5, a6 = a0 + 6, a7 = a0 + 7;
  const double b = 0.999999, c = 1e-9;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      a0 = fma(a0, b, c); a1 = fma(a1, b, c); a2 = fma(a2, b, c); a3 = fma(a3, b, c);
      a4 = fma(a4, b, c); a5 = fma(a5, b, c); a6 = fma(a6, b, c); a7 = fma(a7, b, c);
    }
  }
  double s = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
  if (s == 1234.5) out[threadIdx.x] = s;
}

__global__ void dmma_loop(double* out, int iters) {
  double a = 1.0 + threadIdx.x * 1e-9, b = 0.5;
  double c[8][2];
#pragma unroll
  for (int t = 0; t < 8; ++t) { c[t][0] = 0; c[t][1] = 0; }
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 4; ++j) {
#pragma unroll
      for (int t = 0; t < 8; ++t) {
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                     : "+d"(c[t][0]), "+d"(c[t][1]) : "d"(a), "d"(b));
      }
    }
  }
  double s = 0;
#pragma unroll
  for (int t = 0; t < 8; ++t) s += c[t][0] + c[t][1];
  if (s == 1234.5) out[threadIdx.x] = s;
}

int main() {
  double* out; cudaMalloc(&out, 4096 * sizeof(double));
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int threads = 256, blocks = sms * 8;
  for (int rep = 0; rep < 2; ++rep) {
    int iters = 4000;
    dfma_loop<<<blocks, threads>>>(out, 10);
    cudaEventRecord(e0); dfma_loop<<<blocks, threads>>>(out, iters); cudaEventRecord(e1);
    cudaEventSynchronize(e1); float ms; cudaEventElapsedTime(&ms, e0, e1);
    double fl = 2.0 * 8 * 16 * (double)iters * threads * blocks;
    printf("{\"probe\":\"dfma\",\"tflops\":%.3f,\"ms\":%.3f}\n", fl / ms / 1e9, ms);
    dmma_loop<<<blocks, threads>>>(out, 10);
    cudaEventRecord(e0); dmma_loop<<<blocks, threads>>>(out, iters); cudaEventRecord(e1);
    cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
    fl = 512.0 * 8 * 4 * (double)iters * (threads / 32) * blocks;
    printf("{\"probe\":\"dmma_m8n8k4\",\"tflops\":%.3f,\"ms\":%.3f}\n", fl / ms / 1e9, ms);
  }
  cudaError_t err = cudaGetLastError();
  if (err != cudaSuccess) { printf("error %s\n", cudaGetErrorString(err)); return 1; }
  return 0;
}
