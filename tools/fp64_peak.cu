// FP64 peak probes for the B200 roofline denominator: DFMA pipe and DMMA (mma.sync f64).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/fp64_peak tools/fp64_peak.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void dfma_loop(double* out, int iters, double a, double b) {
  double r[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) r[i] = threadIdx.x * 1e-3 + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) r[i] = fma(r[i], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) s += r[i];
  if (s == 12345.678) out[0] = s;
}

__global__ void dmma_loop(double* out, int iters) {
  double acc[8][2];
#pragma unroll
  for (int i = 0; i < 8; ++i) { acc[i][0] = 0; acc[i][1] = 0; }
  double a = threadIdx.x * 1e-3, b = 1.0 - threadIdx.x * 1e-4;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(acc[i][0]), "+d"(acc[i][1]) : "d"(a), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += acc[i][0] + acc[i][1];
  if (s == 12345.678) out[0] = s;
}

int main() {
  double* d;
  cudaMalloc(&d, 8);
  int dev = 0;
  cudaDeviceProp p;
  cudaGetDeviceProperties(&p, dev);
  int sms = p.multiProcessorCount;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int threads : {256, 512, 1024}) {
    for (int bps : {1, 2, 4}) {
      int iters = 20000;
      dfma_loop<<<sms * bps, threads>>>(d, 100, 1.0000001, 1e-9);
      cudaEventRecord(e0);
      dfma_loop<<<sms * bps, threads>>>(d, iters, 1.0000001, 1e-9);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      double flops = 2.0 * 16 * iters * (double)threads * sms * bps;
      printf("{\"probe\":\"dfma\",\"threads\":%d,\"blocks_per_sm\":%d,\"tflops\":%.3f}\n", threads, bps,
             flops / ms / 1e9);
    }
  }
  for (int threads : {128, 256, 512}) {
    for (int bps : {1, 2, 4}) {
      int iters = 20000;
      dmma_loop<<<sms * bps, threads>>>(d, 100);
      cudaEventRecord(e0);
      dmma_loop<<<sms * bps, threads>>>(d, iters);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      double flops = 2.0 * 256 * 8 * iters * (double)(threads / 32) * sms * bps;
      printf("{\"probe\":\"dmma_m8n8k4\",\"threads\":%d,\"blocks_per_sm\":%d,\"tflops\":%.3f}\n", threads, bps,
             flops / ms / 1e9);
    }
  }
  cudaError_t err = cudaGetLastError();
  printf("err=%s\n", cudaGetErrorString(err));
  return 0;
}
