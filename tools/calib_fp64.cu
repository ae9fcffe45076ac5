// fp64 peak calibration on sm_100a: DMMA (mma.sync m8n8k4 f64) and DFMA throughput.
// Calibration only (not product code). Prints JSON lines.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void dmma_loop(double* out, int iters) {
  double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
  double c[8][2];
#pragma unroll
  for (int i = 0; i < 8; ++i) { c[i][0] = 0; c[i][1] = 0; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1];
  if (s == 12345.678) out[0] = s;
}

__global__ void dfma_loop(double* out, int iters) {
  double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - 1e-12;
  double c[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) c[i] = i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) c[i] = fma(c[i], b, a);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += c[i];
  if (s == 12345.678) out[0] = s;
}

int main() {
  double* d; cudaMalloc(&d, 8);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int wpb : {4, 8, 16}) {
    int iters = 20000;
    for (int blocksPerSM : {1, 2, 4}) {
      int grid = sms * blocksPerSM;
      dmma_loop<<<grid, 32 * wpb>>>(d, 100);
      cudaEventRecord(e0);
      dmma_loop<<<grid, 32 * wpb>>>(d, iters);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      double flops = 2.0 * 256.0 * 8 * iters * (double)grid * wpb;
      printf("{\"kind\":\"dmma\",\"warps_per_block\":%d,\"blocks_per_sm\":%d,\"ms\":%.3f,\"tflops\":%.3f}\n", wpb, blocksPerSM, ms, flops / ms / 1e9);
      dfma_loop<<<grid, 32 * wpb>>>(d, 100);
      cudaEventRecord(e0);
      dfma_loop<<<grid, 32 * wpb>>>(d, iters * 4);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1);
      flops = 2.0 * 8 * iters * 4 * (double)grid * wpb * 32;
      printf("{\"kind\":\"dfma\",\"warps_per_block\":%d,\"blocks_per_sm\":%d,\"ms\":%.3f,\"tflops\":%.3f}\n", wpb, blocksPerSM, ms, flops / ms / 1e9);
    }
  }
  cudaError_t err = cudaGetLastError();
  printf("{\"err\":\"%s\"}\n", cudaGetErrorString(err));
  return 0;
}
