// Probe (not product): FP64 throughput of DFMA vs the FP64 tensor-core MMA
// (mma.sync m8n8k4 f64) on this GPU. nvcc -gencode arch=compute_100a,code=sm_100a
#include <cstdio>
#include <cuda_runtime.h>

__global__ void dfma_loop(double* out, int iters) {
  double a[8], b = 1.0000001, c = 1e-9;
  for (int j = 0; j < 8; ++j) a[j] = threadIdx.x + j;
  for (int i = 0; i < iters; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) a[j] = fma(a[j], b, c);
  double s = 0;
  for (int j = 0; j < 8; ++j) s += a[j];
  if (s == 1.2345) out[0] = s;
}

__global__ void dmma_loop(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
  double c[4][2] = {};
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 4; ++j)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c[j][0]), "+d"(c[j][1]) : "d"(a), "d"(b));
  }
  double s = 0;
  for (int j = 0; j < 4; ++j) s += c[j][0] + c[j][1];
  if (s == 1.2345) out[0] = s;
}

int main() {
  double* d;
  cudaMalloc(&d, 8);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int iters = 4096, threads = 256, blocks = sms * 8;
  for (int rep = 0; rep < 2; ++rep) {
    float ms;
    cudaEventRecord(e0);
    dfma_loop<<<blocks, threads>>>(d, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    const double fl_dfma = 2.0 * 8 * iters * double(threads) * blocks;
    cudaEventRecord(e0);
    dmma_loop<<<blocks, threads>>>(d, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms2;
    cudaEventElapsedTime(&ms2, e0, e1);
    // m8n8k4: 8*8*4 FMA = 512 FMA = 1024 flop per warp-instruction, 4 per iter
    const double fl_dmma = 1024.0 * 4 * iters * double(threads / 32) * blocks;
    printf("DFMA %.2f TFLOP/s   DMMA(m8n8k4) %.2f TFLOP/s  err=%s\n", fl_dfma / ms / 1e9, fl_dmma / ms2 / 1e9,
           cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
