// FP64 DFMA throughput on this GPU (is an FP64 FFT blind rotation viable?).
#include <cstdio>
#include <cuda_runtime.h>
__global__ void dfma_kernel(double* out, int iters, double a, double b) {
  double x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b);
      x4 = fma(x4, a, b); x5 = fma(x5, a, b); x6 = fma(x6, a, b); x7 = fma(x7, a, b);
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}
__global__ void imad_kernel(unsigned* out, int iters, unsigned a, unsigned b) {
  unsigned x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      x0 = x0 * a + b; x1 = x1 * a + b; x2 = x2 * a + b; x3 = x3 * a + b;
      x4 = x4 * a + b; x5 = x5 * a + b; x6 = x6 * a + b; x7 = x7 * a + b;
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}
int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  double* d; unsigned* u;
  cudaMalloc(&d, sizeof(double) * sms * 8 * 1024); cudaMalloc(&u, 4 * sms * 8 * 1024);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int iters = 4096;
  for (int warps : {4, 8, 16, 32}) {
    int blocks = sms * 2, threads = warps * 16;
    dfma_kernel<<<blocks, threads>>>(d, 16, 1.0000001, 0.5);
    cudaEventRecord(e0);
    dfma_kernel<<<blocks, threads>>>(d, iters, 1.0000001, 0.5);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double ops = (double)blocks * threads * iters * 64;
    printf("DFMA warps/SM %2d: %.2f T DFMA/s = %.1f per SM per clk (clock %d MHz)\n", warps, ops / ms / 1e9,
           ops / (ms * 1e-3) / sms / (clk * 1e3), clk / 1000);
    imad_kernel<<<blocks, threads>>>(u, 16, 3, 7);
    cudaEventRecord(e0);
    imad_kernel<<<blocks, threads>>>(u, iters, 3, 7);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    printf("IMAD warps/SM %2d: %.2f T IMAD/s = %.1f per SM per clk\n", warps, ops / ms / 1e9,
           ops / (ms * 1e-3) / sms / (clk * 1e3));
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
