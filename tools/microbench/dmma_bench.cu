// FP64 tensor-core (DMMA, mma.sync m8n8k4 f64) throughput on this GPU, alone
// and issued beside DFMA in the same warps: does the FP64 FFT blind rotation
// have a second FP64 pipe to use?
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o dmma_bench dmma_bench.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

template <int NMMA, int NFMA>
__global__ void mix_kernel(double* out, int iters, double a, double b) {
  double c[8][2];
  double x[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    c[k][0] = threadIdx.x + k;
    c[k][1] = 1.0;
    x[k] = threadIdx.x + k;
  }
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < NMMA; ++k) dmma(c[k][0], c[k][1], a, b);
#pragma unroll
    for (int r = 0; r < NFMA / 8; ++r)
#pragma unroll
      for (int k = 0; k < 8; ++k) x[k] = fma(x[k], a, b);
  }
  double s = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += c[k][0] + c[k][1] + x[k];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int NMMA, int NFMA>
void run(const char* name, int sms, int clk, double* d, int warps) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int iters = 2048, blocks = sms, threads = warps * 32;
  mix_kernel<NMMA, NFMA><<<blocks, threads>>>(d, 16, 1.0000001, 0.5);
  cudaEventRecord(e0);
  mix_kernel<NMMA, NFMA><<<blocks, threads>>>(d, iters, 1.0000001, 0.5);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  const double w = (double)blocks * warps * iters;
  const double mma_flop = w * NMMA * 512.0, fma_flop = w * NFMA * 32 * 2.0;
  const double secs = ms * 1e-3;
  printf("%-28s warps/SM %2d: %7.2f ms  DMMA %6.2f TF/s  DFMA %6.2f TF/s  total %6.2f TF/s  (%.1f DMMA/SM/clk)\n",
         name, warps, ms, mma_flop / secs / 1e12, fma_flop / secs / 1e12, (mma_flop + fma_flop) / secs / 1e12,
         w * NMMA / secs / sms / (clk * 1e3));
}

int main() {
  int sms, clk;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  double* d;
  cudaMalloc(&d, sizeof(double) * sms * 1024);
  for (int warps : {4, 8, 16, 32}) {
    run<8, 0>("dmma only (8 chains)", sms, clk, d, warps);
    run<0, 64>("dfma only (8 chains)", sms, clk, d, warps);
    run<8, 64>("dmma 8 + dfma 64", sms, clk, d, warps);
    run<8, 128>("dmma 8 + dfma 128", sms, clk, d, warps);
    run<4, 128>("dmma 4 + dfma 128", sms, clk, d, warps);
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
