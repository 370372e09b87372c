// field_bench.cu — Goldilocks add/sub variants: correctness vs the reference
// C++ path and throughput inside the real 32-point NTT passes (sm_100a).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --expt-relaxed-constexpr \
//        -I paper_1906_00148_b200/csrc tools/microbench/field_bench.cu -o fb && ./fb
#include <cstdio>
#include <cstdlib>
#include <vector>

#ifndef VARIANT
#define VARIANT 0
#endif

#if VARIANT == 1
#define GL_ADDSUB_PTX 1
#endif
#include "ntt.cuh"

__global__ void ntt_loop(uint64_t* d, int iters) {
  uint64_t x[32];
  for (int q = 0; q < 32; ++q) x[q] = d[(blockIdx.x * blockDim.x + threadIdx.x) * 32 + q];
  for (int it = 0; it < iters; ++it) {
    ntt::fwd<32, 3, true>(x);
    ntt::fwd<32, 6, false>(x);
  }
  for (int q = 0; q < 32; ++q) d[(blockIdx.x * blockDim.x + threadIdx.x) * 32 + q] = gl::canon(x[q]);
}

int main() {
  const int blocks = 148 * 4, threads = 128, iters = 200;
  const size_t n = (size_t)blocks * threads * 32;
  std::vector<uint64_t> h(n), ref(n);
  uint64_t s = 0x1234567;
  for (size_t i = 0; i < n; ++i) {
    s = s * 6364136223846793005ull + 1442695040888963407ull;
    uint64_t v = s ^ (s >> 29);
    if (i % 97 == 0) v = 0xFFFFFFFFFFFFFFFFull - (i % 5);         // non-canonical edge values
    if (i % 89 == 0) v = 0xFFFFFFFF00000001ull + (i % 7);
    h[i] = v;
  }
  // reference on the host (plain C++ path of gl64.cuh)
  for (size_t t = 0; t < n / 32; ++t) {
    uint64_t x[32];
    for (int q = 0; q < 32; ++q) x[q] = h[t * 32 + q];
    for (int it = 0; it < 3; ++it) {
      ntt::fwd<32, 3, true>(x);
      ntt::fwd<32, 6, false>(x);
    }
    for (int q = 0; q < 32; ++q) ref[t * 32 + q] = gl::canon(x[q]);
  }
  uint64_t* d;
  cudaMalloc(&d, n * 8);
  cudaMemcpy(d, h.data(), n * 8, cudaMemcpyHostToDevice);
  ntt_loop<<<blocks, threads>>>(d, 3);
  std::vector<uint64_t> got(n);
  cudaMemcpy(got.data(), d, n * 8, cudaMemcpyDeviceToHost);
  size_t bad = 0;
  for (size_t i = 0; i < n; ++i) bad += got[i] != ref[i];
  cudaMemcpy(d, h.data(), n * 8, cudaMemcpyHostToDevice);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  ntt_loop<<<blocks, threads>>>(d, 10);
  cudaEventRecord(e0);
  ntt_loop<<<blocks, threads>>>(d, iters);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  const double bfly = (double)blocks * threads * iters * 160;  // 2 passes x 80 butterflies
  printf("variant %d: mismatches %zu / %zu ; %.3f ms ; %.1f G butterflies/s ; %s\n", VARIANT, bad, n,
         ms, bfly / ms / 1e6, cudaGetErrorString(cudaGetLastError()));
  return bad != 0;
}
