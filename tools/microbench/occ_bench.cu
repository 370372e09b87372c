// occ_bench.cu — does occupancy pay for the butterfly stream?  The product
// butterflies (ntt::fwd) on 20 warps/SM x 32 values per thread vs 40 warps/SM
// x 16 values per thread (same total butterflies per launch).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --expt-relaxed-constexpr \
//        -DGL_ADDSUB_PTX -I paper_1906_00148_b200/csrc tools/microbench/occ_bench.cu -o ob
#include <cstdio>
#include <vector>

#include "ntt.cuh"

template <int V, int T, int B>
__global__ void __launch_bounds__(T, B) loop(uint64_t* d, int iters) {
  uint64_t x[V];
  const size_t base = ((size_t)blockIdx.x * blockDim.x + threadIdx.x) * V;
  for (int q = 0; q < V; ++q) x[q] = d[base + q];
  for (int it = 0; it < iters; ++it) {
    ntt::fwd<V, (V == 32 ? 3 : 6), true>(x);
    ntt::fwd<V, (V == 32 ? 6 : 12), false>(x);
  }
  for (int q = 0; q < V; ++q) d[base + q] = gl::canon(x[q]);
}

template <int V, int T, int B = 1>
void run(int iters) {
  const int blocks = 148 * B;
  const size_t n = (size_t)blocks * T * V;
  std::vector<uint64_t> h(n);
  uint64_t s = 99;
  for (auto& v : h) { s = s * 6364136223846793005ull + 1442695040888963407ull; v = s ^ (s >> 29); }
  uint64_t* d;
  cudaMalloc(&d, n * 8);
  cudaMemcpy(d, h.data(), n * 8, cudaMemcpyHostToDevice);
  loop<V, T, B><<<blocks, T>>>(d, 2);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float best = 1e9f;
  for (int r = 0; r < 3; ++r) {
    cudaEventRecord(e0);
    loop<V, T, B><<<blocks, T>>>(d, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    best = ms < best ? ms : best;
  }
  const double lg = V == 32 ? 5 : 4;
  const double bfly = (double)blocks * T * iters * 2 * (V / 2) * lg;
  printf("V=%d threads/CTA=%d CTAs/SM=%d: %.3f ms, %.1f G butterflies/s (%s)\n", V, T, B, best, bfly / best / 1e6,
         cudaGetErrorString(cudaGetLastError()));
  cudaFree(d);
}

int main() {
  run<32, 640>(100);
  run<16, 640, 2>(125);
  run<16, 512, 2>(125);
  run<16, 640>(125);
  run<32, 512>(100);
  run<32, 320, 2>(100);
  return 0;
}
