// bfly_bench.cu — throughput of NTT butterfly variants (0 = the product ntt::ct_bfly) inside the real pair of
// 32-point passes (negacyclic theta = 2^3, cyclic omega = 2^6), 20 warps/SM,
// each thread 32 values in registers; correctness checked against the host.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --expt-relaxed-constexpr \
//        -DGL_ADDSUB_PTX -I paper_1906_00148_b200/csrc tools/microbench/bfly_bench.cu -o bb && ./bb
#include <cstdio>
#include <vector>

#include "ntt.cuh"

namespace v {
// variant 3/4 helpers: the shift T = v 2^r as two IMAD.WIDE (FMA pipe)
__device__ __forceinline__ void shift3(uint64_t v, int r, uint32_t& T0, uint32_t& T1, uint32_t& T2) {
  const uint32_t v0 = (uint32_t)v, v1 = (uint32_t)(v >> 32);
  if (r == 0) { T0 = v0; T1 = v1; T2 = 0; return; }
  uint64_t P, W;
  const uint32_t m = 1u << r;
  asm("mul.wide.u32 %0, %1, %2;" : "=l"(P) : "r"(v0), "r"(m));
  asm("mad.wide.u32 %0, %1, %2, %3;" : "=l"(W) : "r"(v1), "r"(m), "l"(P >> 32));
  T0 = (uint32_t)P; T1 = (uint32_t)W; T2 = (uint32_t)(W >> 32);
}
__device__ __forceinline__ uint64_t shl3(uint64_t v, const int s) {
  const int q = s >> 5, r = s & 31;
  uint32_t T0, T1, T2;
  shift3(v, r, T0, T1, T2);
  uint32_t o0, o1;
  if (q == 0) {
    uint32_t w0, w1, c, e0, e1;
    asm("mad.lo.cc.u32 %0, %5, 0xFFFFFFFF, %6;\n\t"
        "madc.hi.cc.u32 %1, %5, 0xFFFFFFFF, %7;\n\t"
        "addc.u32 %2, 0, 0;\n\t"
        "add.cc.u32 %3, %0, 1;\n\t"
        "addc.u32 %4, %1, 0xFFFFFFFF;"
        : "=&r"(w0), "=&r"(w1), "=&r"(c), "=&r"(e0), "=&r"(e1)
        : "r"(T2 + 1), "r"(T0), "r"(T1));
    o0 = c ? w0 : e0;
    o1 = c ? w1 : e1;
  } else if (q == 1) {
    uint32_t s0, H, e0, e1;
    asm("add.cc.u32 %1, %5, %6;\n\t"
        "addc.u32 %2, %1, 0;\n\t"
        "addc.cc.u32 %3, %6, %7;\n\t"
        "addc.u32 %4, 0, 0;\n\t"
        "sub.cc.u32 %0, 0, %3;\n\t"
        "subc.cc.u32 %1, %2, %4;\n\t"
        "subc.u32 %4, 0, 0;\n\t"
        "sub.cc.u32 %0, %0, %4;\n\t"
        "subc.u32 %1, %1, 0;"
        : "=&r"(o0), "=&r"(s0), "=&r"(H), "=&r"(e0), "=&r"(e1)
        : "r"(T0), "r"(T1), "r"(T2));
    o1 = s0;
  } else {
    uint32_t F, fn, g0, g1;
    asm("sub.cc.u32 %2, %6, %8;\n\t"
        "subc.u32 %3, 0, 0;\n\t"
        "add.cc.u32 %4, %6, %7;\n\t"
        "addc.u32 %5, 0, 0;\n\t"
        "sub.cc.u32 %0, 0, %4;\n\t"
        "subc.cc.u32 %1, %2, %5;\n\t"
        "subc.u32 %3, %3, 0;\n\t"
        "sub.cc.u32 %0, %0, %3;\n\t"
        "subc.u32 %1, %1, 0;"
        : "=&r"(o0), "=&r"(o1), "=&r"(F), "=&r"(fn), "=&r"(g0), "=&r"(g1)
        : "r"(T0), "r"(T1), "r"(T2));
  }
  return ((uint64_t)o1 << 32) | o0;
}
__device__ __forceinline__ uint64_t add4(uint64_t x, uint64_t y) {
  uint32_t s0, s1, c;
  asm("add.cc.u32 %0, %3, %5;\n\t"
      "addc.cc.u32 %1, %4, %6;\n\t"
      "addc.u32 %2, 0, 0;"
      : "=&r"(s0), "=&r"(s1), "=&r"(c)
      : "r"((uint32_t)x), "r"((uint32_t)(x >> 32)), "r"((uint32_t)y), "r"((uint32_t)(y >> 32)));
  uint64_t r;
  asm("mad.wide.u32 %0, %1, 0xFFFFFFFF, %2;" : "=l"(r) : "r"(c), "l"(((uint64_t)s1 << 32) | s0));
  return r;
}
template <int VAR>
__device__ __forceinline__ void bfly(uint64_t& lo, uint64_t& hi, int s) {
  if (VAR == 0) { ntt::ct_bfly(lo, hi, s); return; }  // the product butterfly
  const bool ng = s >= 96;
  const int sp = ng ? s - 96 : s;
  const uint64_t u = lo;
  if (sp == 0) {
    lo = ng ? gl::sub(u, hi) : gl::add(u, hi);
    hi = ng ? gl::add(u, hi) : gl::sub(u, hi);
    return;
  }
  const uint64_t t = shl3(hi, sp);
  uint64_t a, b;
  if (VAR == 3) { a = gl::add_le(u, t); b = gl::sub_le(u, t); }
  else { a = add4(u, t); b = gl::sub_le(u, t); }
  lo = ng ? b : a;
  hi = ng ? a : b;
}
template <int L, int SH, bool NEGA, int VAR>
__device__ __forceinline__ void fwd(uint64_t (&a)[L]) {
  constexpr int LG = ntt::ilog2(L);
#pragma unroll
  for (int k = 0; k < LG; ++k) {
    const int len = L >> (k + 1);
#pragma unroll
    for (int b = 0; b < (1 << k); ++b) {
      const int s = ntt::stage_shift<NEGA>(L, SH, k, b);
#pragma unroll
      for (int j = 0; j < len; ++j) bfly<VAR>(a[b * 2 * len + j], a[b * 2 * len + j + len], s);
    }
  }
}
}  // namespace v

template <int VAR>
__global__ void __launch_bounds__(640, 1) ntt_loop(uint64_t* d, int iters) {
  uint64_t x[32];
  const size_t base = ((size_t)blockIdx.x * blockDim.x + threadIdx.x) * 32;
  for (int q = 0; q < 32; ++q) x[q] = d[base + q];
  for (int it = 0; it < iters; ++it) {
    v::fwd<32, 3, true, VAR>(x);
    v::fwd<32, 6, false, VAR>(x);
  }
  for (int q = 0; q < 32; ++q) d[base + q] = gl::canon(x[q]);
}

template <int VAR>
void run(const std::vector<uint64_t>& h, const std::vector<uint64_t>& ref, int blocks, int threads) {
  const size_t n = h.size();
  uint64_t* d;
  cudaMalloc(&d, n * 8);
  cudaMemcpy(d, h.data(), n * 8, cudaMemcpyHostToDevice);
  ntt_loop<VAR><<<blocks, threads>>>(d, 3);
  std::vector<uint64_t> got(n);
  cudaMemcpy(got.data(), d, n * 8, cudaMemcpyDeviceToHost);
  size_t bad = 0;
  for (size_t i = 0; i < n; ++i) bad += got[i] != ref[i];
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int iters = 100;
  ntt_loop<VAR><<<blocks, threads>>>(d, 5);
  cudaEventRecord(e0);
  ntt_loop<VAR><<<blocks, threads>>>(d, iters);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  const double bfly = (double)blocks * threads * iters * 160;
  printf("variant %d: mismatches %zu / %zu ; %.3f ms ; %.1f G butterflies/s ; %s\n", VAR, bad, n, ms,
         bfly / ms / 1e6, cudaGetErrorString(cudaGetLastError()));
  cudaFree(d);
}

int main() {
  const int blocks = 148, threads = 640;
  const size_t n = (size_t)blocks * threads * 32;
  std::vector<uint64_t> h(n), ref(n);
  uint64_t s = 0x1234567;
  for (size_t i = 0; i < n; ++i) {
    s = s * 6364136223846793005ull + 1442695040888963407ull;
    uint64_t v = s ^ (s >> 29);
    if (i % 97 == 0) v = 0xFFFFFFFFFFFFFFFFull - (i % 5);
    if (i % 89 == 0) v = 0xFFFFFFFF00000001ull + (i % 7);
    if (i % 83 == 0) v = (v & 0xFFFFFFFF00000000ull) | (i % 3);
    h[i] = v;
  }
  for (size_t t = 0; t < n / 32; ++t) {
    uint64_t x[32];
    for (int q = 0; q < 32; ++q) x[q] = h[t * 32 + q];
    for (int it = 0; it < 3; ++it) {
      ntt::fwd<32, 3, true>(x);
      ntt::fwd<32, 6, false>(x);
    }
    for (int q = 0; q < 32; ++q) ref[t * 32 + q] = gl::canon(x[q]);
  }
  run<0>(h, ref, blocks, threads);
  run<3>(h, ref, blocks, threads);
  run<4>(h, ref, blocks, threads);
  run<0>(h, ref, blocks, threads);
  return 0;
}
