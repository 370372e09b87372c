// fold_bench.cu — ALU/FMA pipe balance of the butterfly folds (sm_100a).
// Each variant of (shl_le, add_le, sub_le) is checked against the host gl::
// results on edge + random values, then timed inside the 32-point pass pair.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --expt-relaxed-constexpr \
//        -DGL_ADDSUB_PTX -I paper_1906_00148_b200/csrc tools/microbench/fold_bench.cu -o fbb
#include <cstdio>
#include <vector>

#include "ntt.cuh"

namespace v {
// ---- sub_le variants ----
template <int V>
__device__ __forceinline__ uint64_t sub_le(uint64_t x, uint64_t y) {
  if (V == 0) return gl::sub_le(x, y);
  if (V == 2) {  // fold on the FMA pipe: d0 + (-bw)(-1), d1 + bw*1 + carry
    uint32_t d0, d1, bw;
    asm("sub.cc.u32 %0, %3, %5;\n\t"
        "subc.cc.u32 %1, %4, %6;\n\t"
        "subc.u32 %2, 0, 0;\n\t"
        "mad.lo.cc.u32 %0, %2, 0xFFFFFFFF, %0;\n\t"
        "madc.lo.u32 %1, %2, 1, %1;"
        : "=&r"(d0), "=&r"(d1), "=&r"(bw)
        : "r"((uint32_t)x), "r"((uint32_t)(x >> 32)), "r"((uint32_t)y), "r"((uint32_t)(y >> 32)));
    return ((uint64_t)d1 << 32) | d0;
  }
  // V1: d - b EPS = (d + b) - b 2^32 with IMAD.WIDE for the 64-bit add
  uint32_t d0, d1, b;
  asm("sub.cc.u32 %0, %3, %5;\n\t"
      "subc.cc.u32 %1, %4, %6;\n\t"
      "subc.u32 %2, 0, 0;"  // -borrow
      : "=&r"(d0), "=&r"(d1), "=&r"(b)
      : "r"((uint32_t)x), "r"((uint32_t)(x >> 32)), "r"((uint32_t)y), "r"((uint32_t)(y >> 32)));
  uint64_t r;
  const uint32_t nb = 0u - b;  // borrow (0/1)
  asm("mad.wide.u32 %0, %1, 1, %2;" : "=l"(r) : "r"(nb), "l"(((uint64_t)d1 << 32) | d0));
  return r - ((uint64_t)nb << 32);
}
// ---- add_le variants ----
template <int V>
__device__ __forceinline__ uint64_t add_le(uint64_t x, uint64_t y) {
  if (V == 0) return gl::add_le(x, y);
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
// ---- shl_le q = 0 variants (s < 32) ----
template <int V>
__device__ __forceinline__ uint64_t shl_le(uint64_t v, const int s) {
  if (V == 0 || s >= 32 || s == 0) return gl::shl_le(v, s);
  const int r = s;
  const uint32_t v0 = (uint32_t)v, v1 = (uint32_t)(v >> 32);
  const uint32_t T0 = v0 << r, T1 = __funnelshift_l(v0, v1, r), T2 = v1 >> (32 - r);
  uint32_t o0, o1, m;
  if (V == 1) {  // select by IMAD: o = e + c EPS
    uint32_t c, e0, e1, w0, w1;
    asm("mad.lo.cc.u32 %0, %5, 0xFFFFFFFF, %6;\n\t"
        "madc.hi.cc.u32 %1, %5, 0xFFFFFFFF, %7;\n\t"
        "addc.u32 %2, 0, 0;\n\t"
        "add.cc.u32 %3, %0, 1;\n\t"
        "addc.u32 %4, %1, 0xFFFFFFFF;"
        : "=&r"(w0), "=&r"(w1), "=&r"(c), "=&r"(e0), "=&r"(e1)
        : "r"(T2 + 1), "r"(T0), "r"(T1));
    asm("mad.lo.cc.u32 %0, %2, 0xFFFFFFFF, %3;\n\t"
        "madc.hi.u32 %1, %2, 0xFFFFFFFF, %4;"
        : "=&r"(o0), "=&r"(o1)
        : "r"(c), "r"(e0), "r"(e1));
    (void)w0;
    (void)w1;
  } else {  // V2: c from the (T2+1) sum, result (T1:T0) + (T2 + c) EPS
    uint32_t w0, w1;
    asm("mad.lo.cc.u32 %0, %3, 0xFFFFFFFF, %4;\n\t"
        "madc.hi.cc.u32 %1, %3, 0xFFFFFFFF, %5;\n\t"
        "addc.u32 %2, %6, 0;"
        : "=&r"(w0), "=&r"(w1), "=&r"(m)
        : "r"(T2 + 1), "r"(T0), "r"(T1), "r"(T2));
    asm("mad.lo.cc.u32 %0, %2, 0xFFFFFFFF, %3;\n\t"
        "madc.hi.u32 %1, %2, 0xFFFFFFFF, %4;"
        : "=&r"(o0), "=&r"(o1)
        : "r"(m), "r"(T0), "r"(T1));
    (void)w0;
    (void)w1;
  }
  return ((uint64_t)o1 << 32) | o0;
}
// variant code: hundreds = shl, tens = add, ones = sub
template <int VAR>
__device__ __forceinline__ void bfly(uint64_t& lo, uint64_t& hi, int s) {
  constexpr int VS = VAR / 100, VA = (VAR / 10) % 10, VU = VAR % 10;
  const bool ng = s >= 96;
  const int sp = ng ? s - 96 : s;
  const uint64_t u = lo;
  uint64_t a, b;
  if (sp == 0) {
    a = gl::add(u, hi);
    b = gl::sub(u, hi);
  } else {
    const uint64_t t = shl_le<VS>(hi, sp);
    a = add_le<VA>(u, t);
    b = sub_le<VU>(u, t);
  }
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
  float best = 1e9f;
  for (int rep = 0; rep < 3; ++rep) {
    cudaEventRecord(e0);
    ntt_loop<VAR><<<blocks, threads>>>(d, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    best = ms < best ? ms : best;
  }
  const double bfly = (double)blocks * threads * iters * 160;
  printf("variant %03d: mismatches %zu / %zu ; %.3f ms ; %.1f G butterflies/s ; %s\n", VAR, bad, n,
         best, bfly / best / 1e6, cudaGetErrorString(cudaGetLastError()));
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
    if (i % 79 == 0) v = (v | 0xFFFFFFFF00000000ull);
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
  run<2>(h, ref, blocks, threads);
  run<100>(h, ref, blocks, threads);
  run<102>(h, ref, blocks, threads);
  run<0>(h, ref, blocks, threads);
  return 0;
}
