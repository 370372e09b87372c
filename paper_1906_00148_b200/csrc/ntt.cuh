// ntt.cuh — negacyclic NTT of length N = L * L over Goldilocks, built from two
// in-register radix-L passes whose internal twiddles are all powers of two.
//
// Decomposition.  Index m = j1 + L j2.  psi is a primitive
// 2N-th root of unity chosen with psi^L = theta = 2^(96/L) (theta has order
// 2L, a power of two because 2 has order 192 mod p).
//   pass 1 (thread j1, registers j2): y[j1][i] = sum_j2 x[j1 + L j2] theta^((2i+1) j2)
//           a length-L negacyclic NTT with shift twiddles; register q holds i = brev(q)
//   transpose through shared memory
//   twist   (thread i, registers j1): y[j1][i] *= psi^((2i+1) j1)   (general modmul)
//   pass 2: z[i][m] = sum_j1 y'[j1][i] omega^(m j1), omega = psi^(2L) = theta^2
//           a length-L cyclic NTT with shift twiddles; register q holds m = brev(q)
// so z[i][m] = x(psi^(2k+1)) with k = i + L m: the negacyclic NTT evaluated at
// the odd powers of psi.  Storage ("NTT-domain") position of k is q*L + i.
// Only the twist is a general multiplication: L*L - (2L-1) modmuls per
// transform instead of (N/2) log2 N for a radix-2 transform.
//
// The inverse runs the exact reverse (Gentleman-Sande butterflies, inverse
// twiddles) and is unscaled: N^-1 is folded into the bootstrapping key.
#pragma once
#include "gl64.cuh"

namespace ntt {

__host__ __device__ constexpr int brev(int x, int bits) {
  int r = 0;
  for (int b = 0; b < bits; ++b) r |= ((x >> b) & 1) << (bits - 1 - b);
  return r;
}
__host__ __device__ constexpr int ilog2(int x) { return x <= 1 ? 0 : 1 + ilog2(x >> 1); }

// Forward negacyclic length-L NTT in registers; theta = 2^SH has order 2L.
// Out: a[q] = sum_j a_j theta^((2 brev(q) + 1) j).
template <int L, int SH>
__host__ __device__ __forceinline__ void nega_fwd(uint64_t (&a)[L]) {
  constexpr int LG = ilog2(L);
#pragma unroll
  for (int k = 0; k < LG; ++k) {
    const int len = L >> (k + 1);
#pragma unroll
    for (int b = 0; b < (1 << k); ++b) {
      const int x = (2 * brev(b, k) + 1) * len;  // twiddle theta^x
      const int s = (SH * x) % 192;
#pragma unroll
      for (int j = 0; j < len; ++j) {
        const int lo = b * 2 * len + j, hi = lo + len;
        uint64_t t = gl::mul_pow2(a[hi], s);
        uint64_t u = a[lo];
        a[lo] = gl::add(u, t);
        a[hi] = gl::sub(u, t);
      }
    }
  }
}

// Exact inverse of nega_fwd up to the factor L.
template <int L, int SH>
__host__ __device__ __forceinline__ void nega_inv(uint64_t (&a)[L]) {
  constexpr int LG = ilog2(L);
#pragma unroll
  for (int k = LG - 1; k >= 0; --k) {
    const int len = L >> (k + 1);
#pragma unroll
    for (int b = 0; b < (1 << k); ++b) {
      const int x = (2 * brev(b, k) + 1) * len;
      const int s = (192 - (SH * x) % 192) % 192;  // theta^-x
#pragma unroll
      for (int j = 0; j < len; ++j) {
        const int lo = b * 2 * len + j, hi = lo + len;
        uint64_t u = a[lo], v = a[hi];
        a[lo] = gl::add(u, v);
        a[hi] = gl::mul_pow2(gl::sub(u, v), s);
      }
    }
  }
}

// Forward cyclic length-L NTT in registers; omega = 2^SH2 has order L.
// Out: a[q] = sum_j a_j omega^(brev(q) j).
template <int L, int SH2>
__host__ __device__ __forceinline__ void cyc_fwd(uint64_t (&a)[L]) {
  constexpr int LG = ilog2(L);
#pragma unroll
  for (int k = 0; k < LG; ++k) {
    const int len = L >> (k + 1);
#pragma unroll
    for (int b = 0; b < (1 << k); ++b) {
      const int x = brev(b, k) * len;  // omega^x
      const int s = (SH2 * x) % 192;
#pragma unroll
      for (int j = 0; j < len; ++j) {
        const int lo = b * 2 * len + j, hi = lo + len;
        uint64_t t = gl::mul_pow2(a[hi], s);
        uint64_t u = a[lo];
        a[lo] = gl::add(u, t);
        a[hi] = gl::sub(u, t);
      }
    }
  }
}

template <int L, int SH2>
__host__ __device__ __forceinline__ void cyc_inv(uint64_t (&a)[L]) {
  constexpr int LG = ilog2(L);
#pragma unroll
  for (int k = LG - 1; k >= 0; --k) {
    const int len = L >> (k + 1);
#pragma unroll
    for (int b = 0; b < (1 << k); ++b) {
      const int x = brev(b, k) * len;
      const int s = (192 - (SH2 * x) % 192) % 192;
#pragma unroll
      for (int j = 0; j < len; ++j) {
        const int lo = b * 2 * len + j, hi = lo + len;
        uint64_t u = a[lo], v = a[hi];
        a[lo] = gl::add(u, v);
        a[hi] = gl::mul_pow2(gl::sub(u, v), s);
      }
    }
  }
}

// Compile-time description of the transform for a ring dimension N = L^2.
template <int N_>
struct Shape;
template <>
struct Shape<1024> {
  static constexpr int N = 1024, L = 32, SH = 3, SH2 = 6;  // theta = 2^3, omega = 2^6
};
template <>
struct Shape<256> {
  static constexpr int N = 256, L = 16, SH = 6, SH2 = 12;  // theta = 2^6, omega = 2^12
};

// Host-side: psi with psi^L = theta (primitive 2N-th root), and the twist tables
// tw[j1][i] = psi^((2i+1) j1), itw[j1][i] = psi^(-(2i+1) j1).
inline uint64_t find_psi(int N, int L, int SH) {
  const uint64_t g = 7;  // generates F_p^*
  uint64_t psi0 = gl::pow(g, (gl::P - 1) / (2 * (uint64_t)N));
  uint64_t theta = gl::pow(2, SH);
  for (int u = 1; u < 2 * N; u += 2) {
    uint64_t cand = gl::pow(psi0, u);
    if (gl::pow(cand, L) == theta) return cand;
  }
  return 0;
}

inline void make_twists(int N, int L, int SH, uint64_t* tw, uint64_t* itw) {
  uint64_t psi = find_psi(N, L, SH);
  uint64_t ipsi = gl::pow(psi, 2 * (uint64_t)N - 1);
  for (int j1 = 0; j1 < L; ++j1)
    for (int i = 0; i < L; ++i) {
      tw[j1 * L + i] = gl::pow(psi, (uint64_t)(2 * i + 1) * j1);
      itw[j1 * L + i] = gl::pow(ipsi, (uint64_t)(2 * i + 1) * j1);
    }
}

}  // namespace ntt
