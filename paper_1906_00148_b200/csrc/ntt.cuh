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

// t = x * 2^s for a compile-time shift s in [0, 192): returns x * 2^(s mod 96)
// and reports the sign (2^96 = -1) so butterflies swap add/sub instead of
// negating.
__host__ __device__ __forceinline__ uint64_t shift_twiddle(uint64_t x, int s, bool& negative) {
  negative = s >= 96;
  return gl::mul_pow2_pos(x, negative ? s - 96 : s);
}

// CT butterfly (lo, hi) <- (lo + w hi, lo - w hi), w = 2^s.
__host__ __device__ __forceinline__ void ct_bfly(uint64_t& lo, uint64_t& hi, int s) {
  bool ng;
  const uint64_t t = shift_twiddle(hi, s, ng);
  const uint64_t u = lo;
  lo = ng ? gl::sub(u, t) : gl::add(u, t);
  hi = ng ? gl::add(u, t) : gl::sub(u, t);
}

// GS butterfly (lo, hi) <- (lo + hi, (lo - hi) w), w = 2^s; for w = -2^(s-96)
// the difference is taken the other way round instead of negating.
__host__ __device__ __forceinline__ void gs_bfly(uint64_t& lo, uint64_t& hi, int s) {
  const uint64_t u = lo, v = hi;
  lo = gl::add(u, v);
  hi = s >= 96 ? gl::mul_pow2_pos(gl::sub(v, u), s - 96) : gl::mul_pow2_pos(gl::sub(u, v), s);
}

// Twiddle shift of block b at stage k of a length-L transform.
//   negacyclic (theta = 2^SH, order 2L): theta^((2 brev_k(b) + 1) L / 2^(k+1))
//   cyclic     (omega = 2^SH, order L) : omega^(brev_k(b) L / 2^(k+1))
template <bool NEGA>
__host__ __device__ constexpr int stage_shift(int L, int SH, int k, int b) {
  return NEGA ? (SH * (2 * brev(b, k) + 1) * (L >> (k + 1))) % 192
              : (SH * brev(b, k) * (L >> (k + 1))) % 192;
}
__host__ __device__ constexpr int inv_shift(int s) { return (192 - s) % 192; }

// Forward length-L transform in registers (CT, natural in, bit-reversed out).
//   NEGA: a[q] = sum_j a_j theta^((2 brev(q) + 1) j)
//   cyc : a[q] = sum_j a_j omega^(brev(q) j)
template <int L, int SH, bool NEGA>
__host__ __device__ __forceinline__ void fwd(uint64_t (&a)[L]) {
  constexpr int LG = ilog2(L);
#pragma unroll
  for (int k = 0; k < LG; ++k) {
    const int len = L >> (k + 1);
#pragma unroll
    for (int b = 0; b < (1 << k); ++b) {
      const int s = stage_shift<NEGA>(L, SH, k, b);
#pragma unroll
      for (int j = 0; j < len; ++j) ct_bfly(a[b * 2 * len + j], a[b * 2 * len + j + len], s);
    }
  }
}

// Exact inverse of fwd up to the factor L (GS, bit-reversed in, natural out).
template <int L, int SH, bool NEGA>
__host__ __device__ __forceinline__ void inv(uint64_t (&a)[L]) {
  constexpr int LG = ilog2(L);
#pragma unroll
  for (int k = LG - 1; k >= 0; --k) {
    const int len = L >> (k + 1);
#pragma unroll
    for (int b = 0; b < (1 << k); ++b) {
      const int s = inv_shift(stage_shift<NEGA>(L, SH, k, b));
#pragma unroll
      for (int j = 0; j < len; ++j) gs_bfly(a[b * 2 * len + j], a[b * 2 * len + j + len], s);
    }
  }
}

// The inverse split over two threads H = 0, 1 holding halves a[H L/2 + m]:
// stages k = LG-1 .. 1 never cross the halves ...
template <int L, int SH, bool NEGA, int H>
__host__ __device__ __forceinline__ void inv_half(uint64_t (&a)[L / 2]) {
  constexpr int LG = ilog2(L);
#pragma unroll
  for (int k = LG - 1; k >= 1; --k) {
    const int len = L >> (k + 1);
    const int nb = 1 << (k - 1);  // blocks per half
#pragma unroll
    for (int bb = 0; bb < nb; ++bb) {
      const int b = H * nb + bb;
      const int s = inv_shift(stage_shift<NEGA>(L, SH, k, b));
#pragma unroll
      for (int j = 0; j < len; ++j) gs_bfly(a[bb * 2 * len + j], a[bb * 2 * len + j + len], s);
    }
  }
}
// ... and stage 0 pairs element j with j + L/2 (one twiddle for all j).
// Thread H computes the butterflies j in [H L/4, (H+1) L/4): it keeps u (H=0)
// or v (H=1) for those j and receives the other operand from its partner.
// On return lo[m] = out[H L/4 + m], hi[m] = out[H L/4 + m + L/2].
template <int L, int SH, bool NEGA>
__host__ __device__ __forceinline__ void inv_cross(uint64_t (&lo)[L / 4], uint64_t (&hi)[L / 4]) {
  const int s = inv_shift(stage_shift<NEGA>(L, SH, 0, 0));
#pragma unroll
  for (int m = 0; m < L / 4; ++m) gs_bfly(lo[m], hi[m], s);
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
