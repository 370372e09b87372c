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
// The inverse runs both passes as inverse cyclic transforms by decimation in
// time (CT butterflies again, bit-reversed in, natural out); the negacyclic
// pass is then finished by the post-twist theta^(-j2) (a shift), merged into
// the final lift.  It is unscaled: N^-1 is folded into the bootstrapping key.
#pragma once
#include "gl64.cuh"

namespace ntt {

__host__ __device__ constexpr int brev(int x, int bits) {
  int r = 0;
  for (int b = 0; b < bits; ++b) r |= ((x >> b) & 1) << (bits - 1 - b);
  return r;
}
__host__ __device__ constexpr int ilog2(int x) { return x <= 1 ? 0 : 1 + ilog2(x >> 1); }

// CT butterfly (lo, hi) <- (lo + w hi, lo - w hi), w = 2^s, s compile-time in
// [0, 192).  w = -2^(s-96) for s >= 96: the sum and difference swap.  The
// twiddle product is formed <= p (gl::shl_le) so that the sum and difference
// need a single fold each (gl::add_le / sub_le); for w = +-1 the operand is
// lazy and the double-fold add / sub are used.
__host__ __device__ __forceinline__ void ct_bfly(uint64_t& lo, uint64_t& hi, int s) {
  const bool ng = s >= 96;
  const int sp = ng ? s - 96 : s;
  const uint64_t u = lo;
  uint64_t a, b;
  if (sp == 0) {
    a = gl::add(u, hi);
    b = gl::sub(u, hi);
  } else {
    const uint64_t t = gl::shl_le(hi, sp);
    a = gl::add_le(u, t);
    b = gl::sub_le(u, t);
  }
  lo = ng ? b : a;
  hi = ng ? a : b;
}

// Butterfly with twiddle 1 when hi <= p is known (a bounded product feeds it):
// single folds as in ct_bfly.
__host__ __device__ __forceinline__ void ct_bfly_le(uint64_t& lo, uint64_t& hi) {
  const uint64_t u = lo;
  lo = gl::add_le(u, hi);
  hi = gl::sub_le(u, hi);
}

// Twiddle shift of block b at stage k of a length-L forward transform.
//   negacyclic (theta = 2^SH, order 2L): theta^((2 brev_k(b) + 1) L / 2^(k+1))
//   cyclic     (omega = 2^SH, order L) : omega^(brev_k(b) L / 2^(k+1))
template <bool NEGA>
__host__ __device__ constexpr int stage_shift(int L, int SH, int k, int b) {
  return NEGA ? (SH * (2 * brev(b, k) + 1) * (L >> (k + 1))) % 192
              : (SH * brev(b, k) * (L >> (k + 1))) % 192;
}

// Forward length-L transform in registers (CT, natural in, bit-reversed out),
// stages K0 .. log2 L - 1.
//   NEGA: a[q] = sum_j a_j theta^((2 brev(q) + 1) j)
//   cyc : a[q] = sum_j a_j omega^(brev(q) j)
// HI_LE: the inputs a[L/2 ..] of stage 0 are <= p (bounded products), so
// stage-0 butterflies with twiddle 1 fold once.
template <int L, int SH, bool NEGA, int K0 = 0, bool HI_LE = false>
__host__ __device__ __forceinline__ void fwd(uint64_t (&a)[L]) {
  constexpr int LG = ilog2(L);
#pragma unroll
  for (int k = K0; k < LG; ++k) {
    const int len = L >> (k + 1);
#pragma unroll
    for (int b = 0; b < (1 << k); ++b) {
      const int s = stage_shift<NEGA>(L, SH, k, b);
#pragma unroll
      for (int j = 0; j < len; ++j) {
        if (HI_LE && k == 0 && s == 0) ct_bfly_le(a[j], a[j + len]);
        else ct_bfly(a[b * 2 * len + j], a[b * 2 * len + j + len], s);
      }
    }
  }
}

// Inverse cyclic transform by decimation in time (CT butterflies, bit-reversed
// in, natural out), unscaled:  in a[q] = X[brev(q)],  out a[j] = sum_m X[m]
// omega^(-m j), omega = 2^SH2 of order L.  Stage h (half-size 1, 2, .., L/2),
// position j < h in its block: twiddle omega^(-j L / 2h).
__host__ __device__ constexpr int dit_shift(int L, int SH2, int h, int j) {
  return (192 - (SH2 * j * (L / (2 * h))) % 192) % 192;
}
template <int L, int SH2>
__host__ __device__ __forceinline__ void inv_dit(uint64_t (&a)[L]) {
#pragma unroll
  for (int h = 1; h < L; h *= 2) {
#pragma unroll
    for (int blk = 0; blk < L; blk += 2 * h) {
#pragma unroll
      for (int j = 0; j < h; ++j) ct_bfly(a[blk + j], a[blk + j + h], dit_shift(L, SH2, h, j));
    }
  }
}

// The same transform split over two threads H = 0, 1 holding halves
// a[H L/2 + m]: stages h = 1 .. L/4 stay inside a half ...
// (all inputs are <= p: the first stage, twiddle 1 throughout, folds once)
template <int L, int SH2>
__host__ __device__ __forceinline__ void inv_dit_half(uint64_t (&a)[L / 2]) {
#pragma unroll
  for (int h = 1; h < L / 2; h *= 2) {
#pragma unroll
    for (int blk = 0; blk < L / 2; blk += 2 * h) {
#pragma unroll
      for (int j = 0; j < h; ++j) {
        if (h == 1) ct_bfly_le(a[blk + j], a[blk + j + h]);
        else ct_bfly(a[blk + j], a[blk + j + h], dit_shift(L, SH2, h, j));
      }
    }
  }
}
// ... and the last stage pairs j with j + L/2 (twiddle omega^-j).  Thread H
// computes the butterflies j in [H L/4, (H+1) L/4) from u = a[j] and
// v = a[j + L/2]; on return lo[m] = out[H L/4 + m], hi[m] = out[H L/4 + m + L/2].
template <int L, int SH2, int H>
__host__ __device__ __forceinline__ void inv_dit_cross(uint64_t (&lo)[L / 4], uint64_t (&hi)[L / 4]) {
#pragma unroll
  for (int m = 0; m < L / 4; ++m) ct_bfly(lo[m], hi[m], dit_shift(L, SH2, L / 2, H * (L / 4) + m));
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
