// bootstrap_core.cuh — the per-thread steps of one CMux iteration of the blind
// rotation, written as __host__ __device__ functions of
// (warp, lane, shared-memory pointers, registers).  The sm_100a kernel
// (bootstrap.cu) calls them between __syncwarp/__syncthreads; the host
// emulation (host_emu.cpp, tests only) calls them in loops over threads, so
// the exact device arithmetic is checked against the oracle on the CPU too.
//
// One blind-rotation lane (one bootstrapped LWE sample) is one CTA of 4 warps.
// Warp w owns row r = w of the gadget decomposition, r = c*l + j (c = 0 for
// the accumulator's A polynomial, 1 for B; j = digit level) — DESIGN.md R2.
//
// Shared memory of one lane:
//   acc  : uint32[2][N]           the TRLWE accumulator (A, B), torus32
//   buf  : uint64[4][L][L+1]      per-row NTT scratch; storage order q*L + i
//                                  in the first N words, transposed pass-1
//                                  output at i*(L+1) + j1 (padded: no bank
//                                  conflicts for the column reads)
#pragma once
#include "ntt.cuh"

namespace br {

constexpr uint32_t MU = 1u << 29;  // 1/8

struct Geometry {
  uint32_t N, n, l, bg_bits;
  uint32_t lg2N;       // log2(2N)
  uint32_t dec_offset; // sum_j (Bg/2) 2^{32-j bg} + 2^{32-l bg-1}   (R8)
};

__host__ __device__ inline uint32_t modswitch(uint32_t x, uint32_t lg2N) {
  return (x + (1u << (31 - lg2N))) >> (32 - lg2N);  // R7: round half up mod 2N
}

template <class S>
__host__ __device__ __forceinline__ uint64_t* buf_row(uint64_t* buf, int w) {
  return buf + (size_t)w * S::L * (S::L + 1);
}

// ---- forward path of row w ------------------------------------------------

// Load: digit polynomial of row w of D = X^a ACC - ACC, column j1 = lane.
template <class S>
__host__ __device__ __forceinline__ void load_digits(const Geometry& g, int w, int lane,
                                                     const uint32_t* acc, uint32_t a,
                                                     uint64_t (&x)[S::L]) {
  constexpr int L = S::L, N = S::N;
  const int c = w / g.l, j = w % g.l;
  const uint32_t* P = acc + c * N;
  const uint32_t shift = 32 - (j + 1) * g.bg_bits;
  const uint32_t mask = (1u << g.bg_bits) - 1, half = 1u << (g.bg_bits - 1);
#pragma unroll
  for (int j2 = 0; j2 < L; ++j2) {
    const uint32_t m = lane + L * j2;
    const uint32_t idx = (m - a) & (2 * N - 1);  // (X^a P)[m] = +-P[m - a]
    uint32_t v = P[idx & (N - 1)];
    if (idx >= (uint32_t)N) v = 0u - v;
    const uint32_t y = v - P[m] + g.dec_offset;
    const int32_t d = (int32_t)((y >> shift) & mask) - (int32_t)half;
    x[j2] = gl::from_i64(d);
  }
}

// Pass 1 + transposed store: x (coefficients j2 of column j1=lane) -> scratch.
template <class S>
__host__ __device__ __forceinline__ void fwd_pass1_store(int lane, uint64_t (&x)[S::L],
                                                         uint64_t* row) {
  constexpr int L = S::L;
  ntt::nega_fwd<L, S::SH>(x);
#pragma unroll
  for (int q = 0; q < L; ++q) row[ntt::brev(q, ntt::ilog2(L)) * (L + 1) + lane] = x[q];
}

// Pass 2 load: thread i reads its transposed row and applies the twist.
template <class S>
__host__ __device__ __forceinline__ void fwd_pass2_load(int i, const uint64_t* row,
                                                        const uint64_t* tw, uint64_t (&y)[S::L]) {
  constexpr int L = S::L;
  y[0] = row[i * (L + 1)];
#pragma unroll
  for (int j1 = 1; j1 < L; ++j1) y[j1] = gl::mul(row[i * (L + 1) + j1], tw[j1 * L + i]);
}

// Pass 2 + store in NTT storage order (position q*L + i).
template <class S>
__host__ __device__ __forceinline__ void fwd_pass2_store(int i, uint64_t (&y)[S::L], uint64_t* row) {
  constexpr int L = S::L;
  ntt::cyc_fwd<L, S::SH2>(y);
#pragma unroll
  for (int q = 0; q < L; ++q) row[q * L + i] = y[q];
}

// ---- pointwise multiply-accumulate with BK_i --------------------------------
// out_c[p] = sum_r D_r[p] * BK_i[r][c][p] for p = t, t + T, ...; results go to
// rows 0 (c = A) and 1 (c = B) of buf.  bki: uint64[2l][2][N] storage order.
template <class S>
__host__ __device__ __forceinline__ void pointwise(int t, int T, int rows, uint64_t* buf,
                                                   const uint64_t* bki) {
  constexpr int L = S::L, N = S::N;
  constexpr int RS = L * (L + 1);
  for (int p = t; p < N; p += T) {
    uint64_t d[4];
#pragma unroll
    for (int r = 0; r < 4; ++r) d[r] = r < rows ? buf[r * RS + p] : 0;
    uint64_t oa = 0, ob = 0;
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      if (r < rows) {
        oa = gl::add(oa, gl::mul(d[r], bki[(size_t)(r * 2 + 0) * N + p]));
        ob = gl::add(ob, gl::mul(d[r], bki[(size_t)(r * 2 + 1) * N + p]));
      }
    }
    buf[0 * RS + p] = oa;
    buf[1 * RS + p] = ob;
  }
}

// ---- inverse path of output component c = w ---------------------------------

template <class S>
__host__ __device__ __forceinline__ void inv_pass2_load(int i, const uint64_t* row,
                                                        uint64_t (&y)[S::L]) {
  constexpr int L = S::L;
#pragma unroll
  for (int q = 0; q < L; ++q) y[q] = row[q * L + i];
}

template <class S>
__host__ __device__ __forceinline__ void inv_pass2_store(int i, uint64_t (&y)[S::L],
                                                         const uint64_t* itw, uint64_t* row) {
  constexpr int L = S::L;
  ntt::cyc_inv<L, S::SH2>(y);
  row[i * (L + 1)] = y[0];
#pragma unroll
  for (int j1 = 1; j1 < L; ++j1) row[i * (L + 1) + j1] = gl::mul(y[j1], itw[j1 * L + i]);
}

// Pass 1 inverse for column j1 = lane, then lift mod 2^32 and ACC_c += result.
template <class S>
__host__ __device__ __forceinline__ void inv_pass1_acc(int lane, const uint64_t* row,
                                                       uint32_t* accc) {
  constexpr int L = S::L;
  uint64_t x[L];
#pragma unroll
  for (int q = 0; q < L; ++q) x[q] = row[ntt::brev(q, ntt::ilog2(L)) * (L + 1) + lane];
  ntt::nega_inv<L, S::SH>(x);
#pragma unroll
  for (int j2 = 0; j2 < L; ++j2) accc[lane + L * j2] += gl::lift32(x[j2]);
}

// ---- BK transform (setup, K1) ----------------------------------------------
// Load column j1 = lane of a torus32 polynomial with the signed lift.
template <class S>
__host__ __device__ __forceinline__ void load_poly_signed(int lane, const uint32_t* poly,
                                                          uint64_t (&x)[S::L]) {
  constexpr int L = S::L;
#pragma unroll
  for (int j2 = 0; j2 < L; ++j2) x[j2] = gl::from_i64((int32_t)poly[lane + L * j2]);
}

// Pass 2 + N^-1 scaling + store to a global NTT-domain polynomial.
template <class S>
__host__ __device__ __forceinline__ void fwd_pass2_store_scaled(int i, uint64_t (&y)[S::L],
                                                                uint64_t ninv, uint64_t* out) {
  constexpr int L = S::L;
  ntt::cyc_fwd<L, S::SH2>(y);
#pragma unroll
  for (int q = 0; q < L; ++q) out[q * L + i] = gl::canon(gl::mul(y[q], ninv));
}

// ---- test vector and sample extraction ---------------------------------------
// ACC = (0, X^{-bbar} v), v = mu sum_j X^j: coefficient m of X^{-bbar} v is
// +mu if m + bbar lands in [0, N) of the 2N cycle, -mu otherwise.
__host__ __device__ inline uint32_t testvec_coeff(uint32_t m, uint32_t bbar, uint32_t N) {
  // X^{-bbar} X^j = X^{j - bbar}; coefficient m collects j = m + bbar (mod 2N)
  const uint32_t j = (m + bbar) & (2 * N - 1);
  return j < N ? MU : 0u - MU;
}

}  // namespace br
