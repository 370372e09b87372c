// bootstrap_core.cuh — the per-thread steps of one CMux iteration of the blind
// rotation, written as __host__ __device__ functions of
// (lane index, shared-memory pointers, registers).  The sm_100a kernel
// (engine.cu) calls them between barriers; the host emulation (host_emu.cpp,
// tests only) calls them in loops over threads, so the exact device
// arithmetic is checked against the oracle on the CPU as well.
//
// One blind-rotation lane (one bootstrapped LWE sample) is served by 4 warps:
//   forward   warp w computes row r = w of the gadget decomposition (r = c*l+j,
//             c = 0 for the accumulator's A polynomial, 1 for B; R2)
//             and its full forward NTT (32 threads x 32 registers);
//   pointwise all threads of the CTA, BK_i read once per CTA for all lanes;
//   inverse   warps (2c, 2c+1) split the inverse NTT of output component c:
//             thread (H, lane) holds half of a 32-point column, the last
//             butterfly stage exchanges L/4 values through shared memory
//             (decimation-in-time CT butterflies, ntt.cuh).
//
// Shared memory of one lane:
//   acc  : uint32[2][N]          the TRLWE accumulator (A, B), torus32
//   buf  : uint64[4][L][L+1]     per-row NTT storage (order q*L + i in the first
//                                N words) / transposition scratch (i*(L+1) + j1,
//                                padded: conflict-free column access); rows 2, 3
//                                double as the inverse's exchange buffers
//   abar : uint16[n+1]           modulus-switched input sample
#pragma once
#include "ntt.cuh"

namespace br {

constexpr uint32_t MU = 1u << 29;  // 1/8

struct Geometry {
  uint32_t N, n, l, bg_bits;
  uint32_t lg2N;        // log2(2N)
  uint32_t dec_offset;  // sum_j (Bg/2) 2^{32-j bg} + 2^{32-l bg-1}   (R8)
};

__host__ __device__ inline uint32_t modswitch(uint32_t x, uint32_t lg2N) {
  return (x + (1u << (31 - lg2N))) >> (32 - lg2N);  // R7: round half up mod 2N
}

template <class S>
struct Lane {
  static constexpr int L = S::L, N = S::N;
  static constexpr int RS = L * (L + 1);  // words per buf row
  static constexpr size_t bytes(uint32_t n) {
    return (size_t)2 * N * 4 + (size_t)4 * RS * 8 + ((n + 1) * 2 + 15) / 16 * 16;
  }
  uint32_t* acc;
  uint64_t* buf;
  uint16_t* abar;
  __host__ __device__ explicit Lane(uint8_t* base)
      : acc(reinterpret_cast<uint32_t*>(base)),
        buf(reinterpret_cast<uint64_t*>(base + 2 * N * 4)),
        abar(reinterpret_cast<uint16_t*>(base + 2 * N * 4 + 4 * RS * 8)) {}
  __host__ __device__ uint64_t* row(int r) const { return buf + (size_t)r * RS; }
};

// ---- forward path of row w ------------------------------------------------

// Load: digit polynomial of row w of D = X^a ACC - ACC, column j1 = lane, as
// small signed integers (|digit| <= Bg/2).
template <class S>
__host__ __device__ __forceinline__ void load_digits(const Geometry& g, int w, int lane,
                                                     const uint32_t* acc, uint32_t a,
                                                     int32_t (&d)[S::L]) {
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
    d[j2] = (int32_t)((y >> shift) & mask) - (int32_t)half;
  }
}

// Pass 1 (negacyclic, shift twiddles) + transposed store.
template <class S>
__host__ __device__ __forceinline__ void fwd_pass1_store(int lane, uint64_t (&x)[S::L],
                                                         uint64_t* row) {
  constexpr int L = S::L;
  ntt::fwd<L, S::SH, true>(x);
#pragma unroll
  for (int q = 0; q < L; ++q) row[ntt::brev(q, ntt::ilog2(L)) * (L + 1) + lane] = x[q];
}

// Pass 1 of a digit polynomial: stage 0 (pairs j, j + L/2, twiddle theta^(L/2)
// = 2^48) is exact in int64 because the digits are small (|d| 2^48 < 2^57), so
// it needs no modular reduction; the field elements enter at stage 1.
template <class S>
__host__ __device__ __forceinline__ void fwd_pass1_digits_store(int lane, const int32_t (&d)[S::L],
                                                                uint64_t* row) {
  constexpr int L = S::L;
  static_assert(ntt::stage_shift<true>(L, S::SH, 0, 0) == 48, "stage-0 twiddle is 2^48");
  uint64_t x[L];
#pragma unroll
  for (int j = 0; j < L / 2; ++j) {
    const int64_t u = d[j], t = (int64_t)d[j + L / 2] * (int64_t(1) << 48);
    x[j] = gl::from_i64(u + t);
    x[j + L / 2] = gl::from_i64(u - t);
  }
  ntt::fwd<L, S::SH, true, 1>(x);
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
  for (int j1 = 1; j1 < L; ++j1) y[j1] = gl::mul_le(row[i * (L + 1) + j1], tw[j1 * L + i]);
}

// Pass 2 (cyclic, shift twiddles) + store in NTT storage order (q*L + i).
template <class S>
__host__ __device__ __forceinline__ void fwd_pass2_store(int i, uint64_t (&y)[S::L], uint64_t* row) {
  constexpr int L = S::L;
  ntt::fwd<L, S::SH2, false, 0, true>(y);  // y[L/2 ..] are twisted: <= p
#pragma unroll
  for (int q = 0; q < L; ++q) row[q * L + i] = y[q];
}

// ---- pointwise multiply-accumulate with BK_i (lazy: one reduction per output)
// out_c[p] = sum_r D_r[p] * BK_i[r][c][p]; b[r*2 + c] = BK_i[r][c][p].
template <class S>
__host__ __device__ __forceinline__ void pointwise_pos(uint64_t* buf, int p, const uint64_t (&b)[8]) {
  constexpr int RS = Lane<S>::RS;
  uint64_t d[4];
#pragma unroll
  for (int r = 0; r < 4; ++r) d[r] = buf[r * RS + p];
  gl::Acc3 oa, ob;
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    gl::mac(oa, d[r], b[2 * r + 0]);
    gl::mac(ob, d[r], b[2 * r + 1]);
  }
  buf[0 * RS + p] = gl::reduce_acc_le(oa);  // <= p: the inverse's first stage folds once
  buf[1 * RS + p] = gl::reduce_acc_le(ob);
}

// ---- inverse path: output component c, thread (H, lane) ----------------------
// Exchange buffer: row 2 + c of buf, xbuf[(H*L/4 + m)*L + lane].

template <class S, int H>
__host__ __device__ __forceinline__ void inv_a_load(int i, const uint64_t* row, uint64_t (&y)[S::L / 2]) {
  constexpr int L = S::L;
#pragma unroll
  for (int m = 0; m < L / 2; ++m) y[m] = row[(H * (L / 2) + m) * L + i];
}

template <class S, int H, bool NEGA>
__host__ __device__ __forceinline__ void inv_stages_send(int lane, uint64_t (&y)[S::L / 2], uint64_t* xbuf) {
  constexpr int L = S::L;
  ntt::inv_dit_half<L, S::SH2>(y);  // both passes: inverse cyclic, omega = theta^2 = 2^SH2
  // H = 0 sends its lo values for j in [L/4, L/2); H = 1 its hi values for j < L/4
#pragma unroll
  for (int m = 0; m < L / 4; ++m) xbuf[(H * (L / 4) + m) * L + lane] = y[(H == 0 ? L / 4 : 0) + m];
}

template <class S, int H, bool NEGA>
__host__ __device__ __forceinline__ void inv_recv_cross(int lane, const uint64_t (&y)[S::L / 2],
                                                        const uint64_t* xbuf, uint64_t (&lo)[S::L / 4],
                                                        uint64_t (&hi)[S::L / 4]) {
  constexpr int L = S::L;
  const int P = 1 - H;  // partner
#pragma unroll
  for (int m = 0; m < L / 4; ++m) {
    const uint64_t other = xbuf[(P * (L / 4) + m) * L + lane];
    if (H == 0) {
      lo[m] = y[m];
      hi[m] = other;
    } else {
      lo[m] = other;
      hi[m] = y[L / 4 + m];
    }
  }
  ntt::inv_dit_cross<L, S::SH2, H>(lo, hi);
}

// After pass A: untwist and store transposed (thread row i; outputs j1 =
// H*L/4 + m and H*L/4 + m + L/2).
template <class S, int H>
__host__ __device__ __forceinline__ void inv_a_store(int i, const uint64_t (&lo)[S::L / 4],
                                                     const uint64_t (&hi)[S::L / 4],
                                                     const uint64_t* itw, uint64_t* row) {
  constexpr int L = S::L;
#pragma unroll
  for (int m = 0; m < L / 4; ++m) {
    const int j1 = H * (L / 4) + m, j1h = j1 + L / 2;
    // every pass-B input <= p (j1 = 0 is not twisted: bounded by shl_le(x, 0))
    row[i * (L + 1) + j1] = j1 == 0 ? gl::shl_le(lo[m], 0) : gl::mul_le(lo[m], itw[j1 * L + i]);
    row[i * (L + 1) + j1h] = gl::mul_le(hi[m], itw[j1h * L + i]);
  }
}

// Pass B load: column j1 = lane in the nega_fwd output order (register q <-> row brev(q)).
template <class S, int H>
__host__ __device__ __forceinline__ void inv_b_load(int j1, const uint64_t* row, uint64_t (&y)[S::L / 2]) {
  constexpr int L = S::L;
#pragma unroll
  for (int m = 0; m < L / 2; ++m) y[m] = row[ntt::brev(H * (L / 2) + m, ntt::ilog2(L)) * (L + 1) + j1];
}

// After pass B: the negacyclic post-twist theta^(-j2) = -2^(96 - SH j2) (a
// shift, j2 > 0), the centred lift mod 2^32 and ACC_c += result (coefficients
// j1 + L j2).
template <class S>
__host__ __device__ __forceinline__ uint32_t twist_lift(uint64_t x, int j2) {
  if (j2 == 0) return gl::lift32(x);
  return gl::lift32_neg(gl::shl_le(x, 96 - S::SH * j2));
}
template <class S, int H>
__host__ __device__ __forceinline__ void inv_b_acc(int j1, const uint64_t (&lo)[S::L / 4],
                                                   const uint64_t (&hi)[S::L / 4], uint32_t* accc) {
  constexpr int L = S::L;
#pragma unroll
  for (int m = 0; m < L / 4; ++m) {
    const int j2 = H * (L / 4) + m;
    accc[j1 + L * j2] += twist_lift<S>(lo[m], j2);
    accc[j1 + L * (j2 + L / 2)] += twist_lift<S>(hi[m], j2 + L / 2);
  }
}

// ---- BK transform (setup, K1) ----------------------------------------------
template <class S>
__host__ __device__ __forceinline__ void load_poly_signed(int lane, const uint32_t* poly,
                                                          uint64_t (&x)[S::L]) {
  constexpr int L = S::L;
#pragma unroll
  for (int j2 = 0; j2 < L; ++j2) x[j2] = gl::from_i64((int32_t)poly[lane + L * j2]);
}

template <class S>
__host__ __device__ __forceinline__ void fwd_pass2_store_scaled(int i, uint64_t (&y)[S::L],
                                                                uint64_t ninv, uint64_t* out) {
  constexpr int L = S::L;
  ntt::fwd<L, S::SH2, false>(y);
#pragma unroll
  for (int q = 0; q < L; ++q) out[q * L + i] = gl::canon(gl::mul(y[q], ninv));
}

// ---- test vector ---------------------------------------------------------------
// ACC = (0, X^{-bbar} v), v = mu sum_j X^j: coefficient m collects j = m + bbar
// (mod 2N); +mu if that j is in [0, N), -mu otherwise.
__host__ __device__ inline uint32_t testvec_coeff(uint32_t m, uint32_t bbar, uint32_t N) {
  const uint32_t j = (m + bbar) & (2 * N - 1);
  return j < N ? MU : 0u - MU;
}

}  // namespace br
