/*
 * she_rng.h — the seeded synthetic-input generator shared by BOTH the product
 * client library (paper_1906_00148_b200/csrc/client.cpp) and the CPU oracle
 * (oracle/oracle.c).
 *
 * This header holds NO arithmetic of the method (no torus products, no
 * encryption, no bootstrapping).  It only answers "which random number does
 * input object X draw", so that the two independent implementations consume
 * the same random masks, noise samples and secret-key bits (task rule ③:
 * "random numbers the method draws are passed in as inputs, or each side
 * implements the same counter-based generator").
 *
 * Generator: counter-based SplitMix64.  Value #index of stream `stream` under
 * `seed` is mix64(key(seed, stream) + GOLDEN * (index + 1)).
 *
 * Gaussian: Box–Muller from two consecutive counters, rounded to the nearest
 * integer on the 2^32 torus scale (SURVEY.md §8(c) "Gaussian sampling and
 * RNG" reading; the paper's TFHE noise is Gaussian, §4).  Only
 * multiplications surround the libm calls, so no FMA contraction can make the
 * two builds differ; both builds also pass -ffp-contract=off.
 *
 * Index layouts below are the input-object numbering contract (documented in
 * include/she.h and DESIGN.md §3).
 */
#ifndef SHE_RNG_H_
#define SHE_RNG_H_

#include <math.h>
#include <stdint.h>

#define SHE_GOLDEN 0x9E3779B97F4A7C15ULL

/* The integer streams are also compiled for the device (the GPU client of
 * csrc/engine.cu draws its masks here); the Gaussian stays host-only. */
#if defined(__CUDACC__)
#define SHE_RNG_FN __host__ __device__ static inline
#else
#define SHE_RNG_FN static inline
#endif

enum {
  SHE_STREAM_LWE_KEY = 1,   /* s_i, i < n            (bit = u64 & 1)            */
  SHE_STREAM_TRLWE_KEY = 2, /* S_j, j < N            (bit = u64 & 1)            */
  SHE_STREAM_BK_MASK = 3,   /* A coeffs of BK rows  (u32 = u64 >> 32)          */
  SHE_STREAM_BK_NOISE = 4,  /* e coeffs of BK rows  (gaussian, sigma=a_bk*2^32) */
  SHE_STREAM_KSK_MASK = 5,  /* a of KSK entries     (u32)                      */
  SHE_STREAM_KSK_NOISE = 6, /* e of KSK entries     (gaussian, a_lwe)          */
  SHE_STREAM_ENC_MASK = 7,  /* a of fresh ciphertexts                          */
  SHE_STREAM_ENC_NOISE = 8, /* e of fresh ciphertexts                          */
  SHE_STREAM_LVL_MASK = 9,  /* A coeffs of leveled selectors (TRGSW rows, u32)  */
  SHE_STREAM_LVL_NOISE = 10 /* e coeffs of leveled selectors (gaussian, a_bk)   */
};

SHE_RNG_FN uint64_t she_mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

SHE_RNG_FN uint64_t she_rng_u64(uint64_t seed, uint32_t stream, uint64_t index) {
  uint64_t key = she_mix64(seed ^ she_mix64(SHE_GOLDEN * (uint64_t)(stream + 1u)));
  return she_mix64(key + SHE_GOLDEN * (index + 1u));
}

SHE_RNG_FN uint32_t she_rng_u32(uint64_t seed, uint32_t stream, uint64_t index) {
  return (uint32_t)(she_rng_u64(seed, stream, index) >> 32);
}

SHE_RNG_FN uint32_t she_rng_bit(uint64_t seed, uint32_t stream, uint64_t index) {
  return (uint32_t)(she_rng_u64(seed, stream, index) & 1u);
}

/* Rounded Gaussian noise, returned as a torus32 word (two's complement). */
static inline uint32_t she_rng_gauss32(uint64_t seed, uint32_t stream, uint64_t index,
                                       double alpha) {
  uint64_t x = she_rng_u64(seed, stream, 2u * index);
  uint64_t y = she_rng_u64(seed, stream, 2u * index + 1u);
  double u1 = (double)((x >> 11) + 1u) * 0x1.0p-53; /* (0, 1] */
  double u2 = (double)(y >> 11) * 0x1.0p-53;        /* [0, 1) */
  double r = sqrt(-2.0 * log(u1));
  double g = r * cos(6.283185307179586 * u2);
  double sigma = alpha * 4294967296.0;
  long long e = llround(g * sigma);
  return (uint32_t)(uint64_t)e;
}

/* ---- input-object numbering (the contract both sides follow) ---------- */

/* BK row r of TRGSW i (r = c*l + j, c=0 for the A block, 1 for B), coeff m. */
SHE_RNG_FN uint64_t she_idx_bk(uint32_t N, uint32_t l, uint32_t i, uint32_t r, uint32_t m) {
  return ((uint64_t)i * (2u * l) + r) * N + m;
}
/* KSK entry (i < N, j < t, v < base), mask word k < n.  Noise index = entry. */
SHE_RNG_FN uint64_t she_idx_ksk_entry(uint32_t t, uint32_t base, uint32_t i, uint32_t j,
                                         uint32_t v) {
  return ((uint64_t)i * t + j) * base + v;
}
SHE_RNG_FN uint64_t she_idx_ksk_mask(uint32_t n, uint64_t entry, uint32_t k) {
  return entry * n + k;
}
/* Leveled selector number q (a TRGSW, DESIGN.md R-LV): row r, coefficient m
 * numbered as BK row r of TRGSW q: she_idx_bk(N, l, q, r, m). */

/* Fresh ciphertext number q (global ordinal), mask word k < n.  Noise index = q. */
SHE_RNG_FN uint64_t she_idx_enc_mask(uint32_t n, uint64_t q, uint32_t k) {
  return q * n + k;
}

#endif /* SHE_RNG_H_ */
