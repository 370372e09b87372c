// gl64.cuh — arithmetic in the Goldilocks field F_p, p = 2^64 - 2^32 + 1.
//
// The exact negacyclic product of the bootstrapping loop (north_star item 1)
// is computed as an NTT over F_p; the exact integer result is bounded by
// (k+1) l N (Bg/2) 2^31 = 2^52 (C1) < (p-1)/2, so the centred lift mod p
// followed by mod 2^32 is the torus32 product with no rounding at all.
//
// Representation: any uint64 value x in [0, 2^64) stands for x mod p ("lazy"
// form, p ~ 2^64 leaves no headroom for anything else).  gl_canon() maps to
// [0, p).  Identities used:  2^64 = 2^32 - 1 (mod p),  2^96 = -1 (mod p),
// 2^192 = 1: powers of two are "shift twiddles".
//
// All functions are __host__ __device__ so the exact same code is unit-tested
// on the CPU (tests/test_ntt_host.py via libshe_host.so) and runs on sm_100a.
#pragma once
#include <stdint.h>

#ifndef __CUDACC__
#define __host__
#define __device__
#define __forceinline__ inline __attribute__((always_inline))
#endif

namespace gl {

constexpr uint64_t P = 0xFFFFFFFF00000001ull;
constexpr uint64_t EPS = 0xFFFFFFFFull;  // 2^64 mod p

__host__ __device__ __forceinline__ uint64_t mulhi(uint64_t a, uint64_t b) {
#ifdef __CUDA_ARCH__
  return __umul64hi(a, b);
#else
  return (uint64_t)(((unsigned __int128)a * b) >> 64);
#endif
}

__host__ __device__ __forceinline__ uint64_t canon(uint64_t x) { return x >= P ? x - P : x; }

// a + b mod p (lazy in, lazy out).
__host__ __device__ __forceinline__ uint64_t add(uint64_t a, uint64_t b) {
  uint64_t s = a + b;
  if (s < a) {  // carried 2^64 = EPS
    uint64_t s2 = s + EPS;
    if (s2 < s) s2 += EPS;  // second wrap (only for non-canonical inputs)
    s = s2;
  }
  return s;
}

// a - b mod p (lazy in, lazy out).
__host__ __device__ __forceinline__ uint64_t sub(uint64_t a, uint64_t b) {
  uint64_t d = a - b;
  if (a < b) {  // borrowed 2^64: subtract EPS (= add p)
    uint64_t d2 = d - EPS;
    if (d2 > d) d2 -= EPS;
    d = d2;
  }
  return d;
}

__host__ __device__ __forceinline__ uint64_t neg(uint64_t a) { return sub(0, a); }

// (hi:lo) 128-bit value mod p:  lo + hi_lo (2^32 - 1) - hi_hi.
__host__ __device__ __forceinline__ uint64_t reduce128(uint64_t lo, uint64_t hi) {
  uint64_t hh = hi >> 32, hl = hi & 0xFFFFFFFFull;
  uint64_t t0 = lo - hh;
  if (lo < hh) t0 -= EPS;  // borrow: + p (cannot borrow again: t0 >= 2^64 - 2^32)
  uint64_t t1 = (hl << 32) - hl;  // hl * (2^32 - 1), < 2^64
  uint64_t r = t0 + t1;
  if (r < t1) r += EPS;  // carry (cannot carry again)
  return r;
}

// (x2:x1:x0) 96-bit value (x2 < 2^32) mod p: lo + x2 (2^32 - 1).
__host__ __device__ __forceinline__ uint64_t reduce96(uint64_t lo, uint64_t x2) {
  uint64_t t1 = (x2 << 32) - x2;
  uint64_t r = lo + t1;
  if (r < t1) r += EPS;
  return r;
}

__host__ __device__ __forceinline__ uint64_t mul(uint64_t a, uint64_t b) {
  return reduce128(a * b, mulhi(a, b));
}

// x * 2^32 mod p: x1 2^64 + x0 2^32 = x1 (2^32 - 1) + x0 2^32.
__host__ __device__ __forceinline__ uint64_t mul_2_32(uint64_t x) {
  return reduce96(x << 32, x >> 32);
}

// x * 2^s mod p for 0 <= s < 192 (s is a compile-time constant at every call
// site of the NTT, so the branches fold away).
__host__ __device__ __forceinline__ uint64_t mul_pow2(uint64_t x, int s) {
  bool negate = false;
  if (s >= 96) {  // 2^96 = -1
    s -= 96;
    negate = true;
  }
  uint64_t r;
  if (s == 0) {
    r = x;
  } else if (s < 32) {
    r = reduce96(x << s, x >> (64 - s));
  } else if (s == 32) {
    r = mul_2_32(x);
  } else if (s < 64) {
    r = reduce128(x << s, x >> (64 - s));
  } else if (s == 64) {
    r = reduce128(0, x);
  } else {  // 64 < s < 96: (x 2^(s-64)) 2^64, the 2^128 part = -2^32
    uint64_t lo = x << (s - 64), top = x >> (128 - s);  // x 2^(s-64) = top 2^64 + lo
    // value = lo 2^64 + top 2^128 = lo (2^32 - 1) - top 2^32  (top < 2^32)
    uint64_t a = reduce128(0, lo);
    r = sub(a, top << 32);
  }
  return negate ? neg(r) : r;
}

__host__ __device__ inline uint64_t pow(uint64_t b, uint64_t e) {
  uint64_t r = 1;
  while (e) {
    if (e & 1) r = mul(r, b);
    b = mul(b, b);
    e >>= 1;
  }
  return canon(r);
}

// Signed small integer -> F_p.
__host__ __device__ __forceinline__ uint64_t from_i64(int64_t v) {
  return v >= 0 ? (uint64_t)v : (uint64_t)v - EPS;  // 2^64 + v - EPS = p + v
}

// Centred lift of x in F_p to Z, reduced mod 2^32 (torus32).  Valid when the
// exact integer has |value| < (p-1)/2.  (x - p) mod 2^32 = (x - 1) mod 2^32.
__host__ __device__ __forceinline__ uint32_t lift32(uint64_t x) {
  x = canon(x);
  return (uint32_t)x - (x > (P - 1) / 2 ? 1u : 0u);
}

}  // namespace gl
