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
// on the CPU (tests/test_client_and_emu.py via libshe_hostemu.so, built from
// host_emu.cpp) and runs on sm_100a.
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

#if defined(__CUDA_ARCH__) && defined(GL_ADDSUB_PTX)
// a + b mod p (lazy in, lazy out): 64-bit add, fold each carry as +EPS with
// IMAD carry chains (FMA pipe) instead of 64-bit compares and selects.
__device__ __forceinline__ uint64_t add(uint64_t a, uint64_t b) {
  uint32_t s0, s1, c;
  asm("add.cc.u32 %0, %3, %5;\n\t"
      "addc.cc.u32 %1, %4, %6;\n\t"
      "addc.u32 %2, 0, 0;\n\t"
      "mad.lo.cc.u32 %0, %2, 0xFFFFFFFF, %0;\n\t"
      "madc.hi.cc.u32 %1, %2, 0xFFFFFFFF, %1;\n\t"
      "addc.u32 %2, 0, 0;\n\t"
      "mad.lo.cc.u32 %0, %2, 0xFFFFFFFF, %0;\n\t"
      "madc.hi.u32 %1, %2, 0xFFFFFFFF, %1;"
      : "=&r"(s0), "=&r"(s1), "=&r"(c)
      : "r"((uint32_t)a), "r"((uint32_t)(a >> 32)), "r"((uint32_t)b), "r"((uint32_t)(b >> 32)));
  return ((uint64_t)s1 << 32) | s0;
}
// a - b mod p: borrow chains; each borrow subtracts EPS (= adds p).
__device__ __forceinline__ uint64_t sub(uint64_t a, uint64_t b) {
  uint32_t d0, d1, bw;
  asm("sub.cc.u32 %0, %3, %5;\n\t"
      "subc.cc.u32 %1, %4, %6;\n\t"
      "subc.u32 %2, 0, 0;\n\t"
      "sub.cc.u32 %0, %0, %2;\n\t"
      "subc.cc.u32 %1, %1, 0;\n\t"
      "subc.u32 %2, 0, 0;\n\t"
      "sub.cc.u32 %0, %0, %2;\n\t"
      "subc.u32 %1, %1, 0;"
      : "=&r"(d0), "=&r"(d1), "=&r"(bw)
      : "r"((uint32_t)a), "r"((uint32_t)(a >> 32)), "r"((uint32_t)b), "r"((uint32_t)(b >> 32)));
  return ((uint64_t)d1 << 32) | d0;
}
#else
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
#endif

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

__host__ __device__ __forceinline__ uint64_t mul(uint64_t a, uint64_t b) {
  return reduce128(a * b, mulhi(a, b));
}

// (hi:lo) mod p with the result <= p (so a following butterfly with twiddle
// 1 can fold once, see add_le / sub_le).  hl EPS + EPS = (hl : ~hl) costs no
// instruction; w = t0 + hl EPS + EPS with carry c gives c ? w : w - EPS
// (c: w < hl EPS + EPS <= 2^64 - 2^32; !c: w - EPS <= 2^64 - 1 - EPS = p - 1).
__host__ __device__ __forceinline__ uint64_t reduce128_le(uint64_t lo, uint64_t hi) {
#if defined(__CUDA_ARCH__)
  // carry/borrow chains instead of 64-bit compares and selects
  const uint32_t l0 = (uint32_t)lo, l1 = (uint32_t)(lo >> 32);
  const uint32_t h0 = (uint32_t)hi, h1 = (uint32_t)(hi >> 32);
  uint32_t t0, t1, bw, w0, w1, c, e0, e1, r0, r1;
  asm("sub.cc.u32 %0, %10, %13;\n\t"        // t = lo - hh
      "subc.cc.u32 %1, %11, 0;\n\t"
      "subc.u32 %2, 0, 0;\n\t"              // -borrow
      "sub.cc.u32 %0, %0, %2;\n\t"          // + p on a borrow (- EPS mod 2^64)
      "subc.u32 %1, %1, 0;\n\t"
      "add.cc.u32 %3, %0, %14;\n\t"         // w = t + (hl : ~hl) = t + hl EPS + EPS
      "addc.cc.u32 %4, %1, %12;\n\t"
      "addc.u32 %5, 0, 0;\n\t"              // c
      "add.cc.u32 %6, %3, 1;\n\t"           // e = w - EPS
      "addc.u32 %7, %4, 0xFFFFFFFF;\n\t"
      "mad.lo.cc.u32 %8, %5, 0xFFFFFFFF, %6;\n\t"  // c ? w : e  =  e + c EPS
      "madc.hi.u32 %9, %5, 0xFFFFFFFF, %7;"
      : "=&r"(t0), "=&r"(t1), "=&r"(bw), "=&r"(w0), "=&r"(w1), "=&r"(c), "=&r"(e0), "=&r"(e1),
        "=&r"(r0), "=&r"(r1)
      : "r"(l0), "r"(l1), "r"(h0), "r"(h1), "r"(~h0));
  return ((uint64_t)r1 << 32) | r0;
#else
  const uint64_t hh = hi >> 32, hl = hi & 0xFFFFFFFFull;
  uint64_t t0 = lo - hh;
  if (lo < hh) t0 -= EPS;  // borrow: + p (cannot borrow again)
  const uint64_t t1 = (hl << 32) | (~hl & 0xFFFFFFFFull);
  const uint64_t w = t0 + t1;
  return w < t1 ? w : w - EPS;
#endif
}

__host__ __device__ __forceinline__ uint64_t mul_le(uint64_t a, uint64_t b) {
  return reduce128_le(a * b, mulhi(a, b));
}

// ---- butterfly primitives with a bounded twiddle product ----
// The NTT butterflies compute u +- t with t = v 2^s.  If the twiddle product
// is kept <= p (not merely < 2^64), one carry (borrow) fold is always enough:
//   u + t <= 2^64 - 1 + p: after a carry, u + t - 2^64 <= p - 1, + EPS < 2^64;
//   u - t >= -p:           after a borrow, u - t + 2^64 >= EPS, - EPS >= 0.
// shl_le() produces such a product from any 64-bit v.

// x + y for any x and y <= p (lazy result).
__host__ __device__ __forceinline__ uint64_t add_le(uint64_t x, uint64_t y) {
#if defined(__CUDA_ARCH__)
  uint32_t s0, s1, c;
  asm("add.cc.u32 %0, %3, %5;\n\t"
      "addc.cc.u32 %1, %4, %6;\n\t"
      "addc.u32 %2, 0, 0;\n\t"
      "mad.lo.cc.u32 %0, %2, 0xFFFFFFFF, %0;\n\t"
      "madc.hi.u32 %1, %2, 0xFFFFFFFF, %1;"
      : "=&r"(s0), "=&r"(s1), "=&r"(c)
      : "r"((uint32_t)x), "r"((uint32_t)(x >> 32)), "r"((uint32_t)y), "r"((uint32_t)(y >> 32)));
  return ((uint64_t)s1 << 32) | s0;
#else
  const uint64_t s = x + y;
  return s < y ? s + EPS : s;
#endif
}

// x - y for any x and y <= p (lazy result).
__host__ __device__ __forceinline__ uint64_t sub_le(uint64_t x, uint64_t y) {
#if defined(__CUDA_ARCH__)
  uint32_t d0, d1, bw;
  asm("sub.cc.u32 %0, %3, %5;\n\t"
      "subc.cc.u32 %1, %4, %6;\n\t"
      "subc.u32 %2, 0, 0;\n\t"
      "sub.cc.u32 %0, %0, %2;\n\t"
      "subc.u32 %1, %1, 0;"
      : "=&r"(d0), "=&r"(d1), "=&r"(bw)
      : "r"((uint32_t)x), "r"((uint32_t)(x >> 32)), "r"((uint32_t)y), "r"((uint32_t)(y >> 32)));
  return ((uint64_t)d1 << 32) | d0;
#else
  const uint64_t d = x - y;
  return x < y ? d - EPS : d;
#endif
}

// v 2^s mod p for a compile-time 0 <= s < 96 and any 64-bit v; result <= p.
// With r = s mod 32, T = v 2^r = (T2:T1:T0) (T2 < 2^r) and 2^64 = 2^32 - 1,
// 2^96 = -1 (mod p):
//   s <  32: T            = (T1:T0) + T2 EPS.  w = (T1:T0) + (T2+1) EPS with
//            carry c; result c ? w : w - EPS  (c: w < 2^31 EPS < p; !c: w - EPS
//            < 2^64 - EPS = p).
//   s <  64: T 2^32       = (T0 + T1) 2^32 - (T1 + T2).  With T0 + T1 = s1 2^32
//            + s0: = (s0 + s1) 2^32 - (T1 + T2 + s1), H = s0 + s1 < 2^32; R =
//            (H:0) - E lies in [-2^33, 2^64 - 2^32]: add p once if negative.
//   s <  96: T 2^64       = (T0 - T2) 2^32 - (T0 + T1) in (-2^64, 2^64 - 2^32]:
//            add p once if negative (borrow of T0 - T2 or of the 64-bit sub;
//            never both).
// Verified exhaustively on edge values and randomly in tests (host build).
__host__ __device__ __forceinline__ uint64_t shl_le(uint64_t v, const int s) {
  const int q = s >> 5, r = s & 31;
  const uint32_t v0 = (uint32_t)v, v1 = (uint32_t)(v >> 32);
  uint32_t T0, T1, T2;
  if (r == 0) {
    T0 = v0;
    T1 = v1;
    T2 = 0;
  } else {
    T0 = v0 << r;
#if defined(__CUDA_ARCH__)
    T1 = __funnelshift_l(v0, v1, r);
#else
    T1 = (v1 << r) | (v0 >> (32 - r));
#endif
    T2 = v1 >> (32 - r);
  }
#if defined(__CUDA_ARCH__)
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
    o0 = c ? w0 : e0;  // (an IMAD form e + c EPS measured 1.4 % slower in the kernel)
    o1 = c ? w1 : e1;
  } else if (q == 1) {
    uint32_t s0, H, e0, e1;
    asm("add.cc.u32 %1, %5, %6;\n\t"     // s0 = T0 + T1, CF = s1
        "addc.u32 %2, %1, 0;\n\t"        // H = s0 + s1
        "addc.cc.u32 %3, %6, %7;\n\t"    // e0 = T1 + T2 + s1, CF = e1
        "addc.u32 %4, 0, 0;\n\t"         // e1
        "sub.cc.u32 %0, 0, %3;\n\t"      // R = (H:0) - (e1:e0)
        "subc.cc.u32 %1, %2, %4;\n\t"
        "subc.u32 %4, 0, 0;\n\t"         // -borrow
        "sub.cc.u32 %0, %0, %4;\n\t"     // R + p if negative (- EPS mod 2^64)
        "subc.u32 %1, %1, 0;"
        : "=&r"(o0), "=&r"(s0), "=&r"(H), "=&r"(e0), "=&r"(e1)
        : "r"(T0), "r"(T1), "r"(T2));
    o1 = s0;
  } else {
    uint32_t F, fn, g0, g1;
    asm("sub.cc.u32 %2, %6, %8;\n\t"     // F = T0 - T2, CF = borrow
        "subc.u32 %3, 0, 0;\n\t"         // fn = -borrow
        "add.cc.u32 %4, %6, %7;\n\t"     // G = T0 + T1
        "addc.u32 %5, 0, 0;\n\t"
        "sub.cc.u32 %0, 0, %4;\n\t"      // L = (F:0) - G
        "subc.cc.u32 %1, %2, %5;\n\t"
        "subc.u32 %3, %3, 0;\n\t"        // -(borrow_F + borrow_L), at most one is set
        "sub.cc.u32 %0, %0, %3;\n\t"
        "subc.u32 %1, %1, 0;"
        : "=&r"(o0), "=&r"(o1), "=&r"(F), "=&r"(fn), "=&r"(g0), "=&r"(g1)
        : "r"(T0), "r"(T1), "r"(T2));
  }
  return ((uint64_t)o1 << 32) | o0;
#else
  if (q == 0) {
    const uint64_t m = (uint64_t)(T2 + 1) * EPS;
    const uint64_t w = (((uint64_t)T1 << 32) | T0) + m;
    return w < m ? w : w - EPS;
  }
  if (q == 1) {
    const uint64_t S = (uint64_t)T0 + T1;
    const uint32_t s0 = (uint32_t)S, s1 = (uint32_t)(S >> 32);
    const uint64_t H = (uint64_t)(s0 + s1) << 32;
    const uint64_t E = (uint64_t)T1 + T2 + s1;
    return H < E ? H - E - EPS : H - E;
  }
  const uint64_t Hh = (uint64_t)(uint32_t)(T0 - T2) << 32;
  const uint64_t G = (uint64_t)T0 + T1;
  const uint64_t Lv = Hh - G;
  return (T0 < T2 || Hh < G) ? Lv - EPS : Lv;
#endif
}

// x * 2^s mod p for 0 <= s < 192 (2^96 = -1): the bounded product, negated
// for s >= 96 (setup and tests; the butterflies fold the sign into +/-).
__host__ __device__ __forceinline__ uint64_t mul_pow2(uint64_t x, int s) {
  return s >= 96 ? neg(shl_le(x, s - 96)) : shl_le(x, s);
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

// Lazy multiply-accumulate of up to 4 products (< 2^130) with one reduction:
// value = lo + hi 2^64 + top 2^128, and 2^128 = -2^32 (mod p).
struct Acc3 {
  uint64_t lo = 0, hi = 0;
  uint32_t top = 0;
};

__host__ __device__ __forceinline__ void mac(Acc3& A, uint64_t a, uint64_t b) {
#ifdef __CUDA_ARCH__
  const uint64_t l = a * b, h = __umul64hi(a, b);
  asm("add.cc.u64 %0, %0, %3;\n\t"
      "addc.cc.u64 %1, %1, %4;\n\t"
      "addc.u32 %2, %2, 0;"
      : "+l"(A.lo), "+l"(A.hi), "+r"(A.top)
      : "l"(l), "l"(h));
#else
  const unsigned __int128 pr = (unsigned __int128)a * b;
  const unsigned __int128 s = (((unsigned __int128)A.hi << 64) | A.lo) + pr;
  if (s < pr) A.top += 1;
  A.lo = (uint64_t)s;
  A.hi = (uint64_t)(s >> 64);
#endif
}

// As reduce_acc with the result <= p (r <= p; r - t + p <= p when r < t).
__host__ __device__ __forceinline__ uint64_t reduce_acc_le(const Acc3& A) {
  const uint64_t r = reduce128_le(A.lo, A.hi);
#if defined(__CUDA_ARCH__)
  uint32_t d0, d1, bw;
  asm("sub.cc.u32 %0, %3, 0;\n\t"           // r - top 2^32
      "subc.cc.u32 %1, %4, %5;\n\t"
      "subc.u32 %2, 0, 0;\n\t"
      "sub.cc.u32 %0, %0, %2;\n\t"          // + p on a borrow
      "subc.u32 %1, %1, 0;"
      : "=&r"(d0), "=&r"(d1), "=&r"(bw)
      : "r"((uint32_t)r), "r"((uint32_t)(r >> 32)), "r"(A.top));
  return ((uint64_t)d1 << 32) | d0;
#else
  const uint64_t t = (uint64_t)A.top << 32;  // top <= 3
  uint64_t d = r - t;
  if (r < t) d -= EPS;
  return d;
#endif
}

__host__ __device__ __forceinline__ uint64_t reduce_acc(const Acc3& A) {
  const uint64_t r = reduce128(A.lo, A.hi);
  const uint64_t t = (uint64_t)A.top << 32;  // top <= 3
  uint64_t d = r - t;
  if (r < t) d -= EPS;  // + p (single borrow: r - t >= -2^34)
  return d;
}

// Signed small integer -> F_p.
__host__ __device__ __forceinline__ uint64_t from_i64(int64_t v) {
  return v >= 0 ? (uint64_t)v : (uint64_t)v - EPS;  // 2^64 + v - EPS = p + v
}

// Centred lift of x in F_p to Z, reduced mod 2^32 (torus32).  Valid when the
// exact integer has |value| < (p-1)/2.  (x - p) mod 2^32 = (x - 1) mod 2^32.
// Any lazy x works: x >= p implies x > (p-1)/2 and (x - p) = x - 1 mod 2^32.
__host__ __device__ __forceinline__ uint32_t lift32(uint64_t x) {
  return (uint32_t)x - (x > (P - 1) / 2 ? 1u : 0u);
}

// lift32(-t) for t <= p: (p - t) centred and reduced mod 2^32.  p = 1 mod 2^32,
// and p - t > (p-1)/2 exactly when t < (p+1)/2 (t = 0 and t = p both give 0).
__host__ __device__ __forceinline__ uint32_t lift32_neg(uint64_t t) {
  return (0u - (uint32_t)t) + (t >= (P + 1) / 2 ? 1u : 0u);
}

}  // namespace gl
