// fft_core.cuh — FP64 negacyclic FFT of the blind rotation (N = 1024), the
// second engine of K3.
//
// The CMux product sum_r digit_r(X) * BK_{i,r}(X) mod (X^N + 1) (PAPER.md:31,
// TFHE bootstrapping) is computed EXACTLY in double
// precision: BK is split into 16-bit halves (b = 2^16 b_hi + b_lo, |b_*| <=
// 2^15), so every partial product sum is an integer of magnitude <= 4 * 1024 *
// 512 * 2^15 = 2^36, and the FFT round-off on it (<= ~1e-3)
// is far below 1/2: rounding to the nearest integer recovers the exact value,
// and (2^16 C_hi + C_lo) mod 2^32 is the exact torus32 product.
//
// Folding: a real negacyclic polynomial a is evaluated at zeta^(4k+1),
// zeta = exp(i pi / N), through the N/2-point DFT of u_n = (a_n + i a_{n+N/2})
// zeta^n (n < N/2); the inverse takes the conjugate path and reads a_n, a_{n+N/2}
// from the real and imaginary parts.  N/2 = 512 = 16 x 32 in two passes per warp:
//   pass A  thread n1 = lane: 16-point DFT over n2 of points n1 + 32 n2, then
//           the twiddle omega_512^(n1 k2) (times the thread's twist factor);
//   pass B  thread (k2 = t >> 1, h = t & 1): 16-point DFT of the even (h = 0) or
//           odd (h = 1) points n1 of column k2, then one radix-2 step across the
//           thread pair (shfl.xor 1) gives X[k2 + 16 k1] for k1 = 8h + j and
//           16 + 8h + j (j < 8).
// One XOR-swizzled shared-memory transpose (tslot below: conflict-free both
// ways) sits between the passes.  Constant twiddles come from the constant bank
// (compile-time indices); the per-thread pass-A twiddles from a shared table
// filled with sincospi at kernel start (make_tables).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

namespace fft {

constexpr int kN = 1024, kM = 512, kRow = 512;  // complex per scratch row

// Shared-memory swizzles (16-byte accesses are served 8 threads per
// wavefront; each group of 8 must hit 8 distinct 16-byte bank groups):
// transpose slot of (n1, k2): row n1, column k2 ^ s(n1) -- pass A writes
// (k2 fixed, 8 consecutive n1) and pass B reads (n1 = 2m + h, k2 = t >> 1)
// both spread over the 8 groups; frequency k is kept at position
// k ^ (bit 7 of k) << 2 -- the forward's stores (k = k2 + 128 h + 16 j) and
// the inverse's loads (k = lane + 32 m) are conflict-free.
__device__ __forceinline__ int tslot(int n1, int k2) {
#ifdef SHE_CHECKED
  if (n1 < 0 || n1 >= 32 || k2 < 0 || k2 >= 16) {
    printf("tslot(%d, %d) out of the 32 x 16 row\n", n1, k2);
    __trap();
  }
#endif
  return n1 * 16 + (k2 ^ (((n1 & 1) << 2) | ((n1 >> 1) & 3)));
}
__device__ __forceinline__ int fpos(int k) { return k ^ (((k >> 7) & 1) << 2); }

// W128[k] = exp(2 pi i k / 128)
__constant__ double2 c_w128[128] = {
    {1.0, 0.0},
    {0.9987954562051724, 0.049067674327418015},
    {0.9951847266721969, 0.0980171403295606},
    {0.989176509964781, 0.14673047445536175},
    {0.9807852804032304, 0.19509032201612825},
    {0.970031253194544, 0.24298017990326387},
    {0.9569403357322088, 0.29028467725446233},
    {0.9415440651830208, 0.33688985339222005},
    {0.9238795325112867, 0.3826834323650898},
    {0.9039892931234433, 0.4275550934302821},
    {0.881921264348355, 0.47139673682599764},
    {0.8577286100002721, 0.5141027441932217},
    {0.8314696123025452, 0.5555702330196022},
    {0.8032075314806449, 0.5956993044924334},
    {0.773010453362737, 0.6343932841636455},
    {0.7409511253549591, 0.6715589548470183},
    {0.7071067811865476, 0.7071067811865475},
    {0.6715589548470183, 0.7409511253549591},
    {0.6343932841636455, 0.773010453362737},
    {0.5956993044924335, 0.8032075314806448},
    {0.5555702330196023, 0.8314696123025452},
    {0.5141027441932217, 0.8577286100002721},
    {0.4713967368259978, 0.8819212643483549},
    {0.4275550934302822, 0.9039892931234433},
    {0.38268343236508984, 0.9238795325112867},
    {0.33688985339222005, 0.9415440651830208},
    {0.29028467725446233, 0.9569403357322089},
    {0.24298017990326398, 0.970031253194544},
    {0.19509032201612833, 0.9807852804032304},
    {0.14673047445536175, 0.989176509964781},
    {0.09801714032956077, 0.9951847266721968},
    {0.049067674327418126, 0.9987954562051724},
    {0.0, 1.0},
    {-0.04906767432741801, 0.9987954562051724},
    {-0.09801714032956065, 0.9951847266721969},
    {-0.14673047445536164, 0.989176509964781},
    {-0.1950903220161282, 0.9807852804032304},
    {-0.24298017990326387, 0.970031253194544},
    {-0.29028467725446216, 0.9569403357322089},
    {-0.33688985339221994, 0.9415440651830208},
    {-0.3826834323650897, 0.9238795325112867},
    {-0.42755509343028186, 0.9039892931234434},
    {-0.4713967368259977, 0.881921264348355},
    {-0.5141027441932217, 0.8577286100002721},
    {-0.555570233019602, 0.8314696123025455},
    {-0.5956993044924334, 0.8032075314806449},
    {-0.6343932841636454, 0.7730104533627371},
    {-0.6715589548470184, 0.740951125354959},
    {-0.7071067811865475, 0.7071067811865476},
    {-0.7409511253549589, 0.6715589548470186},
    {-0.773010453362737, 0.6343932841636455},
    {-0.8032075314806448, 0.5956993044924335},
    {-0.8314696123025453, 0.5555702330196022},
    {-0.857728610000272, 0.5141027441932218},
    {-0.8819212643483549, 0.47139673682599786},
    {-0.9039892931234433, 0.42755509343028203},
    {-0.9238795325112867, 0.3826834323650899},
    {-0.9415440651830207, 0.33688985339222033},
    {-0.9569403357322088, 0.2902846772544624},
    {-0.970031253194544, 0.24298017990326407},
    {-0.9807852804032304, 0.1950903220161286},
    {-0.989176509964781, 0.1467304744553618},
    {-0.9951847266721968, 0.09801714032956083},
    {-0.9987954562051724, 0.049067674327417966},
    {-1.0, 0.0},
    {-0.9987954562051724, -0.049067674327417724},
    {-0.9951847266721969, -0.09801714032956059},
    {-0.989176509964781, -0.14673047445536158},
    {-0.9807852804032304, -0.19509032201612836},
    {-0.970031253194544, -0.24298017990326382},
    {-0.9569403357322089, -0.2902846772544621},
    {-0.9415440651830208, -0.3368898533922201},
    {-0.9238795325112868, -0.38268343236508967},
    {-0.9039892931234434, -0.4275550934302818},
    {-0.881921264348355, -0.47139673682599764},
    {-0.8577286100002721, -0.5141027441932216},
    {-0.8314696123025455, -0.555570233019602},
    {-0.8032075314806449, -0.5956993044924332},
    {-0.7730104533627371, -0.6343932841636453},
    {-0.7409511253549591, -0.6715589548470184},
    {-0.7071067811865477, -0.7071067811865475},
    {-0.6715589548470187, -0.7409511253549589},
    {-0.6343932841636459, -0.7730104533627367},
    {-0.5956993044924331, -0.803207531480645},
    {-0.5555702330196022, -0.8314696123025452},
    {-0.5141027441932218, -0.857728610000272},
    {-0.47139673682599786, -0.8819212643483549},
    {-0.4275550934302825, -0.9039892931234431},
    {-0.38268343236509034, -0.9238795325112865},
    {-0.33688985339221994, -0.9415440651830208},
    {-0.29028467725446244, -0.9569403357322088},
    {-0.24298017990326412, -0.970031253194544},
    {-0.19509032201612866, -0.9807852804032303},
    {-0.1467304744553623, -0.9891765099647809},
    {-0.09801714032956045, -0.9951847266721969},
    {-0.04906767432741803, -0.9987954562051724},
    {0.0, -1.0},
    {0.04906767432741766, -0.9987954562051724},
    {0.09801714032956009, -0.9951847266721969},
    {0.14673047445536194, -0.9891765099647809},
    {0.1950903220161283, -0.9807852804032304},
    {0.24298017990326376, -0.970031253194544},
    {0.29028467725446205, -0.9569403357322089},
    {0.3368898533922196, -0.9415440651830209},
    {0.38268343236509, -0.9238795325112866},
    {0.42755509343028214, -0.9039892931234433},
    {0.4713967368259976, -0.881921264348355},
    {0.5141027441932216, -0.8577286100002722},
    {0.5555702330196018, -0.8314696123025455},
    {0.5956993044924329, -0.8032075314806453},
    {0.6343932841636456, -0.7730104533627369},
    {0.6715589548470183, -0.7409511253549591},
    {0.7071067811865474, -0.7071067811865477},
    {0.7409511253549589, -0.6715589548470187},
    {0.7730104533627367, -0.6343932841636459},
    {0.803207531480645, -0.5956993044924332},
    {0.8314696123025452, -0.5555702330196022},
    {0.857728610000272, -0.5141027441932219},
    {0.8819212643483548, -0.4713967368259979},
    {0.9039892931234431, -0.42755509343028253},
    {0.9238795325112865, -0.3826834323650904},
    {0.9415440651830208, -0.33688985339222},
    {0.9569403357322088, -0.2902846772544625},
    {0.970031253194544, -0.24298017990326418},
    {0.9807852804032303, -0.19509032201612872},
    {0.9891765099647809, -0.1467304744553624},
    {0.9951847266721969, -0.0980171403295605},
    {0.9987954562051724, -0.04906767432741809}
};

__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 csub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}
__device__ __forceinline__ double2 cmulc(double2 a, double2 b) {  // a * conj(b)
  return make_double2(fma(a.x, b.x, a.y * b.y), fma(a.y, b.x, -a.x * b.y));
}

// W128[e] read at its point of use: the index carries an opaque zero, so the
// compiler cannot hoist the constant-bank loads of a whole transform out of
// the CMux loop into (spilled) registers; the load is one LDC per use, served
// by the constant cache.
__device__ __forceinline__ double2 cw(int e) {
  int z;
  asm volatile("mov.u32 %0, %%laneid;\n\tshr.u32 %0, %0, 5;" : "=r"(z));
  return c_w128[e + z];
}

// a * W128[e]^SIGN for a compile-time e (after unrolling)
template <int SIGN>
__device__ __forceinline__ double2 rot(double2 a, int e) {
  e &= 127;
  if (e == 0) return a;
  if (e == 64) return make_double2(-a.x, -a.y);
  if (e == 32) return SIGN > 0 ? make_double2(-a.y, a.x) : make_double2(a.y, -a.x);
  if (e == 96) return SIGN > 0 ? make_double2(a.y, -a.x) : make_double2(-a.y, a.x);
  return SIGN > 0 ? cmul(a, cw(e)) : cmulc(a, cw(e));
}

__device__ __forceinline__ constexpr int brev4(int k) {
  return ((k & 1) << 3) | ((k & 2) << 1) | ((k & 4) >> 1) | ((k & 8) >> 3);
}

// In-register 16-point DFT, X[k] = sum_n a[n] w16^(SIGN n k), radix-2 DIF:
// natural input, output a[brev4(k)] = X[k].
template <int SIGN>
__device__ __forceinline__ void dft16(double2 (&a)[16]) {
#pragma unroll
  for (int half = 8; half >= 1; half >>= 1) {
#pragma unroll
    for (int s = 0; s < 16; s += 2 * half) {
#pragma unroll
      for (int j = 0; j < half; ++j) {
        const double2 u = a[s + j], v = a[s + j + half];
        a[s + j] = cadd(u, v);
        a[s + j + half] = rot<SIGN>(csub(u, v), j * (64 / half));  // w_(2 half)^j
      }
    }
  }
}

// The same 16-point DFT by radix-2 decimation in time with FMA butterflies
// (variant 3): the input is read through the compile-time relabelling
// b[i] = a[brev4(i)], so the output lands in the same registers as dft16's,
// a[brev4(k)] = X[k].  A butterfly (u, v) -> (u + w v, u - w v) with a general
// twiddle is 4 DFMA for x = u + w v and 2 DFMA for y = 2 u - x: 6 FP64
// instructions instead of DIF's 8; w = +-1, +-i cost 4 DADD.  148 FP64
// instructions per DFT16 instead of 168.
template <int SIGN>
__device__ __forceinline__ void dft16_dit(double2 (&a)[16]) {
#pragma unroll
  for (int s = 1; s <= 8; s <<= 1) {
#pragma unroll
    for (int g0 = 0; g0 < 16; g0 += 2 * s) {
#pragma unroll
      for (int j = 0; j < s; ++j) {
        double2& U = a[brev4(g0 + j)];
        double2& Vr = a[brev4(g0 + j + s)];
        const double2 u = U, v = Vr;
        const int e = (SIGN * j * (64 / s)) & 127;  // w = W128^e = w_(2s)^(SIGN j)
        double2 x, y;
        if (e == 0) {
          x = cadd(u, v);
          y = csub(u, v);
        } else if (e == 64) {
          x = csub(u, v);
          y = cadd(u, v);
        } else if (e == 32) {  // w = i: w v = (-v.y, v.x)
          x = make_double2(u.x - v.y, u.y + v.x);
          y = make_double2(u.x + v.y, u.y - v.x);
        } else if (e == 96) {  // w = -i: w v = (v.y, -v.x)
          x = make_double2(u.x + v.y, u.y - v.x);
          y = make_double2(u.x - v.y, u.y + v.x);
        } else {
          const double2 w = cw(e);
          x.x = fma(w.x, v.x, fma(-w.y, v.y, u.x));
          x.y = fma(w.x, v.y, fma(w.y, v.x, u.y));
          y.x = fma(2.0, u.x, -x.x);
          y.y = fma(2.0, u.y, -x.y);
        }
        U = x;
        Vr = y;
      }
    }
  }
}

// Pass A + transpose + pass B of one 512-point DFT (direction SIGN) on warp-
// private scratch (kRow complex).  In: a[n2] = point lane + 32 n2.  Per-thread
// twiddle after pass A: tw[k2 * 32 + lane] (a shared table, see make_tables).
// Out: x[j] = X[k2 + 16 (8h + j)], y[j] = X[k2 + 16 (16 + 8h + j)],
// (k2, h) = (lane >> 1, lane & 1).
template <int SIGN>
__device__ __forceinline__ void dft512(double2 (&a)[16], int lane, const double2* tw,
                                       double2* scratch, double2 (&x)[8], double2 (&y)[8]) {
  dft16<SIGN>(a);
#pragma unroll
  for (int k2 = 0; k2 < 16; ++k2) {
    const double2 p = tw[k2 * 32 + lane];
    scratch[tslot(lane, k2)] = k2 == 0 && SIGN < 0 ? a[0] : cmul(a[brev4(k2)], p);
  }
  __syncwarp();
  const int k2 = lane >> 1, h = lane & 1;
#pragma unroll
  for (int m = 0; m < 16; ++m) a[m] = scratch[tslot(2 * m + h, k2)];
  dft16<SIGN>(a);
  // exchange: h = 0 keeps E[0..7] and gets O[0..7]; h = 1 keeps O[8..15] and
  // gets E[8..15].  The odd-column twiddle w32^(SIGN k) is applied after the
  // exchange, split between the pair (k = 8h + j = w32^j times i^h), so both
  // threads of a pair do 7 complex products instead of one doing 14.
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const double2 lo = a[brev4(j)], hi = a[brev4(8 + j)];
    const double2 send = h ? lo : hi, keep = h ? hi : lo;
    double2 r;
    r.x = __shfl_xor_sync(0xffffffffu, send.x, 1);
    r.y = __shfl_xor_sync(0xffffffffu, send.y, 1);
    const double2 e = h ? r : keep;
    double2 o = rot<SIGN>(h ? keep : r, 4 * j);
    if (h) o = SIGN > 0 ? make_double2(-o.y, o.x) : make_double2(o.y, -o.x);
    x[j] = cadd(e, o);
    y[j] = csub(e, o);
  }
  __syncwarp();  // scratch reads done before the caller reuses the row
}

// Forward transform of a real polynomial given as (re[m], im[m]) = (a_n,
// a_{n+512}), n = lane + 32 m (m < 16).  Writes X[k] to row[fpos(k)].
__device__ __forceinline__ void forward(const double (&re)[16], const double (&im)[16], int lane,
                                        const double2* tw_fwd, double2* row) {
  double2 a[16];
#pragma unroll
  for (int m = 0; m < 16; ++m) a[m] = rot<1>(make_double2(re[m], im[m]), 2 * m);  // w64^m
  double2 x[8], y[8];
  dft512<1>(a, lane, tw_fwd, row, x, y);
  const int k2 = lane >> 1, h = lane & 1;
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    row[fpos(k2 + 16 * (8 * h + j))] = x[j];
    row[fpos(k2 + 16 * (16 + 8 * h + j))] = y[j];
  }
}

// Inverse transform of X[k] = row[fpos(k)] (1/512 already folded in):
// out_re[j], out_im[j] for the two groups (g = 0, 1) at positions
// n = k2 + 16 (16 g + 8 h + j): a_n = re, a_{n+512} = im.
__device__ __forceinline__ void inverse(const double2* row_in, int lane, const double2* tw_inv,
                                        double2* row, double2 (&x)[8], double2 (&y)[8]) {
  double2 a[16];
#pragma unroll
  for (int m = 0; m < 16; ++m) a[m] = row_in[fpos(lane + 32 * m)];
  __syncwarp();
  dft512<-1>(a, lane, tw_inv, row, x, y);
  const int h = lane & 1;
#pragma unroll
  for (int j = 0; j < 8; ++j) {  // untwist zeta^(-16 k1) = conj(W128[k1])
    x[j] = cmulc(x[j], cw(8 * h + j));
    y[j] = cmulc(y[j], cw(16 + 8 * h + j));
  }
}

// exact small integer -> double (|v| < 2^31) without the conversion unit
__device__ __forceinline__ double i2d(int32_t v) {
  return __hiloint2double(0x43300000, (int)((uint32_t)v ^ 0x80000000u)) - 4503601774854144.0;
}
// round(v) mod 2^32 for |v| < 2^51
__device__ __forceinline__ uint32_t d2u_round(double v) {
  return (uint32_t)__double2loint(v + 6755399441055744.0);
}

// Pass-A twiddle tables [16][32] (k2, lane), each entry from sincospi:
//   forward  zeta^lane w512^(lane k2) = exp(i pi lane (1 + 4 k2) / 1024)
//            (the twist zeta^n = zeta^lane w64^n2 of the folding, its
//            thread-constant factor moved behind the linear pass A);
//   inverse  w512^(-lane k2) zeta^(-k2) = exp(-i pi k2 (4 lane + 1) / 1024)
//            (the untwist's zeta^(-k2) factor of output n = k2 + 16 k1).
__device__ __forceinline__ void make_tables(int t, int nthreads, double2* fwd, double2* inv) {
  for (int e = t; e < 512; e += nthreads) {
    const int k2 = e >> 5, lane = e & 31;
    double s, c;
    sincospi(lane * (1 + 4 * k2) / 1024.0, &s, &c);
    fwd[e] = make_double2(c, s);
    sincospi(-k2 * (4 * lane + 1) / 1024.0, &s, &c);
    inv[e] = make_double2(c, s);
  }
}

// ---------------------------------------------------------------------------
// Variant 2: the same two-pass 512-point DFT with
//  (a) pass-A twiddles from a 9-entry-per-lane table, t(k2) for k2 < 8 and the
//      ratio r8 = t(k2 + 8) / t(k2), so 9 shared loads instead of 16 per
//      transform (8 extra complex products);
//  (b) a select-free pair exchange: lanes n1 = 3 (mod 4) carry a factor -1
//      (folded into t), so the odd thread h = 1 of a column computes
//      Y[k] = E1[k ^ 8] and both threads keep a[brev(j)] and send
//      a[brev(8 + j)]; both then form keep +- c r with c = w^j (h = 0) or
//      1 / w'^(8+j) (h = 1): thread 1's outputs come out scaled by
//      sigma = 1 / w32^(8+j) (x) and -1 / w32^(8+j) (y).  The forward's
//      scaling is undone in the BK setup (BK spectra multiplied by sigma^-2,
//      so that D' B'' = sigma D B / sigma = D B); the inverse's is folded into
//      its untwist constants.  Verified against the exact product on the
//      device (she_fft_product_selftest) and in tests/test_fft_exactness.py.
// ---------------------------------------------------------------------------
constexpr int kTw2 = 9;  // table entries per lane and direction

// v2 tables [9][32] (k2 or 8 = ratio, lane), s(n1) = -1 for n1 = 3 (mod 4):
//   forward  t(k2) = s zeta^lane w512^(lane k2),  ratio w512^(8 lane)
//   inverse  t(k2) = s w512^(-lane k2) zeta^(-k2), ratio exp(-i pi 8 (4 lane + 1) / 1024)
__device__ __forceinline__ void make_tables2(int t, int nthreads, double2* fwd, double2* inv) {
  for (int e = t; e < kTw2 * 32; e += nthreads) {
    const int k2 = e >> 5, lane = e & 31;
    const double sg = (lane & 3) == 3 ? -1.0 : 1.0;
    double s, c;
    if (k2 < 8) {
      sincospi(lane * (1 + 4 * k2) / 1024.0, &s, &c);
      fwd[e] = make_double2(sg * c, sg * s);
      sincospi(-k2 * (4 * lane + 1) / 1024.0, &s, &c);
      inv[e] = make_double2(sg * c, sg * s);
    } else {
      sincospi(lane / 32.0, &s, &c);
      fwd[e] = make_double2(c, s);
      sincospi(-8 * (4 * lane + 1) / 1024.0, &s, &c);
      inv[e] = make_double2(c, s);
    }
  }
}

template <int SIGN>
__device__ __forceinline__ void dft512_v2(double2 (&a)[16], int lane, const double2* tw,
                                          double2* scratch, double2 (&x)[8], double2 (&y)[8]) {
  dft16<SIGN>(a);
  const double2 r8 = tw[8 * 32 + lane];
#pragma unroll
  for (int k2 = 0; k2 < 8; ++k2) {
    const double2 p = tw[k2 * 32 + lane];
    scratch[tslot(lane, k2)] = cmul(a[brev4(k2)], p);
    scratch[tslot(lane, k2 + 8)] = cmul(a[brev4(k2 + 8)], cmul(p, r8));
  }
  __syncwarp();
  const int k2 = lane >> 1;
  int h = lane & 1;
  asm volatile("" : "+r"(h));  // opaque: the selected constants below stay per call (no hoisting)
#pragma unroll
  for (int m = 0; m < 16; ++m) a[m] = scratch[tslot(2 * m + h, k2)];
  dft16<SIGN>(a);
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const double2 keep = a[brev4(j)], send = a[brev4(8 + j)];
    double2 r;
    r.x = __shfl_xor_sync(0xffffffffu, send.x, 1);
    r.y = __shfl_xor_sync(0xffffffffu, send.y, 1);
    // c0 = w32^(SIGN j), c1 = w32^(-SIGN (8 + j)): compile-time constants
    const double2 c = cw(h ? (-SIGN * 4 * (8 + j)) & 127 : (SIGN * 4 * j) & 127);  // one constant-cache load, two addresses per warp
    const double2 t = cmul(r, c);
    x[j] = cadd(keep, t);
    y[j] = csub(keep, t);
  }
  __syncwarp();  // scratch reads done before the caller reuses the row
}

// Forward v2: as forward(); the spectrum at k = k2 + 16 k1 is scaled by
// sigma(k) = w32^(-k1) for k1 & 8, 1 otherwise (see above).
__device__ __forceinline__ void forward_v2(const double (&re)[16], const double (&im)[16], int lane,
                                           const double2* tw_fwd, double2* row) {
  double2 a[16];
#pragma unroll
  for (int m = 0; m < 16; ++m) a[m] = rot<1>(make_double2(re[m], im[m]), 2 * m);  // w64^m
  double2 x[8], y[8];
  dft512_v2<1>(a, lane, tw_fwd, row, x, y);
  const int k2 = lane >> 1, h = lane & 1;
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    row[fpos(k2 + 16 * (8 * h + j))] = x[j];
    row[fpos(k2 + 16 * (16 + 8 * h + j))] = y[j];
  }
}

// Inverse v2 of the TRUE spectrum X[k] = row[fpos(k)]: outputs as inverse();
// the untwist constants absorb thread 1's exchange scaling:
//   h = 0: x * conj(W128[j]),        y * conj(W128[16 + j])
//   h = 1: x * conj(W128[40 + 5 j]), y * conj(W128[(5 j - 8) & 127])
__device__ __forceinline__ void inverse_v2(const double2* row_in, int lane, const double2* tw_inv,
                                           double2* row, double2 (&x)[8], double2 (&y)[8]) {
  double2 a[16];
#pragma unroll
  for (int m = 0; m < 16; ++m) a[m] = row_in[fpos(lane + 32 * m)];
  __syncwarp();
  dft512_v2<-1>(a, lane, tw_inv, row, x, y);
  const int h = lane & 1;
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    x[j] = cmulc(x[j], cw(h ? 40 + 5 * j : j));
    y[j] = cmulc(y[j], cw(h ? (5 * j - 8) & 127 : 16 + j));
  }
}

// ---- the steps of the v2 transform, for the two-stream kernel --------------
// (dft512_v2 split at its shared-memory / FP64 boundaries so that a warp can
// run one lane's FP64 step and another lane's shared-memory step together)
__device__ __forceinline__ void v2_pa_store(const double2 (&a)[16], int lane, const double2* tw,
                                            double2* scratch) {
  const double2 r8 = tw[8 * 32 + lane];
#pragma unroll
  for (int k2 = 0; k2 < 8; ++k2) {
    const double2 p = tw[k2 * 32 + lane];
    scratch[tslot(lane, k2)] = cmul(a[brev4(k2)], p);
    scratch[tslot(lane, k2 + 8)] = cmul(a[brev4(k2 + 8)], cmul(p, r8));
  }
}
__device__ __forceinline__ void v2_pb_load(double2 (&a)[16], int lane, const double2* scratch) {
  const int k2 = lane >> 1, h = lane & 1;
#pragma unroll
  for (int m = 0; m < 16; ++m) a[m] = scratch[tslot(2 * m + h, k2)];
}
template <int SIGN>
__device__ __forceinline__ void v2_exchange(const double2 (&a)[16], int lane, double2 (&x)[8],
                                            double2 (&y)[8]) {
  const int h = lane & 1;
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const double2 keep = a[brev4(j)], send = a[brev4(8 + j)];
    double2 r;
    r.x = __shfl_xor_sync(0xffffffffu, send.x, 1);
    r.y = __shfl_xor_sync(0xffffffffu, send.y, 1);
    const double2 c = cw(h ? (-SIGN * 4 * (8 + j)) & 127 : (SIGN * 4 * j) & 127);  // one constant-cache load, two addresses per warp
    const double2 t = cmul(r, c);
    x[j] = cadd(keep, t);
    y[j] = csub(keep, t);
  }
}
__device__ __forceinline__ void v2_fwd_in(const double (&re)[16], const double (&im)[16],
                                          double2 (&a)[16]) {
#pragma unroll
  for (int m = 0; m < 16; ++m) a[m] = rot<1>(make_double2(re[m], im[m]), 2 * m);  // w64^m
}
__device__ __forceinline__ void v2_fwd_out(const double2 (&x)[8], const double2 (&y)[8], int lane,
                                           double2* row) {
  const int k2 = lane >> 1, h = lane & 1;
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    row[fpos(k2 + 16 * (8 * h + j))] = x[j];
    row[fpos(k2 + 16 * (16 + 8 * h + j))] = y[j];
  }
}
__device__ __forceinline__ void v2_inv_in(const double2* row_in, int lane, double2 (&a)[16]) {
#pragma unroll
  for (int m = 0; m < 16; ++m) a[m] = row_in[fpos(lane + 32 * m)];
}
__device__ __forceinline__ void v2_inv_untwist(int lane, double2 (&x)[8], double2 (&y)[8]) {
  const int h = lane & 1;
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    x[j] = cmulc(x[j], cw(h ? 40 + 5 * j : j));
    y[j] = cmulc(y[j], cw(h ? (5 * j - 8) & 127 : 16 + j));
  }
}

// ---- variant 3: variant 2 with DIT/FMA DFT16s and the FMA pair exchange ----
template <int SIGN>
__device__ __forceinline__ void dft512_v3(double2 (&a)[16], int lane, const double2* tw,
                                          double2* scratch, double2 (&x)[8], double2 (&y)[8]) {
  dft16_dit<SIGN>(a);
  const double2 r8 = tw[8 * 32 + lane];
#pragma unroll
  for (int k2 = 0; k2 < 8; ++k2) {
    const double2 p = tw[k2 * 32 + lane];
    scratch[tslot(lane, k2)] = cmul(a[brev4(k2)], p);
    scratch[tslot(lane, k2 + 8)] = cmul(a[brev4(k2 + 8)], cmul(p, r8));
  }
  __syncwarp();
  const int k2 = lane >> 1, h = lane & 1;
#pragma unroll
  for (int m = 0; m < 16; ++m) a[m] = scratch[tslot(2 * m + h, k2)];
  dft16_dit<SIGN>(a);
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const double2 keep = a[brev4(j)], send = a[brev4(8 + j)];
    double2 r;
    r.x = __shfl_xor_sync(0xffffffffu, send.x, 1);
    r.y = __shfl_xor_sync(0xffffffffu, send.y, 1);
    // c0 = w32^(SIGN j), c1 = w32^(-SIGN (8 + j)): compile-time constants
    const double2 c = cw(h ? (-SIGN * 4 * (8 + j)) & 127 : (SIGN * 4 * j) & 127);  // one constant-cache load, two addresses per warp
    // x = keep + c r (4 DFMA), y = 2 keep - x (2 DFMA)
    x[j].x = fma(c.x, r.x, fma(-c.y, r.y, keep.x));
    x[j].y = fma(c.x, r.y, fma(c.y, r.x, keep.y));
    y[j].x = fma(2.0, keep.x, -x[j].x);
    y[j].y = fma(2.0, keep.y, -x[j].y);
  }
  __syncwarp();  // scratch reads done before the caller reuses the row
}

// Forward v3: as forward_v2 with dft512_v3 (same scaling); the spectrum at k = k2 + 16 k1 is scaled by
// sigma(k) = w32^(-k1) for k1 & 8, 1 otherwise (see above).
__device__ __forceinline__ void forward_v3(const double (&re)[16], const double (&im)[16], int lane,
                                           const double2* tw_fwd, double2* row) {
  double2 a[16];
#pragma unroll
  for (int m = 0; m < 16; ++m) a[m] = rot<1>(make_double2(re[m], im[m]), 2 * m);  // w64^m
  double2 x[8], y[8];
  dft512_v3<1>(a, lane, tw_fwd, row, x, y);
  const int k2 = lane >> 1, h = lane & 1;
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    row[fpos(k2 + 16 * (8 * h + j))] = x[j];
    row[fpos(k2 + 16 * (16 + 8 * h + j))] = y[j];
  }
}

// Inverse v3 (as inverse_v2, dft512_v3) of the TRUE spectrum X[k] = row[fpos(k)]: outputs as inverse();
// the untwist constants absorb thread 1's exchange scaling:
//   h = 0: x * conj(W128[j]),        y * conj(W128[16 + j])
//   h = 1: x * conj(W128[40 + 5 j]), y * conj(W128[(5 j - 8) & 127])
__device__ __forceinline__ void inverse_v3(const double2* row_in, int lane, const double2* tw_inv,
                                           double2* row, double2 (&x)[8], double2 (&y)[8]) {
  double2 a[16];
#pragma unroll
  for (int m = 0; m < 16; ++m) a[m] = row_in[fpos(lane + 32 * m)];
  __syncwarp();
  dft512_v3<-1>(a, lane, tw_inv, row, x, y);
  const int h = lane & 1;
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    x[j] = cmulc(x[j], cw(h ? 40 + 5 * j : j));
    y[j] = cmulc(y[j], cw(h ? (5 * j - 8) & 127 : 16 + j));
  }
}

// ---- the register-layout inverse of the TMEM engine -------
// In-register 16-point DFT by radix-2 decimation in time on bit-reversed
// input: a[brev4(k)] = X[k] on entry, a[n] = sum_k X[k] w16^(SIGN n k) on
// exit (the inverse pairing of dft16: dft16<+1> then dft16_dit_br<-1> is 16x
// the identity).
template <int SIGN>
__device__ __forceinline__ void dft16_dit_br(double2 (&a)[16]) {
#pragma unroll
  for (int s = 1; s <= 8; s <<= 1) {
#pragma unroll
    for (int g0 = 0; g0 < 16; g0 += 2 * s) {
#pragma unroll
      for (int j = 0; j < s; ++j) {
        const double2 u = a[g0 + j], v = rot<SIGN>(a[g0 + j + s], j * (64 / s));  // w_(2s)^(SIGN j)
        a[g0 + j] = cadd(u, v);
        a[g0 + j + s] = csub(u, v);
      }
    }
  }
}

// The same DIT DFT16 on bit-reversed input with FMA butterflies (the variant-3
// arithmetic of dft16_dit): x = u + w v in 4 DFMA, y = 2 u - x in 2 (w = +-1,
// +-i: 4 DADD); 148 FP64 instructions instead of 168.
template <int SIGN>
__device__ __forceinline__ void dft16_dit_br_fma(double2 (&a)[16]) {
#pragma unroll
  for (int s = 1; s <= 8; s <<= 1) {
#pragma unroll
    for (int g0 = 0; g0 < 16; g0 += 2 * s) {
#pragma unroll
      for (int j = 0; j < s; ++j) {
        const double2 u = a[g0 + j], v = a[g0 + j + s];
        const int e = (SIGN * j * (64 / s)) & 127;  // w = W128^e = w_(2s)^(SIGN j)
        double2 x, y;
        if (e == 0) {
          x = cadd(u, v);
          y = csub(u, v);
        } else if (e == 64) {
          x = csub(u, v);
          y = cadd(u, v);
        } else if (e == 32) {  // w = i: w v = (-v.y, v.x)
          x = make_double2(u.x - v.y, u.y + v.x);
          y = make_double2(u.x + v.y, u.y - v.x);
        } else if (e == 96) {  // w = -i: w v = (v.y, -v.x)
          x = make_double2(u.x + v.y, u.y - v.x);
          y = make_double2(u.x - v.y, u.y + v.x);
        } else {
          const double2 w = cw(e);
          x.x = fma(w.x, v.x, fma(-w.y, v.y, u.x));
          x.y = fma(w.x, v.y, fma(w.y, v.x, u.y));
          y.x = fma(2.0, u.x, -x.x);
          y.y = fma(2.0, u.y, -x.y);
        }
        a[g0 + j] = x;
        a[g0 + j + s] = y;
      }
    }
  }
}

// Exact step-by-step inverse (unnormalised: 512 x) of the v2 forward
// transform, taking the spectrum in the REGISTER layout dft512_v2<1> leaves it
// in -- thread (k2, h) = (lane >> 1, lane & 1), x[j] / y[j] at frequencies
// k2 + 16 (8h + j) / k2 + 16 (16 + 8h + j), thread 1's values scaled by
// sigma / -sigma (see dft512_v2) -- and returning the natural layout
// a[n2] = (c_n + i c_{n+512}) for n = lane + 32 n2, untwisted.  The steps, in
// reverse order of the forward:
//   pair step   keep = x + y (= 2 keep'), r = (x - y) conj(c) (= 2 r'), the
//               partner's r is this thread's a[brev(8 + j)];
//   pass B      DIT DFT16 (conjugate) on the bit-reversed registers;
//   transpose   back through the warp's scratch row (the forward's swizzle);
//   pass A      conj(pass-A twiddle) from the forward table, DIT DFT16;
//   twist       conj(w64^n2) (the forward's table carries zeta^lane).
// Because the spectrum never leaves the registers in the forward's layout,
// the inverse needs no shared-memory input row and its output is in natural
// order (consecutive lanes, consecutive coefficients).
template <bool FMA = false>
__device__ __forceinline__ void inverse_tr(const double2 (&x)[8], const double2 (&y)[8], int lane,
                                           const double2* tw, double2* scratch, double2 (&a)[16]) {
  const int k2 = lane >> 1;
  int h = lane & 1;
  asm volatile("" : "+r"(h));  // opaque: keeps the 8 selected constants out of loop-invariant hoisting
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const double2 c = cw(h ? (-4 * (8 + j)) & 127 : (4 * j) & 127);  // one constant-cache load, two addresses per warp
    const double2 t = cmulc(csub(x[j], y[j]), c);
    double2 r;
    r.x = __shfl_xor_sync(0xffffffffu, t.x, 1);
    r.y = __shfl_xor_sync(0xffffffffu, t.y, 1);
    a[brev4(j)] = cadd(x[j], y[j]);
    a[brev4(8 + j)] = r;
  }
  if (FMA) dft16_dit_br_fma<-1>(a);
  else dft16_dit_br<-1>(a);
#pragma unroll
  for (int m = 0; m < 16; ++m) scratch[tslot(2 * m + h, k2)] = a[m];
  __syncwarp();
  const double2 r8 = tw[8 * 32 + lane];
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const double2 p = tw[k * 32 + lane];
    a[brev4(k)] = cmulc(scratch[tslot(lane, k)], p);
    a[brev4(k + 8)] = cmulc(scratch[tslot(lane, k + 8)], cmul(p, r8));
  }
  __syncwarp();  // scratch reads done before the caller reuses the row
  if (FMA) dft16_dit_br_fma<-1>(a);
  else dft16_dit_br<-1>(a);
#pragma unroll
  for (int m = 1; m < 16; ++m) a[m] = rot<-1>(a[m], 2 * m);  // conj(w64^m)
}

// sigma(k)^-2 of the v2 forward (BK setup): w16^(k1) for k1 & 8, 1 otherwise.
__device__ __forceinline__ double2 v2_bk_correction(int k) {
  const int k1 = k >> 4;
  if (!(k1 & 8)) return make_double2(1.0, 0.0);
  double s, c;
  sincospi(k1 / 8.0, &s, &c);
  return make_double2(c, s);
}

}  // namespace fft
