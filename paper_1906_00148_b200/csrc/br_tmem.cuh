// br_tmem.cuh — the TMEM blind-rotation engine (she_ctx_options.fft_engine =
// tmem).  Included by engine.cu inside its anonymous
// namespace (uses GateSrc, lane_form, fbr_load_fields, FLane's layout rules).
//
// The CMux product of the FP64 engine (exact split-BK negacyclic FFT, DESIGN.md
// §4.2b; PAPER.md:31 / :188, TFHE bootstrapping) with the digit spectra and the
// products kept in tensor memory instead of shared memory:
//
//  * Each SM sub-partition (quarter Q = warps Q, Q+4, Q+8, Q+12, which are the
//    warps that can address TMEM lanes 32Q .. 32Q+31) is an independent
//    pipeline of two blind-rotation lanes (slots), with its own named barrier:
//    no CTA-wide barrier inside the CMux loop, so the four quarters drift
//    apart in phase and one quarter's shared-memory steps overlap another's
//    FP64 steps.
//  * Thread t of a quarter owns TMEM row 32Q + t.  A forward transform leaves
//    thread t holding 16 frequencies of its digit row (x[8], y[8], the
//    register layout of dft512_v2); they go to the row with one tcgen05.st
//    (columns slot * 256 + row * 64 + 4 fi).  The pointwise step reads the
//    four digit spectra of frequency slot fi from the same row, multiplies by
//    BK_i (laid out [i][fi][plane][t], so 32 threads read 512 contiguous
//    bytes) and writes the four products in place; the inverse reads its
//    product row back with tcgen05.ld and runs inverse_tr (fft_core.cuh),
//    which takes exactly that register layout and returns natural order.
//    The three shared-memory passes over the spectra of the smem engine
//    (forward output, pointwise, inverse input: 1,024 wavefronts per lane and
//    CMux) leave the L1 data path; TMEM moves ~700 B/clk/SM on its own path
//    (tools/microbench/tmem_bench.cu).
//  * BK_i is read once per quarter (two lanes) instead of once per CTA (four
//    lanes): 512 instead of 256 wavefronts per lane and CMux, loaded through
//    a register ring PD units ahead of use.
//
// smem per quarter: ACC [2 slots][2][N] (16 KB), a-bar [2][512] (2 KB), four
// 8 KB transpose rows (one per warp): 50 KB; + the v2 twiddle tables.
// TMEM: 512 columns x 128 lanes (all of it; one CTA per SM).
#pragma once
#include "dcheck.cuh"
#include "tm_queue.h"

constexpr int kTmSlots = 2;
constexpr size_t kTmAccBytes = (size_t)kTmSlots * 2 * fft::kN * 4;
constexpr size_t kTmAbarBytes = (size_t)kTmSlots * 512 * 2;
constexpr size_t kTmScratchBytes = (size_t)4 * fft::kRow * 16;
constexpr size_t kTmQuarterBytes = kTmAccBytes + kTmAbarBytes + kTmScratchBytes;
constexpr size_t kTmSmemBytes = 4 * kTmQuarterBytes + 2 * fft::kTw2 * 32 * sizeof(double2);
#ifndef SHE_TM_PD
#define SHE_TM_PD 2
#endif
#ifndef SHE_TM_FMA_FWD  // transform 3: FMA butterflies in the forward / inverse (A/B builds)
#define SHE_TM_FMA_FWD 1
#endif
#ifndef SHE_TM_FMA_INV
#define SHE_TM_FMA_INV 1
#endif
constexpr int kTmPrefetch = SHE_TM_PD;  // BK units (4 planes each) in flight ahead of use

// ---- tensor-memory access (tcgen05, 32x32b shape: thread t <-> TMEM lane) ---
// checked build: columns [col, col + ncols) inside the 512 allocated (base
// column 0, asserted at allocation) and a lane field at a quarter boundary
__device__ __forceinline__ void tm_check(uint32_t addr, uint32_t ncols) {
  SHE_DCHECK((addr & 0xFFFFu) + ncols <= 512u && ((addr >> 16) & 31u) == 0 && (addr >> 16) < 128u);
}
__device__ __forceinline__ void tm_st4(uint32_t addr, const double2 (&v)[4]) {
  tm_check(addr, 16);
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(
          addr),
      "r"(__double2loint(v[0].x)), "r"(__double2hiint(v[0].x)), "r"(__double2loint(v[0].y)),
      "r"(__double2hiint(v[0].y)), "r"(__double2loint(v[1].x)), "r"(__double2hiint(v[1].x)),
      "r"(__double2loint(v[1].y)), "r"(__double2hiint(v[1].y)), "r"(__double2loint(v[2].x)),
      "r"(__double2hiint(v[2].x)), "r"(__double2loint(v[2].y)), "r"(__double2hiint(v[2].y)),
      "r"(__double2loint(v[3].x)), "r"(__double2hiint(v[3].x)), "r"(__double2loint(v[3].y)),
      "r"(__double2hiint(v[3].y))
      : "memory");
}
__device__ __forceinline__ void tm_ld4(uint32_t addr, double2 (&v)[4]) {
  tm_check(addr, 16);
  int r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]),
        "=r"(r[15])
      : "r"(addr)
      : "memory");
#pragma unroll
  for (int q = 0; q < 4; ++q)
    v[q] = make_double2(__hiloint2double(r[4 * q + 1], r[4 * q]), __hiloint2double(r[4 * q + 3], r[4 * q + 2]));
}
__device__ __forceinline__ void tm_st1(uint32_t addr, double2 v) {
  tm_check(addr, 4);
  // the b64 -> 2 x b32 split inside the asm, so that ptxas picks the register
  // quad itself instead of copying two pairs into one
  asm volatile(
      "{\n\t.reg .b32 a, b, c, d;\n\tmov.b64 {a, b}, %1;\n\tmov.b64 {c, d}, %2;\n\t"
      "tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {a, b, c, d};\n\t}" ::"r"(addr),
      "d"(v.x), "d"(v.y)
      : "memory");
}
// The four digit spectra (r = 0..3, columns col0 + 64 r) of one frequency slot,
// loaded and waited for in one block (doubles out directly).
__device__ __forceinline__ void tm_ld_rows4(uint32_t col0, double2 (&D)[4]) {
  tm_check(col0 + 192, 4);
  asm volatile(
      "{\n\t.reg .b32 a<16>;\n\t"
      "tcgen05.ld.sync.aligned.32x32b.x4.b32 {a0, a1, a2, a3}, [%8];\n\t"
      "tcgen05.ld.sync.aligned.32x32b.x4.b32 {a4, a5, a6, a7}, [%9];\n\t"
      "tcgen05.ld.sync.aligned.32x32b.x4.b32 {a8, a9, a10, a11}, [%10];\n\t"
      "tcgen05.ld.sync.aligned.32x32b.x4.b32 {a12, a13, a14, a15}, [%11];\n\t"
      "tcgen05.wait::ld.sync.aligned;\n\t"
      "mov.b64 %0, {a0, a1};\n\tmov.b64 %1, {a2, a3};\n\t"
      "mov.b64 %2, {a4, a5};\n\tmov.b64 %3, {a6, a7};\n\t"
      "mov.b64 %4, {a8, a9};\n\tmov.b64 %5, {a10, a11};\n\t"
      "mov.b64 %6, {a12, a13};\n\tmov.b64 %7, {a14, a15};\n\t}"
      : "=d"(D[0].x), "=d"(D[0].y), "=d"(D[1].x), "=d"(D[1].y), "=d"(D[2].x), "=d"(D[2].y), "=d"(D[3].x),
        "=d"(D[3].y)
      : "r"(col0), "r"(col0 + 64), "r"(col0 + 128), "r"(col0 + 192)
      : "memory");
}
__device__ __forceinline__ void tm_ld1(uint32_t addr, double2& v) {
  int r0, r1, r2, r3;
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr)
               : "memory");
  v = make_double2(__hiloint2double(r1, r0), __hiloint2double(r3, r2));
}
__device__ __forceinline__ void tm_st_u16(uint32_t addr, const uint32_t (&v)[16]) {
  tm_check(addr, 16);
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(
          addr),
      "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]),
      "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15])
      : "memory");
}
__device__ __forceinline__ void tm_ld_u16(uint32_t addr, uint32_t (&v)[16]) {
  tm_check(addr, 16);
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
        "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
      : "r"(addr)
      : "memory");
}
__device__ __forceinline__ void tm_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tm_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
// Barrier over the 128 threads of quarter Q (id 1 + Q) with the tcgen05
// ordering fences around it (TMEM writes before, reads after).
__device__ __forceinline__ void tm_quarter_sync(int q) {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  asm volatile("bar.sync %0, 128;" ::"r"(1 + q) : "memory");
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}

// Spectrum of one digit row to TMEM: x[j] at column 8 j, y[j] at 8 j + 4
// (frequency slot fi = 2 j and 2 j + 1), in the order the pair exchange
// produces them.
#ifndef SHE_TM_ST_X16
#define SHE_TM_ST_X16 0
#endif
__device__ __forceinline__ void tm_store_spectrum(uint32_t addr, const double2 (&x)[8], const double2 (&y)[8]) {
  if (SHE_TM_ST_X16) {  // four 16-column stores (needs 16 consecutive registers each)
    tm_st4(addr, {x[0], y[0], x[1], y[1]});
    tm_st4(addr + 16, {x[2], y[2], x[3], y[3]});
    tm_st4(addr + 32, {x[4], y[4], x[5], y[5]});
    tm_st4(addr + 48, {x[6], y[6], x[7], y[7]});
  } else {  // sixteen 4-column stores: no register block to assemble
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      tm_st1(addr + 8 * j, x[j]);
      tm_st1(addr + 8 * j + 4, y[j]);
    }
  }
}
__device__ __forceinline__ void tm_load_spectrum(uint32_t addr, double2 (&x)[8], double2 (&y)[8]) {
  double2 v[4][4];
#pragma unroll
  for (int p = 0; p < 4; ++p) tm_ld4(addr + 16 * p, v[p]);
  tm_wait_ld();
#pragma unroll
  for (int p = 0; p < 4; ++p) {
    x[2 * p] = v[p][0];
    y[2 * p] = v[p][1];
    x[2 * p + 1] = v[p][2];
    y[2 * p + 1] = v[p][3];
  }
}

// Digit fields of BOTH rows (c, j = 0) and (c, j = 1) of ACC_c from one pass
// over the rotation (X^a P)[m] - P[m] + offset (fbr_load_fields, R8): the
// j = 0 fields in u0, the j = 1 fields packed two per register (bg_bits <= 12
// on the FFT engine) for the second transform.
__device__ __forceinline__ void tm_load_fields2(const br::Geometry& g, int lane, const uint32_t* P, uint32_t a,
                                                uint32_t (&u0)[32], uint32_t (&pk1)[16]) {
  constexpr int N = fft::kN;
  const uint32_t sh0 = 32 - g.bg_bits, sh1 = 32 - 2 * g.bg_bits, mask = (1u << g.bg_bits) - 1;
#pragma unroll
  for (int j2 = 0; j2 < 32; ++j2) {
    const uint32_t m = lane + 32 * j2;
    const uint32_t idx = (m - a) & (2 * N - 1);  // (X^a P)[m] = +-P[m - a]
    uint32_t v = P[idx & (N - 1)];
    if (idx >= (uint32_t)N) v = 0u - v;
    const uint32_t y = v - P[m] + g.dec_offset;
    u0[j2] = y >> sh0;
    const uint32_t f1 = (y >> sh1) & mask;
    if (j2 & 1) pk1[j2 >> 1] |= f1 << 16;
    else pk1[j2 >> 1] = f1;
  }
}

// Forward transform of one digit row given as fields u = d + Bg/2 (the
// conversion of fbr_forward_fields) into the TMEM row at addr.
template <bool FMA = false>
__device__ __forceinline__ void tm_forward_fields(const uint32_t (&u)[32], double half, int lane,
                                                  const double2* tw, double2* scratch, uint32_t addr) {
  const double off = 4503599627370496.0 + half;  // 2^52 + Bg/2
  double re[16], im[16];
#pragma unroll
  for (int m = 0; m < 16; ++m) {
    re[m] = __hiloint2double(0x43300000, (int)u[m]) - off;
    im[m] = __hiloint2double(0x43300000, (int)u[m + 16]) - off;
  }
  double2 a[16], x[8], y[8];
  fft::v2_fwd_in(re, im, a);
  if (FMA) fft::dft512_v3<1>(a, lane, tw, scratch, x, y);  // same layout and scaling
  else fft::dft512_v2<1>(a, lane, tw, scratch, x, y);
  tm_store_spectrum(addr, x, y);
}

// Inverse of the product row at addr, rounded to the exact integer and added
// into ACC_o at n = lane + 32 m (re) and n + 512 (im), shifted by sh (16 for
// the hi half).  TRACK: the largest distance to an integer (self-test).
template <bool TRACK, bool FMA = false>
__device__ __forceinline__ void tm_inverse_acc(uint32_t addr, int lane, const double2* tw, double2* scratch,
                                               uint32_t* acc_o, int sh, unsigned long long* worst) {
  double2 x[8], y[8], a[16];
  tm_load_spectrum(addr, x, y);
  fft::inverse_tr<FMA>(x, y, lane, tw, scratch, a);
  double dmax = 0.0;
#pragma unroll
  for (int m = 0; m < 16; ++m) {
    if (TRACK) {
      dmax = fmax(dmax, fabs(a[m].x - rint(a[m].x)));
      dmax = fmax(dmax, fabs(a[m].y - rint(a[m].y)));
    }
    atomicAdd(acc_o + lane + 32 * m, fft::d2u_round(a[m].x) << sh);
    atomicAdd(acc_o + lane + 32 * m + fft::kM, fft::d2u_round(a[m].y) << sh);
  }
  if (TRACK) atomicMax(worst, (unsigned long long)__double_as_longlong(dmax));
}

// A 16-byte read-only global load the compiler keeps in program order (an
// __ldg is an invariant load that may be hoisted arbitrarily far, which turns
// the BK ring below into 256 live registers).
__device__ __forceinline__ double2 ldg_ordered(const double2* p) {
  double2 v;
  asm volatile("ld.global.nc.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(p));
  return v;
}

// BK unit u = f * 4 + q of warp s: the four planes (r, q), r < 4, of frequency
// slot fi = 4 s + f (bkt: [fi][plane][32] for this i, thread t added).
template <int U>
__device__ __forceinline__ void tm_bk_unit(const double2* bk_s, double2 (&b)[4]) {
  constexpr int f = U >> 2, q = U & 3;
#pragma unroll
  for (int r = 0; r < 4; ++r) b[r] = ldg_ordered(bk_s + ((size_t)f * 16 + r * 4 + q) * 32);
}

// Pointwise step of one quarter, warp s: frequency slots fi = 4 s .. 4 s + 3
// of this thread's TMEM row, both slots; the 16 BK units stream through a ring
// of PD + 1 register buffers (the first PD were requested by tm_bk_prefetch).
template <int PD>
struct TmRing {
  double2 b[PD + 1][4];
};
template <int PD, int U = 0>
__device__ __forceinline__ void tm_bk_prefetch(const double2* bk_s, TmRing<PD>& ring) {
  static_assert(PD >= 0 && PD <= 8, "BK prefetch distance");
  if constexpr (U < PD) {
    tm_bk_unit<U>(bk_s, ring.b[U % (PD + 1)]);
    tm_bk_prefetch<PD, U + 1>(bk_s, ring);
  }
}
template <int PD, int NS, int U, int NU = 16>
__device__ __forceinline__ void tm_pw_unit(const double2* bk_s, TmRing<PD>& ring, const double2 (&D)[2][4],
                                           uint32_t row_base, int fi) {
  // unit U + PD into the buffer unit U - 1 used (PD = 0: unit U itself, just in time)
  if (U + PD < NU) tm_bk_unit<(U + PD < NU ? U + PD : 0)>(bk_s, ring.b[(U + PD) % (PD + 1)]);
  constexpr int q = U & 3;
  const double2(&b)[4] = ring.b[U % (PD + 1)];
#pragma unroll
  for (int sl = 0; sl < NS; ++sl) {
    double2 c = fft::cmul(D[sl][0], b[0]);
#pragma unroll
    for (int r = 1; r < 4; ++r) {
      c.x = fma(D[sl][r].x, b[r].x, fma(-D[sl][r].y, b[r].y, c.x));
      c.y = fma(D[sl][r].x, b[r].y, fma(D[sl][r].y, b[r].x, c.y));
    }
    tm_st1(row_base + sl * 256 + q * 64 + 4 * fi, c);
  }
}
// Slot fi = 4 s + F: the four digit spectra of both lanes are read into
// registers first, so the four products can be written in place.  Both
// slots are always computed (an idle slot's columns hold stale values that
// nothing reads), so there is no data-dependent control flow here.
template <int PD, int NS, int F>
__device__ __forceinline__ void tm_pw_slot(const double2* bk_s, TmRing<PD>& ring, uint32_t row_base, int s) {
  const int fi = 4 * s + F;
  double2 D[2][4];
#pragma unroll
  for (int sl = 0; sl < NS; ++sl) tm_ld_rows4(row_base + sl * 256 + 4 * fi, D[sl]);
  tm_pw_unit<PD, NS, 4 * F + 0>(bk_s, ring, D, row_base, fi);
  tm_pw_unit<PD, NS, 4 * F + 1>(bk_s, ring, D, row_base, fi);
  tm_pw_unit<PD, NS, 4 * F + 2>(bk_s, ring, D, row_base, fi);
  tm_pw_unit<PD, NS, 4 * F + 3>(bk_s, ring, D, row_base, fi);
}
// NS = 2: a lane pair (slots 0, 1); NS = 1: slot 0 alone.
template <int PD, int NS>
__device__ __forceinline__ void tm_pointwise(const double2* bk_s, TmRing<PD>& ring, uint32_t row_base, int s) {
  tm_pw_slot<PD, NS, 0>(bk_s, ring, row_base, s);
  tm_pw_slot<PD, NS, 1>(bk_s, ring, row_base, s);
  tm_pw_slot<PD, NS, 2>(bk_s, ring, row_base, s);
  tm_pw_slot<PD, NS, 3>(bk_s, ring, row_base, s);
}
// One lane's pointwise over NF consecutive frequency slots fbase .. fbase +
// NF - 1 (bk_s points at slot fbase): the per-slot pipelines variant.
template <int PD, int NF, int F = 0>
__device__ __forceinline__ void tm_pointwise_range(const double2* bk_s, TmRing<PD>& ring, uint32_t slot_base,
                                                   int fbase) {
  if constexpr (F < NF) {
    const int fi = fbase + F;
    double2 D[2][4];
    tm_ld_rows4(slot_base + 4 * fi, D[0]);
    tm_pw_unit<PD, 1, 4 * F + 0, 4 * NF>(bk_s, ring, D, slot_base, fi);
    tm_pw_unit<PD, 1, 4 * F + 1, 4 * NF>(bk_s, ring, D, slot_base, fi);
    tm_pw_unit<PD, 1, 4 * F + 2, 4 * NF>(bk_s, ring, D, slot_base, fi);
    tm_pw_unit<PD, 1, 4 * F + 3, 4 * NF>(bk_s, ring, D, slot_base, fi);
    tm_pointwise_range<PD, NF, F + 1>(bk_s, ring, slot_base, fbase);
  }
}
#ifndef SHE_TM_INDEP  // 1: the two lanes of a pipeline as two independent 2-warp pipelines
#define SHE_TM_INDEP 0
#endif
__device__ __forceinline__ void tm_slot_sync(int q, int sl) {  // the 64 threads of (quarter, slot)
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  asm volatile("bar.sync %0, 64;" ::"r"(5 + 2 * q + sl) : "memory");
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}

struct TmArgs {
  GateSrc src;
  const uint32_t* lanes;
  const uint32_t* nlanes;
  const double2* bkt;  // [n][16 fi][16 plane][32 t]
  uint32_t* ext;
  uint32_t ext_stride;
  br::Geometry geo;
  uint32_t stagger;  // ns of start delay per quarter index (phase offset)
  // Work queue (see br_fft_tm_kernel, tm_queue.h): sched[0] = next unit,
  // sched[1 + s] = iterations of slot s (a lane pair, or a lane) completed;
  // acc_save[s] = the slot's accumulators between chunks.  chunk = CMux
  // iterations per unit (>= n: the static contiguous split only).
  uint32_t* sched;
  uint32_t* acc_save;
  uint32_t chunk;
  uint32_t wrap;        // 1: the wrap-around schedule instead of the chunk queue (tm_queue.h)
  uint32_t save_slots;  // slots acc_save and sched hold (checked build)
};

// Progress word of a slot (a lane pair, or a lane): the CMux iterations done,
// published with release semantics after the slot's accumulators were written
// back (and fenced), awaited with acquire loads by one thread of the quarter
// that continues the slot.  The unit it waits for is run by a resident CTA
// (one CTA per SM, grid <= SM count) before any unit that waits itself (wrap
// schedule: a pipeline runs its dependency-free first part first; queue: the
// awaited unit was taken earlier and waits only on still earlier units), so
// the wait is finite; the bound turns a broken invariant into a launch error
// instead of a hang.
__device__ __forceinline__ void tm_publish(uint32_t* flag, uint32_t v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(flag), "r"(v) : "memory");
}
__device__ __forceinline__ void tm_await(const uint32_t* flag, uint32_t want) {
  for (uint32_t spins = 0;; ++spins) {
    uint32_t v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(flag) : "memory");
    if (v >= want) return;
    __nanosleep(256);
    if (spins > (1u << 23)) __trap();  // > 2 s
  }
}

__device__ __forceinline__ uint32_t tm_alloc_all(uint32_t* slot, int warp) {
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
                     (uint32_t)__cvta_generic_to_shared(slot))
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  SHE_DCHECK((*slot & 0xFFFFu) == 0 && (*slot >> 16) == 0);  // all 512 columns from column 0
  return *slot;
}
__device__ __forceinline__ void tm_free_all(uint32_t tmem, int warp) {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem) : "memory");
}

// K3, TMEM engine: one persistent CTA of 16 warps per SM, four independent
// quarter pipelines of two lanes each (see the file comment).
//
// Work distribution (tm_queue.h).  A unit is (lane pair or single lane, CMux
// iterations [i0, i1)).  Narrow batches (<= 1 lane per pipeline, or 1.65 .. 2)
// use the static split: pipeline gq runs the contiguous lanes [first, last),
// each for all n iterations.  Wider batches are balanced by splitting units in
// time: a lane is n dependent iterations, so the static split of config 1's
// 4797 lanes over 592 pipelines leaves 61 of them a ninth lane that runs alone
// at the end (wave tail).  Default: the wrap-around schedule
// (every pipeline the same number of iterations; a unit cut at most once, its
// first part run first by one pipeline, its last part run last by the next).
// Option fft_chunk > 0: a device-wide queue of (unit, chunk) items in
// chunk-major order.  Either way the pipeline that ends a part writes the
// accumulators to acc_save and publishes the iteration count; the pipeline
// that continues waits for it, reloads them, recomputes a-bar and goes on
// (or extracts after iteration n).
template <int PD = kTmPrefetch, bool FMA = false>
__global__ void __launch_bounds__(512, 1) br_fft_tm_kernel(TmArgs args) {
  constexpr int N = fft::kN;
  extern __shared__ __align__(16) uint8_t smem[];
  __shared__ uint32_t tmem_slot;
  __shared__ uint32_t unit_info[4][8];
  const GateSrc& src = args.src;
  const br::Geometry& geo = args.geo;
  const uint32_t n = geo.n;
  const int tid = threadIdx.x, lane = tid & 31;
  const int warp = __shfl_sync(0xffffffffu, tid >> 5, 0);  // warp-uniform (uniform datapath)
  const int Q = warp & 3, s = warp >> 2, qt = s * 32 + lane;  // quarter, warp in quarter, thread in quarter
  uint8_t* qb = smem + (size_t)Q * kTmQuarterBytes;
  uint32_t* acc = reinterpret_cast<uint32_t*>(qb);                     // [slot][c][N]
  uint16_t* abar = reinterpret_cast<uint16_t*>(qb + kTmAccBytes);       // [slot][512]
  double2* scratch = reinterpret_cast<double2*>(qb + kTmAccBytes + kTmAbarBytes) + s * fft::kRow;
  double2* tw = reinterpret_cast<double2*>(smem + 4 * kTmQuarterBytes);
  fft::make_tables2(tid, 512, tw, tw + fft::kTw2 * 32);
  const uint32_t tmem = tm_alloc_all(&tmem_slot, warp);  // includes the table barrier
  const uint32_t row_base = __shfl_sync(0xffffffffu, tmem + ((uint32_t)(32 * Q) << 16), 0);

  // the next unit of this pipeline, decoded by its thread 0 (nothing of the
  // queue stays in registers across the CMux loop): lanes base .. base + nsl - 1
  // (nsl = 0: no more work), iterations [i0, i1); [4] = the static split's cursor
  uint32_t* const unit = unit_info[Q];
  if (qt == 0) {
    unit[4] = tmq::first(blockIdx.x * 4 + Q, *args.nlanes, gridDim.x * 4);
    unit[6] = 0;  // the wrap-around schedule's step
  }
#if !SHE_TM_INDEP
  if (args.stagger && Q) __nanosleep(args.stagger * Q);
#endif
  const int sl_f = s >> 1, c_f = s & 1;  // forward: slot, component (rows 2 c + j)
  const int sl_i = s >> 1, o_i = s & 1;  // inverse: slot, output (rows 2 o + half)

  // the gate prologue of the lanes in slots 0 .. nsl - 1: a-bar, then the
  // accumulators (the test vector, or the pair's saved state `resume`)
  auto prologue = [&](uint32_t base, int nsl, const uint32_t* resume) {
    for (int sl = 0; sl < nsl; ++sl) {
      SHE_DCHECK(base + sl < *args.nlanes && n < 512);
      const uint32_t e = args.lanes[base + sl];
      const uint32_t gate = e & 0x7FFFFFFFu, hh = e >> 31;
      SHE_DCHECK(gate < src.count && (hh == 0 || gate_op(src, gate) == SHE_MUX));
      const LaneForm f = lane_form(gate_op(src, gate), (int)hh);
      bool n0, n1;
      const uint32_t* x0 = gate_in(src, gate, 0, n0);
      const uint32_t* x1 = gate_in(src, gate, f.j1, n1);
      const uint32_t k0 = (uint32_t)(n0 ? -f.k0 : f.k0), k1 = (uint32_t)(n1 ? -f.k1 : f.k1);
      for (uint32_t k = qt; k <= n; k += 128) {
        uint32_t v = k0 * x0[k] + k1 * x1[k];
        if (k == n) v += f.kappa;
        abar[sl * 512 + k] = (uint16_t)br::modswitch(v, geo.lg2N);
      }
    }
    tm_quarter_sync(Q);
    if (resume) {  // written by another SM: read through L2
      const uint4* r4 = reinterpret_cast<const uint4*>(resume);
      uint4* a4 = reinterpret_cast<uint4*>(acc);
      for (int m = qt; m < kTmSlots * 2 * N / 4; m += 128) a4[m] = __ldcg(r4 + m);
    } else {
      for (int sl = 0; sl < nsl; ++sl) {
        const uint32_t bbar = abar[sl * 512 + n];
        uint32_t* a = acc + sl * 2 * N;
        for (int m = qt; m < N; m += 128) {
          a[m] = 0;
          a[N + m] = br::testvec_coeff(m, bbar, N);
        }
      }
    }
    tm_quarter_sync(Q);
  };
  // sample extraction of slots 0 .. nsl - 1
  auto extract = [&](uint32_t base, int nsl) {
    for (int sl = 0; sl < nsl; ++sl) {
      const uint32_t* a = acc + sl * 2 * N;
      const uint32_t le = args.lanes[base + sl];  // gate | h << 31
      SHE_DCHECK((le & 0x7FFFFFFFu) < src.count);
      uint32_t* e = args.ext + (size_t)(2 * (le & 0x7FFFFFFFu) + (le >> 31)) * args.ext_stride;
      for (int m = qt; m <= N; m += 128) {
        uint32_t v;
        if (m == 0) v = a[0];
        else if (m < N) v = 0u - a[N - m];
        else v = a[N];
        e[m] = v;
      }
    }
    tm_quarter_sync(Q);
  };

  for (;;) {
    if (qt == 0) {
      const uint32_t total = *args.nlanes, nq = gridDim.x * 4;
      const uint32_t chunk = args.chunk ? args.chunk : n;
      tmq::Unit w;
      const int m = tmq::mode(total, n, args.wrap ? 1u : chunk, nq);
      if (m != tmq::kStatic) {
        if (args.wrap) w = tmq::wrap_unit(blockIdx.x * 4 + Q, unit[6]++, total, n, nq, m);
        else w = tmq::unit(atomicAdd(args.sched, 1u), total, n, chunk, m);
        SHE_DCHECK(args.sched && args.acc_save && w.slot < args.save_slots);
        // the iterations before i0 are done and the accumulators written back
        if (w.nsl && w.i0) tm_await(args.sched + 1 + w.slot, w.i0);
      } else {
        w = tmq::next_static(unit[4], blockIdx.x * 4 + Q, total, nq, n);
        unit[4] = w.base + w.nsl;
      }
      unit[5] = w.slot;
      unit[0] = w.base;
      unit[1] = w.nsl;
      unit[2] = w.i0;
      unit[3] = w.i1;
    }
    tm_quarter_sync(Q);  // unit[] is rewritten only after the barriers below
    const int nsl = (int)unit[1];
    if (nsl == 0) break;
    {
      const uint32_t base = unit[0], i0 = unit[2];
      prologue(base, nsl, i0 ? args.acc_save + (size_t)unit[5] * (kTmSlots * 2 * N) : nullptr);
    }
    const uint32_t i0 = unit[2], i1 = unit[3];

    if (nsl == 2) {  // a lane pair
#if SHE_TM_INDEP
      if (args.stagger && sl_f == 1) __nanosleep(args.stagger);  // slot 1 a phase behind slot 0
#endif
      for (uint32_t i = i0; i < i1; ++i) {
        const int ln = lane;
        double2* const scr = scratch;
        const double2* const twp = tw;
        {  // forward transforms of digit rows 2c, 2c + 1 of slot sl_f
          // both rows' digit fields from one rotation pass; the j = 1 fields wait
          // in the (not yet written) TMEM columns of row 2c + 1 during the first
          // transform instead of in 16 registers
          const uint32_t row0 = row_base + sl_f * 256 + (2 * c_f) * 64, row1 = row0 + 64;
          uint32_t u[32];
          {
            uint32_t pk1[16];
            tm_load_fields2(geo, ln, acc + (sl_f * 2 + c_f) * N, abar[sl_f * 512 + i], u, pk1);
            tm_st_u16(row1, pk1);
          }
          const double half = (double)(1u << (geo.bg_bits - 1));
          tm_forward_fields<FMA && SHE_TM_FMA_FWD>(u, half, ln, twp, scr, row0);
          {
            uint32_t pk1[16];
            tm_wait_st();  // this thread's stash store (long done) before reading it back
            tm_ld_u16(row1, pk1);
            tm_wait_ld();
#pragma unroll
            for (int k = 0; k < 16; ++k) {
              u[2 * k] = pk1[k] & 0xFFFFu;
              u[2 * k + 1] = pk1[k] >> 16;
            }
          }
          tm_forward_fields<FMA && SHE_TM_FMA_FWD>(u, half, ln, twp, scr, row1);
        }
#if SHE_TM_INDEP
        // each slot's two warps: pointwise of their slot over 8 frequency slots each
        const double2* bk_s = args.bkt + ((size_t)i * 16 + 8 * (s & 1)) * 16 * 32 + ln;
        TmRing<PD> ring;
        tm_bk_prefetch<PD>(bk_s, ring);
        tm_wait_st();
        tm_slot_sync(Q, sl_f);
        tm_pointwise_range<PD, 8>(bk_s, ring, row_base + sl_f * 256, 8 * (s & 1));
        tm_wait_st();
        tm_slot_sync(Q, sl_f);
#else
        const double2* bk_s = args.bkt + ((size_t)i * 16 + 4 * s) * 16 * 32 + ln;
        TmRing<PD> ring;
        tm_bk_prefetch<PD>(bk_s, ring);
        tm_wait_st();
        tm_quarter_sync(Q);
        tm_pointwise<PD, 2>(bk_s, ring, row_base, s);
        tm_wait_st();
        tm_quarter_sync(Q);
#endif
        {  // inverse transforms of outputs (o, hi), (o, lo) of slot sl_i
          uint32_t* acc_o = acc + (sl_i * 2 + o_i) * N;
#pragma unroll 1
          for (int half = 0; half < 2; ++half)
            tm_inverse_acc<false, FMA && SHE_TM_FMA_INV>(row_base + sl_i * 256 + (2 * o_i + half) * 64, ln, twp, scr, acc_o,
                                  half ? 0 : 16, nullptr);
        }
        // No quarter barrier here: the next forward of warp s = (slot, c) reads
        // only ACC_c of its slot and writes only rows 2c, 2c + 1 -- exactly what
        // this warp's own inverse (slot, o = c) just wrote and read -- so the
        // four warps may enter the next CMux independently (a warp barrier
        // orders the lanes' shared-memory atomics before their digit loads).
        __syncwarp();
      }
      tm_quarter_sync(Q);  // all ACC complete before the extraction / the write-back
    } else {  // a single lane: all four warps on it (slot 0)
      for (uint32_t i = i0; i < i1; ++i) {
        {  // warp s: forward transform of digit row s
          uint32_t u[32];
          fbr_load_fields(geo, s, lane, acc, abar[i], u);
          tm_forward_fields<FMA && SHE_TM_FMA_FWD>(u, (double)(1u << (geo.bg_bits - 1)), lane, tw, scratch, row_base + s * 64);
        }
        const double2* bk_s = args.bkt + ((size_t)i * 16 + 4 * s) * 16 * 32 + lane;
        TmRing<PD> ring;
        tm_bk_prefetch<PD>(bk_s, ring);
        tm_wait_st();
        tm_quarter_sync(Q);
        tm_pointwise<PD, 1>(bk_s, ring, row_base, s);
        tm_wait_st();
        tm_quarter_sync(Q);
        // warp s: inverse of product row s = (o, half) = (s >> 1, s & 1)
        tm_inverse_acc<false, FMA && SHE_TM_FMA_INV>(row_base + s * 64, lane, tw, scratch, acc + (s >> 1) * N, (s & 1) ? 0 : 16, nullptr);
        tm_quarter_sync(Q);
      }
    }
    const uint32_t base = unit[0];
    if (unit[3] == n) {
      extract(base, (int)unit[1]);
    } else {  // hand the accumulators to whichever pipeline takes the slot's next chunk
      const uint4* a4 = reinterpret_cast<const uint4*>(acc);
      uint4* w4 = reinterpret_cast<uint4*>(args.acc_save + (size_t)unit[5] * (kTmSlots * 2 * N));
      for (int m = qt; m < kTmSlots * 2 * N / 4; m += 128) __stcg(w4 + m, a4[m]);
      __threadfence();
      tm_quarter_sync(Q);
      if (qt == 0) tm_publish(args.sched + 1 + unit[5], unit[3]);
    }
  }
  tm_free_all(tmem, warp);
}

// K1 for the TMEM engine: BK poly (i, w, o) half -> the TRUE spectrum (the v1
// transform: no scaling) / 512, scattered to [i][fi][plane][t] with the
// frequency of (thread t, slot fi) in dft512_v2's register layout as
// tm_store_spectrum places it: (k2, h) = (t >> 1, t & 1), j = fi >> 1,
// k = k2 + 16 (8 h + j) for even fi (x[j]), k2 + 16 (16 + 8 h + j) for odd
// fi (y[j]).  The pointwise product of a (scaled) digit
// spectrum D' = s_p D with it is s_p (D B) / 512, the input inverse_tr
// expects.
__global__ void bk_tm_kernel(const uint32_t* bk, double2* out, uint32_t polys) {
  __shared__ double2 row[fft::kRow];
  __shared__ double2 tw[2 * 512];
  const uint32_t item = blockIdx.x, poly = item >> 1, half = item & 1;
  if (poly >= polys) return;
  const int lane = threadIdx.x;
  fft::make_tables(lane, 32, tw, tw + 512);
  __syncwarp();
  const uint32_t* b = bk + (size_t)poly * fft::kN;
  double re[16], im[16];
#pragma unroll
  for (int m = 0; m < 16; ++m) {
    const int32_t v0 = (int32_t)b[lane + 32 * m], v1 = (int32_t)b[lane + 32 * m + 512];
    const int32_t l0 = (int16_t)(v0 & 0xFFFF), l1 = (int16_t)(v1 & 0xFFFF);
    re[m] = half ? (double)l0 : (double)((v0 - l0) >> 16);
    im[m] = half ? (double)l1 : (double)((v1 - l1) >> 16);
  }
  fft::forward(re, im, lane, tw, row);
  __syncwarp();
  const uint32_t i = poly >> 3, plane = (poly & 7) * 2 + half;
  for (int e = lane; e < fft::kM; e += 32) {
    const int fi = e >> 5, t = e & 31, k2 = t >> 1, h = t & 1;
    const int j = fi >> 1;
    const int k = (fi & 1) ? k2 + 16 * (16 + 8 * h + j) : k2 + 16 * (8 * h + j);
    const double2 v = row[fft::fpos(k)];
    out[(((size_t)i * 16 + fi) * 16 + plane) * 32 + t] = make_double2(v.x * (1.0 / 512), v.y * (1.0 / 512));
  }
}

// Test instrumentation (she_fft_product_selftest, variant 4): the TMEM
// engine's CMux product on caller-given digit rows and BK rows, on its own
// device functions (tm_forward_fields, tm_pointwise, tm_inverse_acc): quarter
// Q of CTA b runs case 4 b + Q in slot 0 (warp s: forward of digit row s,
// inverse of output (s >> 1, s & 1)).
template <bool FMA>
__global__ void __launch_bounds__(512, 1) fft_selftest_tm_kernel(const int32_t* digits, const double2* bkt,
                                                                 uint32_t* out, unsigned long long* worst,
                                                                 uint32_t count) {
  constexpr int N = fft::kN;
  extern __shared__ __align__(16) uint8_t smem[];
  __shared__ uint32_t tmem_slot;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int Q = warp & 3, s = warp >> 2, qt = s * 32 + lane;
  uint8_t* qb = smem + (size_t)Q * kTmQuarterBytes;
  uint32_t* acc = reinterpret_cast<uint32_t*>(qb);
  double2* scratch = reinterpret_cast<double2*>(qb + kTmAccBytes + kTmAbarBytes) + s * fft::kRow;
  double2* tw = reinterpret_cast<double2*>(smem + 4 * kTmQuarterBytes);
  fft::make_tables2(tid, 512, tw, tw + fft::kTw2 * 32);
  const uint32_t tmem = tm_alloc_all(&tmem_slot, warp);
  const uint32_t row_base = tmem + ((uint32_t)(32 * Q) << 16);
  const uint32_t c = blockIdx.x * 4 + Q;
  const bool active = c < count;
  if (active) {
    for (int m = qt; m < 2 * N; m += 128) acc[m] = 0;
    const int32_t* d = digits + ((size_t)c * 4 + s) * N;
    uint32_t uu[32];
#pragma unroll
    for (int j2 = 0; j2 < 32; ++j2) uu[j2] = (uint32_t)(d[lane + 32 * j2] + 2048);
    tm_forward_fields<FMA && SHE_TM_FMA_FWD>(uu, 2048.0, lane, tw, scratch, row_base + s * 64);
  }
  const double2* bk_s = bkt + ((size_t)c * 16 + 4 * s) * 16 * 32 + lane;
  TmRing<kTmPrefetch> ring;
  if (active) tm_bk_prefetch<kTmPrefetch>(bk_s, ring);
  tm_wait_st();
  tm_quarter_sync(Q);
  if (active) tm_pointwise<kTmPrefetch, 1>(bk_s, ring, row_base, s);
  tm_wait_st();
  tm_quarter_sync(Q);
  if (active)
    tm_inverse_acc<true, FMA && SHE_TM_FMA_INV>(row_base + s * 64, lane, tw, scratch, acc + (s >> 1) * N, (s & 1) ? 0 : 16, worst);
  tm_quarter_sync(Q);
  if (active)
    for (int m = qt; m < 2 * N; m += 128) out[(size_t)c * 2 * N + m] = acc[m];
  tm_free_all(tmem, warp);
}
