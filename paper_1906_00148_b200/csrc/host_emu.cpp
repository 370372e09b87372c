// host_emu.cpp — CPU emulation of the device blind-rotation arithmetic, for
// tests only (tests/test_ntt_host.py).  It runs the SAME __host__ __device__
// step functions as the sm_100a kernel (bootstrap_core.cuh), one emulated
// thread at a time, phase by phase, so that the NTT ordering, twiddles, twist
// tables, decomposition and lift are checked against the oracle on a machine
// without a GPU.  It is not part of the product path: the Python binding never
// routes a product call here.
#include <stdint.h>
#include <string.h>

#include <vector>

#include "bootstrap_core.cuh"
#include "tm_queue.h"

namespace {

template <class S>
struct Emu {
  static constexpr int L = S::L, N = S::N;
  std::vector<uint64_t> tw, itw;
  uint64_t ninv;
  Emu() : tw(L * L), itw(L * L) {
    ntt::make_twists(N, L, S::SH, tw.data(), itw.data());
    ninv = gl::pow(N, gl::P - 2);
  }
  // Forward transform of a torus32 polynomial (signed lift) with N^-1 folded.
  void bk_transform(const uint32_t* poly, uint64_t* out) {
    std::vector<uint64_t> row(L * (L + 1));
    for (int lane = 0; lane < L; ++lane) {
      uint64_t x[L];
      br::load_poly_signed<S>(lane, poly, x);
      br::fwd_pass1_store<S>(lane, x, row.data());
    }
    for (int i = 0; i < L; ++i) {
      uint64_t y[L];
      br::fwd_pass2_load<S>(i, row.data(), tw.data(), y);
      br::fwd_pass2_store_scaled<S>(i, y, ninv, out);
    }
  }
};

// The inverse of output component c by the warp pair (2c, 2c+1), phase by
// phase (the device separates the phases with named barriers).
template <class S>
void inverse_component(Emu<S>& E, br::Lane<S>& ln, int c, uint32_t* accc) {
  constexpr int L = S::L;
  uint64_t* row = ln.row(c);
  uint64_t* xb = ln.row(2 + c);
  std::vector<uint64_t> y(2 * L * (L / 2)), lo(2 * L * (L / 4)), hi(2 * L * (L / 4));
  auto Y = [&](int H, int t) { return reinterpret_cast<uint64_t(*)[L / 2]>(&y[(H * L + t) * (L / 2)]); };
  auto LO = [&](int H, int t) { return reinterpret_cast<uint64_t(*)[L / 4]>(&lo[(H * L + t) * (L / 4)]); };
  auto HI = [&](int H, int t) { return reinterpret_cast<uint64_t(*)[L / 4]>(&hi[(H * L + t) * (L / 4)]); };
  // pass A (cyclic inverse over rows)
  for (int t = 0; t < L; ++t) {
    br::inv_a_load<S, 0>(t, row, *Y(0, t));
    br::inv_a_load<S, 1>(t, row, *Y(1, t));
  }
  for (int t = 0; t < L; ++t) {
    br::inv_stages_send<S, 0, false>(t, *Y(0, t), xb);
    br::inv_stages_send<S, 1, false>(t, *Y(1, t), xb);
  }
  for (int t = 0; t < L; ++t) {
    br::inv_recv_cross<S, 0, false>(t, *Y(0, t), xb, *LO(0, t), *HI(0, t));
    br::inv_recv_cross<S, 1, false>(t, *Y(1, t), xb, *LO(1, t), *HI(1, t));
  }
  for (int t = 0; t < L; ++t) {
    br::inv_a_store<S, 0>(t, *LO(0, t), *HI(0, t), E.itw.data(), row);
    br::inv_a_store<S, 1>(t, *LO(1, t), *HI(1, t), E.itw.data(), row);
  }
  // pass B (negacyclic inverse over columns)
  for (int t = 0; t < L; ++t) {
    br::inv_b_load<S, 0>(t, row, *Y(0, t));
    br::inv_b_load<S, 1>(t, row, *Y(1, t));
  }
  for (int t = 0; t < L; ++t) {
    br::inv_stages_send<S, 0, true>(t, *Y(0, t), xb);
    br::inv_stages_send<S, 1, true>(t, *Y(1, t), xb);
  }
  for (int t = 0; t < L; ++t) {
    br::inv_recv_cross<S, 0, true>(t, *Y(0, t), xb, *LO(0, t), *HI(0, t));
    br::inv_recv_cross<S, 1, true>(t, *Y(1, t), xb, *LO(1, t), *HI(1, t));
  }
  for (int t = 0; t < L; ++t) {
    br::inv_b_acc<S, 0>(t, *LO(0, t), *HI(0, t), accc);
    br::inv_b_acc<S, 1>(t, *LO(1, t), *HI(1, t), accc);
  }
}

template <class S>
void pass2_row(Emu<S>& E, uint64_t* row);

template <class S>
void forward_row(Emu<S>& E, br::Lane<S>& ln, int w, const uint64_t (*xs)[S::L]) {
  constexpr int L = S::L;
  uint64_t* row = ln.row(w);
  for (int lane = 0; lane < L; ++lane) {
    uint64_t x[L];
    memcpy(x, xs[lane], sizeof(x));
    br::fwd_pass1_store<S>(lane, x, row);
  }
  pass2_row<S>(E, row);
}

// Pass 2 of a row: every thread loads (with the twist) before any stores.
template <class S>
void pass2_row(Emu<S>& E, uint64_t* row) {
  constexpr int L = S::L;
  std::vector<uint64_t> regs((size_t)L * L);
  for (int lane = 0; lane < L; ++lane) {
    uint64_t y[L];
    br::fwd_pass2_load<S>(lane, row, E.tw.data(), y);
    memcpy(&regs[lane * L], y, sizeof(y));
  }
  for (int lane = 0; lane < L; ++lane) {
    uint64_t y[L];
    memcpy(y, &regs[lane * L], sizeof(y));
    br::fwd_pass2_store<S>(lane, y, row);
  }
}

template <class S>
void blind_rotate(const br::Geometry& g, const uint64_t* bk_ntt, const uint32_t* ct,
                  uint32_t* acc_out) {
  constexpr int L = S::L, N = S::N;
  static Emu<S> E;
  std::vector<uint8_t> smem(br::Lane<S>::bytes(g.n) + 64, 0);
  br::Lane<S> ln(smem.data());
  for (uint32_t k = 0; k <= g.n; ++k) ln.abar[k] = (uint16_t)br::modswitch(ct[k], g.lg2N);
  const uint32_t bbar = ln.abar[g.n];
  for (uint32_t m = 0; m < (uint32_t)N; ++m) {
    ln.acc[m] = 0;
    ln.acc[N + m] = br::testvec_coeff(m, bbar, N);
  }
  std::vector<uint64_t> xs((size_t)L * L);
  for (uint32_t i = 0; i < g.n; ++i) {
    const uint32_t a = ln.abar[i];  // no skip: the device runs a = 0 as well
    for (int w = 0; w < 4; ++w) {
      uint64_t* row = ln.row(w);
      for (int lane = 0; lane < L; ++lane) {  // digits + exact stage 0, as on the device
        int32_t d[L];
        br::load_digits<S>(g, w, lane, ln.acc, a, d);
        br::fwd_pass1_digits_store<S>(lane, d, row);
      }
      pass2_row<S>(E, row);
    }
    const uint64_t* bki = bk_ntt + (size_t)i * 8 * N;
    for (int p = 0; p < N; ++p) {
      uint64_t b[8];
      for (int q = 0; q < 8; ++q) b[q] = bki[(size_t)q * N + p];
      br::pointwise_pos<S>(ln.buf, p, b);
    }
    for (int c = 0; c < 2; ++c) inverse_component<S>(E, ln, c, ln.acc + c * N);
  }
  memcpy(acc_out, ln.acc, sizeof(uint32_t) * 2 * N);
}

br::Geometry geometry(uint32_t N, uint32_t n, uint32_t l, uint32_t bg_bits) {
  br::Geometry g;
  g.N = N;
  g.n = n;
  g.l = l;
  g.bg_bits = bg_bits;
  g.lg2N = 0;
  while ((1u << g.lg2N) < 2 * N) g.lg2N++;
  uint32_t off = 0;
  for (uint32_t j = 1; j <= l; ++j) off += (1u << (bg_bits - 1)) << (32 - j * bg_bits);
  off += 1u << (32 - l * bg_bits - 1);
  g.dec_offset = off;
  return g;
}

}  // namespace

extern "C" {

// out = d * b in Z_{2^32}[X]/(X^N+1) through the device NTT path (row 0 of
// the pointwise with BK row [0][0] = NTT(b), all other rows and outputs 0).
int she_emu_negacyclic_mul(uint32_t N, const int32_t* d, const uint32_t* b, uint32_t* out) {
  auto run = [&](auto shape) {
    using S = decltype(shape);
    constexpr int L = S::L, NN = S::N;
    static Emu<S> E;
    std::vector<uint64_t> bki((size_t)8 * NN, 0);
    E.bk_transform(b, bki.data());
    std::vector<uint8_t> smem(br::Lane<S>::bytes(0) + 64, 0);
    br::Lane<S> ln(smem.data());
    std::vector<uint64_t> xs((size_t)L * L);
    for (int lane = 0; lane < L; ++lane)
      for (int j2 = 0; j2 < L; ++j2) xs[lane * L + j2] = gl::from_i64(d[lane + L * j2]);
    forward_row<S>(E, ln, 0, reinterpret_cast<const uint64_t(*)[L]>(xs.data()));
    for (int p = 0; p < NN; ++p) {
      uint64_t bb[8];
      for (int q = 0; q < 8; ++q) bb[q] = bki[(size_t)q * NN + p];
      br::pointwise_pos<S>(ln.buf, p, bb);
    }
    memset(out, 0, sizeof(uint32_t) * NN);
    inverse_component<S>(E, ln, 0, out);
    return 0;
  };
  if (N == 1024) return run(ntt::Shape<1024>{});
  if (N == 256) return run(ntt::Shape<256>{});
  return -1;
}

// Blind rotation of one LWE sample with the device arithmetic; bk is the
// coefficient-domain key uint32[n][2l][2][N] (transformed here like K1).
int she_emu_blind_rotate(uint32_t N, uint32_t n, uint32_t l, uint32_t bg_bits, const uint32_t* bk,
                         const uint32_t* ct, uint32_t* acc) {
  if (l != 2) return -1;
  br::Geometry g = geometry(N, n, l, bg_bits);
  auto run = [&](auto shape) {
    using S = decltype(shape);
    static Emu<S> E;
    const size_t polys = (size_t)n * 2 * l * 2;
    std::vector<uint64_t> bk_ntt(polys * S::N);
    for (size_t q = 0; q < polys; ++q) E.bk_transform(bk + q * S::N, bk_ntt.data() + q * S::N);
    blind_rotate<S>(g, bk_ntt.data(), ct, acc);
    return 0;
  };
  if (N == 1024) return run(ntt::Shape<1024>{});
  if (N == 256) return run(ntt::Shape<256>{});
  return -1;
}

// Goldilocks helpers exposed for unit tests.
uint64_t she_emu_gl_mul(uint64_t a, uint64_t b) { return gl::canon(gl::mul(a, b)); }
uint64_t she_emu_gl_mul_pow2(uint64_t a, int s) { return gl::canon(gl::mul_pow2(a, s)); }
uint64_t she_emu_gl_add(uint64_t a, uint64_t b) { return gl::canon(gl::add(a, b)); }
uint64_t she_emu_gl_sub(uint64_t a, uint64_t b) { return gl::canon(gl::sub(a, b)); }
// Bounded-product butterfly primitives: raw (non-canonical) results, so the
// tests can check the <= p bound as well as the residue.
uint64_t she_emu_gl_shl_le(uint64_t v, int s) { return gl::shl_le(v, s); }
uint64_t she_emu_gl_add_le(uint64_t a, uint64_t b) { return gl::add_le(a, b); }
uint64_t she_emu_gl_sub_le(uint64_t a, uint64_t b) { return gl::sub_le(a, b); }
uint32_t she_emu_gl_lift32_neg(uint64_t t) { return gl::lift32_neg(t); }

// The TMEM engine's work distribution (tm_queue.h, the kernel's own
// functions): the schedule of one launch written out as rows (base, nsl, i0,
// i1, slot, pipeline).  Queue modes: every unit u < units in order (pipeline =
// 0); static mode: per pipeline gq the units it runs, in order.  Returns the
// number of rows; *mode = tmq::Mode.
uint32_t she_emu_tm_schedule(uint32_t total, uint32_t n, uint32_t chunk, uint32_t pipelines, uint32_t cap,
                             uint32_t* out, int* mode) {
  uint32_t rows = 0;
  const int m = tmq::mode(total, n, chunk, pipelines);
  *mode = m;
  if (m != tmq::kStatic) {
    const uint32_t nu = tmq::units(total, n, chunk, m);
    for (uint32_t u = 0; u < nu && rows < cap; ++u, ++rows) {
      const tmq::Unit w = tmq::unit(u, total, n, chunk, m);
      const uint32_t r[6] = {w.base, w.nsl, w.i0, w.i1, w.slot, 0};
      memcpy(out + 6 * rows, r, sizeof r);
      if (w.slot >= tmq::slots(total, pipelines)) return 0xFFFFFFFFu;
    }
    // one past the end must be "no more work"
    if (tmq::unit(nu, total, n, chunk, m).nsl != 0) return 0xFFFFFFFFu;
    return rows;
  }
  for (uint32_t gq = 0; gq < pipelines; ++gq) {
    uint32_t cursor = tmq::first(gq, total, pipelines);
    for (;;) {
      const tmq::Unit w = tmq::next_static(cursor, gq, total, pipelines, n);
      if (w.nsl == 0 || rows >= cap) break;
      const uint32_t r[6] = {w.base, w.nsl, w.i0, w.i1, 0, gq};
      memcpy(out + 6 * rows, r, sizeof r);
      ++rows;
      cursor = w.base + w.nsl;
    }
  }
  return rows;
}

// The wrap-around schedule (tmq::wrap_unit): per pipeline gq its units in
// execution order as rows (base, nsl, i0, i1, slot, pipeline).  Returns the
// number of rows, or 0xFFFFFFFF if the mode is static; *mode = tmq::Mode.
uint32_t she_emu_tm_wrap_schedule(uint32_t total, uint32_t n, uint32_t pipelines, uint32_t cap, uint32_t* out,
                                  int* mode) {
  const int m = tmq::mode(total, n, 1, pipelines);
  *mode = m;
  if (m == tmq::kStatic) return 0xFFFFFFFFu;
  uint32_t rows = 0;
  for (uint32_t gq = 0; gq < pipelines; ++gq)
    for (uint32_t step = 0;; ++step) {
      const tmq::Unit w = tmq::wrap_unit(gq, step, total, n, pipelines, m);
      if (w.nsl == 0 || rows >= cap) break;
      if (w.slot >= tmq::slots(total, pipelines)) return 0xFFFFFFFEu;
      const uint32_t r[6] = {w.base, w.nsl, w.i0, w.i1, w.slot, gq};
      memcpy(out + 6 * rows, r, sizeof r);
      ++rows;
    }
  return rows;
}
}
