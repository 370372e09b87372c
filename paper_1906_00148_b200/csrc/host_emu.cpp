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

template <class S>
void blind_rotate(const br::Geometry& g, const uint64_t* bk_ntt, const uint32_t* ct,
                  uint32_t* acc) {
  constexpr int L = S::L, N = S::N;
  static Emu<S> E;
  const int rows = 2 * g.l;
  std::vector<uint64_t> buf((size_t)4 * L * (L + 1));
  std::vector<uint64_t> regs((size_t)4 * L * L);
  const uint32_t bbar = br::modswitch(ct[g.n], g.lg2N);
  for (uint32_t m = 0; m < (uint32_t)N; ++m) {
    acc[m] = 0;
    acc[N + m] = br::testvec_coeff(m, bbar, N);
  }
  for (uint32_t i = 0; i < g.n; ++i) {
    const uint32_t a = br::modswitch(ct[i], g.lg2N);
    if (a == 0) continue;  // R9: digits of X^0 ACC - ACC = 0 are all 0
    for (int w = 0; w < rows; ++w)
      for (int lane = 0; lane < L; ++lane) {
        uint64_t x[L];
        br::load_digits<S>(g, w, lane, acc, a, x);
        br::fwd_pass1_store<S>(lane, x, br::buf_row<S>(buf.data(), w));
      }
    for (int w = 0; w < rows; ++w) {
      for (int lane = 0; lane < L; ++lane) {
        uint64_t y[L];
        br::fwd_pass2_load<S>(lane, br::buf_row<S>(buf.data(), w), E.tw.data(), y);
        memcpy(&regs[(w * L + lane) * L], y, sizeof(y));
      }
      for (int lane = 0; lane < L; ++lane) {
        uint64_t y[L];
        memcpy(y, &regs[(w * L + lane) * L], sizeof(y));
        br::fwd_pass2_store<S>(lane, y, br::buf_row<S>(buf.data(), w));
      }
    }
    const uint64_t* bki = bk_ntt + (size_t)i * rows * 2 * N;
    for (int t = 0; t < 128; ++t) br::pointwise<S>(t, 128, rows, buf.data(), bki);
    for (int w = 0; w < 2; ++w) {
      for (int lane = 0; lane < L; ++lane) {
        uint64_t y[L];
        br::inv_pass2_load<S>(lane, br::buf_row<S>(buf.data(), w), y);
        memcpy(&regs[(w * L + lane) * L], y, sizeof(y));
      }
      for (int lane = 0; lane < L; ++lane) {
        uint64_t y[L];
        memcpy(y, &regs[(w * L + lane) * L], sizeof(y));
        br::inv_pass2_store<S>(lane, y, E.itw.data(), br::buf_row<S>(buf.data(), w));
      }
      for (int lane = 0; lane < L; ++lane)
        br::inv_pass1_acc<S>(lane, br::buf_row<S>(buf.data(), w), acc + w * N);
    }
  }
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

// out = d * b in Z_{2^32}[X]/(X^N+1) through the device NTT path.
int she_emu_negacyclic_mul(uint32_t N, const int32_t* d, const uint32_t* b, uint32_t* out) {
  auto run = [&](auto shape) {
    using S = decltype(shape);
    constexpr int L = S::L, NN = S::N;
    static Emu<S> E;
    std::vector<uint64_t> bki((size_t)4 * 2 * NN, 0);  // rows x 2 outputs; only [0][0] used
    E.bk_transform(b, bki.data());
    std::vector<uint64_t> buf((size_t)4 * L * (L + 1), 0);
    uint64_t* row = buf.data();
    for (int lane = 0; lane < L; ++lane) {
      uint64_t x[L];
      for (int j2 = 0; j2 < L; ++j2) x[j2] = gl::from_i64(d[lane + L * j2]);
      br::fwd_pass1_store<S>(lane, x, row);
    }
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
    for (int t = 0; t < 128; ++t) br::pointwise<S>(t, 128, 1, buf.data(), bki.data());
    for (int lane = 0; lane < L; ++lane) {
      uint64_t y[L];
      br::inv_pass2_load<S>(lane, row, y);
      memcpy(&regs[lane * L], y, sizeof(y));
    }
    for (int lane = 0; lane < L; ++lane) {
      uint64_t y[L];
      memcpy(y, &regs[lane * L], sizeof(y));
      br::inv_pass2_store<S>(lane, y, E.itw.data(), row);
    }
    memset(out, 0, sizeof(uint32_t) * NN);
    for (int lane = 0; lane < L; ++lane) br::inv_pass1_acc<S>(lane, row, out);
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
}
