// client.cpp — client side of SHE's threat model (§1-2):
// key generation, bit-wise encryption and decryption, on the
// host.  The server (engine.cu) never sees the secret key.
//
// Randomness comes from the shared seeded generator she_inputs/she_rng.h
// (masks, Gaussian noise, key bits); the arithmetic here is this library's
// own (the oracle has an independent implementation;
// tests/test_client_and_emu.py checks the two produce identical key and
// ciphertext bytes).
#include <omp.h>
#include <stdint.h>
#include <string.h>

#include <new>
#include <vector>

#include "../../she_inputs/she_rng.h"
#include "common.h"

#include "keys.h"

namespace she {

static thread_local std::string g_err;

void set_error(const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_err = buf;
}

static constexpr uint32_t kMu = 1u << 29;  // 1/8 (R4)

// B += X^j * A in Z_2^32[X]/(X^N+1)  (monomial rotate-and-add).
static void add_rotated(uint32_t N, uint32_t j, const uint32_t* A, uint32_t* B) {
  for (uint32_t m = 0; m < N - j; ++m) B[m + j] += A[m];
  for (uint32_t m = N - j; m < N; ++m) B[m + j - N] -= A[m];
}

}  // namespace she

using namespace she;

extern "C" {

const char* she_last_error(void) { return g_err.c_str(); }

size_t she_lwe_stride(const she_params* p) { return p ? lwe_stride(*p) : 0; }

she_status she_keygen(const she_params* p, uint64_t seed, she_secret_key** sk_out,
                      she_cloud_key** ck_out) {
  she_status st = check_params(p);
  if (st != SHE_OK) return st;
  if (!sk_out || !ck_out) return fail(SHE_ERR_ARG, "NULL output pointer");
  she_secret_key* sk = new (std::nothrow) she_secret_key;
  she_cloud_key* ck = new (std::nothrow) she_cloud_key;
  if (!sk || !ck) {
    delete sk;
    delete ck;
    return fail(SHE_ERR_OOM, "host allocation failed");
  }
  const uint32_t N = p->N, n = p->n, l = p->l, t = p->ks_t, base = 1u << p->ks_base_bits;
  sk->p = *p;
  ck->p = *p;
  try {
    sk->s.resize(n);
    sk->S.resize(N);
    ck->bk.assign((size_t)n * 2 * l * 2 * N, 0);
    ck->ksk.assign((size_t)N * t * base * (n + 1), 0);
  } catch (...) {
    delete sk;
    delete ck;
    return fail(SHE_ERR_OOM, "host allocation failed");
  }
  for (uint32_t i = 0; i < n; ++i) sk->s[i] = (uint8_t)she_rng_bit(seed, SHE_STREAM_LWE_KEY, i);
  for (uint32_t j = 0; j < N; ++j) sk->S[j] = (uint8_t)she_rng_bit(seed, SHE_STREAM_TRLWE_KEY, j);
  std::vector<uint32_t> ones;
  for (uint32_t j = 0; j < N; ++j)
    if (sk->S[j]) ones.push_back(j);

  // BK_i = TRGSW_S(s_i): rows r = c*l + j are TRLWE_S(0) + s_i g_j e_c (R1, R2).
#pragma omp parallel for schedule(dynamic)
  for (int64_t ir = 0; ir < (int64_t)n * 2 * l; ++ir) {
    const uint32_t i = (uint32_t)(ir / (2 * l)), r = (uint32_t)(ir % (2 * l));
    uint32_t* A = &ck->bk[((size_t)ir * 2 + 0) * N];
    uint32_t* B = &ck->bk[((size_t)ir * 2 + 1) * N];
    for (uint32_t m = 0; m < N; ++m) {
      A[m] = she_rng_u32(seed, SHE_STREAM_BK_MASK, she_idx_bk(N, l, i, r, m));
      B[m] = she_rng_gauss32(seed, SHE_STREAM_BK_NOISE, she_idx_bk(N, l, i, r, m), p->alpha_bk);
    }
    for (uint32_t j : ones) add_rotated(N, j, A, B);  // B = A*S + e
    if (sk->s[i]) {
      const uint32_t c = r / l, j = r % l;
      (c == 0 ? A : B)[0] += 1u << (32 - (j + 1) * p->bg_bits);
    }
  }

  // KSK[i][j][v] = LWE_s(v S_i 2^{32-(j+1) basebits}), v >= 1 (R3).
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < (int64_t)N; ++i) {
    for (uint32_t j = 0; j < t; ++j)
      for (uint32_t v = 1; v < base; ++v) {
        const uint64_t e = she_idx_ksk_entry(t, base, (uint32_t)i, j, v);
        uint32_t* row = &ck->ksk[e * (n + 1)];
        uint32_t b = she_rng_gauss32(seed, SHE_STREAM_KSK_NOISE, e, p->alpha_lwe);
        if (sk->S[i]) b += v << (32 - (j + 1) * p->ks_base_bits);
        for (uint32_t k = 0; k < n; ++k) {
          row[k] = she_rng_u32(seed, SHE_STREAM_KSK_MASK, she_idx_ksk_mask(n, e, k));
          if (sk->s[k]) b += row[k];
        }
        row[n] = b;
      }
  }
  *sk_out = sk;
  *ck_out = ck;
  return SHE_OK;
}

void she_secret_key_free(she_secret_key* sk) { delete sk; }
void she_cloud_key_free(she_cloud_key* ck) { delete ck; }

she_status she_secret_key_export(const she_secret_key* sk, void* buf, size_t* len) {
  if (!sk || !len) return fail(SHE_ERR_ARG, "NULL argument");
  const size_t need = sk->s.size() + sk->S.size();
  if (!buf) {
    *len = need;
    return SHE_OK;
  }
  if (*len < need) return fail(SHE_ERR_ARG, "buffer too small (%zu < %zu)", *len, need);
  memcpy(buf, sk->s.data(), sk->s.size());
  memcpy((uint8_t*)buf + sk->s.size(), sk->S.data(), sk->S.size());
  *len = need;
  return SHE_OK;
}

she_status she_cloud_key_export(const she_cloud_key* ck, void* buf, size_t* len) {
  if (!ck || !len) return fail(SHE_ERR_ARG, "NULL argument");
  const size_t nb = ck->bk.size() * 4, nk = ck->ksk.size() * 4;
  if (!buf) {
    *len = nb + nk;
    return SHE_OK;
  }
  if (*len < nb + nk) return fail(SHE_ERR_ARG, "buffer too small");
  memcpy(buf, ck->bk.data(), nb);
  memcpy((uint8_t*)buf + nb, ck->ksk.data(), nk);
  *len = nb + nk;
  return SHE_OK;
}

she_status she_cloud_key_import(const she_params* p, const void* buf, size_t len,
                                she_cloud_key** ck_out) {
  she_status st = check_params(p);
  if (st != SHE_OK) return st;
  if (!buf || !ck_out) return fail(SHE_ERR_ARG, "NULL argument");
  const size_t nb = (size_t)p->n * 2 * p->l * 2 * p->N;
  const size_t nk = (size_t)p->N * p->ks_t * (1u << p->ks_base_bits) * (p->n + 1);
  if (len != (nb + nk) * 4) return fail(SHE_ERR_SHAPE, "cloud key length %zu != %zu", len, (nb + nk) * 4);
  she_cloud_key* ck = new (std::nothrow) she_cloud_key;
  if (!ck) return fail(SHE_ERR_OOM, "host allocation failed");
  ck->p = *p;
  ck->bk.assign((const uint32_t*)buf, (const uint32_t*)buf + nb);
  ck->ksk.assign((const uint32_t*)buf + nb, (const uint32_t*)buf + nb + nk);
  *ck_out = ck;
  return SHE_OK;
}

she_status she_encrypt_bits(const she_secret_key* sk, const uint8_t* bits, size_t count,
                            uint64_t seed, uint64_t first_index, uint32_t* out) {
  if (count == 0) return SHE_OK;
  if (!sk || !bits || !out) return fail(SHE_ERR_ARG, "NULL argument");
  const uint32_t n = sk->p.n;
  const size_t stride = lwe_stride(sk->p);
#pragma omp parallel for schedule(static) if (count > 64)
  for (int64_t c = 0; c < (int64_t)count; ++c) {
    const uint64_t q = first_index + (uint64_t)c;
    uint32_t* ct = out + (size_t)c * stride;
    uint32_t b = (bits[c] ? kMu : 0u - kMu) +
                 she_rng_gauss32(seed, SHE_STREAM_ENC_NOISE, q, sk->p.alpha_lwe);
    for (uint32_t k = 0; k < n; ++k) {
      ct[k] = she_rng_u32(seed, SHE_STREAM_ENC_MASK, she_idx_enc_mask(n, q, k));
      if (sk->s[k]) b += ct[k];
    }
    ct[n] = b;
    for (size_t k = n + 1; k < stride; ++k) ct[k] = 0;
  }
  return SHE_OK;
}

she_status she_encrypt_noise(const she_secret_key* sk, size_t count, uint64_t seed,
                             uint64_t first_index, uint32_t* noise) {
  if (count == 0) return SHE_OK;
  if (!sk || !noise) return fail(SHE_ERR_ARG, "NULL argument");
#pragma omp parallel for schedule(static) if (count > 256)
  for (int64_t c = 0; c < (int64_t)count; ++c)
    noise[c] = she_rng_gauss32(seed, SHE_STREAM_ENC_NOISE, first_index + (uint64_t)c,
                               sk->p.alpha_lwe);
  return SHE_OK;
}

she_status she_decrypt_bits(const she_secret_key* sk, const uint32_t* in, size_t count,
                            uint8_t* bits) {
  if (count == 0) return SHE_OK;
  if (!sk || !in || !bits) return fail(SHE_ERR_ARG, "NULL argument");
  const uint32_t n = sk->p.n;
  const size_t stride = lwe_stride(sk->p);
  for (size_t c = 0; c < count; ++c) {
    const uint32_t* ct = in + c * stride;
    uint32_t phase = ct[n];
    for (uint32_t k = 0; k < n; ++k)
      if (sk->s[k]) phase -= ct[k];
    bits[c] = (int32_t)phase >= 0 ? 1 : 0;  // R5
  }
  return SHE_OK;
}

// ---- leveled mode, client side (NEXT-2; reading R-LV) ----------
// Selector number first + idx = TRGSW_S(bit) in the BK row layout: row r =
// c*l + j is TRLWE_S(0) (A from stream 9, B = A*S + e with e from stream 10,
// alpha_bk) plus bit * g_j on component c's constant coefficient (R1, R2).
// out: count x [2l][2][N] (host).
she_status she_lvl_encrypt_selectors(const she_secret_key* sk, const uint8_t* bits, size_t count,
                                     uint64_t seed, uint64_t first_index, uint32_t* out) {
  if (count == 0) return SHE_OK;
  if (!sk || !bits || !out) return fail(SHE_ERR_ARG, "NULL argument");
  const she_params& p = sk->p;
  const uint32_t N = p.N, l = p.l;
  std::vector<uint32_t> ones;
  for (uint32_t j = 0; j < N; ++j)
    if (sk->S[j]) ones.push_back(j);
#pragma omp parallel for schedule(dynamic)
  for (int64_t qr = 0; qr < (int64_t)count * 2 * l; ++qr) {
    const size_t idx = (size_t)(qr / (2 * l));
    const uint32_t q = (uint32_t)(first_index + idx), r = (uint32_t)(qr % (2 * l));
    uint32_t* A = out + ((size_t)qr * 2 + 0) * N;
    uint32_t* B = out + ((size_t)qr * 2 + 1) * N;
    for (uint32_t m = 0; m < N; ++m) {
      A[m] = she_rng_u32(seed, SHE_STREAM_LVL_MASK, she_idx_bk(N, l, q, r, m));
      B[m] = she_rng_gauss32(seed, SHE_STREAM_LVL_NOISE, she_idx_bk(N, l, q, r, m), p.alpha_bk);
    }
    for (uint32_t j : ones) add_rotated(N, j, A, B);  // B = A*S + e
    if (bits[idx]) {
      const uint32_t c = r / l, j = r % l;
      (c == 0 ? A : B)[0] += 1u << (32 - (j + 1) * p.bg_bits);
    }
  }
  return SHE_OK;
}

// Bit of leveled data (TRLWE [2][N], host): R5 on the constant coefficient of
// the phase B - A*S, i.e. B_0 - A_0 S_0 + sum_{m>=1} A_m S_{N-m}.
she_status she_lvl_decrypt(const she_secret_key* sk, const uint32_t* in, size_t count,
                           uint8_t* bits) {
  if (count == 0) return SHE_OK;
  if (!sk || !in || !bits) return fail(SHE_ERR_ARG, "NULL argument");
  const uint32_t N = sk->p.N;
  for (size_t c = 0; c < count; ++c) {
    const uint32_t* A = in + c * 2 * N;
    uint32_t ph = A[N] - (sk->S[0] ? A[0] : 0u);
    for (uint32_t m = 1; m < N; ++m)
      if (sk->S[N - m]) ph += A[m];
    bits[c] = (int32_t)ph >= 0 ? 1 : 0;
  }
  return SHE_OK;
}

// Wire format of a ciphertext batch (NEXT-4; the paper's MSize column,
// PAPER.md:232, :256): 16-byte header {magic "SHEC", n, count (u64)} then
// count x (n + 1) little-endian uint32 words (a[0..n-1], b) — the slot padding
// is not sent.
static const uint32_t kSerMagic = 0x43454853u;  // "SHEC"

size_t she_serialized_bytes(const she_params* p, size_t count) {
  return p ? 16 + count * (size_t)(p->n + 1) * 4 : 0;
}

she_status she_serialize_ciphertexts(const she_params* p, const uint32_t* in, size_t count,
                                     void* buf, size_t* len) {
  if (!p || !len) return fail(SHE_ERR_ARG, "NULL argument");
  const size_t need = she_serialized_bytes(p, count);
  if (!buf) {
    *len = need;
    return SHE_OK;
  }
  if (*len < need) return fail(SHE_ERR_ARG, "buffer of %zu bytes, need %zu", *len, need);
  if (count && !in) return fail(SHE_ERR_ARG, "NULL input");
  uint8_t* o = (uint8_t*)buf;
  const uint32_t hdr[2] = {kSerMagic, p->n};
  const uint64_t cnt = count;
  memcpy(o, hdr, 8);
  memcpy(o + 8, &cnt, 8);
  const size_t stride = lwe_stride(*p), words = p->n + 1;
  for (size_t c = 0; c < count; ++c) memcpy(o + 16 + c * words * 4, in + c * stride, words * 4);
  *len = need;
  return SHE_OK;
}

she_status she_deserialize_ciphertexts(const she_params* p, const void* buf, size_t len,
                                       uint32_t* out, size_t cap, size_t* count) {
  if (!p || !buf || !count) return fail(SHE_ERR_ARG, "NULL argument");
  if (len < 16) return fail(SHE_ERR_SHAPE, "truncated header");
  const uint8_t* b = (const uint8_t*)buf;
  uint32_t hdr[2];
  uint64_t cnt;
  memcpy(hdr, b, 8);
  memcpy(&cnt, b + 8, 8);
  if (hdr[0] != kSerMagic) return fail(SHE_ERR_SHAPE, "not a ciphertext batch");
  if (hdr[1] != p->n) return fail(SHE_ERR_PARAMS, "batch made for n = %u, params n = %u", hdr[1], p->n);
  if (len != she_serialized_bytes(p, cnt)) return fail(SHE_ERR_SHAPE, "length does not match count");
  *count = cnt;
  if (!out) return SHE_OK;
  if (cap < cnt) return fail(SHE_ERR_ARG, "capacity %zu < %llu", cap, (unsigned long long)cnt);
  const size_t stride = lwe_stride(*p), words = p->n + 1;
  for (size_t c = 0; c < cnt; ++c) {
    memcpy(out + c * stride, b + 16 + c * words * 4, words * 4);
    memset(out + c * stride + words, 0, (stride - words) * 4);
  }
  return SHE_OK;
}

}  // extern "C"
