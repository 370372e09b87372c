/*
 * oracle.c — plain, slow, obviously-correct CPU TFHE gate bootstrapping.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.  The
 * product path (paper_1906_00148_b200/) never imports, links or calls it, and
 * it shares no code with the product: the only common file is the seeded
 * input generator she_inputs/she_rng.h, which holds none of the method's
 * arithmetic.
 *
 * What it follows (PAPER.md line, section):
 *   - bit-wise encryption of plaintext words      PAPER.md:142 (§3.2)
 *   - 2-input homomorphic Boolean gates            PAPER.md:110 (§3.1)
 *   - bootstrapping refreshes noise                PAPER.md:31  (§2)
 *   - TFHE TLWE / TRLWE / TRGSW, key switching     PAPER.md:35, :188 (§2, §4)
 * The TFHE internals are not in the paper; the conventions are the readings
 * R1-R10 of SURVEY.md §8(c), restated in DESIGN.md §2, each marked below.
 *
 * Arithmetic: the torus T = R/Z is represented by uint32 (x / 2^32); every
 * operation is mod 2^32 (C unsigned wrap-around).  Polynomial products are
 * SCHOOLBOOK negacyclic products in Z_{2^32}[X]/(X^N+1): no NTT, no FFT, no
 * blocking.  One function per step of the algorithm, in the paper's order.
 *
 * Parity pins (tests/test_oracle_pins.py, -m "not gpu"): truth tables by
 * brute force, trivial-input closed form, decomposition error bound,
 * negacyclic product vs. brute-force polynomial arithmetic, noise variance vs.
 * the closed-form TFHE prediction, keygen/encryption consistency.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#include "../she_inputs/she_rng.h"

typedef struct {
  uint32_t N, k, n, bg_bits, l, ks_base_bits, ks_t;
  double alpha_lwe, alpha_bk;
} orc_params;

/* gate codes (the C-ABI's she_op values; include/she.h) */
enum { ORC_AND, ORC_NAND, ORC_OR, ORC_NOR, ORC_XOR, ORC_XNOR, ORC_MUX, ORC_NOT, ORC_COPY };

#define MU (1u << 29) /* 1/8 on the torus (R4) */

int orc_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}

/* ------------------------------------------------------------------------ */
/* Polynomial primitives in Z_{2^32}[X]/(X^N + 1)                            */
/* ------------------------------------------------------------------------ */

/* out = d * b (negacyclic), d small signed digits, b torus32 coefficients.
 * Written as the definition: X^i * X^j = X^{i+j} if i+j < N, else -X^{i+j-N}. */
void orc_negacyclic_mul(uint32_t N, const int32_t* restrict d, const uint32_t* restrict b,
                        uint32_t* restrict out) {
  memset(out, 0, sizeof(uint32_t) * N);
  for (size_t i = 0; i < N; i++) {
    uint32_t di = (uint32_t)d[i];
    for (size_t j = 0; j < N - i; j++) out[i + j] += di * b[j];      /* X^{i+j}        */
    for (size_t j = N - i; j < N; j++) out[i + j - N] -= di * b[j];  /* -X^{i+j-N}     */
  }
}

/* out += d * b (negacyclic). */
static void negacyclic_mac(uint32_t N, const int32_t* restrict d, const uint32_t* restrict b,
                           uint32_t* restrict out) {
  for (size_t i = 0; i < N; i++) {
    uint32_t di = (uint32_t)d[i];
    if (di == 0) continue;
    for (size_t j = 0; j < N - i; j++) out[i + j] += di * b[j];
    for (size_t j = N - i; j < N; j++) out[i + j - N] -= di * b[j];
  }
}

/* out = X^a * p, a in [0, 2N): multiply by the monomial (X^N = -1). */
void orc_rotate(uint32_t N, uint32_t a, const uint32_t* p, uint32_t* out) {
  for (uint32_t j = 0; j < N; j++) {
    uint32_t e = (j + a) % (2 * N);
    if (e < N)
      out[e] = p[j];
    else
      out[e - N] = (uint32_t)0 - p[j];
  }
}

/* R8 — signed gadget decomposition of one torus32 coefficient x into l
 * digits in [-Bg/2, Bg/2), digit j (1-based) weighs 2^{32 - j*bg_bits}:
 *   y = x + sum_{j=1..l} (Bg/2) 2^{32-j*bg_bits} + 2^{32-l*bg_bits-1}
 *   digit_j = ((y >> (32 - j*bg_bits)) & (Bg-1)) - Bg/2                    */
void orc_decompose(const orc_params* P, uint32_t x, int32_t* digits /* l */) {
  uint32_t Bg = 1u << P->bg_bits, half = Bg / 2, y = x;
  for (uint32_t j = 1; j <= P->l; j++) y += half << (32 - j * P->bg_bits);
  y += 1u << (32 - P->l * P->bg_bits - 1);
  for (uint32_t j = 1; j <= P->l; j++)
    digits[j - 1] = (int32_t)((y >> (32 - j * P->bg_bits)) & (Bg - 1)) - (int32_t)half;
}

/* R7 — modulus switch of a torus32 value to Z_{2N}, rounding half up. */
uint32_t orc_modswitch(uint32_t N, uint32_t x) {
  uint32_t lg = 0;
  while ((1u << lg) < 2 * N) lg++;
  return (uint32_t)((x + (1u << (31 - lg))) >> (32 - lg));
}

/* ------------------------------------------------------------------------ */
/* Client side: keys, encryption, decryption (PAPER.md:31 epsilon / delta)    */
/* ------------------------------------------------------------------------ */

/* Phase of an LWE sample: b - <a, s>. */
uint32_t orc_phase(uint32_t n, const uint8_t* s, const uint32_t* ct) {
  uint32_t acc = ct[n];
  for (uint32_t i = 0; i < n; i++) acc -= ct[i] * (uint32_t)s[i];
  return acc;
}

/* R1 binary uniform keys.  BK_i = TRGSW_S(s_i): 2l rows r = c*l + j; row r is
 * a TRLWE encryption of 0 (A uniform, B = A*S + e) plus s_i * 2^{32-(j+1)bg}
 * added to component c (R2 row order: A-block rows then B-block rows).
 * KSK[i][j][v] = LWE_s(v * S_i * 2^{32-(j+1)*basebits}), v = 1..base-1, each an
 * independent encryption (R3); v = 0 rows are zero.
 *   bk  : uint32[n][2l][2][N]
 *   ksk : uint32[N][t][base][n+1]                                              */
void orc_keygen(const orc_params* P, uint64_t seed, uint8_t* s, uint8_t* S, uint32_t* bk,
                uint32_t* ksk) {
  const uint32_t N = P->N, n = P->n, l = P->l, t = P->ks_t;
  const uint32_t base = 1u << P->ks_base_bits;
  for (uint32_t i = 0; i < n; i++) s[i] = (uint8_t)she_rng_bit(seed, SHE_STREAM_LWE_KEY, i);
  for (uint32_t j = 0; j < N; j++) S[j] = (uint8_t)she_rng_bit(seed, SHE_STREAM_TRLWE_KEY, j);
  int32_t* Sd = (int32_t*)malloc(sizeof(int32_t) * N);
  for (uint32_t j = 0; j < N; j++) Sd[j] = S[j];

#pragma omp parallel for schedule(dynamic)
  for (uint32_t i = 0; i < n; i++) {
    for (uint32_t r = 0; r < 2 * l; r++) {
      uint32_t* A = bk + ((size_t)(i * 2 * l + r) * 2 + 0) * N;
      uint32_t* B = bk + ((size_t)(i * 2 * l + r) * 2 + 1) * N;
      for (uint32_t m = 0; m < N; m++)
        A[m] = she_rng_u32(seed, SHE_STREAM_BK_MASK, she_idx_bk(N, l, i, r, m));
      orc_negacyclic_mul(N, Sd, A, B); /* B = S * A */
      for (uint32_t m = 0; m < N; m++)
        B[m] += she_rng_gauss32(seed, SHE_STREAM_BK_NOISE, she_idx_bk(N, l, i, r, m), P->alpha_bk);
      uint32_t c = r / l, j = r % l;
      uint32_t g = 1u << (32 - (j + 1) * P->bg_bits);
      if (s[i]) (c == 0 ? A : B)[0] += g; /* + s_i * g_j (constant polynomial) */
    }
  }

#pragma omp parallel for schedule(static)
  for (uint32_t i = 0; i < N; i++) {
    for (uint32_t j = 0; j < t; j++) {
      for (uint32_t v = 0; v < base; v++) {
        uint64_t e = she_idx_ksk_entry(t, base, i, j, v);
        uint32_t* row = ksk + e * (n + 1);
        if (v == 0) {
          memset(row, 0, sizeof(uint32_t) * (n + 1));
          continue;
        }
        uint32_t msg = v * (uint32_t)S[i] * (1u << (32 - (j + 1) * P->ks_base_bits));
        uint32_t b = msg + she_rng_gauss32(seed, SHE_STREAM_KSK_NOISE, e, P->alpha_lwe);
        for (uint32_t k = 0; k < n; k++) {
          row[k] = she_rng_u32(seed, SHE_STREAM_KSK_MASK, she_idx_ksk_mask(n, e, k));
          b += row[k] * (uint32_t)s[k];
        }
        row[n] = b;
      }
    }
  }
  free(Sd);
}

/* R4: bit m -> (a, <a,s> + (m ? +1/8 : -1/8) + e).  out: count * stride words;
 * ciphertext #q = first_index + idx draws mask/noise number q. */
void orc_encrypt(const orc_params* P, const uint8_t* s, const uint8_t* bits, size_t count,
                 uint64_t seed, uint64_t first_index, size_t stride, uint32_t* out) {
  const uint32_t n = P->n;
  for (size_t c = 0; c < count; c++) {
    uint64_t q = first_index + c;
    uint32_t* ct = out + c * stride;
    memset(ct, 0, sizeof(uint32_t) * stride);
    uint32_t b = (bits[c] ? MU : (uint32_t)0 - MU) +
                 she_rng_gauss32(seed, SHE_STREAM_ENC_NOISE, q, P->alpha_lwe);
    for (uint32_t k = 0; k < n; k++) {
      ct[k] = she_rng_u32(seed, SHE_STREAM_ENC_MASK, she_idx_enc_mask(n, q, k));
      b += ct[k] * (uint32_t)s[k];
    }
    ct[n] = b;
  }
}

/* R5: m = [ (int32) phase >= 0 ]. */
void orc_decrypt(const orc_params* P, const uint8_t* s, const uint32_t* in, size_t count,
                 size_t stride, uint8_t* bits) {
  for (size_t c = 0; c < count; c++)
    bits[c] = (int32_t)orc_phase(P->n, s, in + c * stride) >= 0;
}

/* ------------------------------------------------------------------------ */
/* Server side: bootstrapping, gates            */
/* ------------------------------------------------------------------------ */

/* Blind rotation of LWE sample c (n+1 words) into ACC (A then B, 2N words):
 *   b~ = ms(b), a~_i = ms(a_i)                                   (R7)
 *   ACC = (0, X^{-b~} v), v = mu * sum_j X^j                     (test vector)
 *   for i < n: ACC += BK_i [x] (X^{a~_i} ACC - ACC)               (CMux)
 * [x] = external product: sum over rows r = (c, j) of
 *       digit_j(D_c) * BK_i[r]  (negacyclic, schoolbook)          (R2, R8)   */
void orc_blind_rotate(const orc_params* P, const uint32_t* bk, const uint32_t* c, uint32_t* acc) {
  const uint32_t N = P->N, n = P->n, l = P->l;
  uint32_t* A = acc;
  uint32_t* B = acc + N;
  uint32_t* tv = (uint32_t*)malloc(sizeof(uint32_t) * N);
  uint32_t* rot = (uint32_t*)malloc(sizeof(uint32_t) * N);
  uint32_t* D = (uint32_t*)malloc(sizeof(uint32_t) * 2 * N);
  int32_t* dig = (int32_t*)malloc(sizeof(int32_t) * 2 * l * N); /* [c][j][m] */
  int32_t* tmp = (int32_t*)malloc(sizeof(int32_t) * l);
  uint32_t* newacc = (uint32_t*)malloc(sizeof(uint32_t) * 2 * N);

  uint32_t bbar = orc_modswitch(N, c[n]);
  for (uint32_t j = 0; j < N; j++) tv[j] = MU;
  memset(A, 0, sizeof(uint32_t) * N);
  orc_rotate(N, (2 * N - bbar) % (2 * N), tv, B);

  for (uint32_t i = 0; i < n; i++) {
    uint32_t abar = orc_modswitch(N, c[i]);
    for (uint32_t comp = 0; comp < 2; comp++) {
      const uint32_t* src = comp == 0 ? A : B;
      orc_rotate(N, abar, src, rot);
      for (uint32_t m = 0; m < N; m++) D[comp * N + m] = rot[m] - src[m];
    }
    for (uint32_t comp = 0; comp < 2; comp++)
      for (uint32_t m = 0; m < N; m++) {
        orc_decompose(P, D[comp * N + m], tmp);
        for (uint32_t j = 0; j < l; j++) dig[(comp * l + j) * N + m] = tmp[j];
      }
    memcpy(newacc, acc, sizeof(uint32_t) * 2 * N);
    for (uint32_t r = 0; r < 2 * l; r++)
      for (uint32_t out = 0; out < 2; out++)
        negacyclic_mac(N, dig + (size_t)r * N, bk + ((size_t)(i * 2 * l + r) * 2 + out) * N,
                       newacc + out * N);
    memcpy(acc, newacc, sizeof(uint32_t) * 2 * N);
  }
  free(tv); free(rot); free(D); free(dig); free(tmp); free(newacc);
}

/* Sample extract of the constant coefficient: a'_0 = A_0, a'_j = -A_{N-j},
 * b' = B_0.  out: N+1 words (key = TRLWE key S). */
void orc_extract(uint32_t N, const uint32_t* acc, uint32_t* out) {
  const uint32_t* A = acc;
  const uint32_t* B = acc + N;
  out[0] = A[0];
  for (uint32_t j = 1; j < N; j++) out[j] = (uint32_t)0 - A[N - j];
  out[N] = B[0];
}

/* R10 — key switch from key S (dim N) to key s (dim n):
 *   out = (0^n, b');  for i < N: y = a'_i + 2^{32 - t*basebits - 1};
 *   for j < t: d = (y >> (32 - (j+1) basebits)) & (base-1); out -= KSK[i][j][d]. */
void orc_keyswitch(const orc_params* P, const uint32_t* ksk, const uint32_t* in, uint32_t* out) {
  const uint32_t N = P->N, n = P->n, t = P->ks_t, bb = P->ks_base_bits;
  const uint32_t base = 1u << bb;
  memset(out, 0, sizeof(uint32_t) * (n + 1));
  out[n] = in[N];
  for (uint32_t i = 0; i < N; i++) {
    uint32_t y = in[i] + (1u << (32 - t * bb - 1));
    for (uint32_t j = 0; j < t; j++) {
      uint32_t d = (y >> (32 - (j + 1) * bb)) & (base - 1);
      if (d == 0) continue;
      const uint32_t* row = ksk + she_idx_ksk_entry(t, base, i, j, d) * (n + 1);
      for (uint32_t k = 0; k <= n; k++) out[k] -= row[k];
    }
  }
}

/* Gate linear forms (checked by brute force in the
 * tests): c = (0, kappa) + k_a a + k_b b. */
static void linear_form(uint32_t n, uint32_t kappa, int32_t ka, const uint32_t* a, int32_t kb,
                        const uint32_t* b, uint32_t* c) {
  for (uint32_t k = 0; k <= n; k++) c[k] = (uint32_t)ka * a[k] + (uint32_t)kb * b[k];
  c[n] += kappa;
}

/* One gate.  a, b, c: input LWEs (stride >= n+1); out: n+1 words
 * (the rest of the slot, up to stride, is zeroed).  MUX(a,b,c) = a ? b : c:
 * u = BR(-1/8 + a + b), v = BR(-1/8 - a + c), out = KS((0, 1/8) + u + v)  (R6). */
void orc_gate(const orc_params* P, const uint32_t* bk, const uint32_t* ksk, int op,
              const uint32_t* a, const uint32_t* b, const uint32_t* c, size_t stride,
              uint32_t* out) {
  const uint32_t N = P->N, n = P->n;
  uint32_t* lin = (uint32_t*)malloc(sizeof(uint32_t) * (n + 1));
  uint32_t* acc = (uint32_t*)malloc(sizeof(uint32_t) * 2 * N);
  uint32_t* ext = (uint32_t*)malloc(sizeof(uint32_t) * (N + 1));
  uint32_t* ext2 = (uint32_t*)malloc(sizeof(uint32_t) * (N + 1));
  memset(out, 0, sizeof(uint32_t) * stride);
  switch (op) {
    case ORC_NOT:
      for (uint32_t k = 0; k <= n; k++) out[k] = (uint32_t)0 - a[k];
      goto done;
    case ORC_COPY:
      for (uint32_t k = 0; k <= n; k++) out[k] = a[k];
      goto done;
    case ORC_AND:  linear_form(n, (uint32_t)0 - MU, 1, a, 1, b, lin); break;
    case ORC_NAND: linear_form(n, MU, -1, a, -1, b, lin); break;
    case ORC_OR:   linear_form(n, MU, 1, a, 1, b, lin); break;
    case ORC_NOR:  linear_form(n, (uint32_t)0 - MU, -1, a, -1, b, lin); break;
    case ORC_XOR:  linear_form(n, 2 * MU, 2, a, 2, b, lin); break;
    case ORC_XNOR: linear_form(n, (uint32_t)0 - 2 * MU, -2, a, -2, b, lin); break;
    case ORC_MUX: {
      linear_form(n, (uint32_t)0 - MU, 1, a, 1, b, lin);
      orc_blind_rotate(P, bk, lin, acc);
      orc_extract(N, acc, ext);
      linear_form(n, (uint32_t)0 - MU, -1, a, 1, c, lin);
      orc_blind_rotate(P, bk, lin, acc);
      orc_extract(N, acc, ext2);
      for (uint32_t k = 0; k <= N; k++) ext[k] += ext2[k];
      ext[N] += MU;
      orc_keyswitch(P, ksk, ext, out);
      goto done;
    }
    default:
      goto done;
  }
  orc_blind_rotate(P, bk, lin, acc);
  orc_extract(N, acc, ext);
  orc_keyswitch(P, ksk, ext, out);
done:
  free(lin); free(acc); free(ext); free(ext2);
}

/* A batch of independent gates, threaded over gates (host cores). */
void orc_gates(const orc_params* P, const uint32_t* bk, const uint32_t* ksk, const uint8_t* ops,
               const uint32_t* a, const uint32_t* b, const uint32_t* c, size_t count,
               size_t stride, uint32_t* out, int nthreads) {
#ifdef _OPENMP
  if (nthreads <= 0) nthreads = omp_get_max_threads();
#pragma omp parallel for schedule(dynamic, 1) num_threads(nthreads)
#endif
  for (long g = 0; g < (long)count; g++)
    orc_gate(P, bk, ksk, ops[g], a + g * stride, b + g * stride, c + g * stride, stride,
             out + g * stride);
}

/* ------------------------------------------------------------------------ */
/* Leveled mode (reading R-LV)              */
/* PAPER.md:188 "We used all 3 levels of TFHE in the LHE mode": selector bits */
/* as TRGSW (the top level), data as TRLWE (level 1), gates as CMux without   */
/* bootstrapping.                                                             */
/* ------------------------------------------------------------------------ */

/* Selector q = TRGSW_S(bit) in the BK row layout (R2): row r = c*l + j is a
 * TRLWE encryption of 0 under S (A from stream 9, B = A*S + e, e from stream
 * 10 with alpha_bk) plus bit * 2^{32-(j+1)bg} on component c's constant
 * coefficient.  out: count x [2l][2][N]; selector idx draws number first+idx. */
void orc_lvl_encrypt_sel(const orc_params* P, const uint8_t* S, const uint8_t* bits, size_t count,
                         uint64_t seed, uint64_t first, uint32_t* out) {
  const uint32_t N = P->N, l = P->l;
  int32_t* Sd = (int32_t*)malloc(sizeof(int32_t) * N);
  for (uint32_t j = 0; j < N; j++) Sd[j] = S[j];
#pragma omp parallel for schedule(dynamic)
  for (long q = 0; q < (long)count; q++) {
    const uint64_t qq = first + (uint64_t)q;
    for (uint32_t r = 0; r < 2 * l; r++) {
      uint32_t* A = out + (((size_t)q * 2 * l + r) * 2 + 0) * N;
      uint32_t* B = A + N;
      for (uint32_t m = 0; m < N; m++)
        A[m] = she_rng_u32(seed, SHE_STREAM_LVL_MASK, she_idx_bk(N, l, (uint32_t)qq, r, m));
      orc_negacyclic_mul(N, Sd, A, B); /* B = S * A */
      for (uint32_t m = 0; m < N; m++)
        B[m] += she_rng_gauss32(seed, SHE_STREAM_LVL_NOISE, she_idx_bk(N, l, (uint32_t)qq, r, m),
                                P->alpha_bk);
      const uint32_t c = r / l, j = r % l;
      if (bits[q]) (c == 0 ? A : B)[0] += 1u << (32 - (j + 1) * P->bg_bits);
    }
  }
  free(Sd);
}

/* CMux(sel, d1, d0) = d0 + sel [x] (d1 - d0) on TRLWE data (A then B, 2N
 * words each): the external product of the CMux step of orc_blind_rotate
 * (rows r = (c, j): digit_j(D_c) * sel[r], signed gadget decomposition R8,
 * schoolbook negacyclic products) with D = d1 - d0 in place of X^a ACC - ACC. */
void orc_lvl_cmux(const orc_params* P, const uint32_t* sel, const uint32_t* d1, const uint32_t* d0,
                  uint32_t* out) {
  const uint32_t N = P->N, l = P->l;
  int32_t* dig = (int32_t*)malloc(sizeof(int32_t) * 2 * l * N);
  int32_t* tmp = (int32_t*)malloc(sizeof(int32_t) * l);
  uint32_t* acc = (uint32_t*)malloc(sizeof(uint32_t) * 2 * N);
  for (uint32_t comp = 0; comp < 2; comp++)
    for (uint32_t m = 0; m < N; m++) {
      orc_decompose(P, d1[comp * N + m] - d0[comp * N + m], tmp);
      for (uint32_t j = 0; j < l; j++) dig[(comp * l + j) * N + m] = tmp[j];
    }
  memcpy(acc, d0, sizeof(uint32_t) * 2 * N);
  for (uint32_t r = 0; r < 2 * l; r++)
    for (uint32_t o = 0; o < 2; o++)
      negacyclic_mac(N, dig + (size_t)r * N, sel + ((size_t)r * 2 + o) * N, acc + o * N);
  memcpy(out, acc, sizeof(uint32_t) * 2 * N);
  free(dig); free(tmp); free(acc);
}

/* A batch of CMuxes (threaded): item i = CMux(sels[sel_idx[i]], d1[i], d0[i]). */
void orc_lvl_cmux_batch(const orc_params* P, const uint32_t* sels, const uint32_t* sel_idx,
                        const uint32_t* d1, const uint32_t* d0, size_t count, uint32_t* out) {
  const size_t T = (size_t)2 * P->N, R = (size_t)2 * P->l * 2 * P->N;
#pragma omp parallel for schedule(dynamic, 1)
  for (long i = 0; i < (long)count; i++)
    orc_lvl_cmux(P, sels + sel_idx[i] * R, d1 + i * T, d0 + i * T, out + i * T);
}

/* Bit of TRLWE data (R5 on the constant coefficient): phase_0 = B_0 - (A S)_0. */
void orc_lvl_decrypt(const orc_params* P, const uint8_t* S, const uint32_t* in, size_t count,
                     uint8_t* bits) {
  const uint32_t N = P->N;
  for (size_t c = 0; c < count; c++) {
    const uint32_t* A = in + c * 2 * N;
    uint32_t ph = A[N];  /* B_0 */
    /* (A S)_0 = A_0 S_0 - sum_{m >= 1} A_m S_{N-m} (negacyclic) */
    ph -= A[0] * (uint32_t)S[0];
    for (uint32_t m = 1; m < N; m++) ph += A[m] * (uint32_t)S[N - m];
    bits[c] = (int32_t)ph >= 0;
  }
}
