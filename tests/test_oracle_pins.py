"""Pins of the CPU oracle against things other than itself (task rule ③).

Each test fixes the oracle to mathematics or to an independent formulation:
  * brute-force polynomial arithmetic (numpy convolution with exact integers),
  * closed forms (trivial-ciphertext bootstrapping, test-vector rotation),
  * exact bounds (gadget decomposition error),
  * exact rational rounding (modulus switch),
  * brute-force truth tables over fresh keys,
  * the closed-form TFHE noise variance (each term isolated by a parameter
    choice that makes it dominant).
References: PAPER.md:31 (bootstrapping), :35 (TFHE), :110 (gates),
:142 (bit-wise encryption), :188 (TFHE setting); readings R1-R10 in
DESIGN.md §2 (= SURVEY.md §8(c)).
"""
from dataclasses import replace
from fractions import Fraction

import numpy as np
import pytest

import oracle
import she_inputs as si

MU = 1 << 29
M32 = (1 << 32) - 1


def negacyclic_ref(d, b):
    """Brute force: full integer convolution, then X^N = -1 folding."""
    N = len(b)
    full = np.convolve(np.asarray(d, dtype=object), np.asarray(b, dtype=object))
    out = [0] * N
    for k, v in enumerate(full):
        if k < N:
            out[k] += v
        else:
            out[k - N] -= v
    return np.array([int(v) % (1 << 32) for v in out], dtype=np.uint32)


def phase_poly(params, acc, S):
    """Phase polynomial B - A*S of a TRLWE (A, B), by exact convolution."""
    N = params.N
    A = acc[:N].astype(np.int64)
    B = acc[N:].astype(np.int64)
    full = np.convolve(A, S.astype(np.int64))
    AS = full[:N].copy()
    AS[: N - 1] -= full[N:]
    return ((B - AS) % (1 << 32)).astype(np.uint32)


def centered(x):
    x = np.asarray(x, dtype=np.int64) & M32
    return np.where(x >= 1 << 31, x - (1 << 32), x)


# --------------------------------------------------------------------------
# polynomial primitives
# --------------------------------------------------------------------------

@pytest.mark.parametrize("N", [8, 16, 256])
def test_negacyclic_mul_matches_bruteforce(N):
    rng = np.random.default_rng(N)
    for _ in range(3):
        d = rng.integers(-512, 512, N)
        b = rng.integers(0, 1 << 32, N, dtype=np.uint64).astype(np.uint32)
        assert np.array_equal(oracle.negacyclic_mul(d, b), negacyclic_ref(d, b))
    # extreme digits and coefficients (SURVEY.md §8(c) pin table)
    for dv in (-512, 511, -128, 127):
        for bv in (0, 1 << 31, M32):
            d = np.full(N, dv)
            b = np.full(N, bv, dtype=np.uint32)
            assert np.array_equal(oracle.negacyclic_mul(d, b), negacyclic_ref(d, b))


def test_negacyclic_monomial_identities():
    N = 64
    e = lambda k: np.eye(N, dtype=np.int64)[k]
    # X * X^{N-1} = X^N = -1
    out = oracle.negacyclic_mul(e(1), e(N - 1).astype(np.uint32))
    assert out[0] == M32 and not out[1:].any()
    # 1 is the identity
    b = np.arange(N, dtype=np.uint32) * 77777
    assert np.array_equal(oracle.negacyclic_mul(e(0), b), b)


@pytest.mark.parametrize("a", [0, 1, 5, 63, 64, 65, 100, 127])
def test_rotate_is_monomial_product(a):
    N = 64
    rng = np.random.default_rng(a)
    p = rng.integers(0, 1 << 32, N, dtype=np.uint64).astype(np.uint32)
    mono = np.zeros(N, dtype=np.int64)
    sign = 1
    k = a
    if k >= N:
        k -= N
        sign = -1
    mono[k] = sign
    assert np.array_equal(oracle.rotate(p, a), negacyclic_ref(mono, p))


@pytest.mark.parametrize("params", [si.C0, si.C1], ids=["C0", "C1"])
def test_decomposition_bound_and_range(params):
    """|x - sum_j d_j 2^{32-j bg}| <= 2^{31 - l bg} (exact bound), digits in
    [-Bg/2, Bg/2), and the digits of 0 are all 0 (R8, R9)."""
    Bg = 1 << params.bg_bits
    rng = np.random.default_rng(7)
    xs = list(rng.integers(0, 1 << 32, 3000, dtype=np.uint64)) + [0, 1, M32, 1 << 31, (1 << 31) - 1]
    bound = 1 << (31 - params.l * params.bg_bits)
    worst = 0
    for x in xs:
        d = oracle.decompose(params, int(x))
        assert all(-Bg // 2 <= v < Bg // 2 for v in d)
        rec = sum(int(v) << (32 - (j + 1) * params.bg_bits) for j, v in enumerate(d))
        err = (int(x) - rec) % (1 << 32)
        err = err - (1 << 32) if err >= 1 << 31 else err
        assert abs(err) <= bound
        worst = max(worst, abs(err))
    assert worst >= bound // 2  # the bound is attained in order of magnitude
    assert not oracle.decompose(params, 0).any()


@pytest.mark.parametrize("N", [256, 1024])
def test_modswitch_is_rounding(N):
    """ms(x) = floor(x * 2N / 2^32 + 1/2) mod 2N, by exact rationals (R7)."""
    lg = (2 * N).bit_length() - 1
    rng = np.random.default_rng(N)
    xs = [int(v) for v in rng.integers(0, 1 << 32, 2000, dtype=np.uint64)]
    xs += [(2 * k + 1) << (31 - lg) for k in range(8)]  # exact halves round up
    xs += [((2 * k + 1) << (31 - lg)) - 1 for k in range(8)]
    xs += [0, M32]
    for x in xs:
        want = int(Fraction(x * 2 * N, 1 << 32) + Fraction(1, 2)) % (2 * N)
        assert oracle.modswitch(N, x) == want


# --------------------------------------------------------------------------
# client side: keys, encryption
# --------------------------------------------------------------------------

def test_keygen_structure_C0():
    """BK row (c, j) of TRGSW(s_i) has phase  e + s_i g_j * (c==B ? 1 : -S)
    (R1, R2); KSK[i][j][v] has phase v S_i 2^{32-2(j+1)} + e (R3)."""
    P = si.C0
    K = oracle.keygen(P, 1000)
    assert set(np.unique(K.s)) <= {0, 1} and 0 < K.s.sum() < P.n
    bk = K.bk.reshape(P.n, 2 * P.l, 2, P.N)
    S = K.S.astype(np.int64)
    sigma_bk = P.alpha_bk * 2.0 ** 32
    for i in (0, 1, 7, P.n - 1):
        for r in range(2 * P.l):
            c, j = divmod(r, P.l)
            g = 1 << (32 - (j + 1) * P.bg_bits)
            ph = centered(phase_poly(P, bk[i, r].reshape(-1), K.S))
            expect = np.zeros(P.N, dtype=np.int64)
            if K.s[i]:
                if c == 1:
                    expect[0] = g
                else:
                    expect = -g * S
            err = centered(ph - expect)
            assert np.abs(err).max() <= 8 * sigma_bk + 1
    base = 1 << P.ks_base_bits
    ksk = K.ksk.reshape(P.N, P.ks_t, base, P.n + 1)
    assert not ksk[:, :, 0, :].any()
    sigma = P.alpha_lwe * 2.0 ** 32
    for i in (0, 3, P.N - 1):
        for j in range(P.ks_t):
            for v in range(1, base):
                ph = oracle.phase(P, K.s, ksk[i, j, v])
                msg = (v * int(K.S[i]) << (32 - (j + 1) * P.ks_base_bits)) & M32
                assert abs(int(centered(ph - msg))) <= 8 * sigma + 1


@pytest.mark.parametrize("params", [si.C0, si.C1], ids=["C0", "C1"])
def test_fresh_encryption_noise(params):
    """phase = +-1/8 + e, Var(e) = (alpha_lwe 2^32)^2 (R4), decrypt is exact (R5)."""
    rng = np.random.default_rng(3)
    s = rng.integers(0, 2, params.n).astype(np.uint8)
    bits = rng.integers(0, 2, 20000).astype(np.uint8)
    cts = oracle.encrypt(params, s, bits, seed=99)
    assert np.array_equal(oracle.decrypt(params, s, cts), bits)
    ph = centered(oracle.phases(params, s, cts))
    e = ph - np.where(bits == 1, MU, -MU)
    var = np.var(e.astype(np.float64))
    pred = (params.alpha_lwe * 2.0 ** 32) ** 2
    assert abs(var / pred - 1) < 0.05
    # the padding words of a slot are zero
    assert not cts[:, params.n + 1:].any()


# --------------------------------------------------------------------------
# bootstrapping: closed forms
# --------------------------------------------------------------------------

def _trivial(params, bit):
    ct = np.zeros(params.stride, dtype=np.uint32)
    ct[params.n] = MU if bit else (-MU) & M32
    return ct


@pytest.mark.parametrize("params", [si.C0, pytest.param(si.C1, marks=pytest.mark.slow)],
                         ids=["C0", "C1"])
def test_trivial_inputs_give_exactly_trivial_outputs(params):
    """a = 0 noiseless inputs: every a~_i = 0, so each CMux adds X^0 ACC - ACC = 0,
    ACC stays (0, X^{-b~} v), the extracted sample is (0, +-mu) and every KS digit
    of 0 + 2^15 is 0: the output is exactly (0^n, +-2^29) with the truth-table sign."""
    K = oracle.keygen(params, 1234)
    ops = [si.AND, si.NAND, si.OR, si.NOR, si.XOR, si.XNOR, si.MUX] if params is si.C0 \
        else [si.AND, si.XOR, si.MUX]
    cases = []
    for op in ops:
        combos = [(x, y, z) for x in (0, 1) for y in (0, 1) for z in (0, 1)] if op == si.MUX \
            else [(x, y, 0) for x in (0, 1) for y in (0, 1)]
        if params is si.C1:
            combos = combos[:2] + combos[-1:]
        for x, y, z in combos:
            cases.append((op, x, y, z))
    opsv = np.array([c[0] for c in cases], dtype=np.uint8)
    A = np.stack([_trivial(params, c[1]) for c in cases])
    B = np.stack([_trivial(params, c[2]) for c in cases])
    C = np.stack([_trivial(params, c[3]) for c in cases])
    out = oracle.gates(K, opsv, A, B, C)
    for row, (op, x, y, z) in zip(out, cases):
        want = int(si.truth(op, x, y, z))
        assert not row[: params.n].any()
        assert row[params.n] == (MU if want else (-MU) & M32)


def test_blind_rotation_is_test_vector_rotation_C0():
    """phase(ACC) = X^{-phibar} v + small, phibar = b~ - sum a~_i s_i mod 2N
    (the constant coefficient is +mu iff phibar in [0, N)); the extracted LWE's
    phase equals the constant coefficient of phase(ACC) exactly."""
    P = si.C0
    K = oracle.keygen(P, 1000)
    rng = np.random.default_rng(11)
    for trial in range(4):
        ct = np.zeros(P.stride, dtype=np.uint32)
        ct[: P.n + 1] = rng.integers(0, 1 << 32, P.n + 1, dtype=np.uint64).astype(np.uint32)
        acc = oracle.blind_rotate(K, ct)
        ph = phase_poly(P, acc, K.S)
        abar = [oracle.modswitch(P.N, int(v)) for v in ct[: P.n]]
        bbar = oracle.modswitch(P.N, int(ct[P.n]))
        phibar = (bbar - sum(a * int(s) for a, s in zip(abar, K.s))) % (2 * P.N)
        # X^{-phibar} v, v = mu * sum_j X^j, by brute force
        tv = np.zeros(P.N, dtype=np.int64)
        for j in range(P.N):
            e = (j - phibar) % (2 * P.N)
            if e < P.N:
                tv[e] += MU
            else:
                tv[e - P.N] -= MU
        err = centered(ph.astype(np.int64) - tv)
        assert np.abs(err).max() < 1 << 24
        assert (tv[0] > 0) == (phibar < P.N)
        ext = oracle.extract(P.N, acc)
        ext_phase = (int(ext[P.N]) - int(np.dot(ext[: P.N].astype(np.uint64),
                                                K.S.astype(np.uint64)))) & M32
        assert ext_phase == int(ph[0])


def test_keyswitch_preserves_phase_C0():
    """phase_s(KS(c)) = phase_S(c) + KS noise (rounding to 16 bits + KSK noise)."""
    P = si.C0
    K = oracle.keygen(P, 1000)
    rng = np.random.default_rng(5)
    sigma = np.sqrt(0.75 * P.N * P.ks_t * (P.alpha_lwe * 2 ** 32) ** 2 + P.N / 2 * 2 ** 32 / 12)
    for _ in range(20):
        ext = rng.integers(0, 1 << 32, P.N + 1, dtype=np.uint64).astype(np.uint32)
        out = oracle.keyswitch(K, ext)
        ph_in = (int(ext[P.N]) - int(np.dot(ext[: P.N].astype(np.uint64),
                                            K.S.astype(np.uint64)))) & M32
        ph_out = oracle.phase(P, K.s, out)
        assert abs(int(centered(ph_out - ph_in))) < 7 * sigma


# --------------------------------------------------------------------------
# gates: brute-force truth tables over fresh keys
# --------------------------------------------------------------------------

def _truth_table_batch(params, key_seed, enc_seed):
    K = oracle.keygen(params, key_seed)
    cases = []
    for op in (si.AND, si.NAND, si.OR, si.NOR, si.XOR, si.XNOR):
        cases += [(op, x, y, 0) for x in (0, 1) for y in (0, 1)]
    cases += [(si.MUX, x, y, z) for x in (0, 1) for y in (0, 1) for z in (0, 1)]
    cases += [(si.NOT, 0, 0, 0), (si.NOT, 1, 0, 0), (si.COPY, 0, 0, 0), (si.COPY, 1, 0, 0)]
    ops = np.array([c[0] for c in cases], dtype=np.uint8)
    bits = np.array([[c[1], c[2], c[3]] for c in cases], dtype=np.uint8)
    cts = oracle.encrypt(params, K.s, bits.ravel(), enc_seed).reshape(len(cases), 3, -1)
    out = oracle.gates(K, ops, cts[:, 0].copy(), cts[:, 1].copy(), cts[:, 2].copy())
    got = oracle.decrypt(params, K.s, out)
    want = np.array([si.truth(*c) for c in cases], dtype=np.uint8)
    return got, want


def test_truth_tables_C0_100_keys():
    """Every op x every input combination x 100 fresh keys decrypts correctly."""
    for k in range(100):
        got, want = _truth_table_batch(si.C0, 10_000 + k, 20_000 + k)
        assert np.array_equal(got, want), f"key {k}"


@pytest.mark.slow
def test_truth_tables_C1_10_keys():
    for k in range(10):
        got, want = _truth_table_batch(si.C1, 30_000 + k, 40_000 + k)
        assert np.array_equal(got, want), f"key {k}"


# --------------------------------------------------------------------------
# noise: closed-form variance, each term made dominant in turn
# --------------------------------------------------------------------------

def predicted_variance(params, s_weight, S_weight, mux=False):
    """Torus-scale output-noise variance of a gate about its mean (
    derived here, the CGGI text is not in the container):
      V_BR = n (k+1) l N E[d^2] a_bk^2 + |s| (1 + |S|) Bg^{-2l} / 12
             E[d^2] = (Bg^2 + 2)/12  (digits uniform in [-Bg/2, Bg/2));
             the decomposition error enters only when s_i = 1 and is multiplied
             by (1, -S), hence (1 + |S|) with |S| the Hamming weight of S.
      V_KS = ((B-1)/B)^2 N t a_lwe^2 + |S| 2^{-2 t basebits} / 12
             digits uniform over {0..B-1}, d = 0 subtracts nothing; for a FIXED
             key the per-entry mean (1/B) sum_v e_v is a constant bias, so the
             variance about the mean keeps (B-1)/B - (B-1)/B^2 = ((B-1)/B)^2.
      out  = V_BR + V_KS, MUX: 2 V_BR + V_KS."""
    P = params
    Bg = 2.0 ** P.bg_bits
    Ed2 = (Bg * Bg + 2) / 12
    v_br = P.n * (P.k + 1) * P.l * P.N * Ed2 * P.alpha_bk ** 2 \
        + s_weight * (1 + S_weight) * Bg ** (-2 * P.l) / 12
    B = 1 << P.ks_base_bits
    v_ks = ((B - 1) / B) ** 2 * P.N * P.ks_t * P.alpha_lwe ** 2 \
        + S_weight * 2.0 ** (-2 * P.ks_t * P.ks_base_bits) / 12
    return (2 * v_br if mux else v_br) + v_ks


NOISE_CASES = {
    "decomposition": si.C0,                                   # Bg^{-2l} term dominates
    "bk_noise": replace(si.C0, alpha_bk=2.0 ** -22),          # a_bk term dominates
    "ks_noise": replace(si.C0, alpha_lwe=2.0 ** -14),         # KSK noise dominates
}


@pytest.mark.parametrize("case", list(NOISE_CASES))
@pytest.mark.parametrize("mux", [False, True], ids=["gate", "mux"])
def test_output_noise_variance(case, mux):
    P = NOISE_CASES[case]
    K = oracle.keygen(P, 777)
    count = 3000 if not mux else 2000
    rng = np.random.default_rng(1)
    if mux:
        ops = np.full(count, si.MUX, dtype=np.uint8)
    else:
        ops = rng.choice(np.array([si.AND, si.NAND, si.OR, si.XOR, si.XNOR], dtype=np.uint8), count)
    bits = rng.integers(0, 2, (count, 3)).astype(np.uint8)
    cts = oracle.encrypt(P, K.s, bits.ravel(), 4242).reshape(count, 3, -1)
    out = oracle.gates(K, ops, cts[:, 0].copy(), cts[:, 1].copy(), cts[:, 2].copy())
    want = np.array([si.truth(o, *b) for o, b in zip(ops, bits)])
    ph = centered(oracle.phases(P, K.s, out))
    err = (ph - np.where(want == 1, MU, -MU)).astype(np.float64) / 2.0 ** 32
    var = float(np.var(err))
    pred = predicted_variance(P, int(K.s.sum()), int(K.S.sum()), mux)
    assert abs(var / pred - 1) < 0.12, (var, pred)
    # the fixed-key KS bias is ~ N(0, (B-1)/B^2 N t a_lwe^2): within 5 sd
    B = 1 << P.ks_base_bits
    bias_sd = np.sqrt((B - 1) / B ** 2 * P.N * P.ks_t * P.alpha_lwe ** 2 + pred / count)
    assert abs(float(np.mean(err))) < 5 * bias_sd
