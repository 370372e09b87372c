"""CPU pins of the leveled mode (DESIGN.md reading
R-LV): client TRGSW selectors, TRLWE data, CMux without bootstrapping.

  * the product client's selectors are byte-identical to the oracle's (same
    seeded streams 9 and 10, independent arithmetic);
  * oracle CMux truth table: decrypt(CMux(sel, d1, d0)) = sel ? d1 : d0 for
    every (sel, d1, d0) bit triple over several keys, and the product client's
    data decryption agrees with the oracle's;
  * closed form: with a NOISELESS selector for 0 the CMux returns d0's phase
    exactly; for 1, d1's phase within the gadget-decomposition bound
    (1 + N) 2^(31 - l bg) / 2 ... (R8);
  * noise growth: a chain of CMuxes with selector 0 on data whose difference
    has uniform digits adds (k+1) l N E[d^2] alpha_bk^2 per CMux (the V_BR
    per-CMux term of DESIGN.md §2), measured over every coefficient.
"""
import dataclasses

import numpy as np
import pytest

import oracle
import she_inputs as si
from paper_1906_00148_b200 import build, she


@pytest.fixture(scope="module", autouse=True)
def built():
    build.build()


def phase(params, S, ct):
    """Phase B - A*S of TRLWE data [2][N] as int64 (torus32 centred)."""
    N = params.N
    A, B = ct[0].astype(np.int64), ct[1].astype(np.int64)
    AS = np.zeros(N, dtype=np.int64)
    for j in np.nonzero(S)[0]:  # negacyclic A * X^j
        r = np.roll(A, j)
        r[:j] = -r[:j]
        AS += r
    ph = (B - AS) & 0xFFFFFFFF
    return np.where(ph >= 1 << 31, ph - (1 << 32), ph)


@pytest.mark.parametrize("params", [si.C0, si.C1], ids=["C0", "C1"])
def test_selectors_match_oracle_bytes(params):
    sk, _ = she.she_keygen(params, 321)
    K = oracle.keygen(params, 321)
    bits = np.random.default_rng(1).integers(0, 2, 5).astype(np.uint8)
    assert np.array_equal(she.lvl_encrypt_selectors(sk, bits, 77, 3),
                          oracle.lvl_encrypt_sel(params, K.S, bits, 77, 3))


@pytest.mark.parametrize("seed", [11, 12, 13])
def test_cmux_truth_table_over_keys(seed):
    P = si.C0
    K = oracle.keygen(P, seed)
    sk, _ = she.she_keygen(P, seed)
    combos = [(s, a, b) for s in (0, 1) for a in (0, 1) for b in (0, 1)]
    sel = oracle.lvl_encrypt_sel(P, K.S, [s for s, _, _ in combos], seed + 100)
    # data: fresh-looking TRLWE (a CMux output of the trivial bits under a
    # noisy selector for 1), so the digits of d1 - d0 are not trivial
    one = oracle.lvl_encrypt_sel(P, K.S, [1] * 16, seed + 200)
    t1 = oracle.lvl_trivial(P, [a for _, a, _ in combos] + [b for _, _, b in combos])
    t0 = oracle.lvl_trivial(P, [1 - a for _, a, _ in combos] + [1 - b for _, _, b in combos])
    data = oracle.lvl_cmux_batch(P, one, np.arange(16), t1, t0)
    out = oracle.lvl_cmux_batch(P, sel, np.arange(8), data[:8], data[8:])
    want = np.array([a if s else b for s, a, b in combos], dtype=np.uint8)
    assert np.array_equal(oracle.lvl_decrypt(P, K.S, out), want)
    assert np.array_equal(she.lvl_decrypt(sk, out), want)


def test_cmux_closed_form_with_noiseless_selectors():
    P = dataclasses.replace(si.C1, alpha_bk=0.0)
    K = oracle.keygen(P, 5)
    rng = np.random.default_rng(2)
    d1 = rng.integers(0, 2**32, (2, P.N), dtype=np.uint64).astype(np.uint32)
    d0 = rng.integers(0, 2**32, (2, P.N), dtype=np.uint64).astype(np.uint32)
    sel = oracle.lvl_encrypt_sel(P, K.S, [0, 1], 9)
    out0 = oracle.lvl_cmux(P, sel[0], d1, d0)
    assert np.array_equal(phase(P, K.S, out0), phase(P, K.S, d0))  # exact
    out1 = oracle.lvl_cmux(P, sel[1], d1, d0)
    err = (phase(P, K.S, out1) - phase(P, K.S, d1) + (1 << 31)) % (1 << 32) - (1 << 31)
    # digit rounding of D = d1 - d0: |D - sum_j d_j g_j| <= 2^(31 - l bg) per
    # coefficient (R8), multiplied by the gadget row of the selector (-e_c)
    # i.e. by (1, S): |err| <= (1 + |S|) 2^(31 - l bg)
    bound = (1 + int(K.S.sum())) * 2 ** (31 - P.l * P.bg_bits)
    assert np.max(np.abs(err)) <= bound
    assert np.max(np.abs(err)) > 0  # the rounding term is really there


def test_cmux_chain_noise_matches_the_external_product_formula():
    P = si.C1
    K = oracle.keygen(P, 7)
    depth = 8
    rng = np.random.default_rng(3)
    zeros = oracle.lvl_encrypt_sel(P, K.S, [0] * depth, 55)
    noise = []
    for chain in range(2):
        d = oracle.lvl_trivial(P, [1])[0]
        for k in range(depth):
            r = rng.integers(0, 2**32, (2, P.N), dtype=np.uint64).astype(np.uint32)
            d = oracle.lvl_cmux(P, zeros[k], r, d)  # selector 0: keeps d, adds noise
        ph = phase(P, K.S, d)
        ph[0] -= 1 << 29  # the message +1/8 on the constant coefficient
        noise.append(ph / 2.0 ** 32)
    v = np.var(np.concatenate(noise))
    Eb = (2 ** (2 * P.bg_bits) + 2) / 12.0
    pred = depth * (P.k + 1) * P.l * P.N * Eb * P.alpha_bk ** 2
    assert 0.85 < v / pred < 1.15, (v, pred)
