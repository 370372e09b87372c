"""TCN baseline: plaintext x ciphertext fixed-point
multipliers by shift-and-add (SPEC.md:238-246 build_pc_mult) on the same
scheduler and engine, the paper's TCN-vs-SHE ablation.

Pins of the TCN term (oracle/network.py term_tcn) that do not restate it:
closed forms (a single-bit multiplier is SHE's shift; x a multiple of 2^7 gives
the exact product x*c/2^7), SPEC's worked examples (x*1 -> x, x*(-1) -> -x),
additivity over disjoint bit sets, and the floor-error bound per set bit.
Then the clear-bit circuits must equal the plaintext network.
"""
import numpy as np
import pytest

import she_inputs as si
from oracle import network as net
from paper_1906_00148_b200 import build, she


@pytest.fixture(scope="module", autouse=True)
def built():
    build.build()


def test_tcn_term_closed_forms_and_spec_examples():
    x = np.arange(-300, 300)
    for e in range(8):  # single-bit multipliers are exactly SHE's shifts (R12)
        for sg in (1, -1):
            c = sg * (1 << (7 - e))
            assert np.array_equal(net.term_tcn(x, c), net.term(x, sg * (e + 1)))
            assert net.log_quantize(c) == sg * (e + 1)
    # SPEC.md:244-246 "x * 1 -> x", "x * (-1) -> -x" (1.0 = 128 / 2^7)
    assert np.array_equal(net.term_tcn(x, 128), x)
    assert np.array_equal(net.term_tcn(x, -128), -x)
    # x = 128 k: every partial product is exact, so the term is the exact product
    k = np.arange(-40, 40)
    for c in (1, 3, 77, 128, 200, 255, -5, -255):
        assert np.array_equal(net.term_tcn(128 * k, c), k * c)
    assert np.array_equal(net.term_tcn(x, 0), 0 * x)


def test_tcn_term_additive_and_bounded():
    rng = np.random.default_rng(3)
    x = rng.integers(0, 1 << 12, 500)
    for _ in range(50):
        c1 = int(rng.integers(0, 256))
        c2 = int(rng.integers(0, 256)) & ~c1  # disjoint bits
        assert np.array_equal(net.term_tcn(x, c1 | c2), net.term_tcn(x, c1) + net.term_tcn(x, c2))
        c = c1 | c2
        pop = bin(c).count("1")
        err = x * c / 128.0 - net.term_tcn(x, c)  # each partial product floors by < 1
        assert np.all(err >= 0) and np.all(err < pop + 1e-9)


@pytest.mark.parametrize("signed,cap", [(False, 16), (True, 16), (True, 7)])
def test_tcn_fc_clear_matches_plaintext(signed, cap):
    rng = np.random.default_rng(10 + cap + signed)
    K, w_in = 23, 8
    x = rng.integers(-(1 << 7) if signed else 0, 1 << 7 if signed else 1 << 8, K)
    wm = rng.integers(-255, 256, (9, K)).astype(np.int16)
    wm[0] = 0
    wm[1, :] = 128
    out, w, st = she.clear_fc_mul_acc(net.bits_of(x, w_in).ravel(), K, w_in, signed, wm, cap)
    assert np.array_equal(net.value_of(out, signed=True), net.fc_tcn(x, wm, cap))
    outr, wr, _ = she.clear_fc_mul_acc(net.bits_of(x, w_in).ravel(), K, w_in, signed, wm, cap,
                                       relu=True)
    assert np.array_equal(net.value_of(outr, signed=False), net.relu(net.fc_tcn(x, wm, cap)))


def test_tcn_conv_clear_matches_plaintext_and_sharding():
    rng = np.random.default_rng(12)
    px = rng.integers(0, 256, (7, 7, 2))
    wm = si.tcn_weights(2, (3, 3, 3, 2), layer=5)
    out, w, _ = she.clear_conv_mul_acc(net.bits_of(px, 8), 7, 7, 2, 8, False, wm, 1, 1, 16,
                                       relu=True)
    assert np.array_equal(net.value_of(out, signed=False), net.relu(net.conv_tcn(px, wm, 1, 1, 16)))
    part, _, _ = she.clear_conv_mul_acc(net.bits_of(px, 8), 7, 7, 2, 8, False, wm, 1, 1, 16,
                                        relu=True, rank=1, world=3)
    flat, pflat = out.reshape(-1, w), part.reshape(-1, w)
    per = -(-flat.shape[0] // 3)
    assert np.array_equal(pflat[per:2 * per], flat[per:2 * per]) and not pflat[:per].any()


def test_tcn_single_bit_multipliers_build_the_she_circuit():
    """c = +-2^(7-e) expands to exactly SHE's term: same gates, same levels."""
    rng = np.random.default_rng(13)
    x = rng.integers(0, 256, 40)
    wq = si.log_quant_weights(3, (6, 40), layer=9)
    e = np.abs(wq.astype(np.int64)) - 1
    wm = np.where(wq == 0, 0, np.sign(wq) * (1 << (7 - np.maximum(e, 0)))).astype(np.int16)
    a, wa, sa = she.clear_fc_shift_acc(net.bits_of(x, 8).ravel(), 40, 8, False, wq, 16)
    b, wb, sb = she.clear_fc_mul_acc(net.bits_of(x, 8).ravel(), 40, 8, False, wm, 16)
    assert wa == wb and np.array_equal(a, b) and sa == sb


def test_tcn_vs_she_config3_ablation():
    """The paper's ablation on the config-3 topology: TCN's 8-bit fixed-point
    multipliers vs their log-quantised (SHE) codes.  Both circuits equal their
    plaintext networks; TCN needs more bootstrapped gates and levels."""
    cfg = 3
    px = si.pixels(cfg, (28, 28, 1)).astype(np.int64)
    m = [si.tcn_weights(cfg, s, layer=i) for i, s in enumerate([(5, 5, 5, 1), (100, 720), (10, 100)])]
    q = [net.log_quantize(mi) for mi in m]
    h, wa, t1 = she.clear_conv_mul_acc(net.bits_of(px, 8), 28, 28, 1, 8, False, m[0], 2, 0, 16, True)
    h, wb, t2 = she.clear_fc_mul_acc(h.reshape(-1), 720, wa, False, m[1], 16, relu=True)
    o, _, t3 = she.clear_fc_mul_acc(h.reshape(-1), 100, wb, False, m[2], 16)
    assert np.array_equal(net.value_of(o, signed=True), net.config3_tcn(px, *m))
    g, wa, s1 = she.clear_conv_shift_acc(net.bits_of(px, 8), 28, 28, 1, 8, False, q[0], 2, 0, 16, True)
    g, wb, s2 = she.clear_fc_shift_acc(g.reshape(-1), 720, wa, False, q[1], 16, relu=True)
    o, _, s3 = she.clear_fc_shift_acc(g.reshape(-1), 100, wb, False, q[2], 16)
    assert np.array_equal(net.value_of(o, signed=True), net.config3(px, *q))
    tcn = sum(t["gates"] for t in (t1, t2, t3))
    she_ = sum(s["gates"] for s in (s1, s2, s3))
    assert tcn > 2.0 * she_
    assert sum(t["levels"] for t in (t1, t2, t3)) > sum(s["levels"] for s in (s1, s2, s3))
