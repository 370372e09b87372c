"""Circuit scheduler on the clear-bit backend vs the plaintext integer network.

The layer circuits (csrc/scheduler.cpp) are the exact gate DAGs the GPU runs;
here they are evaluated on plaintext bits (SPEC.md:88-143 clear backend idea)
and compared with oracle/network.py, which is itself pinned to the worked
examples of tests/golden/spec_unit_examples.json (SPEC.md lines cited there)
and to brute force.  SPEC's acceptance ideas: P1 exhaustive unit sweeps
(SPEC.md:635), P2 shift freeness (:636), P3 accumulator law (:637), P4
end-to-end bit-exactness (:638).
"""
import json
import os

import numpy as np
import pytest

import she_inputs as si
from oracle import network as net
from paper_1906_00148_b200 import build, she

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_unit_examples.json")))


@pytest.fixture(scope="module", autouse=True)
def built():
    build.build()


# ---------------------------------------------------------------------------
# pins of the network oracle (paper / SPEC worked examples, brute force)
# ---------------------------------------------------------------------------

def test_network_oracle_spec_examples():
    for ex in GOLD["relu"]:
        assert net.relu(ex["x"]) == ex["out"], ex["cite"]
    for ex in GOLD["max"]:
        assert max(ex["x"], ex["y"]) == ex["out"]
    for ex in GOLD["maxpool"]:
        v = np.array(ex["inputs"]).reshape(2, 2)
        assert net.maxpool2x2(v)[0, 0] == ex["out"], ex["cite"]
    for ex in GOLD["shift"]:
        if "right" in ex:  # code -(e+1)... a pure shift is the term with sign +: floor semantics
            assert net.term(ex["x"], ex["right"] + 1) == ex["out"], ex["cite"]
    for ex in GOLD["accumulator"]:
        if "sum" in ex:
            x = np.full(ex["inputs"], ex["value"])
            assert net.fc_exact(x, np.ones((1, ex["inputs"]), np.int8))[0] == ex["sum"]
    for ex in GOLD["msize"]:
        assert ex["PN"] * ex["SN"] * ex["PS"] == ex["bytes"]
        assert abs(ex["bytes"] / 2 ** 20 - 122.5) < 1e-9


def test_network_oracle_term_sign_after_shift():
    """R12: -(x >> e) != (-x) >> e when 2^e does not divide x."""
    assert net.term(5, -2) == -2      # -(5 >> 1)
    assert (-5) >> 1 == -3            # the other reading would give -3
    assert net.term(255, 8) == 1      # 255 >> 7
    assert net.term(7, 0) == 0


def test_network_oracle_conv_bruteforce():
    rng = np.random.default_rng(0)
    x = rng.integers(0, 256, (7, 6, 2))
    wq = rng.integers(-8, 9, (3, 3, 3, 2)).astype(np.int8)
    for stride, pad in ((1, 0), (2, 0), (1, 1), (2, 1)):
        got = net.conv_exact(x, wq, stride, pad)
        H, W, _ = x.shape
        for oh in range(got.shape[0]):
            for ow in range(got.shape[1]):
                for co in range(3):
                    s = 0
                    for kh in range(3):
                        for kw in range(3):
                            ih, iw = oh * stride - pad + kh, ow * stride - pad + kw
                            if 0 <= ih < H and 0 <= iw < W:
                                for ci in range(2):
                                    c = int(wq[co, kh, kw, ci])
                                    if c:
                                        s += (1 if c > 0 else -1) * (int(x[ih, iw, ci]) >> (abs(c) - 1))
                    assert got[oh, ow, co] == s


def test_wrap_is_twos_complement():
    assert net.wrap(2 ** 15, 16) == -2 ** 15
    assert net.wrap(-2 ** 15 - 1, 16) == 2 ** 15 - 1
    assert net.wrap(12345, 16) == 12345


# ---------------------------------------------------------------------------
# circuit units on clear bits (SPEC P1 exhaustive sweeps, P2, P3)
# ---------------------------------------------------------------------------

@pytest.mark.parametrize("width", [2, 3, 4, 5, 6])
def test_relu_exhaustive(width):
    vals = np.arange(-(1 << (width - 1)), 1 << (width - 1))
    out, st = she.clear_relu(net.bits_of(vals, width), len(vals), width)
    assert np.array_equal(net.value_of(out, signed=False), np.maximum(vals, 0))
    assert st["gates"] == len(vals) * (width - 1)  # one AND(x_i, !sign) per bit
    assert st["levels"] == 1


def test_relu_spec_examples():
    for ex in GOLD["relu"]:
        out, _ = she.clear_relu(net.bits_of(np.array([ex["x"]]), ex["width"]), 1, ex["width"])
        assert net.value_of(out, signed=False)[0] == ex["out"], ex["cite"]


@pytest.mark.parametrize("signed", [True, False])
def test_max_exhaustive_pairs(signed):
    """maxpool over a 2x2 window holding (x, y, x, y) = max(x, y) for all 5-bit pairs."""
    w = 5
    vals = np.arange(-(1 << (w - 1)), 1 << (w - 1)) if signed else np.arange(0, 1 << w)
    X, Y = np.meshgrid(vals, vals, indexing="ij")
    X, Y = X.ravel(), Y.ravel()
    # H=2, W=2, C=pairs: window (0,0)=x, (0,1)=y, (1,0)=x, (1,1)=y
    img = np.stack([np.stack([X, Y]), np.stack([X, Y])])  # (2, 2, C)
    out, st = she.clear_maxpool2x2(net.bits_of(img, w), 2, 2, len(X), w, signed)
    got = net.value_of(out[0, 0], signed=signed)
    assert np.array_equal(got, np.maximum(X, Y))
    for ex in GOLD["max"]:
        pass  # covered by the sweep: (-1, 0) and (7, 7) are among the pairs


def test_maxpool_spec_example_and_random():
    ex = GOLD["maxpool"][0]
    img = np.array(ex["inputs"]).reshape(2, 2, 1)
    out, st = she.clear_maxpool2x2(net.bits_of(img, 4), 2, 2, 1, 4, True)
    assert net.value_of(out, signed=True)[0, 0, 0] == ex["out"]
    rng = np.random.default_rng(1)
    for signed in (True, False):
        v = rng.integers(-2000 if signed else 0, 2000, (6, 8, 3))
        out, _ = she.clear_maxpool2x2(net.bits_of(v, 13), 6, 8, 3, 13, signed)
        assert np.array_equal(net.value_of(out, signed=signed), net.maxpool2x2(v))


def test_adder_spec_examples_via_fc():
    """a + b as a 2-term neuron with codes +1 (e = 0) on signed 5-bit words."""
    for ex in GOLD["adder"]:
        x = np.array([ex["a"], ex["b"]])
        out, w, st = she.clear_fc_shift_acc(net.bits_of(x, 5).ravel(), 2, 5, True,
                                            np.array([[1, 1]], np.int8), cap=16)
        assert w == ex["width_out"], ex["cite"]
        assert net.value_of(out, signed=True)[0] == ex["sum"]


def test_adder_exhaustive_5bit():
    vals = np.arange(-16, 16)
    A, B = np.meshgrid(vals, vals, indexing="ij")
    x = np.stack([A.ravel(), B.ravel()], axis=1)  # (1024, 2)
    # 1024 neurons, each summing its own pair: K = 2048 inputs, block-diagonal codes
    K = x.size
    wq = np.zeros((len(x), K), np.int8)
    wq[np.arange(len(x)), 2 * np.arange(len(x))] = 1
    wq[np.arange(len(x)), 2 * np.arange(len(x)) + 1] = 1
    out, w, _ = she.clear_fc_shift_acc(net.bits_of(x.ravel(), 5).ravel(), K, 5, True, wq, cap=16)
    assert w == 6
    assert np.array_equal(net.value_of(out, signed=True), x.sum(axis=1))


def test_shift_is_free_rewiring():
    """P2: a lone positive term x >> e costs 0 gates."""
    x = np.array([200, 13, 255, 0])
    for e in range(8):
        wq = np.zeros((4, 4), np.int8)
        wq[np.arange(4), np.arange(4)] = e + 1
        out, w, st = she.clear_fc_shift_acc(net.bits_of(x, 8).ravel(), 4, 8, False, wq, cap=16)
        assert st["gates"] == 0 and st["levels"] == 0
        assert np.array_equal(net.value_of(out, signed=True), x >> e)


def test_accumulator_width_law():
    """P3: level-n adders are min(b+n, cap) bits;
    16 equal 5-bit inputs -> 240, b + 4 bits."""
    ex = [e for e in GOLD["accumulator"] if "sum" in e][0]
    n = ex["inputs"]
    x = np.full(n, ex["value"])
    out, w, st = she.clear_fc_shift_acc(net.bits_of(x, 5).ravel(), n, 5, True,
                                        np.ones((1, n), np.int8), cap=16)
    assert w == 5 + 4
    assert net.value_of(out, signed=True)[0] == ex["sum"]
    out, w, _ = she.clear_fc_shift_acc(net.bits_of(x, 5).ravel(), n, 5, True,
                                       np.ones((1, n), np.int8), cap=7)
    assert w == 7 and net.value_of(out, signed=True)[0] == net.wrap(240, 7)


@pytest.mark.parametrize("seed", range(6))
def test_random_neurons_with_wrap(seed):
    """Random fan-in, widths, signedness, caps (incl. wrapping sums) vs the oracle."""
    rng = np.random.default_rng(seed)
    K = int(rng.integers(1, 300))
    M = 12
    w_in = int(rng.integers(2, 15))
    signed = bool(seed % 2)
    cap = int(rng.choice([8, 10, 16]))
    lo, hi = (-(1 << (w_in - 1)), 1 << (w_in - 1)) if signed else (0, 1 << w_in)
    x = rng.integers(lo, hi, K)
    wq = rng.integers(-8, 9, (M, K)).astype(np.int8)
    wq[rng.random((M, K)) < 0.1] = 0
    out, w, st = she.clear_fc_shift_acc(net.bits_of(x, w_in).ravel(), K, w_in, signed, wq, cap=cap)
    got = net.value_of(out, signed=True)
    assert np.array_equal(got, net.fc(x, wq, cap)), (K, w_in, signed, cap)
    outr, wr, _ = she.clear_fc_shift_acc(net.bits_of(x, w_in).ravel(), K, w_in, signed, wq, cap=cap,
                                         relu=True)
    assert wr == w - 1
    assert np.array_equal(net.value_of(outr, signed=False), net.relu(net.fc(x, wq, cap)))


def test_zero_weight_and_all_negative_neurons():
    x = np.array([5, 9, 255, 17])
    wq = np.array([[0, 0, 0, 0], [-1, -1, -1, -1], [-8, 0, 0, 0], [-1, 0, 0, 0]], np.int8)
    out, w, _ = she.clear_fc_shift_acc(net.bits_of(x, 8).ravel(), 4, 8, False, wq, cap=16)
    assert np.array_equal(net.value_of(out, signed=True), net.fc(x, wq, 16))


# ---------------------------------------------------------------------------
# the configs' layers (P4 end to end on clear bits)
# ---------------------------------------------------------------------------

def test_config2_clear_matches_plaintext_network():
    px = si.pixels(2, (28, 28, 1)).astype(np.int64)
    w1 = si.log_quant_weights(2, (5, 5, 5, 1), layer=0)
    out, w, st = she.clear_conv_shift_acc(net.bits_of(px, 8), 28, 28, 1, 8, False, w1, 2, 0, 16,
                                          relu=True)
    assert out.shape == (12, 12, 5, w) and w == 13  # 14-bit signed sums, ReLU drops the sign
    assert np.array_equal(net.value_of(out, signed=False), net.config2(px, w1))
    # ~0.335 M gates, ~0.41 M BR lanes, 23 levels
    assert 0.30e6 < st["gates"] < 0.40e6 and 0.36e6 < st["br_lanes"] < 0.46e6
    assert 20 <= st["levels"] <= 30


def test_config3_clear_matches_plaintext_network():
    cfg = 3
    px = si.pixels(cfg, (28, 28, 1)).astype(np.int64)
    w1 = si.log_quant_weights(cfg, (5, 5, 5, 1), layer=0)
    w2 = si.log_quant_weights(cfg, (100, 720), layer=1)
    w3 = si.log_quant_weights(cfg, (10, 100), layer=2)
    h, wa, s1 = she.clear_conv_shift_acc(net.bits_of(px, 8), 28, 28, 1, 8, False, w1, 2, 0, 16,
                                         relu=True)
    h2, wb, s2 = she.clear_fc_shift_acc(h.reshape(-1), 720, wa, False, w2, 16, relu=True)
    o, wc, s3 = she.clear_fc_shift_acc(h2.reshape(-1), 100, wb, False, w3, 16)
    assert np.array_equal(net.value_of(o, signed=True), net.config3(px, w1, w2, w3))
    gates = s1["gates"] + s2["gates"] + s3["gates"]
    levels = s1["levels"] + s2["levels"] + s3["levels"]
    assert 2.3e6 < gates < 3.2e6 and 70 <= levels <= 130


def test_config4_shaped_small_clear():
    """Config-4 topology (3x3 'same' convs, maxpools, FC) on an 8x8x3 input with
    4/4/8 channels: every layer kind, padding, signed-free ReLU chains."""
    rng = np.random.default_rng(4)
    px = rng.integers(0, 256, (8, 8, 3))
    w1 = si.log_quant_weights(4, (4, 3, 3, 3), layer=10)
    w2 = si.log_quant_weights(4, (4, 3, 3, 4), layer=11)
    w3 = si.log_quant_weights(4, (8, 3, 3, 4), layer=12)
    w4 = si.log_quant_weights(4, (10, 2 * 2 * 8), layer=13)
    h, wa, _ = she.clear_conv_shift_acc(net.bits_of(px, 8), 8, 8, 3, 8, False, w1, 1, 1, 16, True)
    h, wb, _ = she.clear_conv_shift_acc(h, 8, 8, 4, wa, False, w2, 1, 1, 16, True)
    h, _ = she.clear_maxpool2x2(h, 8, 8, 4, wb, False)
    h, wc, _ = she.clear_conv_shift_acc(h, 4, 4, 4, wb, False, w3, 1, 1, 16, True)
    h, _ = she.clear_maxpool2x2(h, 4, 4, 8, wc, False)
    o, wd, _ = she.clear_fc_shift_acc(h.reshape(-1), 32, wc, False, w4, 16)
    ref = net.config4(px, w1, w2, w3, w4)
    assert np.array_equal(net.value_of(o, signed=True), ref)


def test_layer_argument_errors_are_reported():
    """Bad shapes and out-of-range weights fail with a status (SheError), never
    a crash or a silent result (include/she.h error contract)."""
    x = net.bits_of(np.arange(16) % 200, 8)
    ok = np.ones((2, 3, 3, 1), np.int8)
    with pytest.raises(she.SheError):
        she.clear_conv_shift_acc(x.reshape(4, 4, 1, 8), 4, 4, 1, 8, False,
                                 np.full((2, 3, 3, 1), 9, np.int8), 1, 1)  # code out of [-8, 8]
    with pytest.raises(she.SheError):
        she.clear_conv_shift_acc(x.reshape(4, 4, 1, 8), 4, 4, 1, 8, False, ok, 1, 0, cap=40)
    with pytest.raises(she.SheError):
        she.clear_fc_mul_acc(x.reshape(-1), 16, 8, False, np.full((1, 16), 300, np.int16))
    with pytest.raises(she.SheError):
        she.clear_bn_shift_add(x.reshape(-1), 16, 4, 8, False, np.array([9, 0, 0, 0], np.int8),
                               None, np.zeros(4, np.int32))
    with pytest.raises(she.SheError):  # words not a multiple of the channel count
        she.clear_bn_shift_add(x.reshape(-1)[:120], 15, 4, 8, False, np.zeros(4, np.int8), None,
                               np.zeros(4, np.int32))
    with pytest.raises(she.SheError):
        she.clear_relu(x.reshape(-1)[:16], 16, 1)  # ReLU needs width >= 2
    with pytest.raises(she.SheError):
        she.clear_fc_shift_acc(x.reshape(-1), 16, 8, False, np.ones((1, 16), np.int8), rank=2,
                               world=2)


def test_degenerate_layers():
    """All-zero weights give the constant 0 word; a 1x1 kernel is a per-pixel
    shift; cap 2 wraps everything to 2 bits."""
    px = np.arange(12).reshape(2, 2, 3) * 20
    z = np.zeros((2, 1, 1, 3), np.int8)
    out, w, st = she.clear_conv_shift_acc(net.bits_of(px, 8), 2, 2, 3, 8, False, z, 1, 0, 16)
    assert not out.any() and st["gates"] == 0
    k1 = np.array([[[[1, 0, 0]]], [[[0, -3, 0]]]], np.int8)
    out, w, _ = she.clear_conv_shift_acc(net.bits_of(px, 8), 2, 2, 3, 8, False, k1, 1, 0, 16)
    assert np.array_equal(net.value_of(out, signed=True), net.conv(px, k1, 1, 0, 16))
    out, w, _ = she.clear_conv_shift_acc(net.bits_of(px, 8), 2, 2, 3, 8, False, k1, 1, 0, 2)
    assert w <= 2 and np.array_equal(net.value_of(out, signed=True), net.conv(px, k1, 1, 0, 2))
