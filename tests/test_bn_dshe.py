"""Batch norm lowered to shift + constant, and a DSHE-style deeper net
(PAPER.md T3 :202-203 [C-B-A-C-B-A-P] x k - F - F).

The plaintext BN (oracle/network.py bn_shift_add) is pinned to its
definition's special cases: shift 0 / no sign / bias 0 is the identity (then
the cap's wrap), a positive shift is multiplication by 2^s, a negative one the
floor division SHE uses for its right shifts (R12), the sign flip is
negation; then the clear-bit circuits must equal it, alone and inside a
DSHE-shaped network.
"""
import numpy as np
import pytest

import she_inputs as si
from oracle import network as net
from paper_1906_00148_b200 import build, she


@pytest.fixture(scope="module", autouse=True)
def built():
    build.build()


def test_bn_oracle_special_cases():
    x = np.arange(-600, 600).reshape(-1, 1)
    z = np.zeros(1, np.int64)
    assert np.array_equal(net.bn_shift_add(x, z, z, z, 16), x)
    assert np.array_equal(net.bn_shift_add(x, [3], z, z, 16), 8 * x)
    assert np.array_equal(net.bn_shift_add(x, [-2], z, z, 16), np.floor_divide(x, 4))
    assert np.array_equal(net.bn_shift_add(x, z, [1], [5], 16), 5 - x)
    assert np.array_equal(net.bn_shift_add(x, z, z, z, 8), net.wrap(x, 8))


@pytest.mark.parametrize("signed", [False, True])
@pytest.mark.parametrize("cap,relu", [(16, False), (10, False), (16, True)])
def test_bn_clear_matches_plaintext(signed, cap, relu):
    rng = np.random.default_rng(cap + 2 * signed + relu)
    C, words, w_in = 5, 60, 9
    x = rng.integers(-(1 << 8) if signed else 0, (1 << 8) if signed else (1 << 9), words)
    shift = rng.integers(-8, 9, C).astype(np.int8)
    shift[:3] = [-8, 0, 8]
    neg = rng.integers(0, 2, C).astype(np.uint8)
    bias = rng.integers(-(1 << 12), 1 << 12, C).astype(np.int32)
    out, w, st = she.clear_bn_shift_add(net.bits_of(x, w_in), words, C, w_in, signed, shift, neg,
                                        bias, cap, relu)
    want = net.bn_shift_add(x.reshape(-1, C), shift, neg, bias, cap).ravel()
    if relu:
        assert np.array_equal(net.value_of(out, signed=False), net.relu(want))
    else:
        assert np.array_equal(net.value_of(out, signed=True), want)


def dshe_small(cfg=5, H=12, ch=2, k=2):
    px = si.pixels(cfg, (H, H, 1)).astype(np.int64)
    blocks, cin = [], 1
    for b in range(k):
        wa = si.log_quant_weights(cfg, (ch, 3, 3, cin), layer=10 * b)
        wb = si.log_quant_weights(cfg, (ch, 3, 3, ch), layer=10 * b + 1)
        blocks.append((wa, si.bn_params(cfg, ch, 10 * b), wb, si.bn_params(cfg, ch, 10 * b + 1)))
        cin = ch
    side = H >> k
    fc1 = si.log_quant_weights(cfg, (8, side * side * ch), layer=90)
    fc2 = si.log_quant_weights(cfg, (10, 8), layer=91)
    return px, blocks, fc1, fc2


def run_dshe_clear(px, blocks, fc1, fc2, cap=16):
    H, C, w = px.shape[0], 1, 8
    h = net.bits_of(px, 8)
    levels = gates = 0
    for wa, bna, wb, bnb in blocks:
        for wq, bn in ((wa, bna), (wb, bnb)):
            h, w, s1 = she.clear_conv_shift_acc(h, H, H, C, w, False, wq, 1, 1, cap)
            C = wq.shape[0]
            h, w, s2 = she.clear_bn_shift_add(h.reshape(-1), H * H * C, C, w, True, *bn, cap, True)
            h = h.reshape(H, H, C, w)
            levels += s1["levels"] + s2["levels"]
            gates += s1["gates"] + s2["gates"]
        h, s3 = she.clear_maxpool2x2(h, H, H, C, w, False)
        levels += s3["levels"]
        gates += s3["gates"]
        H //= 2
    h, w, s4 = she.clear_fc_shift_acc(h.reshape(-1), H * H * C, w, False, fc1, cap, relu=True)
    o, w, s5 = she.clear_fc_shift_acc(h.reshape(-1), fc1.shape[0], w, False, fc2, cap)
    return net.value_of(o, signed=True), levels + s4["levels"] + s5["levels"], gates


def test_dshe_small_clear_matches_plaintext_network():
    px, blocks, fc1, fc2 = dshe_small()
    got, levels, gates = run_dshe_clear(px, blocks, fc1, fc2)
    assert np.array_equal(got, net.dshe(px, blocks, fc1, fc2))
    assert levels > 150  # deep: the point of the DSHE workload
