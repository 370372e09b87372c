"""GPU parity of the leveled mode (DESIGN.md R-LV).

  * she_lvl_cmux_batch (the FP64 engine's exact external product without the
    rotation) == oracle.lvl_cmux_batch (schoolbook) word for word, on client
    selectors and arbitrary TRLWE data, including selector reuse;
  * leveled units on client words: decrypted ADD (x + y mod 2^w), MAX (signed
    and unsigned) and ReLU outputs equal the plaintext for every word; CMux
    counts and depths equal the closed forms (6w, 2w - 1 for ADD; 6w, 2w + 2
    for MAX; 2w - 1 CMux and depth 2 for ReLU).
"""
import numpy as np
import pytest

import oracle
import she_inputs as si

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
from paper_1906_00148_b200 import she  # noqa: E402


@pytest.fixture(scope="module")
def lv(cuda):
    P = si.C1
    sk, ck = she.she_keygen(P, si.key_seed(2))
    ctx = she.Context(P, ck, device=0)
    K = oracle.keygen(P, si.key_seed(2))
    return P, sk, ctx, K


def test_cmux_batch_bit_exact_vs_oracle(lv):
    P, sk, ctx, K = lv
    rng = np.random.default_rng(41)
    bits = rng.integers(0, 2, 12).astype(np.uint8)
    sel = she.lvl_encrypt_selectors(sk, bits, 901, 0)
    sel_dev = she.lvl_selectors_to_device(ctx, sel)
    count = 40
    idx = rng.integers(0, 12, count).astype(np.uint32)  # selectors reused
    d1 = rng.integers(0, 2**32, (count, 2, P.N), dtype=np.uint64).astype(np.uint32)
    d0 = rng.integers(0, 2**32, (count, 2, P.N), dtype=np.uint64).astype(np.uint32)
    dev = lambda a: torch.from_numpy(np.ascontiguousarray(a).view(np.int32)).cuda()
    out = she.lvl_cmux_batch(ctx, sel_dev, dev(idx), dev(d1), dev(d0))
    torch.cuda.synchronize()
    got = out.cpu().numpy().view(np.uint32)
    ref = oracle.lvl_cmux_batch(P, oracle.lvl_encrypt_sel(P, K.S, bits, 901, 0), idx, d1, d0)
    assert np.array_equal(got, ref)


def _words(rng, count, w, signed):
    lo, hi = (-(1 << (w - 1)), 1 << (w - 1)) if signed else (0, 1 << w)
    return rng.integers(lo, hi, count)


def _bits(v, w):
    return ((np.asarray(v, np.int64)[:, None] >> np.arange(w)) & 1).astype(np.uint8)


def _value(bits, signed):
    b = bits.astype(np.int64)
    v = (b << np.arange(b.shape[-1])).sum(axis=-1)
    return np.where(b[..., -1] == 1, v - (1 << b.shape[-1]), v) if signed else v


@pytest.mark.parametrize("op, signed", [(0, True), (1, True), (1, False), (2, True)],
                         ids=["add", "max-signed", "max-unsigned", "relu"])
def test_leveled_units_decrypt_to_plaintext(lv, op, signed):
    P, sk, ctx, K = lv
    w, count = 12, 24
    rng = np.random.default_rng(50 + op)
    x = _words(rng, count, w, signed)
    y = _words(rng, count, w, signed)
    bx, by = _bits(x, w), _bits(y, w)
    sel = she.lvl_encrypt_selectors(sk, np.concatenate([bx.ravel(), by.ravel()]), 902 + op, 0)
    sel_dev = she.lvl_selectors_to_device(ctx, sel)
    x_sel = np.arange(count * w, dtype=np.uint32).reshape(count, w)
    y_sel = None if op == 2 else x_sel + count * w
    out, n_cmux, depth = she.lvl_unit(ctx, op, sel_dev, x_sel, y_sel, w, signed)
    torch.cuda.synchronize()
    got_bits = she.lvl_decrypt(sk, out.cpu().numpy().view(np.uint32))
    if op == 0:
        want = (x + y) & ((1 << w) - 1)
        got = _value(got_bits, False)
        assert n_cmux == count * (6 * w - 3) and depth == 2 * w
    elif op == 1:
        want, got = np.maximum(x, y), _value(got_bits, signed)
        assert n_cmux == count * 6 * w and depth == 2 * w + 2
    else:
        want, got = np.maximum(x, 0), _value(got_bits, False)
        assert n_cmux == count * w and depth == 2
    assert np.array_equal(got, want)
