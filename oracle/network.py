"""Plaintext integer shift-accumulate network — TEST INFRASTRUCTURE ONLY (see
oracle/__init__.py).  The decrypted outputs of the encrypted layers must equal
these values exactly.

Semantics (PAPER.md:118 log quantisation, :142 shifts, :147-149 accumulator;
readings R11-R16 of SURVEY.md §8(c)):
  * R11 pixels are unsigned 8-bit values (zero-extended, non-negative);
  * R12 a weight code +-(e+1) contributes sign * floor(x / 2^e), i.e. the
    shift happens before the sign (-(x >> e), not (-x) >> e); code 0 nothing;
  * R13 neuron = the exact integer sum reduced to `cap`-bit two's complement
    (wrap-around, not saturation);
  * ReLU = max(v, 0); max-pool 2x2 stride 2 = max of the four;
  * R14 valid convolution unless `pad` > 0 (zero padding, "same" for 3x3 pad 1);
  * R16 flatten order HWC.
Written as the definitions, with plain loops over the kernel window.
"""
from __future__ import annotations

import numpy as np


def wrap(v, cap: int):
    """Reduce integers to cap-bit two's complement (R13)."""
    v = np.asarray(v, dtype=np.int64)
    m = 1 << cap
    return ((v + (m >> 1)) % m) - (m >> 1)


def wrap_events(v, cap: int) -> int:
    v = np.asarray(v, dtype=np.int64)
    return int(np.sum((v < -(1 << (cap - 1))) | (v >= (1 << (cap - 1)))))


def term(x, code):
    """sign * (x >> e) for code = +-(e+1); 0 for code 0 (R12)."""
    x = np.asarray(x, dtype=np.int64)
    code = np.asarray(code, dtype=np.int64)
    e = np.abs(code) - 1
    t = np.right_shift(x, np.maximum(e, 0))  # floor division by 2^e
    return np.where(code == 0, 0, np.sign(code) * t)


TCN_FRAC = 7  # TCN multipliers c stand for c / 2^7


def term_tcn(x, c):
    """TCN plaintext x ciphertext product (SPEC.md:238-246 build_pc_mult): the
    shift-and-add over the set bits of |c|, sign(c) * sum_{b : bit b of |c|}
    floor(x / 2^(7 - b)); c in [-255, 255]."""
    x = np.asarray(x, dtype=np.int64)
    c = np.asarray(c, dtype=np.int64)
    mag = np.abs(c)
    acc = np.zeros(np.broadcast(x, c).shape, dtype=np.int64)
    for b in range(TCN_FRAC + 1):
        bit = (mag >> b) & 1
        acc = acc + bit * np.right_shift(x, TCN_FRAC - b)
    return np.sign(c) * acc


def log_quantize(c):
    """PAPER.md:118 weightQ = Quantize(log2(weight)): the SHE code +-(e+1) of the
    power of two 2^-e nearest (in log2) to |c| / 2^7; 0 stays 0."""
    c = np.asarray(c, dtype=np.int64)
    mag = np.maximum(np.abs(c), 1)
    e = np.clip(np.rint(TCN_FRAC - np.log2(mag)), 0, 7).astype(np.int64)
    return np.where(c == 0, 0, np.sign(c) * (e + 1)).astype(np.int8)


def conv_exact(x, wq, stride: int, pad: int, term_fn=None):
    """Exact (unwrapped) sums of a conv layer: x (H,W,C) ints, wq (Co,K,K,C) codes."""
    x = np.asarray(x, dtype=np.int64)
    H, W, C = x.shape
    Co, K, _, _ = wq.shape
    xp = np.zeros((H + 2 * pad, W + 2 * pad, C), dtype=np.int64)
    xp[pad:pad + H, pad:pad + W] = x
    Ho = (H + 2 * pad - K) // stride + 1
    Wo = (W + 2 * pad - K) // stride + 1
    out = np.zeros((Ho, Wo, Co), dtype=np.int64)
    for kh in range(K):
        for kw in range(K):
            patch = xp[kh:kh + stride * (Ho - 1) + 1:stride, kw:kw + stride * (Wo - 1) + 1:stride]
            # patch (Ho, Wo, C); weight codes (Co, C) for this tap
            for co in range(Co):
                out[:, :, co] += (term_fn or term)(patch, wq[co, kh, kw][None, None, :]).sum(axis=-1)
    return out


def conv(x, wq, stride: int, pad: int, cap: int):
    return wrap(conv_exact(x, wq, stride, pad), cap)


def fc_exact(x, wq, term_fn=None):
    x = np.asarray(x, dtype=np.int64).ravel()
    return (term_fn or term)(x[None, :], wq).sum(axis=-1)


def fc(x, wq, cap: int):
    return wrap(fc_exact(x, wq), cap)


def conv_tcn(x, wm, stride: int, pad: int, cap: int):
    return wrap(conv_exact(x, wm, stride, pad, term_tcn), cap)


def fc_tcn(x, wm, cap: int):
    return wrap(fc_exact(x, wm, term_tcn), cap)


def config3_tcn(px, m1, m2, m3, cap=16):
    """The config-3 topology with TCN multipliers (the paper's TCN-vs-SHE
    ablation)."""
    h = relu(conv_tcn(px, m1, 2, 0, cap))
    h = relu(fc_tcn(h.ravel(), m2, cap))
    return fc_tcn(h, m3, cap)


def relu(v):
    return np.maximum(np.asarray(v, dtype=np.int64), 0)


def bn_shift_add(v, shift, neg, bias, cap: int):
    """Batch normalisation lowered to a power-of-two scale and a constant
    (SURVEY.md §8(f) NEXT-3): per channel (last axis), wrap_cap(sign * scale +
    bias) with scale = v * 2^s (s >= 0) or floor(v / 2^-s) (s < 0)."""
    v = np.asarray(v, dtype=np.int64)
    shift = np.asarray(shift, dtype=np.int64)
    sign = np.where(np.asarray(neg, dtype=np.int64) != 0, -1, 1)
    scaled = np.where(shift >= 0, v * (2 ** np.maximum(shift, 0)),
                      np.right_shift(v, np.maximum(-shift, 0)))
    return wrap(sign * scaled + np.asarray(bias, dtype=np.int64), cap)


def maxpool2x2(v):
    v = np.asarray(v, dtype=np.int64)
    H, W = v.shape[0] // 2 * 2, v.shape[1] // 2 * 2
    v = v[:H, :W]
    return np.maximum(np.maximum(v[0::2, 0::2], v[0::2, 1::2]),
                      np.maximum(v[1::2, 0::2], v[1::2, 1::2]))


def bits_of(v, width: int) -> np.ndarray:
    """Two's-complement bits, LSB first: (..., width) uint8."""
    v = np.asarray(v, dtype=np.int64)
    return ((v[..., None] >> np.arange(width)) & 1).astype(np.uint8)


def value_of(bits, signed: bool) -> np.ndarray:
    bits = np.asarray(bits, dtype=np.int64)
    w = bits.shape[-1]
    v = (bits << np.arange(w)).sum(axis=-1)
    if signed:
        v = np.where(bits[..., -1] == 1, v - (1 << w), v)
    return v


# ---- the configs' networks (BASELINE.json configs 2-4) ----------------------

def config2(px, w1, cap=16):
    """conv 5x5 s2 1->5 (valid) + ReLU."""
    return relu(conv(px, w1, 2, 0, cap))


def config3(px, w1, w2, w3, cap=16):
    """conv 5x5 s2 1->5 + ReLU; FC 720->100 + ReLU; FC 100->10 (logits)."""
    h = config2(px, w1, cap)
    h = relu(fc(h.ravel(), w2, cap))
    return fc(h, w3, cap)


def config4(px, w1, w2, w3, w4, cap=16):
    """conv3x3 3->32 + ReLU, conv3x3 32->32 + ReLU, maxpool, conv3x3 32->64 + ReLU,
    maxpool, FC 4096->10 ('same' padding for the 3x3 convs, R15)."""
    h = relu(conv(px, w1, 1, 1, cap))
    h = relu(conv(h, w2, 1, 1, cap))
    h = maxpool2x2(h)
    h = relu(conv(h, w3, 1, 1, cap))
    h = maxpool2x2(h)
    return fc(h.ravel(), w4, cap)


def dshe(px, blocks, fc1, fc2, cap=16):
    """DSHE-style deeper net (PAPER.md T3 :202-203, [C-B-A-C-B-A-P] x k - F - F;
    SURVEY.md §8(f) NEXT-3): blocks = [(wa, bna, wb, bnb), ...] with 3x3 'same'
    convs, BN lowered to shift + constant, ReLU, 2x2 max-pool; then FC + ReLU,
    FC (logits)."""
    h = np.asarray(px, dtype=np.int64)
    for wa, bna, wb, bnb in blocks:
        h = relu(bn_shift_add(conv(h, wa, 1, 1, cap), *bna, cap))
        h = relu(bn_shift_add(conv(h, wb, 1, 1, cap), *bnb, cap))
        h = maxpool2x2(h)
    h = relu(fc(h.ravel(), fc1, cap))
    return fc(h, fc2, cap)
