"""GPU parity of the encrypted layer calls.

Two bars (SURVEY.md §8(c) "What pins each part"):
  * decrypted outputs == the plaintext integer network evaluated directly
    (oracle/network.py, pinned in tests/test_scheduler_clear.py), for every
    output word of every layer, and == the clear-bit evaluation of the same
    circuits (wire-level agreement of the scheduler);
  * ciphertexts: seed-sampled gates are recomputed by the CPU oracle from the
    exact input ciphertexts captured from the GPU wire table (she_ctx_capture)
    and must match word for word.
Config 2 (BASELINE.json configs[2]) runs in full at the TFHE default
parameters; the other cases use the C0 parameter set so that many layer
shapes (padding, signed words, max-pool, FC, ReLU) stay fast.
"""
import numpy as np
import pytest

import oracle
import she_inputs as si
from oracle import network as net

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
from paper_1906_00148_b200 import she  # noqa: E402


def dev(a: np.ndarray):
    return torch.from_numpy(np.ascontiguousarray(a).view(np.int32)).cuda()


def host(t) -> np.ndarray:
    return t.cpu().numpy().view(np.uint32)


class LayerEnv:
    def __init__(self, cfg: int, rank: int = 0, world: int = 1):
        self.cfg = cfg
        self.P = si.CONFIG_PARAMS[cfg]
        self.sk, self.ck = she.she_keygen(self.P, si.key_seed(cfg))
        self.ctx = she.Context(self.P, self.ck, device=0, rank=rank, world=world)
        self._K = None

    @property
    def K(self):
        if self._K is None:
            self._K = oracle.keygen(self.P, si.key_seed(self.cfg))
        return self._K

    def encrypt_words(self, vals, width, seed):
        bits = net.bits_of(vals, width)
        cts = she.she_encrypt_bits(self.sk, bits.ravel(), seed, 0)
        return dev(cts.reshape(bits.shape + (self.P.stride,))), bits

    def decrypt_bits(self, t):
        h = host(t)
        return she.she_decrypt_bits(self.sk, h.reshape(-1, self.P.stride)).reshape(h.shape[:-1])


_envs = {}


def env(cfg):
    if cfg not in _envs:
        _envs[cfg] = LayerEnv(cfg)
    return _envs[cfg]


# Seed-sampled gate ciphertexts per default-parameter layer check (SURVEY.md
# §8(c): 256 per config; ~5 s of oracle time on 16 cores).
SAMPLED = 256
CAP = 320


def every_for(gates: int) -> int:
    """Capture period giving ~400 expected picks out of `gates` (cap CAP)."""
    return max(1, gates // 400)


def check_captured(e: LayerEnv, min_gates: int, ctx=None):
    """Seed-sampled ciphertext parity: oracle(captured inputs) == captured output."""
    ops, slots = she.capture_read(ctx or e.ctx, 4096)
    assert len(ops) >= min_gates
    a, b, c, out = (np.ascontiguousarray(slots[:, j]) for j in range(4))
    ref = oracle.gates(e.K, ops, a, b, c)
    bad = np.nonzero((ref != out).any(axis=1))[0]
    assert not len(bad), f"{len(bad)} of {len(ops)} sampled gates differ from the oracle"
    return len(ops)


def test_small_cnn_c0_decrypted_and_sampled_ciphertexts(cuda):
    """Config-4-shaped chain at C0: 3x3 'same' conv + ReLU, max-pool, FC + ReLU, FC."""
    e = env(0)
    rng = np.random.default_rng(si.input_seed(0) + 11)
    px = rng.integers(0, 256, (6, 6, 1))
    w1 = si.log_quant_weights(4, (3, 3, 3, 1), layer=20)
    w2 = si.log_quant_weights(4, (6, 3 * 3 * 3), layer=21)
    w3 = si.log_quant_weights(4, (4, 6), layer=22)
    she.capture(e.ctx, si.sample_seed(0), 37, 256)
    x, _ = e.encrypt_words(px, 8, 777)
    h, wa = she.she_conv_shift_acc(e.ctx, x, 6, 6, 1, 8, False, w1, 1, 1, 16, relu=True)
    ref1 = net.relu(net.conv(px, w1, 1, 1, 16))
    assert np.array_equal(net.value_of(e.decrypt_bits(h), signed=False), ref1)
    clear1, _, _ = she.clear_conv_shift_acc(net.bits_of(px, 8), 6, 6, 1, 8, False, w1, 1, 1, 16,
                                            relu=True)
    assert np.array_equal(e.decrypt_bits(h), clear1)
    p = she.she_maxpool2x2(e.ctx, h, 6, 6, 3, wa, False)
    ref2 = net.maxpool2x2(ref1)
    assert np.array_equal(net.value_of(e.decrypt_bits(p), signed=False), ref2)
    f, wb = she.she_fc_shift_acc(e.ctx, p.reshape(-1, wa, e.P.stride), 27, wa, False, w2, 16,
                                 relu=True)
    ref3 = net.relu(net.fc(ref2.ravel(), w2, 16))
    assert np.array_equal(net.value_of(e.decrypt_bits(f), signed=False), ref3)
    o, wc = she.she_fc_shift_acc(e.ctx, f, 6, wb, False, w3, 16)
    ref4 = net.fc(ref3, w3, 16)
    assert np.array_equal(net.value_of(e.decrypt_bits(o), signed=True), ref4)
    torch.cuda.synchronize()
    check_captured(e, 8)
    she.capture(e.ctx, 0, 0, 0)


def test_signed_relu_and_maxpool_c0(cuda):
    e = env(0)
    rng = np.random.default_rng(5)
    v = rng.integers(-(1 << 9), 1 << 9, (4, 4, 2))
    v[0, 0, 0], v[0, 1, 0], v[1, 0, 0], v[1, 1, 0] = -512, -512, -512, -512  # all-equal minimum
    v[2, 2, 1], v[2, 3, 1], v[3, 2, 1], v[3, 3, 1] = 7, 7, -3, 7  # ties at the maximum
    x, _ = e.encrypt_words(v, 10, 991)
    she.capture(e.ctx, si.sample_seed(0) + 1, 5, 64)
    r = she.she_relu(e.ctx, x.reshape(-1, 10, e.P.stride), v.size, 10)
    assert np.array_equal(net.value_of(e.decrypt_bits(r), signed=False).reshape(v.shape),
                          net.relu(v))
    m = she.she_maxpool2x2(e.ctx, x, 4, 4, 2, 10, True)
    assert np.array_equal(net.value_of(e.decrypt_bits(m), signed=True), net.maxpool2x2(v))
    check_captured(e, 4)
    she.capture(e.ctx, 0, 0, 0)


def test_fc_signed_inputs_with_wrap_c0(cuda):
    """Signed inputs, negative weights, a 6-bit cap that wraps (R13)."""
    e = env(0)
    rng = np.random.default_rng(6)
    x = rng.integers(-(1 << 7), 1 << 7, 12)
    wq = rng.integers(-3, 4, (5, 12)).astype(np.int8)
    ct, _ = e.encrypt_words(x, 8, 1234)
    o, w = she.she_fc_shift_acc(e.ctx, ct, 12, 8, True, wq, cap=6)
    assert w == 6
    exact = net.fc_exact(x, wq)
    assert net.wrap_events(exact, 6) > 0  # the case actually wraps
    assert np.array_equal(net.value_of(e.decrypt_bits(o), signed=True), net.fc(x, wq, 6))


def test_rank_shards_compose_to_the_full_layer_c0(cuda):
    """Neuron-affine sharding: rank r of W computes its contiguous
    share; the shards concatenated are bit-identical to the world-1 ciphertexts."""
    e = env(0)
    rng = np.random.default_rng(8)
    px = rng.integers(0, 256, (5, 5, 1))
    w1 = si.log_quant_weights(2, (3, 3, 3, 1), layer=30)
    x, _ = e.encrypt_words(px, 8, 4321)
    full, w = she.she_conv_shift_acc(e.ctx, x, 5, 5, 1, 8, False, w1, 2, 0, 16)
    full_h = host(full).reshape(-1, w, e.P.stride)
    words = full_h.shape[0]
    got = np.zeros_like(full_h)
    world = 2
    per = (words + world - 1) // world
    for r in range(world):
        ctx_r = she.Context(e.P, e.ck, device=0, rank=r, world=world)
        part, wr = she.she_conv_shift_acc(ctx_r, x, 5, 5, 1, 8, False, w1, 2, 0, 16)
        assert wr == w
        ph = host(part).reshape(-1, w, e.P.stride)
        got[r * per:(r + 1) * per] = ph[r * per:(r + 1) * per]
        ctx_r.close()
    assert np.array_equal(got, full_h)


def test_config2_full_at_default_params(cuda):
    """BASELINE.json configs[2]: 28x28x1 uint8 -> conv 5x5/2 1->5 -> 12x12x5 + ReLU,
    at N=1024, n=500: every decrypted output bit == the plaintext network; at
    least 256 seed-sampled gates (of 339,984) recomputed by the oracle at C1."""
    e = env(2)
    px = si.pixels(2, (28, 28, 1)).astype(np.int64)
    w1 = si.log_quant_weights(2, (5, 5, 5, 1), layer=0)
    x, _ = e.encrypt_words(px, 8, si.input_seed(2))
    she.capture(e.ctx, si.sample_seed(2), every_for(339_984), CAP)
    h, w = she.she_conv_shift_acc(e.ctx, x, 28, 28, 1, 8, False, w1, 2, 0, 16, relu=True)
    st = she.layer_stats(e.ctx)
    assert w == 13 and 0.36e6 < st["br_lanes"] < 0.46e6
    got = net.value_of(e.decrypt_bits(h), signed=False)
    assert np.array_equal(got, net.config2(px, w1))
    assert check_captured(e, SAMPLED) <= CAP
    she.capture(e.ctx, 0, 0, 0)


# ----------------------------------------------------------------------------
# config 4 (BASELINE.json configs[4]) at the default parameters, by tiles
# ----------------------------------------------------------------------------
# The full CIFAR-shaped net is ~0.5-0.7 G bootstrapped gates (hours on one
# GPU), so every layer kind is checked on a seed-independent tile: rank 0 of
# a `world`-way neuron split (the multi-GPU shard API), fed with the client's
# encryption of that layer's exact plaintext input.  Decrypted tile outputs
# must equal the plaintext network; sampled gate ciphertexts must equal the
# oracle's.

@pytest.fixture(scope="module")
def config4_plain():
    cfg = 4
    px = si.pixels(cfg, (32, 32, 3)).astype(np.int64)
    w1 = si.log_quant_weights(cfg, (32, 3, 3, 3), layer=0)
    w2 = si.log_quant_weights(cfg, (32, 3, 3, 32), layer=1)
    w3 = si.log_quant_weights(cfg, (64, 3, 3, 32), layer=2)
    w4 = si.log_quant_weights(cfg, (10, 4096), layer=3)
    h1 = net.relu(net.conv(px, w1, 1, 1, 16))
    h2 = net.relu(net.conv(h1, w2, 1, 1, 16))
    p1 = net.maxpool2x2(h2)
    h3 = net.relu(net.conv(p1, w3, 1, 1, 16))
    p2 = net.maxpool2x2(h3)
    logits = net.fc(p2.ravel(), w4, 16)
    assert np.array_equal(logits, net.config4(px, w1, w2, w3, w4))
    return dict(px=px, w=(w1, w2, w3, w4), h1=h1, h2=h2, p1=p1, h3=h3, p2=p2, logits=logits)


def _tile_ctx(e, world):
    return she.Context(e.P, e.ck, device=0, rank=0, world=world)


def _conv_tile(e, x_plain, w_in, wq, world, seed, gates):
    """Rank 0 of a `world`-way split of a 3x3 'same' conv + ReLU; `gates` is the
    tile's gate count (clear-bit backend) that sets the capture period."""
    H, W, C = x_plain.shape
    ctx = _tile_ctx(e, world)
    x, _ = e.encrypt_words(x_plain, w_in, seed)
    she.capture(ctx, si.sample_seed(4) + seed, every_for(gates), CAP)
    out, w = she.she_conv_shift_acc(ctx, x, H, W, C, w_in, False, wq, 1, 1, 16, relu=True)
    words = out.shape[0] * out.shape[1] * out.shape[2]
    hi = -(-words // world)
    got = net.value_of(e.decrypt_bits(out.reshape(words, w, -1)[:hi]), signed=False)
    ops, slots = she.capture_read(ctx, CAP)
    ctx.close()
    return got, hi, w, ops, slots


def _check_slots(e, ops, slots):
    """At least SAMPLED captured gates, each == the oracle word for word."""
    assert len(ops) >= SAMPLED, f"only {len(ops)} gates captured"
    a, b, c, out = (np.ascontiguousarray(slots[:, j]) for j in range(4))
    ref = oracle.gates(e.K, ops, a, b, c)
    bad = np.nonzero((ref != out).any(axis=1))[0]
    assert not len(bad), f"{len(bad)} of {len(ops)} sampled gates differ from the oracle"


def _bits_needed(v):
    return max(1, int(np.max(v)).bit_length())


def test_config4_conv1_tile(cuda, config4_plain):
    e, d = env(4), config4_plain
    got, hi, w, ops, slots = _conv_tile(e, d["px"], 8, d["w"][0], 128, 41, 78_388)
    assert np.array_equal(got, d["h1"].reshape(-1)[:hi])
    _check_slots(e, ops, slots)


def test_config4_conv2_tile(cuda, config4_plain):
    """32 -> 32 channels, 288 terms per neuron, inputs = ReLU outputs of conv1."""
    e, d = env(4), config4_plain
    wa = she.conv_width(32, 32, 3, 8, False, d["w"][0], 1, 1, 16, relu=True)
    assert _bits_needed(d["h1"]) <= wa
    got, hi, w, ops, slots = _conv_tile(e, d["h1"], wa, d["w"][1], 1024, 42, 129_458)
    assert np.array_equal(got, d["h2"].reshape(-1)[:hi])
    _check_slots(e, ops, slots)


def test_config4_maxpool_tile(cuda, config4_plain):
    e, d = env(4), config4_plain
    wa = she.conv_width(32, 32, 3, 8, False, d["w"][0], 1, 1, 16, relu=True)
    wb = she.conv_width(32, 32, 32, wa, False, d["w"][1], 1, 1, 16, relu=True)
    world = 16
    ctx = _tile_ctx(e, world)
    x, _ = e.encrypt_words(d["h2"], wb, 43)
    she.capture(ctx, si.sample_seed(4) + 43, every_for(67_584), CAP)
    out = she.she_maxpool2x2(ctx, x, 32, 32, 32, wb, False)
    words = 16 * 16 * 32
    hi = -(-words // world)
    got = net.value_of(e.decrypt_bits(out.reshape(words, wb, -1)[:hi]), signed=False)
    ops, slots = she.capture_read(ctx, CAP)
    ctx.close()
    assert np.array_equal(got, d["p1"].reshape(-1)[:hi])
    _check_slots(e, ops, slots)


def test_config4_conv3_tile(cuda, config4_plain):
    e, d = env(4), config4_plain
    wa = she.conv_width(32, 32, 3, 8, False, d["w"][0], 1, 1, 16, relu=True)
    wb = she.conv_width(32, 32, 32, wa, False, d["w"][1], 1, 1, 16, relu=True)
    got, hi, w, ops, slots = _conv_tile(e, d["p1"], wb, d["w"][2], 512, 44, 145_790)
    assert np.array_equal(got, d["h3"].reshape(-1)[:hi])
    _check_slots(e, ops, slots)


def test_config4_fc_logit_tile_wraps(cuda, config4_plain):
    """FC 4096 -> 10: the exact sums exceed 16 bits, so the logits exercise the
    two's-complement wrap of the accumulator cap (R13) on real data."""
    e, d = env(4), config4_plain
    wa = she.conv_width(32, 32, 3, 8, False, d["w"][0], 1, 1, 16, relu=True)
    wb = she.conv_width(32, 32, 32, wa, False, d["w"][1], 1, 1, 16, relu=True)
    wc = she.conv_width(16, 16, 32, wb, False, d["w"][2], 1, 1, 16, relu=True)
    world = 10
    ctx = _tile_ctx(e, world)
    x, _ = e.encrypt_words(d["p2"].ravel(), wc, 45)
    she.capture(ctx, si.sample_seed(4) + 45, every_for(146_522), CAP)
    out, w = she.she_fc_shift_acc(ctx, x, 4096, wc, False, d["w"][3], 16)
    got = net.value_of(e.decrypt_bits(out)[:1], signed=True)
    ops, slots = she.capture_read(ctx, CAP)
    ctx.close()
    _check_slots(e, ops, slots)
    exact = net.fc_exact(d["p2"].ravel(), d["w"][3])
    assert net.wrap_events(exact, 16) > 0
    assert np.array_equal(got, d["logits"][:1])


# ----------------------------------------------------------------------------
# TCN baseline: fixed-point multipliers
# ----------------------------------------------------------------------------

def test_tcn_fc_and_conv_c0_decrypted_and_sampled_ciphertexts(cuda):
    e = env(0)
    rng = np.random.default_rng(21)
    x = rng.integers(-(1 << 7), 1 << 7, 10)
    wm = rng.integers(-255, 256, (4, 10)).astype(np.int16)
    ct, _ = e.encrypt_words(x, 8, 2121)
    she.capture(e.ctx, si.sample_seed(0) + 7, 23, 64)
    o, w = she.she_fc_mul_acc(e.ctx, ct, 10, 8, True, wm, cap=12)
    assert np.array_equal(net.value_of(e.decrypt_bits(o), signed=True), net.fc_tcn(x, wm, 12))
    px = rng.integers(0, 256, (5, 5, 1))
    wc = si.tcn_weights(2, (2, 3, 3, 1), layer=6)
    xc, _ = e.encrypt_words(px, 8, 2222)
    h, wh = she.she_conv_mul_acc(e.ctx, xc, 5, 5, 1, 8, False, wc, 1, 1, 16, relu=True)
    assert np.array_equal(net.value_of(e.decrypt_bits(h), signed=False),
                          net.relu(net.conv_tcn(px, wc, 1, 1, 16)))
    check_captured(e, 4)
    she.capture(e.ctx, 0, 0, 0)


def test_tcn_config2_shape_at_default_params(cuda):
    """Config-2 conv with TCN multipliers at N=1024, n=500 (0.71 M gates)."""
    e = env(2)
    px = si.pixels(2, (28, 28, 1)).astype(np.int64)
    m1 = si.tcn_weights(2, (5, 5, 5, 1), layer=0)
    x, _ = e.encrypt_words(px, 8, si.input_seed(2) + 1)
    h, w = she.she_conv_mul_acc(e.ctx, x, 28, 28, 1, 8, False, m1, 2, 0, 16, relu=True)
    assert np.array_equal(net.value_of(e.decrypt_bits(h), signed=False),
                          net.relu(net.conv_tcn(px, m1, 2, 0, 16)))


# ----------------------------------------------------------------------------
# NEXT-3: batch norm as shift + constant, a DSHE-style deeper chain (C0)
# ----------------------------------------------------------------------------

def test_bn_and_dshe_chain_c0(cuda):
    e = env(0)
    rng = np.random.default_rng(31)
    C, words, w_in = 3, 12, 9
    x = rng.integers(-(1 << 8), 1 << 8, words)
    shift = np.array([-2, 0, 3], np.int8)
    neg = np.array([0, 1, 0], np.uint8)
    bias = np.array([17, -40, 5], np.int32)
    ct, _ = e.encrypt_words(x, w_in, 3131)
    she.capture(e.ctx, si.sample_seed(0) + 9, 11, 64)
    y, w = she.she_bn_shift_add(e.ctx, ct, words, C, w_in, True, shift, neg, bias, cap=14)
    want = net.bn_shift_add(x.reshape(-1, C), shift, neg, bias, 14).ravel()
    assert np.array_equal(net.value_of(e.decrypt_bits(y), signed=True), want)
    check_captured(e, 4)
    she.capture(e.ctx, 0, 0, 0)
    # [C-B-A-C-B-A-P] x 1 - F - F on an 6x6 input, 2 channels
    px = rng.integers(0, 256, (6, 6, 1))
    wa = si.log_quant_weights(5, (2, 3, 3, 1), layer=70)
    wb = si.log_quant_weights(5, (2, 3, 3, 2), layer=71)
    bna, bnb = si.bn_params(5, 2, 70), si.bn_params(5, 2, 71)
    fc1 = si.log_quant_weights(5, (4, 3 * 3 * 2), layer=72)
    fc2 = si.log_quant_weights(5, (3, 4), layer=73)
    h, _ = e.encrypt_words(px, 8, 3232)
    Hc, Cc, wc, sg = 6, 1, 8, False
    for wq, bn in ((wa, bna), (wb, bnb)):
        h, wc = she.she_conv_shift_acc(e.ctx, h, Hc, Hc, Cc, wc, sg, wq, 1, 1, 16)
        Cc = wq.shape[0]
        h, wc = she.she_bn_shift_add(e.ctx, h.reshape(-1, wc, e.P.stride), Hc * Hc * Cc, Cc, wc,
                                     True, *bn, cap=16, relu=True)
        h, sg = h.reshape(Hc, Hc, Cc, wc, e.P.stride), False
    h = she.she_maxpool2x2(e.ctx, h, 6, 6, 2, wc, False)
    h, w1 = she.she_fc_shift_acc(e.ctx, h.reshape(-1, wc, e.P.stride), 18, wc, False, fc1, 16,
                                 relu=True)
    o, w2 = she.she_fc_shift_acc(e.ctx, h, 4, w1, False, fc2, 16)
    want = net.dshe(px, [(wa, bna, wb, bnb)], fc1, fc2)
    assert np.array_equal(net.value_of(e.decrypt_bits(o), signed=True), want)


def test_config3_full_at_default_params(cuda):
    """BASELINE.json configs[3], the bench's net-latency workload, in full at
    N=1024, n=500 (2.67 M gates, ~35 s): the decrypted 16-bit logits equal the
    plaintext network; the hidden layers' outputs too; >= 256 seed-sampled
    gate ciphertexts over the three layers equal the oracle's."""
    e = env(3)
    cfg = 3
    px = si.pixels(cfg, (28, 28, 1)).astype(np.int64)
    w1 = si.log_quant_weights(cfg, (5, 5, 5, 1), layer=0)
    w2 = si.log_quant_weights(cfg, (100, 720), layer=1)
    w3 = si.log_quant_weights(cfg, (10, 100), layer=2)
    x, _ = e.encrypt_words(px, 8, si.input_seed(cfg))
    # >= 256 seed-sampled gate ciphertexts over the whole net (~2.67 M gates)
    she.capture(e.ctx, si.sample_seed(cfg), every_for(2_670_000), CAP)
    h1, wa = she.she_conv_shift_acc(e.ctx, x, 28, 28, 1, 8, False, w1, 2, 0, 16, relu=True)
    ref1 = net.config2(px, w1)
    assert np.array_equal(net.value_of(e.decrypt_bits(h1), signed=False), ref1)
    h2, wb = she.she_fc_shift_acc(e.ctx, h1.reshape(-1, wa, e.P.stride), 720, wa, False, w2, 16,
                                  relu=True)
    ref2 = net.relu(net.fc(ref1.ravel(), w2, 16))
    assert np.array_equal(net.value_of(e.decrypt_bits(h2), signed=False), ref2)
    lo, wc = she.she_fc_shift_acc(e.ctx, h2, 100, wb, False, w3, 16)
    got = net.value_of(e.decrypt_bits(lo), signed=True)
    assert np.array_equal(got, net.config3(px, w1, w2, w3))
    assert net.wrap_events(net.fc_exact(ref2, w3), 16) == 0  # configs 2-3 never wrap
    assert check_captured(e, SAMPLED) <= CAP
    she.capture(e.ctx, 0, 0, 0)
