"""GPU parity of the CUDA gate-bootstrapping path (libshe.so) against the oracle.

Bar (BASELINE.json north_star, task rule ③): output ciphertexts bit-exact
(integer work: no tolerance), decrypted bits equal to the truth table.
  * config 0 (C0, 16 gates): full comparison with the oracle run live;
  * config 1 (C1, 4096 gates, the bench launch configuration): full
    comparison of every gate against tests/golden/config1_oracle_digests.txt
    (written by a committed script that calls only oracle/), plus a
    seed-sampled subset recomputed live by the oracle;
  * edge cases: empty and ragged batches, every op through the uniform-op API,
    NOT/COPY, MUX with aliased inputs, the wire-table level API with negated
    inputs, trivial ciphertexts (closed form), noise variance at C1.
"""
import hashlib
import os

import numpy as np
import pytest

import oracle
import she_inputs as si

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
from paper_1906_00148_b200 import she  # noqa: E402

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
MU = 1 << 29


def dev(a: np.ndarray):
    return torch.from_numpy(np.ascontiguousarray(a).view(np.int32)).cuda()


def host(t) -> np.ndarray:
    return t.cpu().numpy().view(np.uint32)


class Env:
    """Product keys + device context for one config (cached per session)."""

    def __init__(self, cfg: int):
        self.cfg = cfg
        self.P = si.CONFIG_PARAMS[cfg]
        self.sk, self.ck = she.she_keygen(self.P, si.key_seed(cfg))
        self.ctx = she.Context(self.P, self.ck, device=0)
        self._K = None

    @property
    def K(self):  # oracle keys (independent keygen from the same seed)
        if self._K is None:
            self._K = oracle.keygen(self.P, si.key_seed(self.cfg))
        return self._K

    def workload(self, count: int):
        ops = si.gate_ops(self.cfg, count)
        bits = si.gate_input_bits(self.cfg, count)
        cts = she.she_encrypt_bits(self.sk, bits.ravel(), si.input_seed(self.cfg), 0)
        return ops, bits, cts.reshape(count, 3, -1)

    def run_ops(self, ops, a, b, c):
        out = torch.zeros((a.shape[0], self.P.stride), dtype=torch.int32, device="cuda")
        she.she_gate_batch_ops(self.ctx, dev(np.asarray(ops, np.uint8)), dev(a), dev(b), dev(c), out)
        torch.cuda.synchronize()
        return host(out)


_envs = {}


@pytest.fixture(scope="module")
def env0(cuda):
    if 0 not in _envs:
        _envs[0] = Env(0)
    return _envs[0]


@pytest.fixture(scope="module")
def env1(cuda):
    if 1 not in _envs:
        _envs[1] = Env(1)
    return _envs[1]


def digest(words) -> str:
    return hashlib.sha256(np.ascontiguousarray(words, dtype="<u4").tobytes()).hexdigest()[:32]


def read_digests(cfg):
    path = os.path.join(GOLDEN, f"config{cfg}_oracle_digests.txt")
    rows = [ln.split() for ln in open(path) if not ln.startswith("#")]
    return [(int(g), int(op), d, int(bit)) for g, op, d, bit in rows]


# ----------------------------------------------------------------------------
# config 0: full comparison with the oracle, live
# ----------------------------------------------------------------------------

def test_config0_full_parity(env0):
    P = env0.P
    ops, bits, cts = env0.workload(16)
    out = env0.run_ops(ops, cts[:, 0].copy(), cts[:, 1].copy(), cts[:, 2].copy())
    ref = oracle.gates(env0.K, ops, cts[:, 0].copy(), cts[:, 1].copy(), cts[:, 2].copy())
    assert np.array_equal(out, ref)
    want = np.array([si.truth(o, *b) for o, b in zip(ops, bits)])
    assert np.array_equal(she.she_decrypt_bits(env0.sk, out), want)
    # and against the committed oracle digests
    for g, op, d, bit in read_digests(0):
        assert op == ops[g] and digest(out[g, : P.n + 1]) == d and bit == want[g]


def test_config0_truth_tables_all_ops(env0):
    P = env0.P
    cases = []
    for op in (si.AND, si.NAND, si.OR, si.NOR, si.XOR, si.XNOR):
        cases += [(op, x, y, 0) for x in (0, 1) for y in (0, 1)]
    cases += [(si.MUX, x, y, z) for x in (0, 1) for y in (0, 1) for z in (0, 1)]
    cases += [(si.NOT, x, 0, 0) for x in (0, 1)] + [(si.COPY, x, 0, 0) for x in (0, 1)]
    cases = cases * 8
    ops = np.array([c[0] for c in cases], np.uint8)
    bits = np.array([c[1:] for c in cases], np.uint8)
    cts = she.she_encrypt_bits(env0.sk, bits.ravel(), 31337).reshape(len(cases), 3, -1)
    a, b, c = (cts[:, j].copy() for j in range(3))
    out = env0.run_ops(ops, a, b, c)
    ref = oracle.gates(env0.K, ops, a, b, c)
    assert np.array_equal(out, ref)
    want = np.array([si.truth(*c_) for c_ in cases])
    assert np.array_equal(she.she_decrypt_bits(env0.sk, out), want)


def test_trivial_inputs_closed_form(env0):
    """Noiseless a = 0 inputs bootstrap to exactly (0^n, +-2^29)."""
    P = env0.P
    cases = [(op, x, y, z) for op in (si.AND, si.NAND, si.OR, si.NOR, si.XOR, si.XNOR, si.MUX)
             for x in (0, 1) for y in (0, 1) for z in (0, 1)]
    def triv(bit):
        t = np.zeros(P.stride, np.uint32)
        t[P.n] = MU if bit else (-MU) & 0xFFFFFFFF
        return t
    a = np.stack([triv(c[1]) for c in cases])
    b = np.stack([triv(c[2]) for c in cases])
    c = np.stack([triv(c[3]) for c in cases])
    out = env0.run_ops(np.array([c_[0] for c_ in cases], np.uint8), a, b, c)
    for row, case in zip(out, cases):
        assert not row[: P.n].any() and not row[P.n + 1:].any()
        assert row[P.n] == (MU if si.truth(*case) else (-MU) & 0xFFFFFFFF)


@pytest.mark.parametrize("count", [0, 1, 2, 7, 17, 33])
def test_ragged_batches_and_uniform_ops(env0, count):
    P = env0.P
    rng = np.random.default_rng(count)
    for op in (si.AND, si.NAND, si.OR, si.NOR, si.XOR, si.XNOR, si.MUX, si.NOT, si.COPY):
        bits = rng.integers(0, 2, (count, 3)).astype(np.uint8)
        cts = she.she_encrypt_bits(env0.sk, bits.ravel(), 900 + op).reshape(count, 3, P.stride)
        a, b, c = (cts[:, j].copy() for j in range(3))
        out = torch.zeros((count, P.stride), dtype=torch.int32, device="cuda")
        if count:
            she.she_gate_batch(env0.ctx, op, dev(a), dev(b), dev(c), out)
        else:
            empty = torch.zeros((0, P.stride), dtype=torch.int32, device="cuda")
            she.she_gate_batch(env0.ctx, op, empty, empty, empty, out)
        torch.cuda.synchronize()
        got = host(out)
        ref = oracle.gates(env0.K, np.full(count, op, np.uint8), a, b, c)
        assert np.array_equal(got, ref), si.OP_NAMES[op]


def test_device_field_primitives_edge_values(cuda):
    """The hand-written PTX carry/borrow chains of the device Goldilocks
    primitives on edge values that reach their rare branches (a borrow of
    lo - hi_hi, the second fold, inputs in (p, 2^64)), against exact integer
    arithmetic, with the <= p bound of the *_le results."""
    P64 = 2 ** 64 - 2 ** 32 + 1
    edge = [0, 1, 2, 2 ** 32 - 2, 2 ** 32 - 1, 2 ** 32, 2 ** 32 + 1, P64 - 2, P64 - 1, P64,
            P64 + 1, 2 ** 64 - 2, 2 ** 64 - 1, 2 ** 63, 2 ** 63 - 1, 0xFFFFFFFF00000000,
            0xFFFFFFFEFFFFFFFF, 0x80000000FFFFFFFF, 0x00000001FFFFFFFF, 0x00000000FFFFFFFE]
    rng = np.random.default_rng(77)
    rand = [int(v) for v in rng.integers(0, 2 ** 64 - 1, 40, dtype=np.uint64)]
    vals = edge + rand
    pairs = [(x, y) for x in vals for y in vals]
    a = np.array([x for x, _ in pairs], np.uint64)
    b = np.array([y for _, y in pairs], np.uint64)
    c = np.arange(len(pairs), dtype=np.uint32)
    out = she.field_selftest(0, a, b, c)
    for k, (x, y) in enumerate(pairs):
        o = [int(v) for v in out[k]]
        assert o[0] % P64 == (x + y) % P64 and o[1] % P64 == (x - y) % P64
        if y <= P64:
            assert o[2] % P64 == (x + y) % P64 and o[3] % P64 == (x - y) % P64
        assert o[4] % P64 == x * y % P64
        assert o[5] <= P64 and o[5] % P64 == x * y % P64
        assert o[6] <= P64 and o[6] % P64 == (x + y * 2 ** 64) % P64
        top = k & 3
        assert o[7] <= P64 and o[7] % P64 == (x + y * 2 ** 64 + top * 2 ** 128) % P64
        for s_ in range(96):
            assert o[8 + s_] <= P64 and o[8 + s_] % P64 == x * pow(2, s_, P64) % P64, (x, s_)


def test_batch_larger_than_one_launch(env0):
    """Maximum-size path: more gates than one BR+KS launch pair takes (65536,
    csrc/engine.cu kChunk), mixed ops, ragged tail.  Every output decrypts to
    the truth table; a seed-sampled subset on both sides of each chunk seam is
    recomputed by the oracle word for word."""
    P = env0.P
    count = 2 * 65536 + 76  # ragged (not a multiple of the launch size), 4-byte aligned ops
    rng = np.random.default_rng(65537)
    ops = rng.choice(si.BOOTSTRAPPED_MIX, count).astype(np.uint8)
    bits = rng.integers(0, 2, (count, 3)).astype(np.uint8)
    cts = she.she_encrypt_bits(env0.sk, bits.ravel(), 6553).reshape(count, 3, P.stride)
    a, b, c = (cts[:, j].copy() for j in range(3))
    out = env0.run_ops(ops, a, b, c)
    want = np.array([si.truth(o, *bb) for o, bb in zip(ops, bits)])
    assert np.array_equal(she.she_decrypt_bits(env0.sk, out), want)
    pick = np.unique(np.concatenate([[0, 65535, 65536, 131071, 131072, count - 1],
                                     rng.choice(count, 10, replace=False)]))
    ref = oracle.gates(env0.K, ops[pick], a[pick], b[pick], c[pick])
    assert np.array_equal(out[pick], ref)


def test_mux_aliased_inputs(env0):
    P = env0.P
    bits = np.array([0, 1, 1, 0], np.uint8)
    cts = she.she_encrypt_bits(env0.sk, bits, 4444)
    ops = np.full(4, si.MUX, np.uint8)
    out = env0.run_ops(ops, cts, cts, cts)  # MUX(x, x, x) = x
    ref = oracle.gates(env0.K, ops, cts, cts, cts)
    assert np.array_equal(out, ref)
    assert np.array_equal(she.she_decrypt_bits(env0.sk, out), bits)


def test_level_api_negated_inputs(env0):
    """Wire-table level: gate g reads wires[idx & 0x7fffffff], negated if bit 31."""
    P = env0.P
    rng = np.random.default_rng(9)
    W, G = 24, 40
    wbits = rng.integers(0, 2, W).astype(np.uint8)
    wires_h = np.zeros((W + G, P.stride), np.uint32)
    wires_h[:W] = she.she_encrypt_bits(env0.sk, wbits, 5555)
    ops = rng.choice(np.array([si.AND, si.NAND, si.OR, si.NOR, si.XOR, si.XNOR, si.MUX, si.NOT,
                               si.COPY], np.uint8), G)
    idx = rng.integers(0, W, (G, 3)).astype(np.uint32)
    neg = rng.integers(0, 2, (G, 3)).astype(np.uint32)
    ins = idx | (neg << np.uint32(31))
    out_idx = (W + np.arange(G)).astype(np.uint32)
    wires = dev(wires_h)
    she.she_gate_level(env0.ctx, wires, dev(ops), dev(ins.ravel()), dev(out_idx))
    torch.cuda.synchronize()
    got = host(wires)[W:]
    # oracle: negation of an LWE sample is -c (NOT without bootstrapping)
    def lwe(j):
        x = wires_h[idx[:, j]].astype(np.uint64)
        x = np.where(neg[:, j:j + 1] == 1, (-x.astype(np.int64)) & 0xFFFFFFFF, x)
        x[:, P.n + 1:] = 0
        return x.astype(np.uint32)
    ref = oracle.gates(env0.K, ops, lwe(0), lwe(1), lwe(2))
    assert np.array_equal(got, ref)
    vb = wbits[idx] ^ neg.astype(np.uint8)
    want = np.array([si.truth(o, *b) for o, b in zip(ops, vb)])
    assert np.array_equal(she.she_decrypt_bits(env0.sk, got), want)


# ----------------------------------------------------------------------------
# config 1: the bench configuration
# ----------------------------------------------------------------------------

@pytest.fixture(scope="module")
def config1_outputs(env1):
    ops, bits, cts = env1.workload(4096)
    a, b, c = (cts[:, j].copy() for j in range(3))
    out = env1.run_ops(ops, a, b, c)
    return ops, bits, (a, b, c), out


def test_config1_full_parity_vs_oracle_digests(env1, config1_outputs):
    P = env1.P
    ops, bits, _, out = config1_outputs
    rows = read_digests(1)
    assert len(rows) == 4096
    bad = [g for g, op, d, bit in rows if op != ops[g] or digest(out[g, : P.n + 1]) != d]
    assert not bad, f"{len(bad)} gates differ from the oracle, first {bad[:8]}"
    assert not out[:, P.n + 1:].any()
    want = np.array([si.truth(o, *b) for o, b in zip(ops, bits)])
    assert np.array_equal(she.she_decrypt_bits(env1.sk, out), want)


ENGINE_OPTS = {"ntt": dict(engine="ntt"), "fft3": dict(engine="fft", fft_lanes=3),
               "fft2x2": dict(engine="fft", fft_lanes=2), "fft-v1": dict(engine="fft", fft_variant=1),
               "fft-2groups": dict(engine="fft", fft_groups=2),
               "fft5-noprefetch": dict(engine="fft", fft_lanes=5, fft_prefetch=3),
               "ks-imma": dict(ks_kernel="imma"), "ks-cuda": dict(ks_kernel="cuda"),
               "ks-tcgen05": dict(ks_kernel="tcgen05"),
               "fft-2streams": dict(engine="fft", fft_streams=2),
               "fft-v3": dict(engine="fft", fft_variant=3),
               "fft5-v3": dict(engine="fft", fft_lanes=5, fft_prefetch=3, fft_variant=3),
               "fft-smem": dict(engine="fft", fft_store="smem"),
               "fft-tmem-stagger": dict(engine="fft", fft_store="tmem", fft_stagger_ns=20000),
               "fft-tmem-v2": dict(engine="fft", fft_store="tmem", fft_variant=2),
               # TMEM engine work distribution (the default is the chunk queue, 32 iterations):
               # static split only; the chunk queue with a ragged last chunk (500 = 71 x 7 + 3),
               # with 32 iterations given explicitly, with two chunks of 499 + 1; the wrap-around
               # schedule
               "fft-tmem-static": dict(fft_chunk=-1), "fft-tmem-chunk7": dict(fft_chunk=7),
               "fft-tmem-chunk32": dict(fft_chunk=32), "fft-tmem-wrap": dict(fft_chunk=-2),
               "fft-tmem-chunk499": dict(fft_store="tmem", fft_chunk=499)}


@pytest.mark.parametrize("engine", ["ntt", "fft3", "fft2x2", "fft-v1", "fft-2groups",
                                    "fft5-noprefetch", "ks-imma", "ks-cuda", "fft-v3", "fft5-v3",
                                    "ks-tcgen05", "fft-2streams", "fft-smem", "fft-tmem-stagger",
                                    "fft-tmem-v2", "fft-tmem-static", "fft-tmem-chunk7",
                                    "fft-tmem-chunk32", "fft-tmem-wrap", "fft-tmem-chunk499"])
def test_config1_other_blind_rotation_engines(cuda, env1, config1_outputs, engine):
    """The default context of N = 1024 runs the FP64 FFT engine with the
    spectra in tensor memory (br_fft_tm_kernel); the Goldilocks
    NTT engine (she_ctx_options.br_engine = 2), the shared-memory FFT engine
    and its shapes must give the same ciphertexts bit for bit (all products are
    exact): all 4096 config-1 gates against the oracle digests."""
    assert she.br_engine(env1.ctx) == 8  # the TMEM engine
    assert she.br_engine(env0_ctx()) == 0  # N = 256 has no FFT engine
    P = env1.P
    ctx = she.Context(P, env1.ck, device=0, **ENGINE_OPTS[engine])
    assert she.br_engine(ctx) == {"ntt": 0, "fft3": 3, "fft2x2": 2, "fft-v1": 4,
                                  "fft-2groups": 4, "fft5-noprefetch": 5, "ks-imma": 8,
                                  "ks-cuda": 8, "fft-v3": 4, "fft5-v3": 5, "ks-tcgen05": 8,
                                  "fft-2streams": 4, "fft-smem": 4, "fft-tmem-stagger": 8,
                                  "fft-tmem-v2": 8, "fft-tmem-static": 8, "fft-tmem-chunk7": 8,
                                  "fft-tmem-chunk32": 8, "fft-tmem-wrap": 8,
                                  "fft-tmem-chunk499": 8}[engine]
    ops, bits, (a, b, c), _ = config1_outputs
    out = torch.zeros((a.shape[0], P.stride), dtype=torch.int32, device="cuda")
    she.she_gate_batch_ops(ctx, dev(np.asarray(ops, np.uint8)), dev(a), dev(b), dev(c), out)
    torch.cuda.synchronize()
    got = host(out)
    rows = read_digests(1)
    bad = [g for g, op, d, bit in rows if digest(got[g, : P.n + 1]) != d]
    assert not bad, f"{engine}: {len(bad)} gates differ from the oracle, first {bad[:8]}"
    ctx.close()


@pytest.mark.parametrize("chunk", [0, -2], ids=["queue32", "wrap"])
@pytest.mark.parametrize("m", [148, 512, 800, 1000, 2000, 2008])
def test_config1_work_distribution_modes(cuda, env1, config1_outputs, m, chunk):
    """The TMEM engine's work distribution (csrc/tm_queue.h) on prefixes of
    config 1, against the oracle digests: 148 gates (one lane per pipeline,
    static), 512 and 800 gates (~600 / ~940 lanes: single lanes split in time),
    1000 gates (~1170 lanes: one pair per pipeline, static), 2000 and 2008
    gates (lane pairs split in time, an odd / an even lane count); with the
    default chunk queue and with the wrap-around schedule; each twice on the
    same context (the progress words are reset per launch)."""
    P = env1.P
    ops, bits, (a, b, c), _ = config1_outputs
    lanes = si.br_lanes(ops[:m])
    pipelines = 4 * torch.cuda.get_device_properties(0).multi_processor_count
    if m in (512, 800):
        assert pipelines < lanes <= 1.65 * pipelines
    if m >= 2000:
        assert lanes > 2 * pipelines and lanes % 2 == (1 if m == 2000 else 0)
    ctx = env1.ctx if chunk == 0 else she.Context(P, env1.ck, device=0, fft_chunk=chunk)
    rows = read_digests(1)
    for rep in range(2):
        out = torch.zeros((m, P.stride), dtype=torch.int32, device="cuda")
        she.she_gate_batch_ops(ctx, dev(np.asarray(ops[:m], np.uint8)), dev(a[:m]), dev(b[:m]),
                               dev(c[:m]), out)
        torch.cuda.synchronize()
        got = host(out)
        bad = [g for g, op, d, bit in rows[:m] if digest(got[g, : P.n + 1]) != d]
        assert not bad, f"{len(bad)} gates differ from the oracle, first {bad[:8]}"
    if chunk:
        ctx.close()


def env0_ctx():
    if 0 not in _envs:
        _envs[0] = Env(0)
    return _envs[0].ctx


def test_config1_sampled_live_oracle(env1, config1_outputs):
    ops, bits, (a, b, c), out = config1_outputs
    rng = np.random.default_rng(si.sample_seed(1))
    pick = np.sort(rng.choice(4096, 6, replace=False))
    pick = np.union1d(pick, np.nonzero(ops == si.MUX)[0][:2])
    ref = oracle.gates(env1.K, ops[pick], a[pick], b[pick], c[pick])
    assert np.array_equal(out[pick], ref)


def test_config1_noise_variance(env1, config1_outputs):
    """Output noise of 4096 GPU gates vs the closed form (tests/test_oracle_pins)."""
    from test_oracle_pins import predicted_variance
    P = env1.P
    ops, bits, _, out = config1_outputs
    K = env1.K
    want = np.array([si.truth(o, *b) for o, b in zip(ops, bits)])
    ph = oracle.phases(P, K.s, out).astype(np.int64)
    ph = np.where(ph >= 1 << 31, ph - (1 << 32), ph)
    err = (ph - np.where(want == 1, MU, -MU)).astype(np.float64) / 2.0 ** 32
    for mux in (False, True):
        sel = (ops == si.MUX) if mux else (ops != si.MUX)
        pred = predicted_variance(P, int(K.s.sum()), int(K.S.sum()), mux)
        assert abs(np.var(err[sel]) / pred - 1) < 0.15, (mux, np.var(err[sel]), pred)


def test_host_buffer_api_matches_device_api(env1, config1_outputs):
    ops, bits, (a, b, c), out = config1_outputs
    sel = slice(0, 300)
    o2 = np.zeros_like(a[sel])
    she.she_gate_batch_ops_host(env1.ctx, np.ascontiguousarray(ops[sel]), a[sel].copy(),
                                b[sel].copy(), c[sel].copy(), o2)
    assert np.array_equal(o2, out[sel])


def test_bad_arguments_raise(env1):
    P = env1.P
    x = torch.zeros((4, P.stride), dtype=torch.int32, device="cuda")
    with pytest.raises(she.SheError):
        she.she_gate_batch(env1.ctx, 99, x, x, x, torch.zeros_like(x))
    with pytest.raises(she.SheError):
        she.she_gate_batch(env1.ctx, si.AND, x, x, x, x)  # out overlaps inputs



# ----------------------------------------------------------------------------
# client side on the GPU
# ----------------------------------------------------------------------------

@pytest.mark.parametrize("cfg", [0, 1])
def test_gpu_client_matches_host_client(cuda, cfg):
    """Device encryption (masks drawn on the GPU from the shared counter-based
    stream, host-drawn noise) is bit-identical to the ORACLE's encryption
    (oracle.encrypt from the oracle's own keygen of the same seed: an
    independent implementation of R4) and to she_encrypt_bits; device
    decryption equals the oracle's decryption and the host decryption."""
    P = si.CONFIG_PARAMS[cfg]
    sk, _ = she.she_keygen(P, si.key_seed(cfg))
    rng = np.random.default_rng(cfg + 50)
    count = 6272 if cfg == 1 else 1000  # the MNIST image's 784 x 8 bit ciphertexts
    bits = rng.integers(0, 2, count).astype(np.uint8)
    host_ct = she.she_encrypt_bits(sk, bits, 5151, 7)
    noise = she.she_encrypt_noise(sk, count, 5151, 7)
    d_bits = torch.from_numpy(bits).cuda()
    d_noise = torch.from_numpy(noise.view(np.int32)).cuda()
    d_ct = she.she_encrypt_bits_gpu(sk, d_bits, d_noise, 5151, 7)
    torch.cuda.synchronize()
    K = oracle.keygen(P, si.key_seed(cfg))
    ref = oracle.encrypt(P, K.s, bits, 5151, 7)
    assert np.array_equal(host(d_ct), ref), "GPU encryption differs from oracle.encrypt"
    assert np.array_equal(host(d_ct), host_ct)
    back = she.she_decrypt_bits_gpu(sk, d_ct)
    torch.cuda.synchronize()
    assert np.array_equal(back.cpu().numpy(), bits)
    assert np.array_equal(oracle.decrypt(P, K.s, host(d_ct)), bits)
    assert np.array_equal(she.she_decrypt_bits(sk, host_ct), bits)



@pytest.mark.parametrize("ks", ["general", "cuda", "imma", "tcgen05"])
def test_key_switch_kernels_c0(cuda, ks):
    """Every key-switch kernel on the config-0 gates (n = 128: an LWE slot of
    160 words, 5 column tiles of the tensor-core GEMM): bit-exact with the
    oracle.  "general" is ks_kernel (any base / t), "cuda" ks2_kernel, "imma"
    the tensor-core product (ks_imma.cuh)."""
    cfg, count = 0, 16
    P = si.CONFIG_PARAMS[cfg]
    sk, ck = she.she_keygen(P, si.key_seed(cfg))
    ctx = she.Context(P, ck, device=0, ks_kernel=ks)
    ops = si.gate_ops(cfg, count)
    bits = si.gate_input_bits(cfg, count)
    cts = she.she_encrypt_bits(sk, bits.ravel(), si.input_seed(cfg), 0).reshape(count, 3, -1)
    a, b, c = (np.ascontiguousarray(cts[:, j]) for j in range(3))
    out = torch.zeros((count, P.stride), dtype=torch.int32, device="cuda")
    she.she_gate_batch_ops(ctx, dev(ops), dev(a), dev(b), dev(c), out)
    torch.cuda.synchronize()
    K = oracle.keygen(P, si.key_seed(cfg))
    assert np.array_equal(host(out), oracle.gates(K, ops, a, b, c))
    ctx.close()


def test_tensor_core_key_switch_multi_pass_c0(cuda):
    """8,300 config-0 gates: the tensor-core key switch runs in passes of 8,192
    gates (kKsiBatch) with a ragged last pass; every output equals the CUDA-core
    ks2 path's (itself pinned to the oracle above), and a seed-sampled subset
    equals the oracle directly."""
    cfg, count = 0, 8300
    P = si.CONFIG_PARAMS[cfg]
    sk, ck = she.she_keygen(P, si.key_seed(cfg))
    ops = si.gate_ops(cfg, count)
    bits = si.gate_input_bits(cfg, count)
    cts = she.she_encrypt_bits(sk, bits.ravel(), si.input_seed(cfg), 0).reshape(count, 3, -1)
    a, b, c = (np.ascontiguousarray(cts[:, j]) for j in range(3))
    outs = {}
    for ks in ("imma", "cuda", "tcgen05"):
        ctx = she.Context(P, ck, device=0, ks_kernel=ks)
        out = torch.zeros((count, P.stride), dtype=torch.int32, device="cuda")
        she.she_gate_batch_ops(ctx, torch.from_numpy(ops.astype(np.uint8)).cuda(), dev(a), dev(b),
                               dev(c), out)
        torch.cuda.synchronize()
        outs[ks] = host(out)
        ctx.close()
    assert np.array_equal(outs["imma"], outs["cuda"])
    assert np.array_equal(outs["tcgen05"], outs["cuda"])
    rng = np.random.default_rng(si.sample_seed(0) + 3)
    pick = np.sort(rng.choice(count, 24, replace=False))
    pick[-1] = count - 1  # the last gate of the ragged pass
    K = oracle.keygen(P, si.key_seed(cfg))
    ref = oracle.gates(K, ops[pick], a[pick], b[pick], c[pick])
    assert np.array_equal(outs["imma"][pick], ref)
    want = np.array([si.truth(o, *bb) for o, bb in zip(ops, bits)])
    assert np.array_equal(she.she_decrypt_bits(sk, outs["imma"]), want)
