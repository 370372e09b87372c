"""CPU tests of the product library's host side (no GPU needed).

  * libshe.so loads and exports every function include/she.h declares;
  * the product client (keygen / encrypt / decrypt, csrc/client.cpp) produces
    byte-identical keys and ciphertexts to the oracle's independent client
    (oracle/oracle.c) from the same seeds — so the GPU path and the oracle
    consume identical inputs;
  * the device arithmetic, compiled for the host (csrc/host_emu.cpp runs the
    same __host__ __device__ step functions as the sm_100a kernel), is
    bit-exact with the oracle's schoolbook: the negacyclic NTT product
    (random and extreme inputs) and a whole blind rotation at C0 and C1.
"""
import ctypes
import os
import re

import numpy as np
import pytest

import oracle
import she_inputs as si
from paper_1906_00148_b200 import build, she

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module", autouse=True)
def built():
    build.build()


def test_library_exports_every_declared_symbol():
    header = open(os.path.join(ROOT, "include", "she.h")).read()
    header = re.sub(r"/\*.*?\*/", "", header, flags=re.S)
    names = sorted(set(re.findall(r"\b(she_[a-z0-9_]+)\s*\(", header)))
    assert len(names) >= 20
    lib = ctypes.CDLL(build.LIB)
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing


@pytest.mark.parametrize("params", [si.C0, si.C1], ids=["C0", "C1"])
def test_client_keys_match_oracle_bytes(params):
    sk, ck = she.she_keygen(params, 4321)
    K = oracle.keygen(params, 4321)
    skb = np.frombuffer(sk.export(), dtype=np.uint8)
    assert np.array_equal(skb[: params.n], K.s) and np.array_equal(skb[params.n:], K.S)
    w = ck.export()
    assert np.array_equal(w[: len(K.bk)], K.bk)
    assert np.array_equal(w[len(K.bk):], K.ksk)
    ck2 = she.CloudKey.import_(params, w)
    assert np.array_equal(ck2.export(), w)


@pytest.mark.parametrize("params", [si.C0, si.C1], ids=["C0", "C1"])
def test_client_encrypt_decrypt_matches_oracle(params):
    sk, _ = she.she_keygen(params, 99)
    K = oracle.keygen(params, 99)
    bits = np.random.default_rng(1).integers(0, 2, 500).astype(np.uint8)
    c1 = she.she_encrypt_bits(sk, bits, seed=7, first_index=123)
    c2 = oracle.encrypt(params, K.s, bits, 7, 123)
    assert np.array_equal(c1, c2)
    assert np.array_equal(she.she_decrypt_bits(sk, c1), bits)
    assert np.array_equal(she.she_decrypt_bits(sk, c2), oracle.decrypt(params, K.s, c2))


def test_bad_params_rejected():
    from dataclasses import replace
    for bad in (replace(si.C1, N=512), replace(si.C1, l=3), replace(si.C1, k=2),
                replace(si.C1, ks_base_bits=3)):
        with pytest.raises(she.SheError):
            she.she_keygen(bad, 1)


# ---- host emulation of the device arithmetic --------------------------------

def emu():
    L = ctypes.CDLL(build.build_emu())
    L.she_emu_gl_mul.restype = ctypes.c_uint64
    L.she_emu_gl_mul.argtypes = [ctypes.c_uint64] * 2
    L.she_emu_gl_mul_pow2.restype = ctypes.c_uint64
    L.she_emu_gl_mul_pow2.argtypes = [ctypes.c_uint64, ctypes.c_int]
    for f in ("she_emu_gl_add", "she_emu_gl_sub", "she_emu_gl_add_le", "she_emu_gl_sub_le"):
        getattr(L, f).restype = ctypes.c_uint64
        getattr(L, f).argtypes = [ctypes.c_uint64] * 2
    L.she_emu_gl_shl_le.restype = ctypes.c_uint64
    L.she_emu_gl_shl_le.argtypes = [ctypes.c_uint64, ctypes.c_int]
    L.she_emu_gl_lift32_neg.restype = ctypes.c_uint32
    L.she_emu_gl_lift32_neg.argtypes = [ctypes.c_uint64]
    return L


P64 = 2 ** 64 - 2 ** 32 + 1


def test_goldilocks_field_ops():
    L = emu()
    rng = np.random.default_rng(0)
    edge = [0, 1, 2, P64 - 1, P64, P64 + 1, 2 ** 64 - 1, 2 ** 63, 2 ** 32 - 1, 2 ** 32]
    vals = edge + [int(v) for v in rng.integers(0, 2 ** 63, 200, dtype=np.uint64) * 2 + 1]
    for a in vals[:40]:
        for b in vals[:40]:
            assert L.she_emu_gl_mul(a, b) == a * b % P64
            assert L.she_emu_gl_add(a, b) == (a + b) % P64
            assert L.she_emu_gl_sub(a, b) == (a - b) % P64
    for s in range(192):
        for x in vals[:16]:
            assert L.she_emu_gl_mul_pow2(x, s) == x * pow(2, s, P64) % P64, (s, x)


def test_bounded_butterfly_primitives():
    """shl_le: v 2^s mod p with the result <= p for EVERY 64-bit v (the bound the
    single-fold add_le / sub_le rely on); add_le / sub_le exact for y <= p;
    lift32_neg(t) = centred lift of -t.  Edge values hit every fold branch."""
    L = emu()
    rng = np.random.default_rng(1)
    edge = [0, 1, 2, 2 ** 32 - 2, 2 ** 32 - 1, 2 ** 32, 2 ** 32 + 1, P64 - 2, P64 - 1, P64,
            P64 + 1, 2 ** 64 - 2, 2 ** 64 - 1, 2 ** 63, 2 ** 63 - 1, 0xFFFFFFFF00000000,
            0xFFFFFFFEFFFFFFFF, 0x80000000FFFFFFFF, 0x7FFFFFFF80000000, 0x00000001FFFFFFFF]
    rand = [int(v) for v in rng.integers(0, 2 ** 64 - 1, 60, dtype=np.uint64)]
    hi_max = [(v | 0xFFFFFFFF00000000) for v in rand[:20]]
    lo_small = [(v & 0xFFFFFFFF00000000) | k for k, v in enumerate(rand[20:40])]
    vals = edge + rand + hi_max + lo_small
    for s in range(96):
        for v in vals:
            t = L.she_emu_gl_shl_le(v, s)
            assert t <= P64 and t % P64 == v * pow(2, s, P64) % P64, (s, v)
    ys = [y for y in vals if y <= P64]
    for x in vals:
        for y in ys:
            a, d = L.she_emu_gl_add_le(x, y), L.she_emu_gl_sub_le(x, y)
            assert a % P64 == (x + y) % P64 and d % P64 == (x - y) % P64, (x, y)
    half = (P64 - 1) // 2
    for t in ys + [half, half + 1, half + 2]:
        y = (-t) % P64
        want = (y - P64 if y > half else y) % 2 ** 32
        assert L.she_emu_gl_lift32_neg(t) == want, t


@pytest.mark.parametrize("N", [256, 1024])
def test_device_ntt_product_matches_schoolbook(N):
    L = emu()
    rng = np.random.default_rng(N)
    u32p = ctypes.POINTER(ctypes.c_uint32)
    i32p = ctypes.POINTER(ctypes.c_int32)
    half = 512 if N == 1024 else 128
    cases = [(rng.integers(-half, half, N), rng.integers(0, 2 ** 32, N, dtype=np.uint64))]
    for dv in (-half, half - 1):
        for bv in (0, 2 ** 31, 2 ** 32 - 1):
            cases.append((np.full(N, dv), np.full(N, bv, dtype=np.uint64)))
    for d, b in cases:
        d = np.ascontiguousarray(d, dtype=np.int32)
        b = np.ascontiguousarray(b.astype(np.uint32))
        out = np.zeros(N, dtype=np.uint32)
        assert L.she_emu_negacyclic_mul(N, d.ctypes.data_as(i32p), b.ctypes.data_as(u32p),
                                        out.ctypes.data_as(u32p)) == 0
        assert np.array_equal(out, oracle.negacyclic_mul(d, b))


@pytest.mark.parametrize("params", [si.C0, si.C1], ids=["C0", "C1"])
def test_device_blind_rotation_matches_oracle(params):
    L = emu()
    u32p = ctypes.POINTER(ctypes.c_uint32)
    K = oracle.keygen(params, 1000)
    ct = oracle.encrypt(params, K.s, [1], 5)[0]
    acc = np.zeros(2 * params.N, dtype=np.uint32)
    assert L.she_emu_blind_rotate(params.N, params.n, params.l, params.bg_bits,
                                  K.bk.ctypes.data_as(u32p), ct.ctypes.data_as(u32p),
                                  acc.ctypes.data_as(u32p)) == 0
    assert np.array_equal(acc, oracle.blind_rotate(K, ct))



@pytest.mark.parametrize("params", [si.C0, si.C1], ids=["C0", "C1"])
def test_encrypt_noise_is_the_host_clients_noise(params):
    """she_encrypt_noise (the noise the GPU client is handed) equals the noise
    inside the host client's ciphertexts: e = b - <a, s> - (m ? mu : -mu)."""
    import oracle
    sk, _ = she.she_keygen(params, 7)
    bits = np.array([0, 1, 1, 0, 1] * 7, np.uint8)
    cts = she.she_encrypt_bits(sk, bits, 4242, 100)
    noise = she.she_encrypt_noise(sk, len(bits), 4242, 100)
    K = oracle.keygen(params, 7)
    mu = np.where(bits == 1, 1 << 29, (1 << 32) - (1 << 29)).astype(np.uint64)
    ph = oracle.phases(params, K.s, cts).astype(np.uint64)
    assert np.array_equal((ph - mu) % (1 << 32), noise.astype(np.uint64))


@pytest.mark.parametrize("opts, why", [
    (dict(engine="fft"), "FFT engine at N = 256"),
    (dict(engine="ntt", fft_lanes=3), "fft_lanes for the NTT engine"),
    (dict(ntt_shape=(9, 9)), "uninstantiated NTT shape"),
    (dict(fft_lanes=7), "unknown FFT lane count"),
    (dict(fft_chunk=32), "fft_chunk at N = 256 (NTT engine)"),
    (dict(fft_chunk=-3), "fft_chunk out of range"),
], ids=["fft-at-N256", "lanes-for-ntt", "shape-9x9", "lanes-7", "chunk-for-ntt", "chunk-range"])
def test_ctx_options_rejected_before_any_device_work(opts, why):
    """she_ctx_create_ex validates she_ctx_options on the host (SHE_ERR_ARG)
    before it touches CUDA, so these run without a GPU."""
    P = si.C0
    _, ck = she.she_keygen(P, 5)
    with pytest.raises(she.SheError) as e:
        she.Context(P, ck, device=0, **opts)
    assert e.value.status == -1, why


def test_ctx_options_reserved_and_params_checked():
    P = si.C0
    _, ck = she.she_keygen(P, 5)
    opt = she.she_ctx_options.of()
    opt.reserved[0] = 1
    h = ctypes.c_void_p()
    st = she.lib().she_ctx_create_ex(ctypes.byref(she.she_params.of(P)), ck.handle, 0, 0, 1,
                                     ctypes.byref(opt), ctypes.byref(h))
    assert st == -1
    import dataclasses
    big = dataclasses.replace(P, n=600)
    st = she.lib().she_ctx_create_ex(ctypes.byref(she.she_params.of(big)), ck.handle, 0, 0, 1,
                                     None, ctypes.byref(h))
    assert st == -2  # n > 511: SHE_ERR_PARAMS (include/she.h she_params)


@pytest.mark.parametrize("params", [si.C0, si.C1], ids=["C0", "C1"])
def test_ciphertext_serialization_roundtrip_and_size(params):
    """NEXT-4: the wire format carries n + 1 words per ciphertext (the paper's
    MSize arithmetic: bits x ciphertext bytes), round-trips
    bit for bit and is read by an independent parser (numpy) the same way."""
    sk, _ = she.she_keygen(params, 77)
    bits = np.random.default_rng(3).integers(0, 2, 100).astype(np.uint8)
    cts = she.she_encrypt_bits(sk, bits, 5, 0)
    data = she.serialize(params, cts)
    assert len(data) == 16 + 100 * (params.n + 1) * 4
    hdr = np.frombuffer(data[:8], dtype="<u4")
    assert hdr[0] == 0x43454853 and hdr[1] == params.n
    assert int(np.frombuffer(data[8:16], dtype="<u8")[0]) == 100
    body = np.frombuffer(data[16:], dtype="<u4").reshape(100, params.n + 1)
    assert np.array_equal(body, cts[:, : params.n + 1])
    back = she.deserialize(params, data)
    assert np.array_equal(back, cts)
    assert np.array_equal(she.she_decrypt_bits(sk, back), bits)
    with pytest.raises(she.SheError):
        she.deserialize(params, data[:-4])
    # the MNIST image of config 3: 784 pixels x 8 bit-wise ciphertexts
    assert she.lib().she_serialized_bytes(ctypes.byref(she.she_params.of(si.C1)), 6272) == \
        16 + 6272 * 501 * 4
