"""CPU oracle for SHE's bootstrapped-gate hot path — TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` legs may import this package.  The product
(``paper_1906_00148_b200``) never imports it and shares no code with it (the
only common file is the seeded input generator ``she_inputs/she_rng.h``).

``oracle.c`` is plain C: schoolbook negacyclic products mod 2^32, one function
per step of TFHE gate bootstrapping (
readings R1-R10 of SURVEY.md §8(c) / DESIGN.md §2).  ``network.py`` is the
plaintext integer shift-accumulate network.

Pins: tests/test_oracle_pins.py (brute-force truth tables, closed forms,
bounds, noise variance).  Functions with no pin say "parity unpinned" here and
in DESIGN.md — currently none.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "oracle.c")
ROOT = os.path.dirname(HERE)

# Two builds: AVX-512 (x86-64-v4) and AVX2 (x86-64-v3); the GPU box's host CPU
# may differ from the build box.  No -ffast-math; -ffp-contract=off keeps the
# shared Gaussian sampler bit-identical to the product client library.
_VARIANTS = {"v4": "-march=x86-64-v4", "v3": "-march=x86-64-v3"}
CFLAGS = ["-O3", "-fopenmp", "-fPIC", "-shared", "-ffp-contract=off", "-std=c11"]


def lib_path(variant: str) -> str:
    return os.path.join(HERE, f"liboracle_{variant}.so")


def build(force: bool = False) -> None:
    for v, march in _VARIANTS.items():
        out = lib_path(v)
        if not force and os.path.exists(out) and os.path.getmtime(out) >= max(
                os.path.getmtime(SRC),
                os.path.getmtime(os.path.join(ROOT, "she_inputs", "she_rng.h"))):
            continue
        cmd = ["gcc", *CFLAGS, march, SRC, "-o", out, "-lm"]
        subprocess.run(cmd, check=True)


def _cpu_has_avx512() -> bool:
    try:
        with open("/proc/cpuinfo") as f:
            flags = f.read()
        return all(x in flags for x in ("avx512f", "avx512bw", "avx512vl", "avx512dq"))
    except OSError:
        return False


COMPILER_FLAGS = " ".join(CFLAGS)
MU = 1 << 29  # +-1/8 on the 2^32 torus scale (R4)
_lib = None


def lib() -> ctypes.CDLL:
    global _lib
    if _lib is None:
        build()
        variant = "v4" if _cpu_has_avx512() else "v3"
        _lib = ctypes.CDLL(lib_path(variant))
        _setup(_lib)
        _lib.variant = variant
    return _lib


class OrcParams(ctypes.Structure):
    _fields_ = [("N", ctypes.c_uint32), ("k", ctypes.c_uint32), ("n", ctypes.c_uint32),
                ("bg_bits", ctypes.c_uint32), ("l", ctypes.c_uint32),
                ("ks_base_bits", ctypes.c_uint32), ("ks_t", ctypes.c_uint32),
                ("alpha_lwe", ctypes.c_double), ("alpha_bk", ctypes.c_double)]


def _p(params) -> OrcParams:
    return OrcParams(params.N, params.k, params.n, params.bg_bits, params.l,
                     params.ks_base_bits, params.ks_t, params.alpha_lwe, params.alpha_bk)


_u8p = ctypes.POINTER(ctypes.c_uint8)
_u32p = ctypes.POINTER(ctypes.c_uint32)
_i32p = ctypes.POINTER(ctypes.c_int32)
_pp = ctypes.POINTER(OrcParams)


def _setup(L):
    L.orc_threads.restype = ctypes.c_int
    L.orc_negacyclic_mul.argtypes = [ctypes.c_uint32, _i32p, _u32p, _u32p]
    L.orc_rotate.argtypes = [ctypes.c_uint32, ctypes.c_uint32, _u32p, _u32p]
    L.orc_decompose.argtypes = [_pp, ctypes.c_uint32, _i32p]
    L.orc_modswitch.argtypes = [ctypes.c_uint32, ctypes.c_uint32]
    L.orc_modswitch.restype = ctypes.c_uint32
    L.orc_phase.argtypes = [ctypes.c_uint32, _u8p, _u32p]
    L.orc_phase.restype = ctypes.c_uint32
    L.orc_keygen.argtypes = [_pp, ctypes.c_uint64, _u8p, _u8p, _u32p, _u32p]
    L.orc_encrypt.argtypes = [_pp, _u8p, _u8p, ctypes.c_size_t, ctypes.c_uint64,
                              ctypes.c_uint64, ctypes.c_size_t, _u32p]
    L.orc_decrypt.argtypes = [_pp, _u8p, _u32p, ctypes.c_size_t, ctypes.c_size_t, _u8p]
    L.orc_blind_rotate.argtypes = [_pp, _u32p, _u32p, _u32p]
    L.orc_extract.argtypes = [ctypes.c_uint32, _u32p, _u32p]
    L.orc_keyswitch.argtypes = [_pp, _u32p, _u32p, _u32p]
    L.orc_gate.argtypes = [_pp, _u32p, _u32p, ctypes.c_int, _u32p, _u32p, _u32p,
                           ctypes.c_size_t, _u32p]
    L.orc_gates.argtypes = [_pp, _u32p, _u32p, _u8p, _u32p, _u32p, _u32p, ctypes.c_size_t,
                            ctypes.c_size_t, _u32p, ctypes.c_int]
    L.orc_lvl_encrypt_sel.argtypes = [_pp, _u8p, _u8p, ctypes.c_size_t, ctypes.c_uint64,
                                      ctypes.c_uint64, _u32p]
    L.orc_lvl_cmux.argtypes = [_pp, _u32p, _u32p, _u32p, _u32p]
    L.orc_lvl_cmux_batch.argtypes = [_pp, _u32p, _u32p, _u32p, _u32p, ctypes.c_size_t, _u32p]
    L.orc_lvl_decrypt.argtypes = [_pp, _u8p, _u32p, ctypes.c_size_t, _u8p]


def _ptr(a: np.ndarray, t):
    assert a.flags["C_CONTIGUOUS"]
    return a.ctypes.data_as(t)


def threads() -> int:
    return int(lib().orc_threads())


# ---- primitives -------------------------------------------------------------

def negacyclic_mul(d: np.ndarray, b: np.ndarray) -> np.ndarray:
    d = np.ascontiguousarray(d, dtype=np.int32)
    b = np.ascontiguousarray(b, dtype=np.uint32)
    out = np.zeros(len(b), dtype=np.uint32)
    lib().orc_negacyclic_mul(len(b), _ptr(d, _i32p), _ptr(b, _u32p), _ptr(out, _u32p))
    return out


def rotate(p: np.ndarray, a: int) -> np.ndarray:
    p = np.ascontiguousarray(p, dtype=np.uint32)
    out = np.zeros_like(p)
    lib().orc_rotate(len(p), a, _ptr(p, _u32p), _ptr(out, _u32p))
    return out


def decompose(params, x: int) -> np.ndarray:
    d = np.zeros(params.l, dtype=np.int32)
    lib().orc_decompose(ctypes.byref(_p(params)), ctypes.c_uint32(x & 0xFFFFFFFF), _ptr(d, _i32p))
    return d


def modswitch(N: int, x: int) -> int:
    return int(lib().orc_modswitch(N, x & 0xFFFFFFFF))


def phase(params, s: np.ndarray, ct: np.ndarray) -> int:
    s = np.ascontiguousarray(s, dtype=np.uint8)
    ct = np.ascontiguousarray(ct, dtype=np.uint32)
    return int(lib().orc_phase(params.n, _ptr(s, _u8p), _ptr(ct, _u32p)))


def phases(params, s: np.ndarray, cts: np.ndarray) -> np.ndarray:
    """Vectorised phase b - <a, s> mod 2^32 of an array of LWE slots."""
    cts = np.asarray(cts, dtype=np.uint32)
    a = cts[..., : params.n].astype(np.uint64)
    dot = (a * np.asarray(s, dtype=np.uint64)).sum(axis=-1) & 0xFFFFFFFF
    return ((cts[..., params.n].astype(np.uint64) - dot) & 0xFFFFFFFF).astype(np.uint32)


# ---- client -----------------------------------------------------------------

class Keys:
    def __init__(self, params, s, S, bk, ksk):
        self.params, self.s, self.S, self.bk, self.ksk = params, s, S, bk, ksk


def keygen(params, seed: int) -> Keys:
    P = params
    base = 1 << P.ks_base_bits
    s = np.zeros(P.n, dtype=np.uint8)
    S = np.zeros(P.N, dtype=np.uint8)
    bk = np.zeros(P.n * 2 * P.l * 2 * P.N, dtype=np.uint32)
    ksk = np.zeros(P.N * P.ks_t * base * (P.n + 1), dtype=np.uint32)
    lib().orc_keygen(ctypes.byref(_p(P)), seed, _ptr(s, _u8p), _ptr(S, _u8p), _ptr(bk, _u32p),
                     _ptr(ksk, _u32p))
    return Keys(P, s, S, bk, ksk)


def encrypt(params, s, bits, seed: int, first_index: int = 0, stride: int | None = None):
    stride = stride or params.stride
    bits = np.ascontiguousarray(bits, dtype=np.uint8).ravel()
    out = np.zeros((len(bits), stride), dtype=np.uint32)
    lib().orc_encrypt(ctypes.byref(_p(params)), _ptr(np.ascontiguousarray(s, np.uint8), _u8p),
                      _ptr(bits, _u8p), len(bits), seed, first_index, stride, _ptr(out, _u32p))
    return out


def encrypt_ordinals(params, s, bits, seed: int, ordinals, stride: int | None = None):
    """Encrypt bits[i] as ciphertext number ordinals[i] (arbitrary numbering)."""
    stride = stride or params.stride
    bits = np.asarray(bits, dtype=np.uint8).ravel()
    ordinals = np.asarray(ordinals, dtype=np.uint64).ravel()
    out = np.zeros((len(bits), stride), dtype=np.uint32)
    # runs of consecutive ordinals are encrypted in one call
    i = 0
    while i < len(bits):
        j = i + 1
        while j < len(bits) and ordinals[j] == ordinals[j - 1] + 1:
            j += 1
        out[i:j] = encrypt(params, s, bits[i:j], seed, int(ordinals[i]), stride)
        i = j
    return out


def decrypt(params, s, cts) -> np.ndarray:
    cts = np.ascontiguousarray(cts, dtype=np.uint32)
    count = cts.shape[0]
    bits = np.zeros(count, dtype=np.uint8)
    lib().orc_decrypt(ctypes.byref(_p(params)), _ptr(np.ascontiguousarray(s, np.uint8), _u8p),
                      _ptr(cts, _u32p), count, cts.shape[1], _ptr(bits, _u8p))
    return bits


# ---- server steps -----------------------------------------------------------

def blind_rotate(keys: Keys, ct: np.ndarray) -> np.ndarray:
    P = keys.params
    ct = np.ascontiguousarray(ct, dtype=np.uint32)
    acc = np.zeros(2 * P.N, dtype=np.uint32)
    lib().orc_blind_rotate(ctypes.byref(_p(P)), _ptr(keys.bk, _u32p), _ptr(ct, _u32p),
                           _ptr(acc, _u32p))
    return acc


def extract(N: int, acc: np.ndarray) -> np.ndarray:
    acc = np.ascontiguousarray(acc, dtype=np.uint32)
    out = np.zeros(N + 1, dtype=np.uint32)
    lib().orc_extract(N, _ptr(acc, _u32p), _ptr(out, _u32p))
    return out


def keyswitch(keys: Keys, ext: np.ndarray) -> np.ndarray:
    P = keys.params
    ext = np.ascontiguousarray(ext, dtype=np.uint32)
    out = np.zeros(P.n + 1, dtype=np.uint32)
    lib().orc_keyswitch(ctypes.byref(_p(P)), _ptr(keys.ksk, _u32p), _ptr(ext, _u32p),
                        _ptr(out, _u32p))
    return out


def gates(keys: Keys, ops, a, b, c, nthreads: int = 0) -> np.ndarray:
    """Batch of gates; a, b, c: (count, stride) uint32 LWE slots."""
    P = keys.params
    ops = np.ascontiguousarray(ops, dtype=np.uint8)
    a = np.ascontiguousarray(a, dtype=np.uint32)
    b = np.ascontiguousarray(b, dtype=np.uint32)
    c = np.ascontiguousarray(c, dtype=np.uint32)
    count, stride = a.shape
    out = np.zeros((count, stride), dtype=np.uint32)
    if count:
        lib().orc_gates(ctypes.byref(_p(P)), _ptr(keys.bk, _u32p), _ptr(keys.ksk, _u32p),
                        _ptr(ops, _u8p), _ptr(a, _u32p), _ptr(b, _u32p), _ptr(c, _u32p),
                        count, stride, _ptr(out, _u32p), nthreads)
    return out


# ---- leveled mode (NEXT-2; reading R-LV) ------------------------------

def lvl_encrypt_sel(params, S, bits, seed: int, first: int = 0) -> np.ndarray:
    """Selectors TRGSW_S(bit): uint32 [count][2l][2][N] (streams 9, 10)."""
    bits = np.ascontiguousarray(bits, dtype=np.uint8).ravel()
    S = np.ascontiguousarray(S, dtype=np.uint8)
    out = np.zeros((len(bits), 2 * params.l, 2, params.N), dtype=np.uint32)
    if len(bits):
        lib().orc_lvl_encrypt_sel(ctypes.byref(_p(params)), _ptr(S, _u8p), _ptr(bits, _u8p),
                                  len(bits), seed, first, _ptr(out, _u32p))
    return out


def lvl_cmux(params, sel, d1, d0) -> np.ndarray:
    """CMux(sel, d1, d0) = d0 + sel [x] (d1 - d0) on TRLWE data [2][N]."""
    sel = np.ascontiguousarray(sel, dtype=np.uint32)
    d1 = np.ascontiguousarray(d1, dtype=np.uint32)
    d0 = np.ascontiguousarray(d0, dtype=np.uint32)
    out = np.zeros((2, params.N), dtype=np.uint32)
    lib().orc_lvl_cmux(ctypes.byref(_p(params)), _ptr(sel, _u32p), _ptr(d1, _u32p),
                       _ptr(d0, _u32p), _ptr(out, _u32p))
    return out


def lvl_cmux_batch(params, sels, sel_idx, d1, d0) -> np.ndarray:
    sels = np.ascontiguousarray(sels, dtype=np.uint32)
    sel_idx = np.ascontiguousarray(sel_idx, dtype=np.uint32)
    d1 = np.ascontiguousarray(d1, dtype=np.uint32)
    d0 = np.ascontiguousarray(d0, dtype=np.uint32)
    out = np.zeros_like(d1)
    if len(sel_idx):
        lib().orc_lvl_cmux_batch(ctypes.byref(_p(params)), _ptr(sels, _u32p), _ptr(sel_idx, _u32p),
                                 _ptr(d1, _u32p), _ptr(d0, _u32p), len(sel_idx), _ptr(out, _u32p))
    return out


def lvl_decrypt(params, S, cts) -> np.ndarray:
    cts = np.ascontiguousarray(cts, dtype=np.uint32)
    S = np.ascontiguousarray(S, dtype=np.uint8)
    c2 = cts.reshape(-1, 2 * params.N)
    bits = np.zeros(c2.shape[0], dtype=np.uint8)
    if len(bits):
        lib().orc_lvl_decrypt(ctypes.byref(_p(params)), _ptr(S, _u8p), _ptr(c2, _u32p), len(bits),
                              _ptr(bits, _u8p))
    return bits.reshape(cts.shape[:-2])


def lvl_trivial(params, bits) -> np.ndarray:
    """Noiseless TRLWE data (A = 0, B = +-1/8 on the constant coefficient)."""
    bits = np.asarray(bits, dtype=np.uint8).ravel()
    out = np.zeros((len(bits), 2, params.N), dtype=np.uint32)
    out[:, 1, 0] = np.where(bits == 1, MU, (1 << 32) - MU).astype(np.uint32)
    return out
