"""Thin Python binding of libshe.so (include/she.h): argument marshalling only.

Every step of the hot path runs in the CUDA kernels of libshe.so; this module
converts numpy arrays / torch tensors to pointers and raises on error.  There
is no CPU fallback: if libshe.so is missing or a call fails, it raises.

Device buffers are torch tensors of dtype int32 holding torch-allocated CUDA
memory (bit patterns of the uint32 torus words); host buffers are numpy
uint32 / uint8 arrays.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libshe.so")

SHE_AND, SHE_NAND, SHE_OR, SHE_NOR, SHE_XOR, SHE_XNOR, SHE_MUX, SHE_NOT, SHE_COPY = range(9)

_STATUS = {0: "SHE_OK", -1: "SHE_ERR_ARG", -2: "SHE_ERR_PARAMS", -3: "SHE_ERR_SHAPE",
           -4: "SHE_ERR_CUDA", -5: "SHE_ERR_NCCL", -6: "SHE_ERR_OOM", -7: "SHE_ERR_STATE"}


class SheError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{_STATUS.get(status, status)}: {msg}")
        self.status = status


class she_params(ctypes.Structure):
    _fields_ = [("N", ctypes.c_uint32), ("k", ctypes.c_uint32), ("n", ctypes.c_uint32),
                ("bg_bits", ctypes.c_uint32), ("l", ctypes.c_uint32),
                ("ks_base_bits", ctypes.c_uint32), ("ks_t", ctypes.c_uint32),
                ("alpha_lwe", ctypes.c_double), ("alpha_bk", ctypes.c_double)]

    @classmethod
    def of(cls, p) -> "she_params":
        return cls(p.N, p.k, p.n, p.bg_bits, p.l, p.ks_base_bits, p.ks_t, p.alpha_lwe, p.alpha_bk)


class she_ctx_options(ctypes.Structure):
    """include/she.h she_ctx_options: engine selection (all engines are exact)."""
    _fields_ = [("br_engine", ctypes.c_int), ("fft_lanes", ctypes.c_int),
                ("ntt_lanes", ctypes.c_int), ("ntt_ctas", ctypes.c_int),
                ("ks_kernel", ctypes.c_int), ("fft_variant", ctypes.c_int),
                ("fft_groups", ctypes.c_int), ("fft_prefetch", ctypes.c_int),
                ("fft_streams", ctypes.c_int), ("fft_store", ctypes.c_int),
                ("fft_stagger_ns", ctypes.c_int), ("fft_chunk", ctypes.c_int),
                ("reserved", ctypes.c_int * 1)]

    ENGINES = {"default": 0, "fft": 1, "ntt": 2}

    @classmethod
    def of(cls, engine="default", fft_lanes=0, ntt_shape=(0, 0), ks_kernel="default",
           fft_variant=0, fft_groups=0, fft_prefetch=0, fft_streams=0, fft_store="default",
           fft_stagger_ns=0, fft_chunk=0):
        return cls(cls.ENGINES[engine], fft_lanes, ntt_shape[0], ntt_shape[1],
                   {"default": 0, "general": 1, "cuda": 2, "imma": 3, "tcgen05": 4}[ks_kernel], fft_variant,
                   fft_groups, fft_prefetch, fft_streams,
                   {"default": 0, "smem": 1, "tmem": 2}[fft_store], fft_stagger_ns, fft_chunk)


class she_circuit_stats(ctypes.Structure):
    _fields_ = [(k, ctypes.c_uint64) for k in
                ("gates", "br_lanes", "levels", "max_level_width", "min_level_width", "tiles")]

    def as_dict(self) -> dict:
        return {k: int(getattr(self, k)) for k, _ in self._fields_}


_lib = None
_vp = ctypes.c_void_p
_sz = ctypes.c_size_t


def lib() -> ctypes.CDLL:
    """Load the in-tree libshe.so; raise (never fall back) if it is missing."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} missing: run paper_1906_00148_b200.build (no CPU fallback)")
        L = ctypes.CDLL(LIB_PATH)
        P = ctypes.POINTER(she_params)
        sig = {
            "she_lwe_stride": ([P], _sz),
            "she_last_error": ([], ctypes.c_char_p),
            "she_keygen": ([P, ctypes.c_uint64, ctypes.POINTER(_vp), ctypes.POINTER(_vp)], ctypes.c_int),
            "she_secret_key_free": ([_vp], None),
            "she_cloud_key_free": ([_vp], None),
            "she_secret_key_export": ([_vp, _vp, ctypes.POINTER(_sz)], ctypes.c_int),
            "she_cloud_key_export": ([_vp, _vp, ctypes.POINTER(_sz)], ctypes.c_int),
            "she_cloud_key_import": ([P, _vp, _sz, ctypes.POINTER(_vp)], ctypes.c_int),
            "she_encrypt_bits": ([_vp, _vp, _sz, ctypes.c_uint64, ctypes.c_uint64, _vp], ctypes.c_int),
            "she_decrypt_bits": ([_vp, _vp, _sz, _vp], ctypes.c_int),
            "she_ctx_create": ([P, _vp, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.POINTER(_vp)],
                               ctypes.c_int),
            "she_ctx_create_ex": ([P, _vp, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                   ctypes.POINTER(she_ctx_options), ctypes.POINTER(_vp)], ctypes.c_int),
            "she_ctx_destroy": ([_vp], ctypes.c_int),
            "she_ctx_synchronize": ([_vp], ctypes.c_int),
            "she_gate_batch": ([_vp, ctypes.c_int, _vp, _vp, _vp, _vp, _sz, _vp], ctypes.c_int),
            "she_gate_batch_ops": ([_vp, _vp, _vp, _vp, _vp, _vp, _sz, _vp], ctypes.c_int),
            "she_gate_batch_ops_host": ([_vp, _vp, _vp, _vp, _vp, _vp, _sz, _vp], ctypes.c_int),
            "she_gate_level": ([_vp, _vp, _vp, _vp, _vp, _sz, _vp], ctypes.c_int),
            "she_ctx_enable_timing": ([_vp, ctypes.c_int], ctypes.c_int),
            "she_ctx_timing": ([_vp, ctypes.c_int, ctypes.POINTER(ctypes.c_double),
                                ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_uint64),
                                ctypes.POINTER(ctypes.c_uint64)], ctypes.c_int),
            "she_bench_modmul_peak": ([ctypes.c_int, ctypes.POINTER(ctypes.c_double),
                                       ctypes.POINTER(ctypes.c_double)], ctypes.c_int),
            "she_bench_fp64_peak": ([ctypes.c_int, ctypes.POINTER(ctypes.c_double),
                                     ctypes.POINTER(ctypes.c_double)], ctypes.c_int),
            "she_ctx_br_engine": ([_vp, ctypes.POINTER(ctypes.c_int)], ctypes.c_int),
            "she_ctx_kernel_launches": ([_vp, ctypes.c_int, ctypes.POINTER(ctypes.c_uint64)], ctypes.c_int),
            "she_conv_shift_acc": ([_vp, _vp] + [ctypes.c_int] * 5 + [_vp] + [ctypes.c_int] * 6
                                   + [_vp, ctypes.POINTER(ctypes.c_int), _vp], ctypes.c_int),
            "she_fc_shift_acc": ([_vp, _vp, ctypes.c_int, ctypes.c_int, ctypes.c_int, _vp,
                                  ctypes.c_int, ctypes.c_int, ctypes.c_int, _vp,
                                  ctypes.POINTER(ctypes.c_int), _vp], ctypes.c_int),
            "she_conv_mul_acc": ([_vp, _vp] + [ctypes.c_int] * 5 + [_vp] + [ctypes.c_int] * 6
                                 + [_vp, ctypes.POINTER(ctypes.c_int), _vp], ctypes.c_int),
            "she_fc_mul_acc": ([_vp, _vp, ctypes.c_int, ctypes.c_int, ctypes.c_int, _vp,
                                ctypes.c_int, ctypes.c_int, ctypes.c_int, _vp,
                                ctypes.POINTER(ctypes.c_int), _vp], ctypes.c_int),
            "she_clear_conv_mul_acc": ([_vp] + [ctypes.c_int] * 5 + [_vp] + [ctypes.c_int] * 6
                                       + [_vp, ctypes.POINTER(ctypes.c_int), ctypes.c_int,
                                          ctypes.c_int, ctypes.POINTER(she_circuit_stats)],
                                       ctypes.c_int),
            "she_clear_fc_mul_acc": ([_vp, ctypes.c_int, ctypes.c_int, ctypes.c_int, _vp,
                                      ctypes.c_int, ctypes.c_int, ctypes.c_int, _vp,
                                      ctypes.POINTER(ctypes.c_int), ctypes.c_int, ctypes.c_int,
                                      ctypes.POINTER(she_circuit_stats)], ctypes.c_int),
            "she_relu": ([_vp, _vp, _sz, ctypes.c_int, _vp, _vp], ctypes.c_int),
            "she_bn_shift_add": ([_vp, _vp, _sz, ctypes.c_int, ctypes.c_int, ctypes.c_int, _vp,
                                  _vp, _vp, ctypes.c_int, ctypes.c_int, _vp,
                                  ctypes.POINTER(ctypes.c_int), _vp], ctypes.c_int),
            "she_clear_bn_shift_add": ([_vp, _sz, ctypes.c_int, ctypes.c_int, ctypes.c_int, _vp,
                                        _vp, _vp, ctypes.c_int, ctypes.c_int, _vp,
                                        ctypes.POINTER(ctypes.c_int), ctypes.c_int, ctypes.c_int,
                                        ctypes.POINTER(she_circuit_stats)], ctypes.c_int),
            "she_maxpool2x2": ([_vp, _vp] + [ctypes.c_int] * 5 + [_vp, _vp], ctypes.c_int),
            "she_ctx_layer_stats": ([_vp, ctypes.POINTER(she_circuit_stats)], ctypes.c_int),
            "she_field_selftest": ([ctypes.c_int, _vp, _vp, _vp, _sz, _vp], ctypes.c_int),
            "she_serialized_bytes": ([P, _sz], _sz),
            "she_lvl_encrypt_selectors": ([_vp, _vp, _sz, ctypes.c_uint64, ctypes.c_uint64, _vp],
                                          ctypes.c_int),
            "she_lvl_decrypt": ([_vp, _vp, _sz, _vp], ctypes.c_int),
            "she_lvl_selector_bytes": ([], _sz),
            "she_lvl_selectors_to_device": ([_vp, _vp, _sz, _vp, _vp], ctypes.c_int),
            "she_lvl_cmux_batch": ([_vp, _vp, _vp, _vp, _vp, _vp, _sz, _vp], ctypes.c_int),
            "she_lvl_unit": ([_vp, ctypes.c_int, _vp, _vp, _vp, _sz, ctypes.c_int, ctypes.c_int, _vp,
                              ctypes.POINTER(ctypes.c_uint64), ctypes.POINTER(ctypes.c_uint32), _vp],
                             ctypes.c_int),
            "she_serialize_ciphertexts": ([P, _vp, _sz, _vp, ctypes.POINTER(_sz)], ctypes.c_int),
            "she_deserialize_ciphertexts": ([P, _vp, _sz, _vp, _sz, ctypes.POINTER(_sz)],
                                            ctypes.c_int),
            "she_fft_product_selftest": ([ctypes.c_int, ctypes.c_int, _vp, _vp, _sz, _vp,
                                          ctypes.POINTER(ctypes.c_double)], ctypes.c_int),
            "she_encrypt_noise": ([_vp, _sz, ctypes.c_uint64, ctypes.c_uint64, _vp], ctypes.c_int),
            "she_encrypt_bits_gpu": ([_vp, _vp, _vp, _sz, ctypes.c_uint64, ctypes.c_uint64, _vp,
                                      ctypes.c_int, _vp], ctypes.c_int),
            "she_decrypt_bits_gpu": ([_vp, _vp, _sz, _vp, ctypes.c_int, _vp], ctypes.c_int),
            "she_ctx_capture": ([_vp, ctypes.c_uint64, ctypes.c_uint32, _sz], ctypes.c_int),
            "she_ctx_capture_read": ([_vp, _vp, _vp, _sz, ctypes.POINTER(_sz)], ctypes.c_int),
            "she_clear_conv_shift_acc": ([_vp] + [ctypes.c_int] * 5 + [_vp] + [ctypes.c_int] * 6
                                         + [_vp, ctypes.POINTER(ctypes.c_int), ctypes.c_int,
                                            ctypes.c_int, ctypes.POINTER(she_circuit_stats)],
                                         ctypes.c_int),
            "she_clear_fc_shift_acc": ([_vp, ctypes.c_int, ctypes.c_int, ctypes.c_int, _vp,
                                        ctypes.c_int, ctypes.c_int, ctypes.c_int, _vp,
                                        ctypes.POINTER(ctypes.c_int), ctypes.c_int, ctypes.c_int,
                                        ctypes.POINTER(she_circuit_stats)], ctypes.c_int),
            "she_clear_relu": ([_vp, _sz, ctypes.c_int, _vp, ctypes.c_int, ctypes.c_int,
                                ctypes.POINTER(she_circuit_stats)], ctypes.c_int),
            "she_clear_maxpool2x2": ([_vp] + [ctypes.c_int] * 5 + [_vp, ctypes.c_int, ctypes.c_int,
                                     ctypes.POINTER(she_circuit_stats)], ctypes.c_int),
        }
        for name, (args, res) in sig.items():
            fn = getattr(L, name)
            fn.argtypes = args
            fn.restype = res
        _lib = L
    return _lib


def _check(status: int) -> None:
    if status != 0:
        raise SheError(status, lib().she_last_error().decode(errors="replace"))


def _np_ptr(a: np.ndarray) -> int:
    assert a.flags["C_CONTIGUOUS"]
    return a.ctypes.data


def _dev_ptr(t) -> int | None:
    if t is None:
        return None
    if not t.is_cuda or not t.is_contiguous():
        raise ValueError("device buffers must be contiguous CUDA tensors")
    return t.data_ptr()


def _stream_ptr(stream) -> int | None:
    if stream is None:
        import torch
        return torch.cuda.current_stream().cuda_stream
    return getattr(stream, "cuda_stream", stream)


def stride(params) -> int:
    return int(lib().she_lwe_stride(ctypes.byref(she_params.of(params))))


# ---- client side -------------------------------------------------------------

class SecretKey:
    def __init__(self, handle: int, params):
        self.handle, self.params = handle, params

    def __del__(self):
        if getattr(self, "handle", None) and _lib is not None:
            _lib.she_secret_key_free(self.handle)
            self.handle = None

    def export(self) -> bytes:
        n = _sz(0)
        _check(lib().she_secret_key_export(self.handle, None, ctypes.byref(n)))
        buf = np.zeros(n.value, dtype=np.uint8)
        _check(lib().she_secret_key_export(self.handle, _np_ptr(buf), ctypes.byref(n)))
        return buf.tobytes()


class CloudKey:
    def __init__(self, handle: int, params):
        self.handle, self.params = handle, params

    def __del__(self):
        if getattr(self, "handle", None) and _lib is not None:
            _lib.she_cloud_key_free(self.handle)
            self.handle = None

    def export(self) -> np.ndarray:
        n = _sz(0)
        _check(lib().she_cloud_key_export(self.handle, None, ctypes.byref(n)))
        buf = np.zeros(n.value // 4, dtype=np.uint32)
        _check(lib().she_cloud_key_export(self.handle, _np_ptr(buf), ctypes.byref(n)))
        return buf

    @classmethod
    def import_(cls, params, words: np.ndarray) -> "CloudKey":
        words = np.ascontiguousarray(words, dtype=np.uint32)
        h = _vp()
        _check(lib().she_cloud_key_import(ctypes.byref(she_params.of(params)), _np_ptr(words),
                                          words.nbytes, ctypes.byref(h)))
        return cls(h.value, params)


def she_keygen(params, seed: int):
    sk, ck = _vp(), _vp()
    _check(lib().she_keygen(ctypes.byref(she_params.of(params)), seed, ctypes.byref(sk),
                            ctypes.byref(ck)))
    return SecretKey(sk.value, params), CloudKey(ck.value, params)


def she_encrypt_bits(sk: SecretKey, bits, seed: int, first_index: int = 0) -> np.ndarray:
    bits = np.ascontiguousarray(bits, dtype=np.uint8).ravel()
    out = np.zeros((len(bits), stride(sk.params)), dtype=np.uint32)
    if len(bits):
        _check(lib().she_encrypt_bits(sk.handle, _np_ptr(bits), len(bits), seed, first_index,
                                      _np_ptr(out)))
    return out


def she_decrypt_bits(sk: SecretKey, cts) -> np.ndarray:
    cts = np.ascontiguousarray(cts, dtype=np.uint32)
    cts2 = cts.reshape(-1, cts.shape[-1])
    assert cts2.shape[-1] == stride(sk.params)
    bits = np.zeros(cts2.shape[0], dtype=np.uint8)
    if len(bits):
        _check(lib().she_decrypt_bits(sk.handle, _np_ptr(cts2), cts2.shape[0], _np_ptr(bits)))
    return bits.reshape(cts.shape[:-1])


def serialize(params, cts) -> bytes:
    """Wire format of a ciphertext batch (she.h she_serialize_ciphertexts)."""
    cts = np.ascontiguousarray(cts, dtype=np.uint32).reshape(-1, stride(params))
    P = she_params.of(params)
    n = _sz(0)
    _check(lib().she_serialize_ciphertexts(ctypes.byref(P), None, cts.shape[0], None, ctypes.byref(n)))
    buf = np.zeros(n.value, dtype=np.uint8)
    _check(lib().she_serialize_ciphertexts(ctypes.byref(P), _np_ptr(cts), cts.shape[0], _np_ptr(buf),
                                           ctypes.byref(n)))
    return buf.tobytes()


def deserialize(params, data: bytes) -> np.ndarray:
    P = she_params.of(params)
    buf = np.frombuffer(data, dtype=np.uint8).copy()
    cnt = _sz(0)
    _check(lib().she_deserialize_ciphertexts(ctypes.byref(P), _np_ptr(buf), buf.size, None, 0,
                                             ctypes.byref(cnt)))
    out = np.zeros((max(cnt.value, 1), stride(params)), dtype=np.uint32)
    _check(lib().she_deserialize_ciphertexts(ctypes.byref(P), _np_ptr(buf), buf.size, _np_ptr(out),
                                             cnt.value, ctypes.byref(cnt)))
    return out[:cnt.value]


# ---- server side -------------------------------------------------------------

class Context:
    """she_ctx: device keys (BK in the engine's transform domain, KSK) on one
    CUDA device.  Keyword options (she_ctx_options): engine = "default" | "fft"
    | "ntt", fft_lanes, ntt_shape = (G, B), ks_kernel = "default" | "general"."""

    def __init__(self, params, ck: CloudKey, device: int = 0, rank: int = 0, world: int = 1,
                 **options):
        h = _vp()
        opt = she_ctx_options.of(**options)
        _check(lib().she_ctx_create_ex(ctypes.byref(she_params.of(params)), ck.handle, device, rank,
                                       world, ctypes.byref(opt), ctypes.byref(h)))
        self.handle, self.params, self.device = h.value, params, device
        self.stride = stride(params)

    def close(self):
        h = getattr(self, "handle", None)
        if h and lib is not None:  # module globals are gone at interpreter teardown
            lib().she_ctx_destroy(h)
            self.handle = None

    __del__ = close

    def synchronize(self):
        _check(lib().she_ctx_synchronize(self.handle))

    def enable_timing(self, on: bool = True):
        _check(lib().she_ctx_enable_timing(self.handle, int(on)))

    def timing(self, reset: bool = False) -> dict:
        br, ks = ctypes.c_double(), ctypes.c_double()
        nb, nk = ctypes.c_uint64(), ctypes.c_uint64()
        _check(lib().she_ctx_timing(self.handle, int(reset), ctypes.byref(br), ctypes.byref(ks),
                                    ctypes.byref(nb), ctypes.byref(nk)))
        return {"br_ms": br.value, "ks_ms": ks.value, "br_launches": nb.value,
                "ks_launches": nk.value}

    def kernel_launches(self, reset: bool = False) -> int:
        """Kernels launched by this context's gate passes (she_ctx_kernel_launches)."""
        c = ctypes.c_uint64()
        _check(lib().she_ctx_kernel_launches(self.handle, int(reset), ctypes.byref(c)))
        return c.value


def modmul_peak(device: int = 0) -> tuple[float, float]:
    """K6: measured Goldilocks modmul/s on all SMs (and the kernel's ms)."""
    r, ms = ctypes.c_double(), ctypes.c_double()
    _check(lib().she_bench_modmul_peak(device, ctypes.byref(r), ctypes.byref(ms)))
    return r.value, ms.value


def fp64_peak(device: int = 0) -> tuple[float, float]:
    """K7: measured FP64 instructions/s on all SMs (and the kernel's ms)."""
    r, ms = ctypes.c_double(), ctypes.c_double()
    _check(lib().she_bench_fp64_peak(device, ctypes.byref(r), ctypes.byref(ms)))
    return r.value, ms.value


def br_engine(ctx: Context) -> int:
    """G > 0: FP64 FFT blind rotation with G lanes per CTA; 0: Goldilocks NTT."""
    g = ctypes.c_int()
    _check(lib().she_ctx_br_engine(ctx.handle, ctypes.byref(g)))
    return g.value


def she_gate_batch(ctx: Context, op: int, a, b, c, out, stream=None) -> None:
    count = a.shape[0]
    _check(lib().she_gate_batch(ctx.handle, op, _dev_ptr(a), _dev_ptr(b), _dev_ptr(c),
                                _dev_ptr(out), count, _stream_ptr(stream)))


def she_gate_batch_ops(ctx: Context, ops, a, b, c, out, stream=None) -> None:
    count = a.shape[0]
    _check(lib().she_gate_batch_ops(ctx.handle, _dev_ptr(ops), _dev_ptr(a), _dev_ptr(b),
                                    _dev_ptr(c), _dev_ptr(out), count, _stream_ptr(stream)))


def she_gate_batch_ops_host(ctx: Context, ops: np.ndarray, a: np.ndarray, b: np.ndarray,
                            c: np.ndarray, out: np.ndarray, stream=None) -> None:
    """Host buffers (ideally pinned): copy in, evaluate, copy out, synchronise."""
    count = a.shape[0]
    _check(lib().she_gate_batch_ops_host(ctx.handle, ops.ctypes.data, a.ctypes.data,
                                         b.ctypes.data, c.ctypes.data, out.ctypes.data, count,
                                         _stream_ptr(stream)))


def she_gate_level(ctx: Context, wires, ops, ins, out_idx, stream=None) -> None:
    """ops: uint8 codes (any dtype view of the bytes); ins: 3 x uint32 per gate;
    out_idx: one uint32 slot index per gate (its length is the gate count)."""
    count = out_idx.numel()
    _check(lib().she_gate_level(ctx.handle, _dev_ptr(wires), _dev_ptr(ops), _dev_ptr(ins),
                                _dev_ptr(out_idx), count, _stream_ptr(stream)))


# ---- layer calls (device) ------------------------------------------------------

def _codes(wq) -> np.ndarray:
    return np.ascontiguousarray(wq, dtype=np.int8)


def conv_width(H, W, C, w_in, in_signed, wq, stride, pad, cap=16, relu=False) -> int:
    wq = _codes(wq)
    Co, K = wq.shape[0], wq.shape[1]
    w = ctypes.c_int(0)
    _check(lib().she_conv_shift_acc(None, None, H, W, C, w_in, int(in_signed), _np_ptr(wq), Co, K,
                                    stride, pad, cap, int(relu), None, ctypes.byref(w), None))
    return w.value


def fc_width(K, w_in, in_signed, wq, cap=16, relu=False) -> int:
    wq = _codes(wq)
    w = ctypes.c_int(0)
    _check(lib().she_fc_shift_acc(None, None, K, w_in, int(in_signed), _np_ptr(wq), wq.shape[0],
                                  cap, int(relu), None, ctypes.byref(w), None))
    return w.value


def she_conv_shift_acc(ctx: Context, x, H, W, C, w_in, in_signed, wq, stride, pad, cap=16,
                       relu=False, out=None, stream=None):
    """x: device slots [H][W][C][w_in][stride]; returns (out [Ho][Wo][Co][w][stride], w)."""
    import torch
    wq = _codes(wq)
    Co, K = wq.shape[0], wq.shape[1]
    Ho, Wo = (H + 2 * pad - K) // stride + 1, (W + 2 * pad - K) // stride + 1
    w = ctypes.c_int(conv_width(H, W, C, w_in, in_signed, wq, stride, pad, cap, relu))
    if out is None:
        out = torch.zeros((Ho, Wo, Co, w.value, ctx.stride), dtype=torch.int32, device=x.device)
    _check(lib().she_conv_shift_acc(ctx.handle, _dev_ptr(x), H, W, C, w_in, int(in_signed),
                                    _np_ptr(wq), Co, K, stride, pad, cap, int(relu), _dev_ptr(out),
                                    ctypes.byref(w), _stream_ptr(stream)))
    return out, w.value


def she_fc_shift_acc(ctx: Context, x, K, w_in, in_signed, wq, cap=16, relu=False, out=None,
                     stream=None):
    import torch
    wq = _codes(wq)
    M = wq.shape[0]
    w = ctypes.c_int(fc_width(K, w_in, in_signed, wq, cap, relu))
    if out is None:
        out = torch.zeros((M, w.value, ctx.stride), dtype=torch.int32, device=x.device)
    _check(lib().she_fc_shift_acc(ctx.handle, _dev_ptr(x), K, w_in, int(in_signed), _np_ptr(wq), M,
                                  cap, int(relu), _dev_ptr(out), ctypes.byref(w),
                                  _stream_ptr(stream)))
    return out, w.value


def she_relu(ctx: Context, x, words, width, out=None, stream=None):
    import torch
    if out is None:
        out = torch.zeros((words, width - 1, ctx.stride), dtype=torch.int32, device=x.device)
    _check(lib().she_relu(ctx.handle, _dev_ptr(x), words, width, _dev_ptr(out), _stream_ptr(stream)))
    return out


def she_maxpool2x2(ctx: Context, x, H, W, C, w, in_signed, out=None, stream=None):
    import torch
    if out is None:
        out = torch.zeros((H // 2, W // 2, C, w, ctx.stride), dtype=torch.int32, device=x.device)
    _check(lib().she_maxpool2x2(ctx.handle, _dev_ptr(x), H, W, C, w, int(in_signed), _dev_ptr(out),
                                _stream_ptr(stream)))
    return out


def layer_stats(ctx: Context) -> dict:
    st = she_circuit_stats()
    _check(lib().she_ctx_layer_stats(ctx.handle, ctypes.byref(st)))
    return st.as_dict()


def capture(ctx: Context, seed: int, every: int, max_gates: int) -> None:
    """Sample layer gates for ciphertext parity (test instrumentation, she.h)."""
    _check(lib().she_ctx_capture(ctx.handle, seed, every, max_gates))


def capture_read(ctx: Context, cap: int):
    """-> (ops uint8[k], slots uint32[k][4][stride]: a, b, c as read, out)."""
    ops = np.zeros(max(cap, 1), np.uint8)
    slots = np.zeros((max(cap, 1), 4, ctx.stride), np.uint32)
    n = ctypes.c_size_t(0)
    _check(lib().she_ctx_capture_read(ctx.handle, _np_ptr(ops), _np_ptr(slots), cap, ctypes.byref(n)))
    k = min(n.value, cap)
    return ops[:k], slots[:k]


# ---- clear-bit backend (host bits; scheduler tests and gate counts) -------------

def clear_conv_shift_acc(bits, H, W, C, w_in, in_signed, wq, stride, pad, cap=16, relu=False,
                         rank=0, world=1):
    """bits: uint8 [H][W][C][w_in]; returns (bits [Ho][Wo][Co][w], w, stats)."""
    wq = _codes(wq)
    bits = np.ascontiguousarray(bits, dtype=np.uint8)
    Co, K = wq.shape[0], wq.shape[1]
    Ho, Wo = (H + 2 * pad - K) // stride + 1, (W + 2 * pad - K) // stride + 1
    w = ctypes.c_int(conv_width(H, W, C, w_in, in_signed, wq, stride, pad, cap, relu))
    out = np.zeros((Ho, Wo, Co, w.value), dtype=np.uint8)
    st = she_circuit_stats()
    _check(lib().she_clear_conv_shift_acc(_np_ptr(bits), H, W, C, w_in, int(in_signed), _np_ptr(wq),
                                          Co, K, stride, pad, cap, int(relu), _np_ptr(out),
                                          ctypes.byref(w), rank, world, ctypes.byref(st)))
    return out, w.value, st.as_dict()


def clear_fc_shift_acc(bits, K, w_in, in_signed, wq, cap=16, relu=False, rank=0, world=1):
    wq = _codes(wq)
    bits = np.ascontiguousarray(bits, dtype=np.uint8)
    M = wq.shape[0]
    w = ctypes.c_int(fc_width(K, w_in, in_signed, wq, cap, relu))
    out = np.zeros((M, w.value), dtype=np.uint8)
    st = she_circuit_stats()
    _check(lib().she_clear_fc_shift_acc(_np_ptr(bits), K, w_in, int(in_signed), _np_ptr(wq), M, cap,
                                        int(relu), _np_ptr(out), ctypes.byref(w), rank, world,
                                        ctypes.byref(st)))
    return out, w.value, st.as_dict()


def clear_relu(bits, words, width, rank=0, world=1):
    bits = np.ascontiguousarray(bits, dtype=np.uint8)
    out = np.zeros((words, width - 1), dtype=np.uint8)
    st = she_circuit_stats()
    _check(lib().she_clear_relu(_np_ptr(bits), words, width, _np_ptr(out), rank, world,
                                ctypes.byref(st)))
    return out, st.as_dict()


def clear_maxpool2x2(bits, H, W, C, w, in_signed, rank=0, world=1):
    bits = np.ascontiguousarray(bits, dtype=np.uint8)
    out = np.zeros((H // 2, W // 2, C, w), dtype=np.uint8)
    st = she_circuit_stats()
    _check(lib().she_clear_maxpool2x2(_np_ptr(bits), H, W, C, w, int(in_signed), _np_ptr(out),
                                      rank, world, ctypes.byref(st)))
    return out, st.as_dict()


# ---- TCN baseline: fixed-point multipliers (she.h she_*_mul_acc) -------------

def _mults(wm) -> np.ndarray:
    return np.ascontiguousarray(wm, dtype=np.int16)


def conv_mul_width(H, W, C, w_in, in_signed, wm, stride, pad, cap=16, relu=False) -> int:
    wm = _mults(wm)
    Co, K = wm.shape[0], wm.shape[1]
    w = ctypes.c_int(0)
    _check(lib().she_conv_mul_acc(None, None, H, W, C, w_in, int(in_signed), _np_ptr(wm), Co, K,
                                  stride, pad, cap, int(relu), None, ctypes.byref(w), None))
    return w.value


def fc_mul_width(K, w_in, in_signed, wm, cap=16, relu=False) -> int:
    wm = _mults(wm)
    w = ctypes.c_int(0)
    _check(lib().she_fc_mul_acc(None, None, K, w_in, int(in_signed), _np_ptr(wm), wm.shape[0],
                                cap, int(relu), None, ctypes.byref(w), None))
    return w.value


def she_conv_mul_acc(ctx: Context, x, H, W, C, w_in, in_signed, wm, stride, pad, cap=16,
                     relu=False, out=None, stream=None):
    import torch
    wm = _mults(wm)
    Co, K = wm.shape[0], wm.shape[1]
    Ho, Wo = (H + 2 * pad - K) // stride + 1, (W + 2 * pad - K) // stride + 1
    w = ctypes.c_int(conv_mul_width(H, W, C, w_in, in_signed, wm, stride, pad, cap, relu))
    if out is None:
        out = torch.zeros((Ho, Wo, Co, w.value, ctx.stride), dtype=torch.int32, device=x.device)
    _check(lib().she_conv_mul_acc(ctx.handle, _dev_ptr(x), H, W, C, w_in, int(in_signed),
                                  _np_ptr(wm), Co, K, stride, pad, cap, int(relu), _dev_ptr(out),
                                  ctypes.byref(w), _stream_ptr(stream)))
    return out, w.value


def she_fc_mul_acc(ctx: Context, x, K, w_in, in_signed, wm, cap=16, relu=False, out=None,
                   stream=None):
    import torch
    wm = _mults(wm)
    M = wm.shape[0]
    w = ctypes.c_int(fc_mul_width(K, w_in, in_signed, wm, cap, relu))
    if out is None:
        out = torch.zeros((M, w.value, ctx.stride), dtype=torch.int32, device=x.device)
    _check(lib().she_fc_mul_acc(ctx.handle, _dev_ptr(x), K, w_in, int(in_signed), _np_ptr(wm), M,
                                cap, int(relu), _dev_ptr(out), ctypes.byref(w),
                                _stream_ptr(stream)))
    return out, w.value


def clear_conv_mul_acc(bits, H, W, C, w_in, in_signed, wm, stride, pad, cap=16, relu=False,
                       rank=0, world=1):
    wm = _mults(wm)
    bits = np.ascontiguousarray(bits, dtype=np.uint8)
    Co, K = wm.shape[0], wm.shape[1]
    Ho, Wo = (H + 2 * pad - K) // stride + 1, (W + 2 * pad - K) // stride + 1
    w = ctypes.c_int(conv_mul_width(H, W, C, w_in, in_signed, wm, stride, pad, cap, relu))
    out = np.zeros((Ho, Wo, Co, w.value), dtype=np.uint8)
    st = she_circuit_stats()
    _check(lib().she_clear_conv_mul_acc(_np_ptr(bits), H, W, C, w_in, int(in_signed), _np_ptr(wm),
                                        Co, K, stride, pad, cap, int(relu), _np_ptr(out),
                                        ctypes.byref(w), rank, world, ctypes.byref(st)))
    return out, w.value, st.as_dict()


def clear_fc_mul_acc(bits, K, w_in, in_signed, wm, cap=16, relu=False, rank=0, world=1):
    wm = _mults(wm)
    bits = np.ascontiguousarray(bits, dtype=np.uint8)
    M = wm.shape[0]
    w = ctypes.c_int(fc_mul_width(K, w_in, in_signed, wm, cap, relu))
    out = np.zeros((M, w.value), dtype=np.uint8)
    st = she_circuit_stats()
    _check(lib().she_clear_fc_mul_acc(_np_ptr(bits), K, w_in, int(in_signed), _np_ptr(wm), M, cap,
                                      int(relu), _np_ptr(out), ctypes.byref(w), rank, world,
                                      ctypes.byref(st)))
    return out, w.value, st.as_dict()


# ---- batch normalisation as shift + constant (she.h she_bn_shift_add) --------

def _bn_args(shift, neg, bias):
    shift = np.ascontiguousarray(shift, dtype=np.int8)
    neg = np.ascontiguousarray(np.zeros_like(shift, dtype=np.uint8) if neg is None else neg,
                               dtype=np.uint8)
    bias = np.ascontiguousarray(bias, dtype=np.int32)
    return shift, neg, bias


def bn_width(words, C, w_in, in_signed, shift, neg, bias, cap=16, relu=False) -> int:
    shift, neg, bias = _bn_args(shift, neg, bias)
    w = ctypes.c_int(0)
    _check(lib().she_bn_shift_add(None, None, words, C, w_in, int(in_signed), _np_ptr(shift),
                                  _np_ptr(neg), _np_ptr(bias), cap, int(relu), None,
                                  ctypes.byref(w), None))
    return w.value


def she_bn_shift_add(ctx: Context, x, words, C, w_in, in_signed, shift, neg, bias, cap=16,
                     relu=False, out=None, stream=None):
    """x: device [words][w_in][stride] (HWC); returns (out [words][w][stride], w)."""
    import torch
    shift, neg, bias = _bn_args(shift, neg, bias)
    w = ctypes.c_int(bn_width(words, C, w_in, in_signed, shift, neg, bias, cap, relu))
    if out is None:
        out = torch.zeros((words, w.value, ctx.stride), dtype=torch.int32, device=x.device)
    _check(lib().she_bn_shift_add(ctx.handle, _dev_ptr(x), words, C, w_in, int(in_signed),
                                  _np_ptr(shift), _np_ptr(neg), _np_ptr(bias), cap, int(relu),
                                  _dev_ptr(out), ctypes.byref(w), _stream_ptr(stream)))
    return out, w.value


def clear_bn_shift_add(bits, words, C, w_in, in_signed, shift, neg, bias, cap=16, relu=False,
                       rank=0, world=1):
    shift, neg, bias = _bn_args(shift, neg, bias)
    bits = np.ascontiguousarray(bits, dtype=np.uint8)
    w = ctypes.c_int(bn_width(words, C, w_in, in_signed, shift, neg, bias, cap, relu))
    out = np.zeros((words, w.value), dtype=np.uint8)
    st = she_circuit_stats()
    _check(lib().she_clear_bn_shift_add(_np_ptr(bits), words, C, w_in, int(in_signed),
                                        _np_ptr(shift), _np_ptr(neg), _np_ptr(bias), cap,
                                        int(relu), _np_ptr(out), ctypes.byref(w), rank, world,
                                        ctypes.byref(st)))
    return out, w.value, st.as_dict()


def field_selftest(device: int, a, b, c) -> np.ndarray:
    """Device field primitives on (a, b, c) triples (test instrumentation, she.h)."""
    a = np.ascontiguousarray(a, dtype=np.uint64)
    b = np.ascontiguousarray(b, dtype=np.uint64)
    c = np.ascontiguousarray(c, dtype=np.uint32)
    out = np.zeros((len(a), 104), dtype=np.uint64)
    _check(lib().she_field_selftest(device, _np_ptr(a), _np_ptr(b), _np_ptr(c), len(a), _np_ptr(out)))
    return out


def fft_product_selftest(device: int, digits, bk, variant: int = 0):
    """FP64-engine CMux product on given inputs (test instrumentation, she.h):
    digits int32 [count][4][1024], bk uint32 [count][4][2][1024] ->
    (out uint32 [count][2][1024], worst distance to an integer)."""
    digits = np.ascontiguousarray(digits, dtype=np.int32)
    bk = np.ascontiguousarray(bk, dtype=np.uint32)
    count = digits.shape[0]
    assert digits.shape == (count, 4, 1024) and bk.shape == (count, 4, 2, 1024)
    out = np.zeros((count, 2, 1024), dtype=np.uint32)
    worst = ctypes.c_double(0.0)
    _check(lib().she_fft_product_selftest(device, variant, _np_ptr(digits), _np_ptr(bk), count,
                                          _np_ptr(out), ctypes.byref(worst)))
    return out, worst.value


# ---- client side on the GPU (she.h, NEXT-4) -----------------------------------

def she_encrypt_noise(sk: SecretKey, count: int, seed: int, first_index: int = 0) -> np.ndarray:
    noise = np.zeros(max(count, 1), np.uint32)
    _check(lib().she_encrypt_noise(sk.handle, count, seed, first_index, _np_ptr(noise)))
    return noise[:count]


def she_encrypt_bits_gpu(sk: SecretKey, bits, noise, seed: int, first_index: int = 0,
                         out=None, stream=None):
    """bits: device uint8 tensor [count]; noise: device int32 tensor [count]
    (she_encrypt_noise); returns device int32 [count][stride]."""
    import torch
    count = bits.numel()
    if out is None:
        out = torch.empty((count, stride(sk.params)), dtype=torch.int32, device=bits.device)
    _check(lib().she_encrypt_bits_gpu(sk.handle, _dev_ptr(bits), _dev_ptr(noise), count, seed,
                                      first_index, _dev_ptr(out), bits.device.index or 0,
                                      _stream_ptr(stream)))
    return out


def she_decrypt_bits_gpu(sk: SecretKey, cts, out=None, stream=None):
    """cts: device int32 [count][stride]; returns device uint8 [count]."""
    import torch
    count = cts.shape[0]
    if out is None:
        out = torch.empty((count,), dtype=torch.uint8, device=cts.device)
    _check(lib().she_decrypt_bits_gpu(sk.handle, _dev_ptr(cts), count, _dev_ptr(out),
                                      cts.device.index or 0, _stream_ptr(stream)))
    return out


# ---- leveled mode (she.h she_lvl_*; NEXT-2, reading R-LV) ----------

SHE_LVL_ADD, SHE_LVL_MAX, SHE_LVL_RELU = 0, 1, 2


def lvl_encrypt_selectors(sk: SecretKey, bits, seed: int, first_index: int = 0) -> np.ndarray:
    """Client: bits -> TRGSW selectors, uint32 [count][2l][2][N] (host)."""
    P = sk.params
    bits = np.ascontiguousarray(bits, dtype=np.uint8).ravel()
    out = np.zeros((len(bits), 2 * P.l, 2, P.N), dtype=np.uint32)
    if len(bits):
        _check(lib().she_lvl_encrypt_selectors(sk.handle, _np_ptr(bits), len(bits), seed,
                                               first_index, _np_ptr(out)))
    return out


def lvl_decrypt(sk: SecretKey, cts) -> np.ndarray:
    """Client: TRLWE data [..][2][N] (host) -> bits."""
    P = sk.params
    cts = np.ascontiguousarray(cts, dtype=np.uint32)
    flat = cts.reshape(-1, 2 * P.N)
    bits = np.zeros(flat.shape[0], dtype=np.uint8)
    if len(bits):
        _check(lib().she_lvl_decrypt(sk.handle, _np_ptr(flat), len(bits), _np_ptr(bits)))
    return bits.reshape(cts.shape[:-2])


def lvl_selectors_to_device(ctx: Context, sel: np.ndarray, stream=None):
    """Upload + FFT-transform selectors; returns the device buffer (torch uint8)."""
    import torch
    sel = np.ascontiguousarray(sel, dtype=np.uint32)
    count = sel.shape[0]
    out = torch.empty(max(count, 1) * int(lib().she_lvl_selector_bytes()), dtype=torch.uint8,
                      device=f"cuda:{ctx.device}")
    _check(lib().she_lvl_selectors_to_device(ctx.handle, _np_ptr(sel), count, _dev_ptr(out),
                                             _stream_ptr(stream)))
    return out


def lvl_cmux_batch(ctx: Context, sel_dev, sel_idx, d1, d0, out=None, stream=None):
    """out[i] = sel[sel_idx[i]] ? d1[i] : d0[i] (device int32 [count][2][N])."""
    import torch
    if out is None:
        out = torch.empty_like(d1)
    _check(lib().she_lvl_cmux_batch(ctx.handle, _dev_ptr(sel_dev), _dev_ptr(sel_idx), _dev_ptr(d1),
                                    _dev_ptr(d0), _dev_ptr(out), sel_idx.numel(),
                                    _stream_ptr(stream)))
    return out


def lvl_unit(ctx: Context, op: int, sel_dev, x_sel, y_sel, width: int, signed: bool, stream=None):
    """Leveled ADD / MAX / RELU on client words; returns (out device int32
    [count][w_out][2][N], cmux_count, depth)."""
    import torch
    x_sel = np.ascontiguousarray(x_sel, dtype=np.uint32)
    count = x_sel.shape[0]
    y_sel = None if y_sel is None else np.ascontiguousarray(y_sel, dtype=np.uint32)
    wout = width - 1 if op == SHE_LVL_RELU else width
    N = ctx.params.N
    out = torch.zeros((count, wout, 2, N), dtype=torch.int32, device=f"cuda:{ctx.device}")
    n_cmux, depth = ctypes.c_uint64(0), ctypes.c_uint32(0)
    _check(lib().she_lvl_unit(ctx.handle, op, _dev_ptr(sel_dev), _np_ptr(x_sel),
                              None if y_sel is None else _np_ptr(y_sel), count, width, int(signed),
                              _dev_ptr(out), ctypes.byref(n_cmux), ctypes.byref(depth),
                              _stream_ptr(stream)))
    return out, int(n_cmux.value), int(depth.value)
