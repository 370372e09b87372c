"""Seeded synthetic-input generators shared by the product tests, the oracle
tests and bench.py.

This module holds no arithmetic of the method: it only defines parameter sets
(BASELINE.json ``configs``), seeds, and the counter-based random streams that
draw plaintext inputs (gate ops, input bits, pixels, log-quantised weights).
The C twin of the generator is ``she_rng.h`` (same SplitMix64 definition),
used for key material and encryption randomness by both the product client
library and the oracle.

Input recipe:
  * keys        seed 1000+cfg
  * input bits  seed 2000+cfg, stream 16, index = 3*gate + slot
  * encryption  seed 2000+cfg, ordinal = 3*gate + slot
  * gate ops    seed 4000+cfg, stream 17, uniform over the six bootstrapped ops
  * pixels      seed 2000+cfg, stream 18
  * weights     seed 3000+cfg, stream 19 (zero w.p. 0.1, else sign +-1, e in 0..7)
  * oracle sample seed 5000+cfg, stream 20
"""
from __future__ import annotations

import os
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
RNG_HEADER = os.path.join(HERE, "she_rng.h")

GOLDEN = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)

STREAM_INPUT_BITS = 16
STREAM_OPS = 17
STREAM_PIXELS = 18
STREAM_WEIGHTS = 19
STREAM_SAMPLE = 20

# op codes of the C-ABI (include/she.h she_op)
AND, NAND, OR, NOR, XOR, XNOR, MUX, NOT, COPY = range(9)
OP_NAMES = ["AND", "NAND", "OR", "NOR", "XOR", "XNOR", "MUX", "NOT", "COPY"]
# BASELINE.json configs[0..1]: "ops uniform over NAND/AND/OR/XOR/XNOR/MUX"
BOOTSTRAPPED_MIX = np.array([NAND, AND, OR, XOR, XNOR, MUX], dtype=np.uint8)


def mix64(z: np.ndarray) -> np.ndarray:
    z = np.asarray(z, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = (z ^ (z >> np.uint64(30))) * _M1
        z = (z ^ (z >> np.uint64(27))) * _M2
    return z ^ (z >> np.uint64(31))


def rng_u64(seed: int, stream: int, index) -> np.ndarray:
    """Value #index of (seed, stream); identical to she_rng_u64 in she_rng.h."""
    idx = np.asarray(index, dtype=np.uint64)
    with np.errstate(over="ignore"):
        key = mix64(np.uint64(seed) ^ mix64(GOLDEN * np.uint64(stream + 1)))
        return mix64(key + GOLDEN * (idx + np.uint64(1)))


@dataclass(frozen=True)
class Params:
    """TFHE gate-bootstrapping parameters (BASELINE.json configs; k = 1)."""
    N: int
    n: int
    bg_bits: int
    l: int
    ks_base_bits: int
    ks_t: int
    alpha_lwe: float
    alpha_bk: float
    k: int = 1

    @property
    def stride(self) -> int:
        """Words per LWE slot: n+1 padded to a multiple of 32 (include/she.h)."""
        return (self.n + 1 + 31) // 32 * 32

    @property
    def name(self) -> str:
        return "C0" if self.N == 256 else "C1"


# configs[0]: toy plumbing
C0 = Params(N=256, n=128, bg_bits=8, l=2, ks_base_bits=2, ks_t=8,
            alpha_lwe=2.0 ** -20, alpha_bk=2.0 ** -30)
# configs[1..4]: "TFHE-library default gate params"
C1 = Params(N=1024, n=500, bg_bits=10, l=2, ks_base_bits=2, ks_t=8,
            alpha_lwe=2.44e-5, alpha_bk=3.73e-9)

CONFIG_PARAMS = {0: C0, 1: C1, 2: C1, 3: C1, 4: C1}
CONFIG_GATES = {0: 16, 1: 4096}


def key_seed(cfg: int) -> int:
    return 1000 + cfg


def input_seed(cfg: int) -> int:
    return 2000 + cfg


def weight_seed(cfg: int) -> int:
    return 3000 + cfg


def ops_seed(cfg: int) -> int:
    return 4000 + cfg


def sample_seed(cfg: int) -> int:
    return 5000 + cfg


def gate_ops(cfg: int, count: int) -> np.ndarray:
    """Per-gate op, uniform over the six bootstrapped ops (configs 0-1)."""
    r = rng_u64(ops_seed(cfg), STREAM_OPS, np.arange(count, dtype=np.uint64))
    return BOOTSTRAPPED_MIX[(r % np.uint64(6)).astype(np.int64)]


def gate_input_bits(cfg: int, count: int) -> np.ndarray:
    """bits[g, slot] for slot a=0, b=1, c=2 (c only read by MUX)."""
    idx = np.arange(3 * count, dtype=np.uint64)
    bits = (rng_u64(input_seed(cfg), STREAM_INPUT_BITS, idx) & np.uint64(1)).astype(np.uint8)
    return bits.reshape(count, 3)


def gate_input_ordinals(count: int) -> np.ndarray:
    """Encryption ordinal of (gate, slot): 3*gate + slot."""
    return np.arange(3 * count, dtype=np.uint64).reshape(count, 3)


def truth(op: int, a, b, c=None):
    """Plain Boolean semantics of the C-ABI ops (MUX(s,a,b) = s ? a : b with
    s=a-slot, a=b-slot, b=c-slot)."""
    a = np.asarray(a, dtype=np.uint8)
    b = np.asarray(b, dtype=np.uint8)
    if op == AND:
        return a & b
    if op == NAND:
        return 1 - (a & b)
    if op == OR:
        return a | b
    if op == NOR:
        return 1 - (a | b)
    if op == XOR:
        return a ^ b
    if op == XNOR:
        return 1 - (a ^ b)
    if op == MUX:
        c = np.asarray(c, dtype=np.uint8)
        return np.where(a == 1, b, c).astype(np.uint8)
    if op == NOT:
        return 1 - a
    if op == COPY:
        return a.copy()
    raise ValueError(op)


def br_lanes(ops: np.ndarray) -> int:
    """Blind-rotation lanes a gate batch needs (MUX = 2, NOT/COPY = 0)."""
    ops = np.asarray(ops)
    return int(np.sum(np.where(ops == MUX, 2, np.where(ops >= NOT, 0, 1))))


# ---- network inputs (configs 2-4) -------------------------------------------

def pixels(cfg: int, shape) -> np.ndarray:
    """uint8 pixels uniform in [0, 255] (stand-in for MNIST / CIFAR-10 images)."""
    size = int(np.prod(shape))
    r = rng_u64(input_seed(cfg), STREAM_PIXELS, np.arange(size, dtype=np.uint64))
    return (r >> np.uint64(56)).astype(np.uint8).reshape(shape)


def log_quant_weights(cfg: int, shape, layer: int = 0) -> np.ndarray:
    """Log-quantised weights as int8 codes: 0 = zero weight, else +-(e+1) meaning
    sign * 2^-e, e in 0..7 (BASELINE.json configs[2]: 10% zero, sign uniform,
    e uniform).  PAPER.md:118 (weightQ = round(log2 w))."""
    size = int(np.prod(shape))
    base = np.uint64(layer) << np.uint64(40)
    r = rng_u64(weight_seed(cfg), STREAM_WEIGHTS, base + np.arange(size, dtype=np.uint64))
    u = (r >> np.uint64(11)).astype(np.float64) * 2.0 ** -53
    zero = u < 0.1
    sign = np.where(((r >> np.uint64(3)) & np.uint64(1)) == 1, -1, 1)
    e = (r & np.uint64(7)).astype(np.int64)
    code = np.where(zero, 0, sign * (e + 1)).astype(np.int8)
    return code.reshape(shape)


def tcn_weights(cfg: int, shape, layer: int = 0) -> np.ndarray:
    """Fixed-point multipliers for the TCN baseline:
    int16 c in [-255, 255] standing for c / 2^7.  Same stream, sign and zero
    pattern as log_quant_weights; the magnitude is 2^(7 - t) rounded, with t
    uniform in [-0.5, 7.5) (so its nearest power of two spreads over the same
    exponents e in 0..7 as the SHE weights), clipped to [1, 255]."""
    size = int(np.prod(shape))
    base = np.uint64(layer) << np.uint64(40)
    r = rng_u64(weight_seed(cfg), STREAM_WEIGHTS, base + np.arange(size, dtype=np.uint64))
    u = (r >> np.uint64(11)).astype(np.float64) * 2.0 ** -53
    zero = u < 0.1
    sign = np.where(((r >> np.uint64(3)) & np.uint64(1)) == 1, -1, 1)
    t = ((r >> np.uint64(16)) & np.uint64(0xFFFFFF)).astype(np.float64) / 2.0 ** 24 * 8.0 - 0.5
    mag = np.clip(np.rint(2.0 ** (7.0 - t)), 1, 255).astype(np.int64)
    return np.where(zero, 0, sign * mag).astype(np.int16).reshape(shape)


def bn_params(cfg: int, C: int, layer: int = 0):
    """Synthetic batch-norm folding for the BN layers:
    per channel a power-of-two scale shift in [-2, 1], a sign flip w.p. 1/8 and
    an integer bias uniform in [-64, 64]."""
    base = (np.uint64(1) << np.uint64(52)) + (np.uint64(layer) << np.uint64(40))
    r = rng_u64(weight_seed(cfg), STREAM_WEIGHTS, base + np.arange(C, dtype=np.uint64))
    shift = ((r & np.uint64(3)).astype(np.int64) - 2).astype(np.int8)
    neg = (((r >> np.uint64(8)) & np.uint64(7)) == 0).astype(np.uint8)
    bias = (((r >> np.uint64(16)) % np.uint64(129)).astype(np.int64) - 64).astype(np.int32)
    return shift, neg, bias
