"""Device pin of the FP64 FFT engine's exactness.

she_fft_product_selftest runs the CMux product of br_fft_kernel — the setup
transform of BK into 16-bit halves (bk_fft_kernel), the forward FFT of the
digit rows, the pointwise sum, the inverse FFT, the rounding and the hi/lo
recombination, i.e. the same device functions the blind rotation calls — on
caller-given digit rows and BK rows.  The result must equal the oracle's
schoolbook negacyclic products (oracle.negacyclic_mul, summed over the four
rows, mod 2^32) word for word, on random inputs and on the worst-magnitude
inputs SURVEY.md §8(c) names: digits -Bg/2 and Bg/2 - 1, BK words 0, 2^31,
2^32 - 1 and the halves' extremes 0x7FFF7FFF / 0x80008000, with signs aligned
so that one output coefficient sums |d| |b| over all 4 x 1024 terms (the
2^36 bound of the reading).  The kernel also reports the largest distance of
any pre-rounding value to its integer, which must stay below 1/2 (the margin
the reading claims is > 100x).
"""
import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
from paper_1906_00148_b200 import she  # noqa: E402

N = 1024
HALF = 512  # Bg / 2 at the default parameters (Bg = 2^10)


def expected(digits, bk):
    """sum_r digits[r] * bk[r][o] mod (X^N + 1) mod 2^32 by the oracle's
    schoolbook product (PAPER.md:31 bootstrapping)."""
    out = np.zeros((2, N), dtype=np.uint64)
    for r in range(4):
        for o in range(2):
            out[o] += oracle.negacyclic_mul(digits[r], bk[r, o]).astype(np.uint64)
    return (out & 0xFFFFFFFF).astype(np.uint32)


def aligned_digits(bk_signs, k):
    """Digits of magnitude Bg/2 whose sign makes every term of output
    coefficient k add with the same sign: term m of coefficient k multiplies
    d[m] by b[(k - m) mod N] with a factor -1 when m > k (negacyclic wrap)."""
    m = np.arange(N)
    wrap = np.where(m > k, -1, 1)
    s = wrap * bk_signs[(k - m) % N]
    return np.where(s >= 0, HALF - 1, -HALF).astype(np.int32)


def signed16(v):
    lo = ((v & 0xFFFF) ^ 0x8000) - 0x8000
    return lo, (v.astype(np.int64) - lo) >> 16


def cases():
    rng = np.random.default_rng(20261020)
    out = []
    # random digits in [-Bg/2, Bg/2) and random torus32 BK
    for _ in range(4):
        d = rng.integers(-HALF, HALF, size=(4, N), dtype=np.int32)
        b = rng.integers(0, 2**32, size=(4, 2, N), dtype=np.uint64).astype(np.uint32)
        out.append(("random", d, b))
    consts = [0x00000000, 0x80000000, 0xFFFFFFFF, 0x7FFF7FFF, 0x80008000, 0x7FFF8000, 0x80007FFF]
    for c in consts:
        b = np.full((4, 2, N), c, dtype=np.uint32)
        # d_0 = -Bg/2, d_m = Bg/2 - 1: coefficient 0 sums |d||b| over every term
        d = np.full((4, N), HALF - 1, dtype=np.int32)
        d[:, 0] = -HALF
        out.append((f"const {c:#010x}, coefficient-0 aligned digits", d, b))
        out.append((f"const {c:#010x}, digits all -Bg/2", np.full((4, N), -HALF, np.int32), b))
        alt = np.where(np.arange(N) % 2 == 0, HALF - 1, -HALF).astype(np.int32)
        out.append((f"const {c:#010x}, alternating extreme digits", np.tile(alt, (4, 1)), b))
    # random extreme halves (|b_lo|, |b_hi| near 2^15) with digits aligned on
    # the signed low half (lo half) and on the high half for several k
    for k in (0, 1, 511, 512, 1023):
        hi = rng.choice([-0x8000, 0x7FFF], size=(4, 2, N)).astype(np.int64)
        lo = rng.choice([-0x8000, 0x7FFF], size=(4, 2, N)).astype(np.int64)
        b = ((hi << 16) + lo).astype(np.int64) & 0xFFFFFFFF
        b = b.astype(np.uint32)
        which = k % 2  # align on the lo half for even k, the hi half for odd k
        d = np.stack([aligned_digits(np.sign(signed16(b[r, 0])[which]), k) for r in range(4)])
        out.append((f"extreme halves, aligned on {'hi' if which else 'lo'} at k={k}", d, b))
    out.append(("zero digits", np.zeros((4, N), np.int32),
                rng.integers(0, 2**32, size=(4, 2, N), dtype=np.uint64).astype(np.uint32)))
    return out


@pytest.mark.parametrize("variant", [2, 1, 3, 4, 5],
                         ids=["v2", "v1-round1", "v3-dit-fma", "tmem", "tmem-fma"])
def test_fft_product_selftest_matches_schoolbook_on_extreme_inputs(cuda, variant):
    cs = cases()
    digits = np.stack([d for _, d, _ in cs])
    bk = np.stack([b for _, _, b in cs])
    got, worst = she.fft_product_selftest(0, digits, bk, variant)
    bad = [name for (name, d, b), g in zip(cs, got) if not np.array_equal(g, expected(d, b))]
    assert not bad, f"device FFT product differs from the schoolbook product: {bad}"
    print(f"\nvariant {variant}: worst distance to an integer before rounding: {worst:.3e} "
          f"over {len(cs)} cases")
    assert worst < 0.5
    # the reading's margin: worst-case bound ~1.1e-3, i.e.
    # more than 100x below 1/2
    assert worst < 5e-3


def test_fft_product_selftest_rejects_bad_arguments(cuda):
    assert she.lib().she_fft_product_selftest(0, 0, None, None, 1, None, None) == -1  # SHE_ERR_ARG
    assert she.lib().she_fft_product_selftest(0, 0, None, None, 0, None, None) == 0   # count 0: no-op
