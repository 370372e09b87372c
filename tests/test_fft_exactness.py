"""CPU pins of the reading behind the FP64 FFT engine.

The CMux product sum_r d_r * b_r mod (X^1024 + 1), with digits |d| <= 512
(Bg = 2^10) and torus32 BK coefficients split as b = 2^16 b_hi + b_lo
(|b_*| <= 2^15), is recovered EXACTLY by a double-precision folded FFT
(512 complex points) followed by rounding: the round-off stays far below 1/2.
These tests check that claim with numpy's FFT (an independent implementation
of the same arithmetic class, not the CUDA code) against exact integer
negacyclic products, on random and on worst-case-magnitude inputs, and show
that without the split the result is not exact.  The GPU engine itself is
pinned bit for bit against the oracle in tests/test_gpu_gates.py.
"""
import numpy as np
import pytest

N, M = 1024, 512
ZETA = np.exp(1j * np.pi * np.arange(M) / N)  # zeta^n, zeta = exp(i pi / N)


def negacyclic_exact(a, b):
    """Schoolbook a * b mod (X^N + 1) in int64 (|result| < 2^63 asserted)."""
    full = np.convolve(a.astype(np.int64), b.astype(np.int64))
    out = full[:N].copy()
    out[: N - 1] -= full[N:]
    return out


def fold_fft(a):
    return np.fft.fft((a[:M] + 1j * a[M:]) * ZETA)


def unfold_ifft(A):
    u = np.fft.ifft(A) / ZETA
    return np.concatenate([u.real, u.imag])


def split16(b):
    b = b.astype(np.int64)
    lo = ((b & 0xFFFF) ^ 0x8000) - 0x8000
    return (b - lo) >> 16, lo


def cmux_product_fft(d, bk):
    """sum_r d[r] * bk[r] mod (X^N + 1) mod 2^32 by the split FFT, plus the
    largest distance of any rounded value from an integer."""
    hi_lo = [split16(b) for b in bk]
    D = [fold_fft(x.astype(np.float64)) for x in d]
    res, worst = np.zeros(N, np.int64), 0.0
    for half, shift in ((0, 16), (1, 0)):
        acc = sum(D[r] * fold_fft(hi_lo[r][half].astype(np.float64)) for r in range(len(d)))
        c = unfold_ifft(acc)
        r = np.rint(c)
        worst = max(worst, float(np.max(np.abs(c - r))))
        res += r.astype(np.int64) << shift
    return res & 0xFFFFFFFF, worst


def cmux_product_exact(d, bk):
    return sum(negacyclic_exact(x, b.astype(np.int64)) for x, b in zip(d, bk)) & 0xFFFFFFFF


@pytest.mark.parametrize("seed", [1, 2, 3])
def test_split_fft_product_is_exact_random(seed):
    rng = np.random.default_rng(seed)
    d = [rng.integers(-512, 512, N) for _ in range(4)]
    bk = [rng.integers(-2**31, 2**31, N) for _ in range(4)]
    got, worst = cmux_product_fft(d, bk)
    assert np.array_equal(got, cmux_product_exact(d, bk))
    assert worst < 1e-3


@pytest.mark.parametrize("kind", ["all_min", "alternating", "aligned_signs"])
def test_split_fft_product_is_exact_worst_magnitude(kind):
    """Inputs that drive one output coefficient to the bound 4 * 1024 * 512 * 2^15."""
    n = np.arange(N)
    if kind == "all_min":
        d = [np.full(N, -512) for _ in range(4)]
        bk = [np.full(N, -2**31) for _ in range(4)]
    elif kind == "alternating":
        d = [np.where(n % 2 == 0, -512, 511) for _ in range(4)]
        bk = [np.where(n % 2 == 0, -2**31, 2**31 - 1) for _ in range(4)]
    else:  # b_j = sign so that coefficient 0 of d * b sums |d||b| (negacyclic wrap)
        d = [np.full(N, -512) for _ in range(4)]
        s = np.where(n == 0, 1, -1)
        bk = [(s * (2**31 - 1)).astype(np.int64) for _ in range(4)]
        bk = [np.where(b > 0, b, -(2**31) + 0 * b) for b in bk]
    got, worst = cmux_product_fft(d, bk)
    assert np.array_equal(got, cmux_product_exact(d, bk))
    assert worst < 5e-3


def test_without_the_split_the_fft_is_not_exact():
    """Full 32-bit BK coefficients: sums reach ~2^52 and the FFT result is no
    longer the exact integer product (the reason for the split)."""
    d = [np.full(N, -512) for _ in range(4)]
    bk = [np.full(N, -2**31 + 12345) for _ in range(4)]
    D = [fold_fft(x.astype(np.float64)) for x in d]
    acc = sum(D[r] * fold_fft(bk[r].astype(np.float64)) for r in range(4))
    got = np.rint(unfold_ifft(acc)).astype(np.int64) & 0xFFFFFFFF
    assert not np.array_equal(got, cmux_product_exact(d, bk))
