"""CPU model of the TMEM engine's transform pair (csrc/br_tmem.cuh,
fft_core.cuh dft512_v2 / inverse_tr), step for step in numpy with the warp's 32
threads as array rows: the forward leaves thread t = (k2, h) holding the spectrum
at the frequencies bk_tm_kernel assumes (with the v2 scaling sigma on the odd
thread), inverse_tr on that register layout is the exact inverse (x 512), and
forward -> pointwise with the TRUE BK spectrum / 512 -> inverse_tr is the
negacyclic product.  The device runs the same steps (pinned on the GPU by
she_fft_product_selftest variants 4/5 and the config-1 gate digests); this
test pins the algebra of the layout, the exchange and the inverse on the CPU,
against numpy's FFT and a schoolbook negacyclic product."""
import numpy as np
import pytest

N, M = 1024, 512


def W(e):  # W128^e
    return np.exp(2j * np.pi * (e % 128) / 128)


def brev4(k):
    return ((k & 1) << 3) | ((k & 2) << 1) | ((k & 4) >> 1) | ((k & 8) >> 3)


def tslot(n1, k2):
    return n1 * 16 + (k2 ^ (((n1 & 1) << 2) | ((n1 >> 1) & 3)))


def rot(a, e, sign):
    return a * W(e) if sign > 0 else a * np.conj(W(e))


def dft16(a, sign):  # DIF, natural in, a[brev4(k)] = X[k] out
    a = a.copy()
    half = 8
    while half >= 1:
        for s in range(0, 16, 2 * half):
            for j in range(half):
                u, v = a[s + j], a[s + j + half]
                a[s + j] = u + v
                a[s + j + half] = rot(u - v, j * (64 // half), sign)
        half //= 2
    return a


def dft16_dit_br(a, sign):  # DIT, a[brev4(k)] = X[k] in, natural out
    a = a.copy()
    s = 1
    while s <= 8:
        for g0 in range(0, 16, 2 * s):
            for j in range(s):
                u, v = a[g0 + j], rot(a[g0 + j + s], j * (64 // s), sign)
                a[g0 + j], a[g0 + j + s] = u + v, u - v
        s *= 2
    return a


def tables():  # make_tables2, forward half: t(k2) (k2 < 8) and the ratio r8
    tw = np.zeros(9 * 32, complex)
    for e in range(9 * 32):
        k2, lane = e >> 5, e & 31
        sg = -1.0 if (lane & 3) == 3 else 1.0
        tw[e] = sg * np.exp(1j * np.pi * lane * (1 + 4 * k2) / 1024) if k2 < 8 else \
            np.exp(1j * np.pi * lane / 32)
    return tw


TW = tables()


def exch_c(h, j):  # the pair-exchange constant of thread h, step j (SIGN = +1)
    return W(-4 * (8 + j)) if h else W(4 * j)


def forward(coef):
    """dft512_v2<1> after v2_fwd_in: returns x, y [32][8] (thread, j)."""
    A = [dft16(np.array([(coef[l + 32 * m] + 1j * coef[512 + l + 32 * m]) * W(2 * m)
                         for m in range(16)]), 1) for l in range(32)]
    scr = np.zeros(512, complex)
    for l in range(32):
        r8 = TW[8 * 32 + l]
        for k2 in range(8):
            p = TW[k2 * 32 + l]
            scr[tslot(l, k2)] = A[l][brev4(k2)] * p
            scr[tslot(l, k2 + 8)] = A[l][brev4(k2 + 8)] * p * r8
    B = [dft16(np.array([scr[tslot(2 * m + (l & 1), l >> 1)] for m in range(16)]), 1)
         for l in range(32)]
    x = np.zeros((32, 8), complex)
    y = np.zeros((32, 8), complex)
    for l in range(32):
        for j in range(8):
            keep, r = B[l][brev4(j)], B[l ^ 1][brev4(8 + j)]  # shfl.xor 1 of a[brev(8 + j)]
            t = r * exch_c(l & 1, j)
            x[l, j], y[l, j] = keep + t, keep - t
    return x, y


def inverse_tr(x, y):
    """fft::inverse_tr: register layout in, natural order out (x 512)."""
    A = [np.zeros(16, complex) for _ in range(32)]
    T = np.zeros((32, 8), complex)
    for l in range(32):
        for j in range(8):
            T[l, j] = (x[l, j] - y[l, j]) * np.conj(exch_c(l & 1, j))
            A[l][brev4(j)] = x[l, j] + y[l, j]
    for l in range(32):
        for j in range(8):
            A[l][brev4(8 + j)] = T[l ^ 1, j]
    A = [dft16_dit_br(a, -1) for a in A]
    scr = np.zeros(512, complex)
    for l in range(32):
        for m in range(16):
            scr[tslot(2 * m + (l & 1), l >> 1)] = A[l][m]
    out = np.zeros((32, 16), complex)
    for l in range(32):
        r8 = TW[8 * 32 + l]
        a = np.zeros(16, complex)
        for k in range(8):
            p = TW[k * 32 + l]
            a[brev4(k)] = scr[tslot(l, k)] * np.conj(p)
            a[brev4(k + 8)] = scr[tslot(l, k + 8)] * np.conj(p * r8)
        a = dft16_dit_br(a, -1)
        out[l] = [a[m] * np.conj(W(2 * m)) for m in range(16)]
    return out


def unfold(out):
    c = np.zeros(N)
    for l in range(32):
        for m in range(16):
            c[l + 32 * m], c[512 + l + 32 * m] = out[l, m].real, out[l, m].imag
    return c


def k_of(t, j, which):  # the frequency bk_tm_kernel assigns to thread t, x[j] / y[j]
    k2, h = t >> 1, t & 1
    return k2 + 16 * (8 * h + j) if which == "x" else k2 + 16 * (16 + 8 * h + j)


def true_spectrum(c):  # folded negacyclic spectrum: DFT512 of (c_n + i c_{n+512}) zeta^n
    zeta = np.exp(1j * np.pi / N)
    u = (c[:M] + 1j * c[M:]) * zeta ** np.arange(M)
    return np.fft.ifft(u) * M  # sum_n u_n exp(+2 pi i n k / 512)


def negacyclic(a, b):
    full = np.convolve(a, b)
    out = full[:N].copy()
    out[: len(full) - N] -= full[N:]
    return out


@pytest.fixture(scope="module")
def rng():
    return np.random.default_rng(20261021)


def test_forward_register_layout_and_scaling(rng):
    c = rng.integers(-512, 512, N).astype(float)
    x, y = forward(c)
    X = true_spectrum(c)
    for t in range(32):
        h = t & 1
        for j in range(8):
            sigma = W(-4 * (8 + j))  # the odd thread's scaling
            sx, sy = (1, 1) if h == 0 else (sigma, -sigma)
            assert abs(x[t, j] - sx * X[k_of(t, j, "x")]) < 1e-9 * np.abs(X).max()
            assert abs(y[t, j] - sy * X[k_of(t, j, "y")]) < 1e-9 * np.abs(X).max()
    # the 32 x 16 positions cover every frequency once
    ks = sorted(k_of(t, j, w) for t in range(32) for j in range(8) for w in "xy")
    assert ks == list(range(M))


def test_inverse_tr_is_the_exact_inverse(rng):
    c = rng.integers(-2**20, 2**20, N).astype(float)
    x, y = forward(c)
    back = unfold(inverse_tr(x, y)) / 512
    assert np.max(np.abs(back - c)) < 1e-6


@pytest.mark.parametrize("kind", ["random", "extreme"])
def test_pointwise_with_true_spectrum_gives_the_negacyclic_product(rng, kind):
    if kind == "random":
        d = rng.integers(-512, 512, N)
        b = rng.integers(-2**15, 2**15, N)
    else:  # aligned extremes: coefficient 0 of the product sums |d| |b|
        b = np.where(rng.integers(0, 2, N) == 1, 2**15 - 1, -2**15)
        d = np.zeros(N, np.int64)
        d[0] = 511 if b[0] > 0 else -512
        d[1:] = np.where(b[:0:-1] < 0, 511, -512)  # X^i X^(N-i) = -1 flips the sign
    x, y = forward(d.astype(float))
    B = true_spectrum(b.astype(float)) / 512
    px, py = np.zeros_like(x), np.zeros_like(y)
    for t in range(32):
        for j in range(8):
            px[t, j] = x[t, j] * B[k_of(t, j, "x")]
            py[t, j] = y[t, j] * B[k_of(t, j, "y")]
    got = unfold(inverse_tr(px, py))
    want = negacyclic(d.astype(np.int64), b.astype(np.int64)).astype(float)
    assert np.array_equal(np.rint(got), want)
    assert np.max(np.abs(got - want)) < 1e-3
