"""Host logic of the tridiagonal column pass (sr_tri.cuh), no GPU: the constants the library
tabulates (sr_sb_tri_constants) drive a plain numpy replay of the kernels' chunked recurrences, which must
reproduce (a) a dense solve of the cyclic tridiagonal column system and (b) the column part of the oracle's
FFT solve (Eq. 31-33): rfft along the rows, this solve per spectrum column, irfft == orc.solve."""
import numpy as np
import pytest


@pytest.fixture(scope="module")
def S():
    from paper_2003_12693_b200 import build
    build.build()
    from paper_2003_12693_b200 import srsb
    return srsb


def chunked_solve(d, consts, L):
    """The parallel form of sr_tri.cuh written out serially: local recurrences per chunk, carry sums over
    mmax neighbouring chunks (cyclic) with the closure factor, then the true forward / backward recurrences."""
    r, kappa, rho, clos, mmax = consts
    M = len(d)
    C = M // L
    ch = d.reshape(C, L)
    Bf = np.zeros(C, dtype=d.dtype)
    Bb = np.zeros(C, dtype=d.dtype)
    for c in range(C):
        y = z = 0.0
        for j in range(L):
            y = r * y + ch[c, j]
            z = r * z + ch[c, L - 1 - j]
        Bf[c], Bb[c] = y, z
    x = np.zeros((C, L), dtype=d.dtype)
    for c in range(C):
        y = z = 0.0
        w = 1.0
        for m in range(1, mmax + 1):
            y += w * Bf[(c - m) % C]
            z += w * Bb[(c + m) % C]
            w *= rho
        y *= clos
        z *= clos
        Y = np.zeros(L, dtype=d.dtype)
        for j in range(L):
            y = r * y + ch[c, j]
            Y[j] = y
        for j in range(L - 1, -1, -1):
            x[c, j] = kappa * (Y[j] + r * z)
            z = r * z + ch[c, j]
    return x.reshape(M)


@pytest.mark.parametrize("M,L,tau,mu,k2,N", [(16, 16, 0.05, 8.0, 0, 64), (64, 16, 0.05, 8.0, 3, 64), (1024, 16, 0.05, 8.0, 0, 1024),
                                           (64, 16, 5.0, 20.0, 1, 128), (16, 16, 5.0, 8.0, 0, 32), (128, 16, 0.0, 8.0, 5, 64),
                                           (512, 32, 0.05, 8.0, 128, 256), (256, 16, 0.25, 8.0, 0, 512), (128, 8, 1.0, 8.0, 64, 128)])
def test_constants_reproduce_the_dense_cyclic_tridiagonal_solve(S, M, L, tau, mu, k2, N):
    consts = S.tri_constants(tau, mu, N, k2, L, M // L)
    a = float(np.float32(tau)) * float(np.float32(mu))     # the ABI carries tau, mu as float32
    c = 1 + a * (4 - 2 * np.cos(2 * np.pi * k2 / N))
    A = np.zeros((M, M))
    for i in range(M):
        A[i, i] += c
        A[i, (i - 1) % M] -= a
        A[i, (i + 1) % M] -= a
    d = np.random.default_rng(M + k2).standard_normal(M)
    ref = np.linalg.solve(A, d)
    assert np.max(np.abs(chunked_solve(d, consts, L) - ref)) <= 1e-12 * max(1.0, np.max(np.abs(ref)))
    r, kappa, rho, clos, mmax = consts
    assert 0 <= r < 1 and 1 <= mmax <= M // L
    assert kappa == pytest.approx(1 / np.sqrt(c * c - 4 * a * a), rel=1e-14)
    assert a * r * r - c * r + a == pytest.approx(0.0, abs=1e-12)          # r is the small root of a r^2 - c r + a
    assert mmax == M // L or rho ** mmax <= 2.0 ** -48 * (1 + 1e-9)                       # truncated below fp32 rounding ...
    assert clos == (1.0 if mmax < M // L else pytest.approx(1 / (1 - rho ** (M // L))))   # ... or closed exactly


def test_row_fft_plus_column_solves_is_the_oracle_solve(S, orc):
    """Eq. (33) as the library computes it: FFT along the rows only, the cyclic tridiagonal system per spectrum
    column (complex right-hand sides: real and imaginary parts separately), inverse FFT."""
    M, N, tau, mu, L = 64, 32, float(np.float32(0.05)), 8.0, 16
    F = np.random.default_rng(3).standard_normal((M, N))
    spec = np.fft.rfft(F, axis=1)                      # [M][N/2 + 1]
    for k2 in range(N // 2 + 1):
        consts = S.tri_constants(tau, mu, N, k2, L, M // L)
        col = spec[:, k2]
        spec[:, k2] = chunked_solve(col.real.copy(), consts, L) + 1j * chunked_solve(col.imag.copy(), consts, L)
    phi = np.fft.irfft(spec, n=N, axis=1)
    assert np.max(np.abs(phi - orc.solve(F, tau, mu))) < 1e-12


def test_bad_arguments(S):
    with pytest.raises(S.SrsbError):
        S.tri_constants(0.05, 8.0, 64, 40, 16, 4)      # k2 > N/2
    with pytest.raises(S.SrsbError):
        S.tri_constants(0.05, 0.0, 64, 0, 16, 4)       # mu = 0
