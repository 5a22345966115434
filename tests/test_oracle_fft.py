"""Pins of the oracle's recursive radix-2 FFT: brute-force O(n^2) DFT, numpy.fft, Parseval, modes."""
import cmath
import math

import numpy as np
import pytest


def brute_dft(x, sign=-1):
    n = len(x)
    return [sum(x[m] * cmath.exp(sign * 2j * math.pi * k * m / n) for m in range(n)) for k in range(n)]


@pytest.mark.parametrize("n", [1, 2, 4, 8, 16, 32])
def test_fft_vs_bruteforce(orc, n):
    rng = np.random.default_rng(n)
    x = rng.standard_normal(n) + 1j * rng.standard_normal(n)
    X = orc.fft(x)
    ref = np.array(brute_dft(list(x)))
    assert np.max(np.abs(X - ref)) <= 1e-12 * max(1.0, np.max(np.abs(ref)))
    xi = orc.fft(X, inverse=True)
    assert np.max(np.abs(xi - x)) <= 1e-12


@pytest.mark.parametrize("M,N", [(1, 1), (2, 4), (4, 2), (8, 16), (16, 16), (4, 32)])
def test_fft2_vs_bruteforce_and_numpy(orc, M, N):
    rng = np.random.default_rng(M * 100 + N)
    x = rng.standard_normal((M, N)) + 1j * rng.standard_normal((M, N))
    X = orc.fft2(x)
    # brute force 2-D DFT
    ref = np.zeros((M, N), dtype=complex)
    for k1 in range(M):
        for k2 in range(N):
            s = 0j
            for m in range(M):
                for n in range(N):
                    s += x[m, n] * cmath.exp(-2j * math.pi * (k1 * m / M + k2 * n / N))
            ref[k1, k2] = s
    scale = max(1.0, np.max(np.abs(ref)))
    assert np.max(np.abs(X - ref)) <= 1e-12 * scale
    assert np.max(np.abs(X - np.fft.fft2(x))) <= 1e-12 * scale
    assert np.max(np.abs(orc.fft2(X, inverse=True) - x)) <= 1e-12


def test_parseval_and_single_mode(orc):
    rng = np.random.default_rng(7)
    x = rng.standard_normal(256) + 1j * rng.standard_normal(256)
    X = orc.fft(x)
    assert np.sum(np.abs(X) ** 2) == pytest.approx(256 * np.sum(np.abs(x) ** 2), rel=1e-12)
    k = 37
    mode = np.exp(2j * np.pi * k * np.arange(256) / 256)
    Y = orc.fft(mode)
    expect = np.zeros(256, dtype=complex)
    expect[k] = 256
    assert np.max(np.abs(Y - expect)) < 1e-10


def test_rejects_non_power_of_two(orc):
    with pytest.raises(ValueError):
        orc.fft(np.ones(6))
