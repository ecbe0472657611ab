"""The PSNR / SSIM harness of the quality protocol (tests/quality.py) against SPEC's examples
(S:389-402): closed forms, identities, sign of anticorrelation and a window-by-window brute force."""
import numpy as np
import pytest

from quality import psnr, ssim, ssim_brute


def test_psnr_closed_forms():
    a = np.zeros((16, 16))
    assert psnr(a, a) == float("inf")
    assert abs(psnr(a, a + 0.1) - 20.0) <= 1e-12           # uniform error 0.1, peak 1 -> 20 dB
    rng = np.random.default_rng(0)
    x, y = rng.uniform(size=(2, 20, 30))
    direct = 10 * np.log10(1.0 / (((x - y) ** 2).sum() / x.size))
    assert abs(psnr(x, y) - direct) <= 1e-9
    assert psnr(x, y) == psnr(y, x)


def test_ssim_identities_and_brute_force():
    rng = np.random.default_rng(1)
    a, b = rng.uniform(size=(2, 32, 32))
    assert abs(ssim(a, a) - 1.0) <= 1e-12
    chk = 0.4 * (np.indices((32, 32)).sum(0) % 2 * 2 - 1.0)  # constant-free pattern: zero mean per window
    assert ssim(chk, -chk) < 0                               # image vs its negative
    assert abs(ssim(a, b) - ssim_brute(a, b)) <= 1e-9
    c = 0.5 * a + 0.3 * b
    assert abs(ssim(a, c) - ssim_brute(a, c)) <= 1e-9
    with pytest.raises(ValueError):
        ssim(a, b[:-1])
