"""Image-quality metrics for the SR-vs-interpolation protocol (test harness, not product code):
PSNR and SSIM as SPEC defines them: PSNR = 10 log10(peak^2 / MSE); SSIM = mean over all
8 x 8 windows (valid positions) of the standard structural similarity with C1 = (0.01 L)^2,
C2 = (0.03 L)^2, L = the intensity range (1 for [0, 1] images), window statistics with 1/64 weights."""
import numpy as np


def psnr(a, b, peak: float = 1.0) -> float:
    mse = float(np.mean((np.asarray(a, np.float64) - np.asarray(b, np.float64)) ** 2))
    return float("inf") if mse == 0 else 10.0 * np.log10(peak * peak / mse)


def _box(x, win):
    c = np.cumsum(np.cumsum(np.pad(x, ((1, 0), (1, 0))), 0), 1)
    return (c[win:, win:] - c[:-win, win:] - c[win:, :-win] + c[:-win, :-win]) / (win * win)


def ssim(a, b, win: int = 8, L: float = 1.0) -> float:
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    if a.shape != b.shape:
        raise ValueError("dimension mismatch")
    C1, C2 = (0.01 * L) ** 2, (0.03 * L) ** 2
    ma, mb = _box(a, win), _box(b, win)
    va = _box(a * a, win) - ma * ma
    vb = _box(b * b, win) - mb * mb
    cov = _box(a * b, win) - ma * mb
    s = ((2 * ma * mb + C1) * (2 * cov + C2)) / ((ma * ma + mb * mb + C1) * (va + vb + C2))
    return float(s.mean())


def ssim_brute(a, b, win: int = 8, L: float = 1.0) -> float:
    """The same definition, window by window with plain loops (pin for ssim())."""
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    C1, C2 = (0.01 * L) ** 2, (0.03 * L) ** 2
    vals = []
    for i in range(a.shape[0] - win + 1):
        for j in range(a.shape[1] - win + 1):
            wa, wb = a[i:i + win, j:j + win].ravel(), b[i:i + win, j:j + win].ravel()
            ma, mb = wa.mean(), wb.mean()
            va, vb = ((wa - ma) ** 2).mean(), ((wb - mb) ** 2).mean()
            cov = ((wa - ma) * (wb - mb)).mean()
            vals.append(((2 * ma * mb + C1) * (2 * cov + C2)) / ((ma * ma + mb * mb + C1) * (va + vb + C2)))
    return float(np.mean(vals))
