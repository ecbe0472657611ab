"""Pins for the fp64 CPU oracle (oracle/flmisr_oracle.c) against things other than itself:
textbook polyphase slicing, scipy.ndimage, brute-force dense matrices, finite differences,
closed forms, SPEC worked examples (tests/golden/) and scipy.sparse.linalg.cg.

Each test names the DESIGN.md reading / paper passage it pins.  No GPU needed."""
import json
import os

import numpy as np
import pytest
import scipy.ndimage as ndi
import scipy.sparse.linalg as spla

from paper_2108_04315_b200 import synth

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def gold(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


def problem(orc, lr=8, mag=2, psf=None, shifts=None, **kw):
    psf = synth.gaussian_psf() if psf is None else psf
    shifts = synth.shift_pattern(mag) if shifts is None else np.asarray(shifts, dtype=np.float64)
    return orc.Problem(k=len(shifts), lr_h=lr, lr_w=kw.pop("lr_w", lr), shifts=shifts, psf=psf, mag=mag, **kw)


# ----------------------------------------------------------------------------- forward A_i
@pytest.mark.parametrize("mag", [2, 3])
def test_forward_delta_psf_is_polyphase_slicing(orc, mag):
    """PSF = delta with integer phases: A_i x = x[s_y::r, s_x::r] (reading 3; textbook polyphase)."""
    pb = problem(orc, lr=7, mag=mag, psf=synth.delta_psf())
    x = np.random.default_rng(1).uniform(size=(pb.H, pb.W))
    y = orc.forward(pb, x)
    for i, (dy, dx) in enumerate(pb.shifts):
        sy, sx = int(round(mag * dy)), int(round(mag * dx))
        np.testing.assert_array_equal(y[i], x[sy::mag, sx::mag])


def test_forward_flux_constant_image(orc):
    """Constant image -> the same constant in every frame incl. borders (clamp + sum h = 1)."""
    shifts = [[0, 0], [0.25, -0.4], [0.7, 0.5], [-0.3, 1.1]]
    pb = problem(orc, lr=9, mag=2, shifts=shifts, psf=synth.gaussian_psf(0.8, 5))
    y = orc.forward(pb, np.full((pb.H, pb.W), 0.37))
    np.testing.assert_allclose(y, 0.37, rtol=0, atol=1e-15)


@pytest.mark.parametrize("shift", [(0.0, 0.0), (0.5, 0.0), (0.25, 0.75), (0.3, -0.45), (1.0, 0.5)])
def test_forward_matches_scipy_shift_then_blur_then_sample(orc, shift):
    """A = D B M built from library routines: M = scipy.ndimage.shift (order 1, linear),
    B = scipy.ndimage.correlate, D = [::r].  Reading 19: identical away from the border (the
    composed kernel clamps once, the sequential form clamps twice); identical everywhere at zero shift."""
    mag = 2
    psf = synth.gaussian_psf(0.6, 3)
    pb = problem(orc, lr=12, mag=mag, shifts=[shift], psf=psf)
    x = np.random.default_rng(2).uniform(size=(pb.H, pb.W))
    ty, tx = mag * shift[0], mag * shift[1]
    m = ndi.shift(x, (-ty, -tx), order=1, mode="nearest", prefilter=False)  # m(u) = x(u + t)
    b = ndi.correlate(m, psf, mode="nearest")
    ref = b[0::mag, 0::mag]
    y = orc.forward(pb, x)[0]
    zero = ty == 0 and tx == 0
    sl = (slice(None), slice(None)) if zero else (slice(2, -2), slice(2, -2))
    np.testing.assert_allclose(y[sl], ref[sl], rtol=0, atol=1e-13)


def _dense(orc, pb):
    N, M = pb.H * pb.W, pb.k * pb.lr_h * pb.lr_w
    A = np.zeros((M, N))
    for n in range(N):
        e = np.zeros(N)
        e[n] = 1.0
        A[:, n] = orc.forward(pb, e.reshape(pb.H, pb.W)).ravel()
    At = np.zeros((N, M))
    for m in range(M):
        e = np.zeros(M)
        e[m] = 1.0
        At[:, m] = orc.adjoint(pb, e.reshape(pb.k, pb.lr_h, pb.lr_w)).ravel()
    return A, At


def test_adjoint_is_dense_transpose(orc):
    """Brute force on 8x8 HR: the adjoint applied to unit LR vectors is the transpose of the
    forward applied to unit HR vectors (S:37-63 spmv_transpose); fractional shifts and border folding."""
    pb = problem(orc, lr=4, mag=2, shifts=[[0, 0], [0.3, 0.5], [0.5, 0.9], [-0.25, 0.0]])
    A, At = _dense(orc, pb)
    np.testing.assert_allclose(At, A.T, rtol=0, atol=1e-15)
    # row sums = 1 (row-stochastic), every entry >= 0
    np.testing.assert_allclose(A.sum(axis=1), 1.0, atol=1e-14)
    assert (A >= 0).all()


@pytest.mark.parametrize("mag,lr", [(2, 16), (3, 10)])
def test_adjoint_identity(orc, mag, lr):
    """<Ax, y> = <x, A^T y> to 1e-12 relative in fp64 (north_star asks 1e-6)."""
    pb = problem(orc, lr=lr, mag=mag, psf=synth.gaussian_psf(0.5, 5))
    rng = np.random.default_rng(3)
    x = rng.standard_normal((pb.H, pb.W))
    y = rng.standard_normal((pb.k, pb.lr_h, pb.lr_w))
    lhs = np.vdot(orc.forward(pb, x), y)
    rhs = np.vdot(x, orc.adjoint(pb, y))
    assert abs(lhs - rhs) <= 1e-12 * (abs(lhs) + 1e-30)


# ----------------------------------------------------------------------------- values
def test_data_term_worked_example_S194(orc):
    g = gold("s194_data_term.json")
    pb = orc.Problem(k=1, lr_h=1, lr_w=2, shifts=np.zeros((1, 2)), psf=np.ones((1, 1)), mag=1,
                     p_norm=2, lam=0.0)
    x = np.array(g["x"]).reshape(1, 2)
    y = np.array(g["y"]).reshape(1, 1, 2)
    D, _ = orc.value(pb, x, y)
    assert D == g["value"]
    np.testing.assert_array_equal(orc.grad(pb, x, y).ravel(), g["gradient"])


def test_btv_worked_example_S203(orc):
    g = gold("s203_btv.json")
    img = np.array(g["image"])
    pb = orc.Problem(k=1, lr_h=2, lr_w=2, shifts=np.zeros((1, 2)), psf=np.ones((1, 1)), mag=1,
                     eps=g["eps"], btv_alpha=g["btv_alpha"], btv_window=g["btv_window"])
    _, R = orc.value(pb, img, img[None])
    assert abs(R - g["value"]) < 1e-15


def test_btv_zero_on_constant_and_nonnegative(orc):
    """R(const) = 0 and grad R(const) = 0; R >= 0."""
    pb = problem(orc, lr=6, mag=2, lam=1.0)
    c = np.full((pb.H, pb.W), 0.42)
    y = orc.forward(pb, c)
    D, R = orc.value(pb, c, y)
    assert R == 0.0 and D == 0.0
    np.testing.assert_allclose(orc.grad(pb, c, y), 0.0, atol=1e-15)
    x = np.random.default_rng(4).uniform(size=(pb.H, pb.W))
    assert orc.value(pb, x, y)[1] > 0


def test_btv_offset_set_and_weights(orc):
    """Q = {(dy,dx) in [0,w-1]^2} minus (0,0), gamma = alpha^(dx+dy) (Eq. prior): a single
    unit step edge between columns 0|1 of a 1-row image sees only dx=1 pairs (gamma=alpha) with
    dx>=1 crossing it; brute force on a 1x4 row with w=3 gives alpha*psi(1) + alpha^2*2*psi(1)."""
    eps = 1e-3
    pb = orc.Problem(k=1, lr_h=1, lr_w=4, shifts=np.zeros((1, 2)), psf=np.ones((1, 1)), mag=1,
                     btv_alpha=0.4, btv_window=3, eps=eps)
    x = np.array([[0.0, 1.0, 1.0, 1.0]])
    _, R = orc.value(pb, x, x[None])
    s1 = np.sqrt(1 + eps * eps) - eps
    assert abs(R - (0.4 * s1 + 0.16 * s1)) < 1e-15  # pairs (0,1) dx=1 and (0,2) dx=2


# ----------------------------------------------------------------------------- gradient
@pytest.mark.parametrize("p_norm,lam", [(1, 0.0), (1, 0.05), (2, 0.0), (2, 0.3)])
def test_gradient_central_fd_16x16(orc, p_norm, lam):
    """Central FD, h = 1e-6, on 16x16 HR: <= 1e-6 rel L2 and <= 1e-4 per coordinate (north_star)."""
    pb = problem(orc, lr=8, mag=2, p_norm=p_norm, lam=lam, shifts=[[0, 0], [0, .5], [.5, .5], [.5, .1]])
    rng = np.random.default_rng(5 + p_norm)
    x = rng.uniform(size=(pb.H, pb.W))
    y = rng.uniform(size=(pb.k, pb.lr_h, pb.lr_w))
    g = orc.grad(pb, x, y)
    h = 1e-6
    fd = np.zeros_like(x)
    for n in range(x.size):
        xp = x.copy().ravel(); xp[n] += h
        xm = x.copy().ravel(); xm[n] -= h
        fd.ravel()[n] = (orc.objective(pb, xp, y) - orc.objective(pb, xm, y)) / (2 * h)
    assert np.linalg.norm(g - fd) <= 1e-6 * np.linalg.norm(fd)
    assert np.max(np.abs(g - fd) / np.maximum(np.abs(fd), 1e-2)) <= 1e-4


# ----------------------------------------------------------------------------- curvature
@pytest.mark.parametrize("p_norm,lam", [(1, 0.05), (2, 0.05)])
def test_curvature_fd_of_gradient(orc, p_norm, lam):
    """delta = p^T Hess J p = d/dh <p, grad J(x + h p)> at h = 0 (central FD, h = 1e-6)."""
    pb = problem(orc, lr=8, mag=2, p_norm=p_norm, lam=lam)
    rng = np.random.default_rng(9)
    x = rng.uniform(size=(pb.H, pb.W))
    y = rng.uniform(size=(pb.k, pb.lr_h, pb.lr_w))
    p = rng.standard_normal((pb.H, pb.W))
    h = 1e-6
    fd = (np.vdot(p, orc.grad(pb, x + h * p, y)) - np.vdot(p, orc.grad(pb, x - h * p, y))) / (2 * h)
    d = orc.curv(pb, x, y, p)
    assert abs(d - fd) <= 1e-6 * abs(fd)


def test_curvature_closed_form_quadratic(orc):
    """p = 2, lambda = 0: delta = 2 ||A p||^2 exactly."""
    pb = problem(orc, lr=8, mag=2, p_norm=2, lam=0.0)
    rng = np.random.default_rng(10)
    x = rng.uniform(size=(pb.H, pb.W))
    y = rng.uniform(size=(pb.k, pb.lr_h, pb.lr_w))
    p = rng.standard_normal((pb.H, pb.W))
    ap = orc.forward(pb, p)
    assert abs(orc.curv(pb, x, y, p) - 2 * np.vdot(ap, ap)) <= 1e-12 * np.vdot(ap, ap)


# ----------------------------------------------------------------------------- init
def test_init_x0_bilinear_matches_scipy_zoom_grid(orc):
    """x0 = bilerp(y_0, (u - t_0)/r) with clamped LR indices == scipy.ndimage.map_coordinates
    (order 1, mode 'nearest') at the same coordinates (reading 14)."""
    pb = problem(orc, lr=9, mag=2, shifts=[[0.5, 0.25], [0, 0], [0, .5], [.5, 0]])
    y = np.random.default_rng(11).uniform(size=(pb.k, pb.lr_h, pb.lr_w))
    x0 = orc.init_x0(pb, y)
    ty, tx = 2 * 0.5, 2 * 0.25
    uu, vv = np.meshgrid((np.arange(pb.H) - ty) / 2, (np.arange(pb.W) - tx) / 2, indexing="ij")
    ref = ndi.map_coordinates(y[0], [uu, vv], order=1, mode="nearest")
    np.testing.assert_allclose(x0, ref, atol=1e-14)


# ----------------------------------------------------------------------------- SCG
def test_scg_quadratic_1d_worked_trace(orc):
    """S:339 worked example with the closed form of tests/golden/scg_quadratic_1d.json."""
    g = gold("scg_quadratic_1d.json")
    pb = orc.Problem(k=1, lr_h=1, lr_w=1, shifts=np.zeros((1, 2)), psf=np.ones((1, 1)), mag=1,
                     p_norm=2, lam=0.0)
    y = np.array([[[3.0]]])
    x1, tr1, _ = orc.scg(pb, y, 1, x0=np.zeros((1, 1)))
    assert abs(x1[0, 0] - g["x1"]) <= 4e-16 * 3
    assert abs(tr1[1, 3] - g["alpha0"]) <= 1e-16
    assert tr1[1, 4] == g["lambda_seq"][1]
    x2, tr2, _ = orc.scg(pb, y, 2, x0=np.zeros((1, 1)))
    assert abs(abs(x2[0, 0] - 3.0) - g["abs_x2_minus_3"]) <= 1e-15
    x3, tr3, st = orc.scg(pb, y, 3, x0=np.zeros((1, 1)))
    assert x3[0, 0] == 3.0                       # converged within 2-3 iterations
    assert list(tr3[1:, 4]) == g["lambda_seq"][1:1 + len(tr3) - 1]
    assert list(tr3[:, 5]) == [1.0] * len(tr3)   # every step accepted


def test_scg_equals_textbook_cg_on_quadratic(orc):
    """p = 2, lambda_BTV = 0, invertible PSF: SCG with exact curvature reproduces CG on
    2 A^T A x = 2 A^T y (scipy.sparse.linalg.cg, same x0) iterate for iterate."""
    pb = problem(orc, lr=6, mag=2, p_norm=2, lam=0.0)
    rng = np.random.default_rng(12)
    y = rng.uniform(size=(pb.k, pb.lr_h, pb.lr_w))
    A, _ = _dense(orc, pb)
    x0 = orc.init_x0(pb, y)
    its = []
    spla.cg(2 * A.T @ A, 2 * A.T @ y.ravel(), x0=x0.ravel(), rtol=1e-30, atol=0, maxiter=12,
            callback=lambda xk: its.append(xk.copy()))
    for n in (1, 3, 6, 12):
        xs, _, _ = orc.scg(pb, y, n, x0=x0)
        ref = its[n - 1]
        assert np.linalg.norm(xs.ravel() - ref) <= 1e-4 * np.linalg.norm(ref), n


def test_exact_recovery_delta_psf(orc):
    """Noise-free, PSF = delta, K = r^2 distinct integer phases, p = 2, lambda = 0: H = 2I and x* is
    recovered to <= 1e-12 within 3 iterations (north_star 'exact recovery').  Frames by slicing."""
    mag = 2
    pb = problem(orc, lr=16, mag=mag, psf=synth.delta_psf(), p_norm=2, lam=0.0)
    xs = synth.phantom(pb.H, pb.W, seed=3)
    y = np.stack([xs[int(mag * dy)::mag, int(mag * dx)::mag] for dy, dx in pb.shifts])
    x, tr, st = orc.scg(pb, y, 3)
    assert np.linalg.norm(x - xs) <= 1e-12 * np.linalg.norm(xs)


def test_exact_recovery_gaussian_psf(orc):
    """Noise-free, Gaussian sigma=0.5 PSF (invertible: Nyquist response 0.574), p = 2, lambda = 0:
    the unique minimiser x* is reached to ~1e-8 (CG with condition number <= 9.2)."""
    pb = problem(orc, lr=12, mag=2, p_norm=2, lam=0.0)
    xs = synth.phantom(pb.H, pb.W, seed=4)
    y = orc.forward(pb, xs)
    x, tr, st = orc.scg(pb, y, 80)
    assert np.linalg.norm(x - xs) <= 1e-8 * np.linalg.norm(xs)


def test_monotone_objective_over_accepted_steps(orc):
    """f_c non-increasing over accepted steps (P:404 'almost converged after 5')."""
    y, sh, _ = synth.make_stack(24, 2, seed=21)
    pb = problem(orc, lr=24, mag=2, shifts=sh)
    x, tr, st = orc.scg(pb, y, 20)
    f = tr[:, 1]
    assert np.all(np.diff(f) <= 0)
    assert st["accepted"] >= 1
    # the objective falls substantially within the paper's 20 iterations.  The stronger
    # "almost converged after 5" proxy does NOT hold at eps = 1e-3 on this
    # phantom (reading 8 note): it is recorded, not asserted.
    assert f[-1] <= 0.6 * f[0]


# ----------------------------------------------------------------------------- consensus
def test_partition_additivity(orc):
    """sum_h f_h equals the centralised J to 1e-10 (P:404 'the sum of the 4
    distributed objectives equals the centralized one')."""
    pb = problem(orc, lr=16, mag=2)
    rng = np.random.default_rng(13)
    x = rng.uniform(size=(pb.H, pb.W))
    y = rng.uniform(size=(pb.k, pb.lr_h, pb.lr_w))
    f = orc.objective(pb, x, y)
    for g in (2, 3, 4, 8):
        parts = [orc.value_rows(pb, x, y, *orc.band_bounds(pb.H, g, 2, h)) for h in range(g)]
        assert abs(sum(parts) - f) <= 1e-10 * abs(f)


@pytest.mark.parametrize("g", [2, 4, 8])
def test_band_simulation_equals_centralised(orc, g):
    """g bands with eta = 2 halo rows and the inner-outer border exchange follow the
    centralised SCG to 1e-10, i.e. no seam."""
    y, sh, _ = synth.make_stack(32, 2, seed=22)
    pb = problem(orc, lr=32, mag=2, shifts=sh)
    x1, tr1, _ = orc.scg(pb, y, 8, g=1)
    xg, trg, _ = orc.scg(pb, y, 8, g=g, eta=2)
    assert np.linalg.norm(xg - x1) <= 1e-10 * np.linalg.norm(x1)
    np.testing.assert_allclose(trg[:, 1], tr1[:, 1], rtol=1e-10)


def test_band_simulation_insufficient_halo_is_detected(orc):
    """eta = 1 < max(2R, w-1) = 2 reads a row the band does not hold (NaN poisoning)."""
    y, sh, _ = synth.make_stack(16, 2, seed=23)
    pb = problem(orc, lr=16, mag=2, shifts=sh)
    x, tr, st = orc.scg(pb, y, 2, g=2, eta=1)
    assert st["rc"] == -2 or not np.all(np.isfinite(x))


def test_fd_curvature_mode_agrees_with_exact(orc):
    """Paper-literal FD probe (sigma0 = 1e-4) vs exact curvature (reading 16)."""
    y, sh, _ = synth.make_stack(16, 2, seed=24)
    pb = problem(orc, lr=16, mag=2, shifts=sh)
    xe, tre, _ = orc.scg(pb, y, 10, curv_mode=orc.CURV_EXACT)
    xf, trf, _ = orc.scg(pb, y, 10, curv_mode=orc.CURV_FD)
    assert np.linalg.norm(xf - xe) <= 1e-3 * np.linalg.norm(xe)


# ----------------------------------------------------------------------------- interpolation fusion
def test_interp_fuse_single_frame_is_bilinear(orc):
    """k = 1, zero shift -> plain bilinear upsampling except at the frame's own sites."""
    pb = problem(orc, lr=9, mag=2, shifts=[[0.0, 0.0]])
    y = np.random.default_rng(30).uniform(size=(1, 9, 9))
    out = orc.interp_fuse(pb, y)
    np.testing.assert_allclose(out, orc.init_x0(pb, y), atol=1e-15)
    np.testing.assert_array_equal(out[0::2, 0::2], y[0])


def test_interp_fuse_complete_phases_is_exact_inverse(orc):
    """K = r^2 distinct integer phases of a sliced image reassemble it exactly."""
    for mag in (2, 3):
        pb = problem(orc, lr=7, mag=mag, psf=synth.delta_psf())
        x = np.random.default_rng(31).uniform(size=(pb.H, pb.W))
        y = orc.forward(pb, x)
        np.testing.assert_array_equal(orc.interp_fuse(pb, y), x)


def test_interp_fuse_partial_coverage(orc):
    """Two of four phases: their sites are exact, the others bilinear from frame 0."""
    pb = problem(orc, lr=8, mag=2, psf=synth.delta_psf(), shifts=[[0, 0], [0.5, 0.5]])
    x = np.random.default_rng(32).uniform(size=(pb.H, pb.W))
    y = orc.forward(pb, x)
    out = orc.interp_fuse(pb, y)
    np.testing.assert_array_equal(out[0::2, 0::2], x[0::2, 0::2])
    np.testing.assert_array_equal(out[1::2, 1::2], x[1::2, 1::2])
    x0 = orc.init_x0(pb, y)
    np.testing.assert_array_equal(out[0::2, 1::2], x0[0::2, 1::2])


# ----------------------------------------------------------------------------- NEXT-4 variants
def _psi(t, eps=1e-3):
    return np.sqrt(t * t + eps * eps) - eps


@pytest.mark.parametrize("offsets", [0, 1])
def test_btv_offsets_2x2_closed_form(orc, offsets):
    """w = 2 on [[a, b], [c, d]]: the quadrant has d = (0,1), (1,0), (1,1); Farsiu's set
    (m in [0,1], l in [-1,1], l + m >= 0) adds the anti-diagonal (1,-1) with gamma = alpha^2:
    R = alpha [psi(a-b) + psi(c-d) + psi(a-c) + psi(b-d)] + alpha^2 [psi(a-d) (+ psi(b-c))]."""
    a, b, c, d = 0.9, 0.1, 0.35, 0.6
    al = 0.4
    pb = orc.Problem(k=1, lr_h=2, lr_w=2, shifts=np.zeros((1, 2)), psf=np.ones((1, 1)), mag=1,
                     btv_alpha=al, btv_window=2, btv_offsets=offsets)
    x = np.array([[a, b], [c, d]])
    _, R = orc.value(pb, x, x[None])
    ref = al * (_psi(a - b) + _psi(c - d) + _psi(a - c) + _psi(b - d)) + al ** 2 * _psi(a - d)
    if offsets:
        ref += al ** 2 * _psi(b - c)
    assert abs(R - ref) <= 1e-15


def test_btv_farsiu_w3_weights(orc):
    """Farsiu w = 3 on a 3x3 image with a single bright centre pixel: every pair touching the centre
    has |diff| = 1; the offsets reaching it are the 11 of the set, each counted from both sides when
    valid.  Brute force from the set {(m, l): 0 <= m <= 2, -2 <= l <= 2, l + m >= 0} \\ {(0,0)}."""
    al, eps = 0.4, 1e-3
    pb = orc.Problem(k=1, lr_h=3, lr_w=3, shifts=np.zeros((1, 2)), psf=np.ones((1, 1)), mag=1,
                     btv_alpha=al, btv_window=3, btv_offsets=1, eps=eps)
    x = np.zeros((3, 3))
    x[1, 1] = 1.0
    _, R = orc.value(pb, x, x[None])
    offs = [(m, l) for m in range(3) for l in range(-2, 3) if l + m >= 0 and (m, l) != (0, 0)]
    assert len(offs) == 11
    ref = 0.0
    for m, l in offs:
        for (u, v) in [(1 - m, 1 - l), (1, 1)]:          # centre as second or first endpoint
            u2, v2 = u + m, v + l
            if 0 <= u < 3 and 0 <= v < 3 and 0 <= u2 < 3 and 0 <= v2 < 3 and (u, v) != (u2, v2):
                ref += al ** (abs(l) + m) * _psi(x[u, v] - x[u2, v2], eps)
    assert abs(R - ref) <= 1e-15


def test_gradient_and_curvature_fd_farsiu(orc):
    """Farsiu offsets: central-FD gradient (<= 1e-6 rel L2) and curvature (<= 1e-6) on 16x16."""
    pb = problem(orc, lr=8, mag=2, p_norm=1, lam=0.3, shifts=[[0, 0], [0, .5], [.5, .5], [.5, .1]])
    pb.btv_offsets = 1
    rng = np.random.default_rng(31)
    x = rng.uniform(size=(pb.H, pb.W))
    y = rng.uniform(size=(pb.k, pb.lr_h, pb.lr_w))
    g = orc.grad(pb, x, y)
    h = 1e-6
    fd = np.zeros_like(x)
    for n in range(x.size):
        xp = x.copy().ravel(); xp[n] += h
        xm = x.copy().ravel(); xm[n] -= h
        fd.ravel()[n] = (orc.objective(pb, xp, y) - orc.objective(pb, xm, y)) / (2 * h)
    assert np.linalg.norm(g - fd) <= 1e-6 * np.linalg.norm(fd)
    p = rng.standard_normal((pb.H, pb.W))
    cfd = (np.vdot(p, orc.grad(pb, x + h * p, y)) - np.vdot(p, orc.grad(pb, x - h * p, y))) / (2 * h)
    assert abs(orc.curv(pb, x, y, p) - cfd) <= 1e-6 * abs(cfd)


def test_band_simulation_farsiu_equals_centralised(orc):
    """The anti-diagonal offsets keep the halo at w - 1 rows: g = 4 bands with eta = 2 == g = 1."""
    y, sh, _ = synth.make_stack(32, 2, seed=32)
    pb = problem(orc, lr=32, mag=2, shifts=sh)
    pb.btv_offsets = 1
    x1, tr1, _ = orc.scg(pb, y, 6, g=1)
    xg, trg, _ = orc.scg(pb, y, 6, g=4, eta=2)
    assert np.linalg.norm(xg - x1) <= 1e-10 * np.linalg.norm(x1)


@pytest.mark.parametrize("rules", [1, 2, 3])
def test_scg_rule_variants_equal_cg_on_quadratic(orc, rules):
    """On a strictly convex quadratic PR+ never triggers (beta = <r,r>/mu > 0) and the Netlab scale
    rules keep lambda negligible, so every variant reproduces textbook CG (scipy) like Moller's."""
    pb = problem(orc, lr=6, mag=2, p_norm=2, lam=0.0)
    rng = np.random.default_rng(12)
    y = rng.uniform(size=(pb.k, pb.lr_h, pb.lr_w))
    A, _ = _dense(orc, pb)
    x0 = orc.init_x0(pb, y)
    its = []
    spla.cg(2 * A.T @ A, 2 * A.T @ y.ravel(), x0=x0.ravel(), rtol=1e-30, atol=0, maxiter=12,
            callback=lambda xk: its.append(xk.copy()))
    for n in (1, 3, 6, 12):
        xs, _, _ = orc.scg(pb, y, n, x0=x0, rules=rules)
        assert np.linalg.norm(xs.ravel() - its[n - 1]) <= 1e-4 * np.linalg.norm(its[n - 1]), n


def test_netlab_lambda_rule_1d(orc):
    """J(x) = (x - 3)^2 from x0 = 0, lambda_1 = 1e-6: the first step is accepted with Delta ~ 1 > 0.75,
    so Moller divides lambda by 4 and Netlab halves it (exact fp64 scalings of 1e-6); x1 agrees."""
    pb = orc.Problem(k=1, lr_h=1, lr_w=1, shifts=np.zeros((1, 2)), psf=np.ones((1, 1)), mag=1,
                     p_norm=2, lam=0.0)
    y = np.array([[[3.0]]])
    xm, trm, _ = orc.scg(pb, y, 1, x0=np.zeros((1, 1)))
    xn, trn, _ = orc.scg(pb, y, 1, x0=np.zeros((1, 1)), rules=orc.RULE_NETLAB)
    assert trm[1, 4] == 1e-6 / 4 and trn[1, 4] == 1e-6 / 2
    assert xm[0, 0] == xn[0, 0]


def test_pr_plus_monotone_on_robust_problem(orc):
    """PR+ and Netlab variants on the robust (Charbonnier) problem: f non-increasing over accepted
    steps and a substantial decrease within 20 passes (same bar as Moller's)."""
    y, sh, _ = synth.make_stack(24, 2, seed=21)
    pb = problem(orc, lr=24, mag=2, shifts=sh)
    for rules in (1, 2, 3):
        x, tr, st = orc.scg(pb, y, 20, rules=rules)
        assert np.all(np.diff(tr[:, 1]) <= 0)
        assert tr[-1, 1] <= 0.6 * tr[0, 1]
