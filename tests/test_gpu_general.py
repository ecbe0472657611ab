"""General-geometry path (flmisr_general.cu) vs the fp64 oracle, through the C ABI.

Geometries outside the polyphase fast path: missing and repeated integer phases, per-frame
fractional phases (a different kappa_i per frame, reading 19), negative shifts and shifts of more
than one HR pixel, K = 1, mag 3, a 5x5 PSF.  Same bars as the fast path (north_star): per-operator
relative L2 <= 1e-5, final image after 20 SCG passes <= 1e-3."""
import numpy as np
import pytest

from paper_2108_04315_b200 import synth

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2108_04315_b200 import flmisr  # noqa: E402


def rel(a, b):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


_rng = np.random.default_rng(2108)
CASES = {
    # name: (lr_h, lr_w, mag, psf, shifts (LR px), p_norm, lam, w)
    "missing_phase": (29, 35, 2, synth.gaussian_psf(), synth.shift_pattern(2)[:3], 1, 0.05, 3),
    "repeated_neg": (24, 31, 2, synth.gaussian_psf(),
                     np.array([[0, 0], [0, .5], [-.5, 0], [.5, .5], [0, .5], [1.0, -0.5]]), 1, 0.05, 3),
    "fractional": (33, 27, 2, synth.gaussian_psf(), np.round(_rng.uniform(-0.6, 0.9, (5, 2)), 3), 1, 0.05, 3),
    "single_frame": (30, 30, 2, synth.gaussian_psf(), np.array([[0.25, 0.0]]), 1, 0.05, 2),
    "mag3_psf5_p2": (17, 22, 3, synth.gaussian_psf(0.9, 5), np.round(_rng.uniform(0, 1, (7, 2)), 3), 2, 0.2, 3),
    "delta_w1": (21, 19, 2, synth.delta_psf(), np.array([[0, 0], [0.5, 0.5], [0.3, 0.1]]), 1, 0.05, 1),
    # integer phases outside [-(R+1), mag-1+R]: always the unfused kernels
    "far_shift": (26, 23, 2, synth.gaussian_psf(),
                  np.array([[0, 0], [2.0, -1.5], [0.5, 0.5], [-1.0, 1.5], [1.5, 0.0], [0.0, -0.5]]), 1, 0.05, 3),
    # mag 4: the fused gather's one-residue-class-per-thread form (at most one tap per axis and class)
    "mag4_quarter": (12, 17, 4, synth.gaussian_psf(),
                     np.array([[a / 4 + 0.05 * (b % 2), b / 4 + 0.04 * (a % 2)] for a in range(4) for b in range(4)]),
                     1, 0.05, 3),
    # mag 1 (deblurring + sub-pixel registration, no zoom) and many frames (K = 12, 3 chunks of 4)
    "mag1": (40, 52, 1, synth.gaussian_psf(), np.array([[0, 0], [0.5, 0.25], [-0.3, 0.6]]), 1, 0.05, 3),
    "k12": (20, 26, 2, synth.gaussian_psf(), np.round(_rng.uniform(0, 1, (12, 2)), 3), 1, 0.05, 3),
}
FUSABLE = {"far_shift": False}
# f-trace tolerance of the full runs (default 1e-4).  These two geometries are less well conditioned:
# a 1e-7 relative perturbation of y moves the oracle's own fp64 f trace by 4.4e-5 (far_shift) and
# 9.8e-5 (mag4_quarter) -- the rho'' regime of DESIGN.md reading 23 -- so fp32 rounding is held to 1e-3
# there; the final-image bar stays north_star's 1e-3.
TRACE_RTOL = {"far_shift": 1e-3, "mag4_quarter": 1e-3}


@pytest.fixture(params=["fused", "unfused"])
def impl(request, monkeypatch):
    """The fused tiled kernels (flmisr_general3.cu) and the unfused ones (flmisr_general.cu,
    FLMISR_GEN2=1 at plan time) on the same cases."""
    if request.param == "unfused":
        monkeypatch.setenv("FLMISR_GEN2", "1")
    return request.param


def make(orc, name, n_iter=20, impl=None):
    """A plan on the general-geometry kernels (FLMISR_NO_PC=1: geometries the per-phase streaming path
    also covers -- missing phases at x2 -- stay on the kernels this module tests; tests/test_gpu_pc.py
    runs them on the per-phase path)."""
    import os
    lr_h, lr_w, mag, psf, sh, pn, lam, w = CASES[name]
    k = len(sh)
    prev = os.environ.get("FLMISR_NO_PC")
    os.environ["FLMISR_NO_PC"] = "1"
    try:
        pl = flmisr.Plan(k=k, lr_h=lr_h, lr_w=lr_w, shifts=sh, psf=psf, mag=mag, p_norm=pn, lam=lam,
                         btv_window=w, n_iter=n_iter)
    finally:
        if prev is None:
            del os.environ["FLMISR_NO_PC"]
        else:
            os.environ["FLMISR_NO_PC"] = prev
    if impl is None:
        assert pl.fast_path in (0, 3)
    else:
        assert pl.fast_path == (3 if impl == "fused" and FUSABLE.get(name, True) else 0)
    pb = orc.Problem(k=k, lr_h=lr_h, lr_w=lr_w, shifts=sh, psf=psf, mag=mag, p_norm=pn, lam=lam, btv_window=w)
    return pl, pb


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32)).cuda()


@pytest.mark.parametrize("name", list(CASES))
def test_forward(orc, name):
    pl, pb = make(orc, name)
    x = synth.random_fields((pb.H, pb.W), 1)
    out = torch.zeros((pb.k, pb.lr_h, pb.lr_w), device="cuda")
    pl.debug(flmisr.OP_FORWARD, in0=dev(x), out=out)
    assert rel(out.cpu().numpy(), orc.forward(pb, x.astype(np.float64))) <= 1e-5


@pytest.mark.parametrize("name", list(CASES))
def test_adjoint(orc, name):
    pl, pb = make(orc, name)
    w = synth.random_fields((pb.k, pb.lr_h, pb.lr_w), 2, -1, 1)
    out = torch.zeros((pb.H, pb.W), device="cuda")
    pl.debug(flmisr.OP_ADJOINT, in0=dev(w), out=out)
    assert rel(out.cpu().numpy(), orc.adjoint(pb, w.astype(np.float64))) <= 1e-5


@pytest.mark.parametrize("name", list(CASES))
def test_gradient_and_value(orc, name, impl):
    pl, pb = make(orc, name, impl=impl)
    x = synth.random_fields((pb.H, pb.W), 3)
    y = synth.random_fields((pb.k, pb.lr_h, pb.lr_w), 4)
    out = torch.zeros((pb.H, pb.W), device="cuda")
    D, R, rr, _ = pl.debug(flmisr.OP_GRAD, lr=dev(y), in0=dev(x), out=out)
    g = orc.grad(pb, x.astype(np.float64), y.astype(np.float64))
    assert rel(out.cpu().numpy(), -g) <= 1e-5
    Dr, Rr = orc.value(pb, x.astype(np.float64), y.astype(np.float64))
    assert abs(D - Dr) <= 1e-5 * abs(Dr)
    assert abs(R - Rr) <= 1e-5 * abs(Rr) + 1e-12
    assert abs(rr - np.vdot(g, g)) <= 1e-5 * np.vdot(g, g)


@pytest.mark.parametrize("name", list(CASES))
def test_curvature(orc, name, impl):
    pl, pb = make(orc, name, impl=impl)
    x = synth.random_fields((pb.H, pb.W), 5)
    y = synth.random_fields((pb.k, pb.lr_h, pb.lr_w), 6)
    p = synth.random_fields((pb.H, pb.W), 7, -1, 1)
    delta, pp, mu, _ = pl.debug(flmisr.OP_CURV, lr=dev(y), in0=dev(x), in1=dev(p))
    ref = orc.curv(pb, x.astype(np.float64), y.astype(np.float64), p.astype(np.float64))
    assert abs(delta - ref) <= 1e-5 * abs(ref) + curv_rounding_bound(orc, pb, x, y, p)
    p64 = p.astype(np.float64)
    assert abs(pp - np.vdot(p64, p64)) <= 1e-6 * np.vdot(p64, p64)


def curv_rounding_bound(orc, pb, x, y, p, u=2.0 ** -24, sigmas=6.0):
    """Propagated fp32 rounding of the data curvature sum_i rho''(e_i) (A p)_i^2 (reading 23).

    For the Charbonnier penalty rho''(e) = eps^2 / (e^2 + eps^2)^(3/2) is ill-conditioned near e = 0:
    d rho''/de = -3 eps^2 e / (e^2 + eps^2)^(5/2), ~1/eps^2 at |e| ~ eps.  Each fp32 residual carries the
    rounding of a kd^2-term dot product, |de| ~ u (sqrt(kd^2) |z| + |y|); the per-pixel effects have
    independent signs, so their RMS times `sigmas` bounds the sum.  Squared L2 (rho'' = 2) has no term."""
    if pb.p_norm == 2:
        return 0.0
    x, y, p = (a.astype(np.float64) for a in (x, y, p))
    z, ap = orc.forward(pb, x), orc.forward(pb, p)
    e = z - y
    ntap = (pb.psf.shape[0] + 1) * (pb.psf.shape[1] + 1)
    de = 2 * u * (np.sqrt(ntap) * np.abs(z) + np.abs(y))
    d3 = 3 * pb.eps ** 2 * np.abs(e) / (e * e + pb.eps ** 2) ** 2.5
    return sigmas * float(np.sqrt(np.sum((d3 * de * ap * ap) ** 2)))


@pytest.mark.parametrize("name", ["missing_phase", "repeated_neg", "fractional", "delta_w1"])
def test_interpolation_fusion(orc, name):
    """integer-phase frames inserted at their HR sites (first frame wins), bilinear elsewhere.
    Inserted sites are copies (exact); bilinear sites carry fp32 vs fp64 interpolation rounding."""
    pl, pb = make(orc, name)
    y = synth.random_fields((pb.k, pb.lr_h, pb.lr_w), 9)
    out = torch.zeros((pb.H, pb.W), device="cuda")
    pl.debug(flmisr.OP_INTERP, lr=dev(y), out=out)
    ref = orc.interp_fuse(pb, y.astype(np.float64))
    np.testing.assert_allclose(out.cpu().numpy(), ref, rtol=0, atol=2e-6)


@pytest.mark.parametrize("name", list(CASES))
def test_reconstruct_matches_oracle(orc, name, impl):
    lr_h, lr_w, mag, psf, sh, pn, lam, w = CASES[name]
    truth = synth.phantom(mag * lr_h, mag * lr_w, seed=61)
    y = synth.detector_stack(truth, mag, sh, 1 / 255, seed=61).astype(np.float32)
    pl, pb = make(orc, name, n_iter=20, impl=impl)
    hr, rep = pl.reconstruct(dev(y))
    xo, tr, st = orc.scg(pb, y.astype(np.float64), 20)
    assert rel(hr.cpu().numpy(), xo) <= 1e-3
    assert rep["accepted"] == st["accepted"]
    np.testing.assert_allclose(rep["trace"][:, 1], tr[:, 1], rtol=TRACE_RTOL.get(name, 1e-4))
    np.testing.assert_array_equal(rep["trace"][:, 5], tr[:, 5])


@pytest.mark.parametrize("shape", [(64, 64), (37, 50)])
def test_general_path_agrees_with_fast_path(orc, shape, monkeypatch):
    """On a polyphase-complete stack the general kernels (FLMISR_FORCE_GENERAL) and the fast path
    compute the same operator: both match the oracle, and the full runs agree."""
    lr_h, lr_w = shape
    sh = synth.shift_pattern(2)
    truth = synth.phantom(2 * lr_h, 2 * lr_w, seed=62)
    y = synth.detector_stack(truth, 2, sh, 1 / 255, seed=62).astype(np.float32)
    pb = orc.Problem(k=4, lr_h=lr_h, lr_w=lr_w, shifts=sh, psf=synth.gaussian_psf())
    outs = []
    for force in (False, True):
        if force:
            monkeypatch.setenv("FLMISR_FORCE_GENERAL", "1")
        pl = flmisr.Plan(k=4, lr_h=lr_h, lr_w=lr_w, shifts=sh, psf=synth.gaussian_psf(), n_iter=20)
        assert pl.fast_path == (3 if force else 2)
        hr, _ = pl.reconstruct(dev(y))
        outs.append(hr.cpu().numpy())
    xo, _, _ = orc.scg(pb, y.astype(np.float64), 20)
    for o in outs:
        assert rel(o, xo) <= 1e-3
    assert rel(outs[1], outs[0]) <= 1e-3


def test_general_host_entry_and_determinism(orc):
    lr_h, lr_w, mag, psf, sh, pn, lam, w = CASES["fractional"]
    y = synth.random_fields((len(sh), lr_h, lr_w), 63)
    pl, _ = make(orc, "fractional", n_iter=8)
    a, ra = pl.reconstruct(dev(y))
    b, rb = pl.reconstruct(dev(y))
    assert torch.equal(a, b)
    np.testing.assert_array_equal(ra["trace"], rb["trace"])
    hh, _ = pl.reconstruct_host(y)
    np.testing.assert_array_equal(hh, a.cpu().numpy())
