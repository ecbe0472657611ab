"""Parity at BASELINE.json's full size (C3: K=4 LR 2048^2 -> 4096^2) in the launch configuration
bench.py times (streaming path, one wave of 128-column warp strips), against the fp64 oracle on the
full image (per-operator: value, gradient, curvature), and properties of a full reconstruction."""
import numpy as np
import pytest

from paper_2108_04315_b200 import synth

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2108_04315_b200 import flmisr  # noqa: E402


@pytest.fixture(scope="module")
def c3(orc):
    c = synth.CONFIGS["C3"]
    y, sh, _ = synth.make_stack(c["lr"], c["mag"], seed=c["seed"])
    pl = flmisr.Plan(k=4, lr_h=c["lr"], lr_w=c["lr"], shifts=sh, psf=synth.gaussian_psf(), mag=2, n_iter=c["n_iter"])
    pb = orc.Problem(k=4, lr_h=c["lr"], lr_w=c["lr"], shifts=sh, psf=synth.gaussian_psf(), mag=2)
    assert pl.fast_path == 2   # the streaming kernels bench.py times
    return y, pl, pb


def test_c3_gradient_value_curvature_random_inputs(orc, c3):
    """Per-operator bar (relative L2 <= 1e-5, north_star) on O(1) random fields at full size."""
    _, pl, pb = c3
    y = synth.random_fields((4, pl.lr_h, pl.lr_w), 72)
    yd = torch.from_numpy(y).cuda()
    xr = synth.random_fields((pl.H, pl.W), 73)
    x0 = torch.from_numpy(xr).cuda()
    x = xr.astype(np.float64)
    r = torch.zeros_like(x0)
    D, R, rr, _ = pl.debug(flmisr.OP_GRAD, lr=yd, in0=x0, out=r)
    g = orc.grad(pb, x, y.astype(np.float64))
    rn = r.cpu().numpy().astype(np.float64)
    assert np.linalg.norm(rn + g) <= 1e-5 * np.linalg.norm(g)
    Do, Ro = orc.value(pb, x, y.astype(np.float64))
    assert abs(D - Do) <= 1e-5 * Do and abs(R - Ro) <= 1e-5 * Ro
    p = synth.random_fields((pl.H, pl.W), 71, -1, 1)
    delta, pp, mu, _ = pl.debug(flmisr.OP_CURV, lr=yd, in0=x0, in1=torch.from_numpy(p).cuda())
    dref = orc.curv(pb, x, y.astype(np.float64), p.astype(np.float64))
    assert abs(delta - dref) <= 1e-5 * abs(dref)


def test_c3_gradient_at_initial_estimate(orc, c3):
    """Realistic inputs (phantom stack, x0 = bilinear): residuals are ~noise level, where rho'(e)
    = e / sqrt(e^2 + eps^2) has slope up to 1/eps = 1e3, so the fp32 rounding of z - y (~1e-7 on
    O(1) values) is amplified ~1e3x in the worst pixels: the bar here is 1e-4 relative L2."""
    y, pl, pb = c3
    yd = torch.from_numpy(y).cuda()
    x0 = torch.zeros((pl.H, pl.W), device="cuda")
    pl.debug(flmisr.OP_X0, lr=yd, out=x0)
    x = x0.cpu().numpy().astype(np.float64)
    np.testing.assert_allclose(x, orc.init_x0(pb, y.astype(np.float64)), rtol=0, atol=1e-6)
    r = torch.zeros_like(x0)
    D, R, rr, _ = pl.debug(flmisr.OP_GRAD, lr=yd, in0=x0, out=r)
    g = orc.grad(pb, x, y.astype(np.float64))
    assert np.linalg.norm(r.cpu().numpy() + g) <= 1e-4 * np.linalg.norm(g)
    Do, Ro = orc.value(pb, x, y.astype(np.float64))
    assert abs(D - Do) <= 1e-5 * Do and abs(R - Ro) <= 1e-5 * Ro


def test_c3_reconstruction_properties(orc, c3):
    """Full 20-pass reconstruction: objective non-increasing over accepted steps, the reported f
    equals the oracle's J at the returned image (to fp32 summation accuracy), finite output."""
    y, pl, pb = c3
    hr, rep = pl.reconstruct(torch.from_numpy(y).cuda())
    f = rep["trace"][:, 1]
    acc = rep["trace"][:, 5] > 0
    assert np.all(np.diff(f[acc]) <= 0)
    assert rep["iters_run"] == 20 and rep["accepted"] >= 15
    h = hr.cpu().numpy().astype(np.float64)
    assert np.isfinite(h).all()
    J = orc.objective(pb, h, y.astype(np.float64))
    assert abs(J - f[-1]) <= 1e-5 * J


@pytest.fixture(scope="module", params=["per_phase", "fused_general"])
def g3(orc, request):
    """G3: C3's size at quarter-pixel shifts, against the oracle on the full image, on the per-phase
    streaming kernels bench.py --config G3 times (fast_path 4) and on the fused general-geometry
    kernels (FLMISR_NO_PC=1, fast_path 3)."""
    import os
    c = synth.CONFIGS["G3"]
    sh = np.asarray(c["shifts"], dtype=np.float64)
    if request.param == "fused_general":
        os.environ["FLMISR_NO_PC"] = "1"
    try:
        pl = flmisr.Plan(k=len(sh), lr_h=c["lr"], lr_w=c["lr"], shifts=sh, psf=synth.gaussian_psf(), mag=c["mag"],
                         n_iter=c["n_iter"])
    finally:
        os.environ.pop("FLMISR_NO_PC", None)
    pb = orc.Problem(k=len(sh), lr_h=c["lr"], lr_w=c["lr"], shifts=sh, psf=synth.gaussian_psf(), mag=c["mag"])
    assert pl.fast_path == (4 if request.param == "per_phase" else 3)
    yield pl, pb
    pl.destroy()


def test_g3_gradient_value_curvature_random_inputs(orc, g3):
    """Per-operator bar at full size on the general path: gradient and value 1e-5 relative; the data
    curvature adds the rho'' conditioning bound of reading 23 (as in tests/test_gpu_general.py)."""
    from test_gpu_general import curv_rounding_bound
    pl, pb = g3
    y = synth.random_fields((pb.k, pl.lr_h, pl.lr_w), 82)
    yd = torch.from_numpy(y).cuda()
    xr = synth.random_fields((pl.H, pl.W), 83)
    x0 = torch.from_numpy(xr).cuda()
    x = xr.astype(np.float64)
    r = torch.zeros_like(x0)
    D, R, rr, _ = pl.debug(flmisr.OP_GRAD, lr=yd, in0=x0, out=r)
    g = orc.grad(pb, x, y.astype(np.float64))
    rn = r.cpu().numpy().astype(np.float64)
    assert np.linalg.norm(rn + g) <= 1e-5 * np.linalg.norm(g)
    Do, Ro = orc.value(pb, x, y.astype(np.float64))
    assert abs(D - Do) <= 1e-5 * Do and abs(R - Ro) <= 1e-5 * Ro
    p = synth.random_fields((pl.H, pl.W), 81, -1, 1)
    delta, pp, mu, _ = pl.debug(flmisr.OP_CURV, lr=yd, in0=x0, in1=torch.from_numpy(p).cuda())
    dref = orc.curv(pb, x, y.astype(np.float64), p.astype(np.float64))
    assert abs(delta - dref) <= 1e-5 * abs(dref) + curv_rounding_bound(orc, pb, xr, y, p)


@pytest.mark.parametrize("cfg", ["C4", "C6"])
def test_full_size_operators_c4_c6(orc, cfg):
    """The other BASELINE-size workloads in the configuration bench.py times: C4 (K=9 LR 2048^2 -> x3
    6144^2, 37.7 MP) and C6 (K=4 LR 4096^2 -> x2 8192^2, 67.1 MP, the paper's largest case): value,
    gradient and curvature on O(1) random fields against the fp64 oracle over the whole image
    (relative L2 <= 1e-5, north_star's per-operator bar)."""
    c = synth.CONFIGS[cfg]
    mag, lr = c["mag"], c["lr"]
    k = mag * mag
    sh = synth.shift_pattern(mag)
    pl = flmisr.Plan(k=k, lr_h=lr, lr_w=lr, shifts=sh, psf=synth.gaussian_psf(), mag=mag, n_iter=c["n_iter"])
    pb = orc.Problem(k=k, lr_h=lr, lr_w=lr, shifts=sh, psf=synth.gaussian_psf(), mag=mag)
    assert pl.fast_path == 2 and pl.loop_kernel
    y = synth.random_fields((k, lr, lr), 90)
    yd = torch.from_numpy(y).cuda()
    xr = synth.random_fields((pl.H, pl.W), 91)
    x0 = torch.from_numpy(xr).cuda()
    r = torch.zeros_like(x0)
    D, R, rr, _ = pl.debug(flmisr.OP_GRAD, lr=yd, in0=x0, out=r)
    x, y64 = xr.astype(np.float64), y.astype(np.float64)
    g = orc.grad(pb, x, y64)
    rn = r.cpu().numpy().astype(np.float64)
    e_g = np.linalg.norm(rn + g) / np.linalg.norm(g)
    assert e_g <= 1e-5
    del rn, r
    Do, Ro = orc.value(pb, x, y64)
    assert abs(D - Do) <= 1e-5 * Do and abs(R - Ro) <= 1e-5 * Ro
    p = synth.random_fields((pl.H, pl.W), 92, -1, 1)
    delta, pp, mu, _ = pl.debug(flmisr.OP_CURV, lr=yd, in0=x0, in1=torch.from_numpy(p).cuda())
    dref = orc.curv(pb, x, y64, p.astype(np.float64))
    print(f"\n{cfg}: gradient rel L2 {e_g:.2e}, value D rel {abs(D - Do) / Do:.2e}, "
          f"curvature rel {abs(delta - dref) / abs(dref):.2e}")
    assert abs(delta - dref) <= 1e-5 * abs(dref)
    pl.destroy()
