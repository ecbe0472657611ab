"""Per-pixel parity of the operators on well-conditioned inputs, fast path and general path.

The relative-L2 bars of test_gpu_parity.py / test_gpu_general.py average over the image, so a wrong
fold at one corner or a dropped tap in one border row could hide under 1e-5 at 128^2 and above.
Here every pixel is checked (max-abs), with the image-border rows/columns (the clamp folds of
reading 4 and the valid-pairs rule of reading 5) reported separately.

Inputs: x uniform in [0, 1] and y = A x + m with |m| in [0.02, 0.5] and a random sign, so every
residual satisfies |e| >= 20 eps.  There rho'(e) and rho''(e) are well conditioned (DESIGN.md
reading 23: the fp32 rounding of e near |e| ~ eps is amplified ~1/eps), and the plain north_star bar
applies to the curvature on the general path too (no propagated-rounding allowance)."""
import numpy as np
import pytest

from paper_2108_04315_b200 import synth

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2108_04315_b200 import flmisr  # noqa: E402
import test_gpu_general as gen  # noqa: E402
import test_gpu_parity as fast  # noqa: E402

ALL = [("fast", n) for n in fast.CASES] + [("general", n) for n in gen.CASES]


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32)).cuda()


def _make(orc, kind, name, impl):
    if kind == "fast":
        return fast.make(orc, name)
    return gen.make(orc, name, impl=impl)


def _inputs(orc, pb, seed):
    rng = np.random.default_rng(seed)
    x = rng.uniform(0, 1, (pb.H, pb.W)).astype(np.float32)
    z = orc.forward(pb, x.astype(np.float64))
    m = rng.uniform(0.02, 0.5, z.shape) * rng.choice([-1.0, 1.0], z.shape)
    y = (z + m).astype(np.float32)
    p = rng.uniform(-1, 1, (pb.H, pb.W)).astype(np.float32)
    e = orc.forward(pb, x.astype(np.float64)) - y.astype(np.float64)
    assert np.abs(e).min() >= 10 * pb.eps
    return x, y, p


def _border_mask(H, W, width=3):
    m = np.zeros((H, W), bool)
    m[:width], m[-width:], m[:, :width], m[:, -width:] = True, True, True, True
    return m


@pytest.fixture(params=["fused", "unfused"])
def impl(request, monkeypatch):
    if request.param == "unfused":
        monkeypatch.setenv("FLMISR_GEN2", "1")
    return request.param


@pytest.mark.parametrize("kind,name", ALL)
def test_gradient_pixelwise(orc, kind, name, impl):
    if kind == "fast" and impl == "unfused":
        pytest.skip("the unfused variant is a general-path option")
    pl, pb = _make(orc, kind, name, impl)
    x, y, _ = _inputs(orc, pb, 11)
    out = torch.zeros((pb.H, pb.W), device="cuda")
    D, R, rr, _ = pl.debug(flmisr.OP_GRAD, lr=dev(y), in0=dev(x), out=out)
    g = -orc.grad(pb, x.astype(np.float64), y.astype(np.float64))
    err = np.abs(out.cpu().numpy().astype(np.float64) - g)
    bm = _border_mask(pb.H, pb.W)
    scale = np.abs(g).max()
    print(f"\n{kind}/{name}/{impl}: grad max-abs err interior {err[~bm].max():.2e} border {err[bm].max():.2e} "
          f"(max |g| {scale:.2f})")
    assert err.max() <= 1e-5 * scale, np.unravel_index(np.argmax(err), err.shape)
    Dr, Rr = orc.value(pb, x.astype(np.float64), y.astype(np.float64))
    assert abs(D - Dr) <= 1e-5 * abs(Dr)
    assert abs(R - Rr) <= 1e-5 * abs(Rr) + 1e-12


@pytest.mark.parametrize("kind,name", ALL)
def test_curvature_plain_bar(orc, kind, name, impl):
    """north_star's 1e-5 per-operator bar with no rounding allowance."""
    if kind == "fast" and impl == "unfused":
        pytest.skip("the unfused variant is a general-path option")
    pl, pb = _make(orc, kind, name, impl)
    x, y, p = _inputs(orc, pb, 12)
    delta, pp, mu, _ = pl.debug(flmisr.OP_CURV, lr=dev(y), in0=dev(x), in1=dev(p))
    ref = orc.curv(pb, x.astype(np.float64), y.astype(np.float64), p.astype(np.float64))
    print(f"\n{kind}/{name}/{impl}: curvature rel err {abs(delta - ref) / abs(ref):.2e}")
    assert abs(delta - ref) <= 1e-5 * abs(ref)


@pytest.mark.parametrize("kind,name", ALL)
def test_forward_adjoint_pixelwise(orc, kind, name):
    pl, pb = _make(orc, kind, name, None)
    rng = np.random.default_rng(13)
    x = rng.uniform(0, 1, (pb.H, pb.W)).astype(np.float32)
    out = torch.zeros((pb.k, pb.lr_h, pb.lr_w), device="cuda")
    pl.debug(flmisr.OP_FORWARD, in0=dev(x), out=out)
    ref = orc.forward(pb, x.astype(np.float64))
    assert np.abs(out.cpu().numpy() - ref).max() <= 1e-6 * np.abs(ref).max()
    w = rng.uniform(-1, 1, (pb.k, pb.lr_h, pb.lr_w)).astype(np.float32)
    outa = torch.zeros((pb.H, pb.W), device="cuda")
    pl.debug(flmisr.OP_ADJOINT, in0=dev(w), out=outa)
    refa = orc.adjoint(pb, w.astype(np.float64))
    err = np.abs(outa.cpu().numpy() - refa)
    bm = _border_mask(pb.H, pb.W)
    scale = orc.adjoint(pb, np.abs(w).astype(np.float64)).max()   # sum of |terms| at the worst pixel
    assert err.max() <= 1e-6 * scale, (err[bm].max(), err[~bm].max(), scale)
