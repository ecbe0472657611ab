"""Streaming capture-reconstruct pipeline (flmisr_pipeline_*).

Every view streamed through the pipeline (H2D -> SCG -> D2H, overlapped across views) must equal,
byte for byte, the same plan's flmisr_reconstruct on that view (same kernels, deterministic sums),
for fp32 and 16-bit detector input, pinned and pageable host buffers, and through a numeric failure
in the middle of the stream."""
import numpy as np
import pytest

from paper_2108_04315_b200 import synth

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2108_04315_b200 import flmisr  # noqa: E402


def views(n, lr=48, lr_w=52, seed=90):
    sh = synth.shift_pattern(2)
    out = []
    for j in range(n):
        truth = synth.phantom(2 * lr, 2 * lr_w, seed=seed + j)
        out.append(synth.detector_stack(truth, 2, sh, 1 / 255, seed=seed + j).astype(np.float32))
    return out, sh


def plan(sh, lr=48, lr_w=52, n_iter=12, **kw):
    return flmisr.Plan(k=len(sh), lr_h=lr, lr_w=lr_w, shifts=sh, psf=synth.gaussian_psf(), n_iter=n_iter, **kw)


def direct(pl, y):
    hr, _ = pl.reconstruct(torch.from_numpy(y).cuda())
    return hr.cpu().numpy()


@pytest.mark.parametrize("depth,pinned", [(2, True), (3, False), (4, True)])
def test_pipeline_matches_direct_reconstruct(depth, pinned):
    ys, sh = views(7)
    pl = plan(sh)
    ref = [direct(pl, y) for y in ys]
    if pinned:
        ins = [torch.from_numpy(y).pin_memory() for y in ys]
        outs = [torch.empty((pl.H, pl.W)).pin_memory() for _ in ys]
    else:
        ins = [y.copy() for y in ys]
        outs = [np.empty((pl.H, pl.W), np.float32) for _ in ys]
    pipe = flmisr.Pipeline(pl, depth=depth)
    for a, b in zip(ins, outs):
        pipe.submit(a, b)
    rep = pipe.wait()
    assert rep["done"] == len(ys)
    for o, r in zip(outs, ref):
        np.testing.assert_array_equal(np.asarray(o), r)
    pipe.destroy()
    # the plan is usable directly again once the pipeline is gone
    np.testing.assert_array_equal(direct(pl, ys[0]), ref[0])


def test_pipeline_u16_input_equals_scaled_fp32():
    """16-bit codes converted on the device (value = scale * code in fp32) == the fp32 frames."""
    ys, sh = views(4, seed=95)
    scale = np.float32(1.0 / 65535.0)
    codes = [np.clip(np.rint(y * 65535.0), 0, 65535).astype(np.uint16) for y in ys]
    pl = plan(sh)
    ref = [direct(pl, (c.astype(np.float32) * scale).astype(np.float32)) for c in codes]
    pipe = flmisr.Pipeline(pl, depth=2, input_u16=True, u16_scale=float(scale))
    outs = [np.empty((pl.H, pl.W), np.float32) for _ in codes]
    for c, o in zip(codes, outs):
        pipe.submit(c, o)
    assert pipe.wait()["done"] == len(codes)
    for o, r in zip(outs, ref):
        np.testing.assert_array_equal(o, r)


def test_pipeline_odd_sizes_u16_tail():
    """K*h*w not a multiple of 8 (the conversion kernel's vector width): ragged tail path."""
    sh = synth.shift_pattern(2)
    rng = np.random.default_rng(5)
    codes = rng.integers(0, 65536, size=(4, 13, 21), dtype=np.uint16)
    pl = plan(sh, lr=13, lr_w=21, n_iter=5)
    scale = np.float32(1.0 / 65535.0)
    ref = direct(pl, (codes.astype(np.float32) * scale).astype(np.float32))
    pipe = flmisr.Pipeline(pl, depth=2, input_u16=True, u16_scale=float(scale))
    out = np.empty((pl.H, pl.W), np.float32)
    pipe.submit(codes, out)
    pipe.wait()
    np.testing.assert_array_equal(out, ref)


def test_pipeline_reports_numeric_failure_and_continues():
    ys, sh = views(4, seed=99)
    bad = ys[1].copy()
    bad[2, 5, 7] = np.nan
    pl = plan(sh)
    ref3 = direct(pl, ys[3])
    pipe = flmisr.Pipeline(pl, depth=2)
    outs = [np.empty((pl.H, pl.W), np.float32) for _ in range(4)]
    for y, o in zip([ys[0], bad, ys[2], ys[3]], outs):
        pipe.submit(y, o)
    with pytest.raises(flmisr.FlmisrError) as ei:
        pipe.wait()
    assert ei.value.status == flmisr.ERR_NUMERIC
    np.testing.assert_array_equal(outs[3], ref3)
    pipe.submit(ys[3], outs[0])
    assert pipe.wait()["done"] == 5
    np.testing.assert_array_equal(outs[0], ref3)


def test_pipeline_general_geometry():
    sh = np.array([[0, 0], [0.3, 0.1], [0.5, 0.5]])
    rng = np.random.default_rng(7)
    ys = [rng.uniform(0, 1, (3, 20, 23)).astype(np.float32) for _ in range(3)]
    pl = flmisr.Plan(k=3, lr_h=20, lr_w=23, shifts=sh, psf=synth.gaussian_psf(), n_iter=6)
    assert pl.fast_path == 3
    ref = [direct(pl, y) for y in ys]
    pipe = flmisr.Pipeline(pl, depth=2)
    outs = [np.empty((pl.H, pl.W), np.float32) for _ in ys]
    for y, o in zip(ys, outs):
        pipe.submit(y, o)
    pipe.wait()
    for o, r in zip(outs, ref):
        np.testing.assert_array_equal(o, r)


def test_pipeline_argument_errors():
    _, sh = views(1)
    pl = plan(sh)
    with pytest.raises(flmisr.FlmisrError) as ei:
        flmisr.Pipeline(pl, depth=1)
    assert ei.value.status == flmisr.ERR_SHAPE
    pipe = flmisr.Pipeline(pl, depth=2)
    with pytest.raises(flmisr.FlmisrError):
        pipe.submit(np.zeros((4, 48, 52), np.float32), None)
