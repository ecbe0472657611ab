"""C-ABI checks that need no GPU: the library loads, exports every symbol include/flmisr.h
declares, and rejects invalid configurations before any GPU work."""
import os
import re

import numpy as np
import pytest

from paper_2108_04315_b200 import build as fbuild
from paper_2108_04315_b200 import synth

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def fl():
    fbuild.build()
    import torch  # noqa: F401  (maps the torch-bundled libnccl.so.2 like a real caller)
    from paper_2108_04315_b200 import flmisr
    return flmisr


def test_exports_every_declared_symbol(fl):
    hdr = open(os.path.join(ROOT, "include", "flmisr.h")).read()
    declared = set(re.findall(r"^\s*(?:flmisr_status|const char\*)\s+(flmisr_\w+)\(", hdr, re.M))
    assert {"flmisr_plan", "flmisr_reconstruct", "flmisr_destroy"} <= declared
    for name in declared:
        assert hasattr(fl._lib, name), name
    assert declared == set(fl.EXPORTS)


def cfg(**kw):
    base = dict(k=4, lr_h=16, lr_w=16, shifts=synth.shift_pattern(2), psf=synth.gaussian_psf(), mag=2)
    base.update(kw)
    return base


@pytest.mark.parametrize("kw,msg", [
    (dict(psf=np.ones((3, 3))), "sum to 1"),
    (dict(psf=np.ones((2, 2)) / 4), "odd"),
    (dict(psf=-synth.gaussian_psf() + 2 / 9), ">= 0"),
    (dict(k=0, shifts=np.zeros((0, 2))), "k must be"),
    (dict(p_norm=3), "p_norm"),
    (dict(l1_eps=0.0), "l1_eps"),
    (dict(btv_alpha=1.0), "btv_alpha"),
    (dict(btv_window=4), "btv_window"),
    (dict(lam=-1.0), "lambda"),
    (dict(mag=5), "mag"),
    # general geometries run on one GPU; bands need the polyphase fast path
    (dict(k=3, shifts=synth.shift_pattern(2)[:3], world=2, rank=0, nccl_id=b"\0" * 128), "row-band partitioning"),
    (dict(shifts=np.array([[0, 0], [0, .5], [.5, .5], [.5, .5]]), world=2, rank=1, nccl_id=b"\0" * 128),
     "row-band partitioning"),
    (dict(k=65, shifts=np.zeros((65, 2))), "k <= 64"),
    (dict(btv_offsets=2), "btv_offsets"),
    (dict(scg_rules=4), "scg_rules"),
    (dict(curv_mode=2), "curv_mode"),
    (dict(curv_mode=1, scg_sigma0=0.0), "scg_sigma0"),
    (dict(curv_mode=1, world=2, rank=0, nccl_id=b"\0" * 128), "world must be 1"),
    (dict(btv_offsets=1, world=2, rank=0, nccl_id=b"\0" * 128), "world must be 1"),
    (dict(x0_mode=2), "x0_mode"),
    (dict(x0_mode=1, shifts=synth.shift_pattern(2) + 0.1, world=2, rank=0, nccl_id=b"\0" * 128),
     "x0_mode = 1 with fractional HR shifts needs world == 1"),
    (dict(det_rows=4), "det_rows"),
    (dict(det_rows=2), "det_rows"),
    (dict(det_rows=-1), "det_rows"),
    (dict(det_rows=5000), "det_rows"),
])
def test_config_errors_raised_before_gpu_work(fl, kw, msg):
    c = cfg(**kw)
    with pytest.raises(fl.FlmisrError) as ei:
        fl.Plan(**c)
    assert ei.value.status == fl.ERR_CONFIG
    assert msg in str(ei.value)


def test_band_too_small_names_minimum_height(fl):
    c = cfg(lr_h=2, lr_w=16, world=4, rank=0, nccl_id=b"\0" * 128)
    with pytest.raises(fl.FlmisrError) as ei:
        fl.Plan(**c)
    assert ei.value.status == fl.ERR_CONFIG
    assert "minimum HR height" in str(ei.value)


def test_det_band_too_small_names_tile_minimum(fl):
    """det mode: every band must hold at least one lcm(det_rows, mag) tile row block"""
    c = cfg(lr_h=8, lr_w=16, world=4, rank=0, nccl_id=b"\0" * 128, det_rows=6)
    with pytest.raises(fl.FlmisrError) as ei:
        fl.Plan(**c)
    assert ei.value.status == fl.ERR_CONFIG
    assert "minimum HR height 24" in str(ei.value)


def test_peer_entry_points_reject_bad_arguments_without_a_gpu(fl):
    """The peer-memory band loop's entry points validate before touching a device."""
    import ctypes as C
    buf = C.create_string_buffer(fl.PEER_BLOB_BYTES)
    assert fl._lib.flmisr_peer_export(None, C.cast(buf, C.c_void_p)) == -2          # FLMISR_ERR_SHAPE
    assert "plan" in fl.last_error()
    assert fl._lib.flmisr_peer_connect(None, C.cast(buf, C.c_void_p)) == -2
    arr = (C.c_void_p * 1)(None)
    assert fl._lib.flmisr_reconstruct_virtual_peer(arr, 1, None, None, None, None) == -2
    assert "2 <= g <= 8" in fl.last_error()
    arr9 = (C.c_void_p * 9)(*([None] * 9))
    assert fl._lib.flmisr_reconstruct_virtual_peer(arr9, 9, None, None, None, None) == -2


def test_interp_fuse_and_binding_checks_without_a_gpu(fl):
    """flmisr_interp_fuse rejects a NULL plan / NULL buffers before any device work; the binding
    rejects wrong dtypes, devices and sizes before the C call."""
    assert fl._lib.flmisr_interp_fuse(None, None, None, None) == -2
    assert "plan" in fl.last_error()
    import torch
    with pytest.raises(ValueError, match="dtype"):
        fl._ptr(torch.zeros(4, dtype=torch.float64), 4, None, "x")
    with pytest.raises(ValueError, match="elements"):
        fl._ptr(np.zeros(3, np.float32), 4, None, "x")
    with pytest.raises(ValueError, match="expected cuda:0"):
        fl._ptr(torch.zeros(4), 4, 0, "x")
    with pytest.raises(ValueError, match="contiguous"):
        fl._ptr(np.zeros((4, 4), np.float32)[:, ::2], 8, None, "x")
