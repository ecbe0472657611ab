"""Thin Python binding of the C ABI in include/flmisr.h (argument marshalling only).

Every step of the reconstruction runs in the sm_100a kernels of libflmisr.so; this module only
converts torch tensors / numpy arrays into pointers and the config struct.  There is no CPU
fallback: if the library is missing the import of this module fails loudly.

Names follow the C ABI: ``plan`` / ``reconstruct`` / ``destroy``.
"""
from __future__ import annotations

import ctypes as C
import os
import weakref

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("FLMISR_LIB", os.path.join(_HERE, "libflmisr.so"))

OK, ERR_CONFIG, ERR_SHAPE, ERR_CUDA, ERR_NCCL, ERR_NUMERIC = 0, -1, -2, -3, -4, -5
OP_FORWARD, OP_ADJOINT, OP_GRAD, OP_CURV, OP_VALUE, OP_X0, OP_INTERP = range(7)


class FlmisrError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"flmisr status {status}: {msg}")
        self.status = status


class Config(C.Structure):
    _fields_ = [
        ("k", C.c_int32), ("lr_h", C.c_int32), ("lr_w", C.c_int32),
        ("shifts", C.POINTER(C.c_double)),
        ("psf", C.POINTER(C.c_double)), ("psf_h", C.c_int32), ("psf_w", C.c_int32),
        ("mag", C.c_int32), ("p_norm", C.c_int32),
        ("l1_eps", C.c_double), ("lam", C.c_double), ("btv_alpha", C.c_double),
        ("btv_window", C.c_int32), ("n_iter", C.c_int32),
        ("scg_sigma0", C.c_double), ("scg_lambda0", C.c_double),
        ("rank", C.c_int32), ("world", C.c_int32),
        ("nccl_unique_id", C.c_void_p), ("device", C.c_int32),
        ("btv_offsets", C.c_int32), ("curv_mode", C.c_int32), ("scg_rules", C.c_int32),
        ("x0_mode", C.c_int32),
        ("det_rows", C.c_int32),
    ]


class Report(C.Structure):
    _fields_ = [("iters_run", C.c_int32), ("accepted", C.c_int32), ("converged_at", C.c_int32),
                ("failed_stage", C.c_int32), ("failed_iter", C.c_int32),
                ("f_trace", C.POINTER(C.c_double))]


EXPORTS = ("flmisr_plan", "flmisr_reconstruct", "flmisr_reconstruct_async", "flmisr_finish",
           "flmisr_profile", "flmisr_reconstruct_host", "flmisr_destroy", "flmisr_last_error",
           "flmisr_nccl_unique_id", "flmisr_plan_info", "flmisr_debug_apply", "flmisr_band",
           "flmisr_plan_virtual", "flmisr_reconstruct_virtual", "flmisr_pipeline_create",
           "flmisr_pipeline_submit", "flmisr_pipeline_wait", "flmisr_pipeline_destroy",
           "flmisr_reconstruct_virtual_peer", "flmisr_peer_export", "flmisr_peer_connect", "flmisr_interp_fuse")
PEER_BLOB_BYTES = 256   # FLMISR_PEER_BLOB_BYTES


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: build it with `python -m paper_2108_04315_b200.build` "
                          "(there is no CPU fallback)")
    lib = C.CDLL(LIB_PATH)
    vp = C.c_void_p
    lib.flmisr_plan.argtypes = [C.POINTER(Config), C.POINTER(vp)]
    lib.flmisr_reconstruct.argtypes = [vp, vp, vp, vp, vp, C.POINTER(Report)]
    lib.flmisr_reconstruct_host.argtypes = [vp, vp, vp, C.POINTER(Report)]
    lib.flmisr_reconstruct_async.argtypes = [vp, vp, vp, vp, vp]
    lib.flmisr_finish.argtypes = [vp, C.POINTER(Report)]
    lib.flmisr_profile.argtypes = [vp, C.c_int32, C.POINTER(C.c_double)]
    lib.flmisr_destroy.argtypes = [vp]
    lib.flmisr_last_error.restype = C.c_char_p
    lib.flmisr_nccl_unique_id.argtypes = [vp]
    lib.flmisr_plan_info.argtypes = [vp] + [C.POINTER(C.c_int32)] * 6
    lib.flmisr_debug_apply.argtypes = [vp, C.c_int32, vp, vp, vp, vp, C.POINTER(C.c_double)]
    lib.flmisr_band.argtypes = [C.c_int32] * 4 + [C.POINTER(C.c_int32)] * 2
    lib.flmisr_plan_virtual.argtypes = [C.POINTER(Config), C.POINTER(vp)]
    lib.flmisr_reconstruct_virtual.argtypes = [C.POINTER(vp), C.c_int32, vp, vp, vp, C.POINTER(Report)]
    lib.flmisr_reconstruct_virtual_peer.argtypes = [C.POINTER(vp), C.c_int32, vp, vp, vp, C.POINTER(Report)]
    lib.flmisr_peer_export.argtypes = [vp, vp]
    lib.flmisr_peer_connect.argtypes = [vp, vp]
    lib.flmisr_pipeline_create.argtypes = [vp, C.c_int32, C.c_int32, C.c_float, C.POINTER(vp)]
    lib.flmisr_pipeline_submit.argtypes = [vp, vp, vp]
    lib.flmisr_pipeline_wait.argtypes = [vp, C.POINTER(C.c_int64), C.POINTER(Report)]
    lib.flmisr_pipeline_destroy.argtypes = [vp]
    lib.flmisr_interp_fuse.argtypes = [vp, vp, vp, vp]
    for f in EXPORTS:
        if f == "flmisr_last_error":
            continue
        getattr(lib, f).restype = C.c_int
    return lib


_lib = _load()


def _check(st: int):
    if st != OK:
        raise FlmisrError(st, _lib.flmisr_last_error().decode())


def last_error() -> str:
    return _lib.flmisr_last_error().decode()


def nccl_unique_id() -> bytes:
    buf = C.create_string_buffer(128)
    _check(_lib.flmisr_nccl_unique_id(C.cast(buf, C.c_void_p)))
    return buf.raw


def band(H: int, world: int, rank: int, mag: int):
    """flmisr_band: owned HR rows [lo, hi) of `rank` (Eq. subfunction)."""
    lo, hi = C.c_int32(), C.c_int32()
    _check(_lib.flmisr_band(H, world, rank, mag, C.byref(lo), C.byref(hi)))
    return lo.value, hi.value


def broadcast_unique_id(group=None) -> bytes:
    """Rank 0 draws an ncclUniqueId and broadcasts its 128 bytes over the torch process group
    (any backend, e.g. gloo); every rank returns the same bytes."""
    import torch
    import torch.distributed as dist
    dev = torch.device("cuda", torch.cuda.current_device()) if dist.get_backend(group) == "nccl" else "cpu"
    buf = torch.zeros(128, dtype=torch.uint8, device=dev)
    if dist.get_rank(group) == 0:
        buf = torch.frombuffer(bytearray(nccl_unique_id()), dtype=torch.uint8).clone().to(dev)
    dist.broadcast(buf, src=0, group=group)
    return bytes(buf.cpu().tolist())


def _stream_handle(stream, device):
    """cudaStream_t for the C ABI.  torch's default stream has handle 0, which the ABI reads as 'the
    plan's own stream'; map it to cudaStreamLegacy (0x1) so the work stays ordered with torch ops."""
    import torch
    h = stream.cuda_stream if stream is not None else torch.cuda.current_stream(device).cuda_stream
    return C.c_void_p(h if h else 1)


def _ptr(t, numel=None, device=None, what="buffer", dtype="float32"):
    """Pointer of a contiguous torch tensor or numpy array.  numel: the element count the C ABI will
    read or write; device: the CUDA ordinal a device tensor must live on (None: a host array is
    expected).  A wrong dtype, device, size or layout raises ValueError before any C call."""
    if t is None:
        return None
    if hasattr(t, "data_ptr"):
        if not t.is_contiguous():
            raise ValueError(f"{what}: tensor must be contiguous")
        if str(t.dtype) != f"torch.{dtype}":
            raise ValueError(f"{what}: dtype {t.dtype}, expected {dtype}")
        if device is not None and (t.device.type != "cuda" or t.device.index != device):
            raise ValueError(f"{what}: tensor on {t.device}, expected cuda:{device}")
        if device is None and t.device.type != "cpu":
            raise ValueError(f"{what}: tensor on {t.device}, expected a host tensor")
        if numel is not None and t.numel() != numel:
            raise ValueError(f"{what}: {t.numel()} elements, expected {numel}")
        return C.c_void_p(t.data_ptr())
    if isinstance(t, np.ndarray):
        if device is not None:
            raise ValueError(f"{what}: numpy array given where a cuda:{device} tensor is expected")
        if not t.flags["C_CONTIGUOUS"]:
            raise ValueError(f"{what}: array must be C-contiguous")
        if t.dtype != np.dtype(dtype):
            raise ValueError(f"{what}: dtype {t.dtype}, expected {dtype}")
        if numel is not None and t.size != numel:
            raise ValueError(f"{what}: {t.size} elements, expected {numel}")
        return t.ctypes.data_as(C.c_void_p)
    raise TypeError(type(t))


class Plan:
    """flmisr_plan(): one plan per (geometry, parameters, rank); reusable across projections."""

    def __init__(self, k, lr_h, lr_w, shifts, psf, mag=2, p_norm=1, l1_eps=1e-3, lam=0.05,
                 btv_alpha=0.4, btv_window=3, n_iter=20, scg_sigma0=1e-4, scg_lambda0=1e-6,
                 rank=0, world=1, nccl_id: bytes | None = None, device=0, virtual=False,
                 btv_offsets=0, scg_rules=0, curv_mode=0, x0_mode=0, det_rows=0):
        self.shifts = np.ascontiguousarray(np.asarray(shifts, dtype=np.float64).reshape(k, 2))
        self.psf = np.ascontiguousarray(np.asarray(psf, dtype=np.float64))
        self._id = C.create_string_buffer(nccl_id, 128) if nccl_id is not None else None
        cfg = Config(k, lr_h, lr_w, self.shifts.ctypes.data_as(C.POINTER(C.c_double)),
                     self.psf.ctypes.data_as(C.POINTER(C.c_double)), self.psf.shape[0], self.psf.shape[1],
                     mag, p_norm, l1_eps, lam, btv_alpha, btv_window, n_iter, scg_sigma0, scg_lambda0,
                     rank, world, C.cast(self._id, C.c_void_p) if self._id is not None else None, device,
                     btv_offsets, curv_mode, scg_rules, x0_mode, det_rows)
        self.k, self.lr_h, self.lr_w, self.mag, self.n_iter = k, lr_h, lr_w, mag, n_iter
        self.rank, self.world, self.device = rank, world, device
        self._pipes = weakref.WeakSet()   # pipelines driving this plan (destroyed first)
        self._h = C.c_void_p()
        _check((_lib.flmisr_plan_virtual if virtual else _lib.flmisr_plan)(C.byref(cfg), C.byref(self._h)))
        vals = [C.c_int32() for _ in range(6)]
        _check(_lib.flmisr_plan_info(self._h, *[C.byref(v) for v in vals]))
        self.H, self.W, self.row_lo, self.row_hi, self.fast_path, self.loop_kernel = [v.value for v in vals]

    def destroy(self):
        for pipe in list(getattr(self, "_pipes", ())):
            pipe.destroy()
        if self._h:
            _lib.flmisr_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.destroy()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.destroy()

    def _report(self, rep: Report, trace: np.ndarray) -> dict:
        return dict(iters_run=rep.iters_run, accepted=rep.accepted, converged_at=rep.converged_at,
                    failed_stage=rep.failed_stage, failed_iter=rep.failed_iter,
                    trace=trace[: rep.iters_run + 1].copy())

    # argument checks of the device entry points (include/flmisr.h: full LR frames in, x0 H x W,
    # hr_out H x W on rank 0 / the owned band elsewhere, fp32, on the plan's device)
    def _out_numel(self):
        return self.H * self.W if self.rank == 0 or self.world == 1 else (self.row_hi - self.row_lo) * self.W

    def _lr_ptr(self, t):
        return _ptr(t, self.k * self.lr_h * self.lr_w, self.device, "lr_stack")

    def _hr_ptr(self, t, what):
        return _ptr(t, self.H * self.W, self.device, what)

    def _out_ptr(self, t):
        if t is not None and t.numel() == self.H * self.W:
            return _ptr(t, self.H * self.W, self.device, "hr_out")
        return _ptr(t, self._out_numel(), self.device, "hr_out")

    def reconstruct(self, lr_stack, x0=None, out=None, stream=None, raise_numeric=True):
        """flmisr_reconstruct on device tensors: lr_stack (k, lr_h, lr_w) fp32 CUDA; returns (hr, report)."""
        import torch
        if out is None:
            out = torch.empty((self.H, self.W), dtype=torch.float32, device=lr_stack.device)
        trace = np.zeros((self.n_iter + 1, 6))
        rep = Report(0, 0, 0, 0, 0, trace.ctypes.data_as(C.POINTER(C.c_double)))
        s = _stream_handle(stream, lr_stack.device)
        st = _lib.flmisr_reconstruct(self._h, self._lr_ptr(lr_stack), self._hr_ptr(x0, "x0"),
                                     self._out_ptr(out), s, C.byref(rep))
        if st != OK and (raise_numeric or st != ERR_NUMERIC):
            _check(st)
        return out, self._report(rep, trace)

    def interp_fuse(self, lr_stack, out=None, stream=None):
        """flmisr_interp_fuse: the multi-image interpolation fusion image (asynchronous on `stream`)."""
        import torch
        if out is None:
            out = torch.empty((self.H, self.W), dtype=torch.float32, device=lr_stack.device)
        _check(_lib.flmisr_interp_fuse(self._h, self._lr_ptr(lr_stack), self._hr_ptr(out, "hr_out"),
                                       _stream_handle(stream, lr_stack.device)))
        return out

    def reconstruct_async(self, lr_stack, out, x0=None, stream=None):
        """flmisr_reconstruct_async: enqueue only; pair with finish()."""
        s = _stream_handle(stream, lr_stack.device)
        _check(_lib.flmisr_reconstruct_async(self._h, self._lr_ptr(lr_stack), self._hr_ptr(x0, "x0"),
                                             self._out_ptr(out), s))

    def finish(self, raise_numeric=True):
        trace = np.zeros((self.n_iter + 1, 6))
        rep = Report(0, 0, 0, 0, 0, trace.ctypes.data_as(C.POINTER(C.c_double)))
        st = _lib.flmisr_finish(self._h, C.byref(rep))
        if st != OK and (raise_numeric or st != ERR_NUMERIC):
            _check(st)
        return self._report(rep, trace)

    def profile(self, enable: int = -1) -> dict:
        """flmisr_profile: enable=1 on+reset, 0 off+reset, -1 read.  Returns the counters before the call."""
        out = (C.c_double * 8)()
        _check(_lib.flmisr_profile(self._h, enable, out))
        names = ("value_grad", "update_curv", "setup_finalize", "reconstruct")
        return {n: dict(launches=int(out[2 * i]), ms=out[2 * i + 1]) for i, n in enumerate(names)}

    def reconstruct_host(self, lr_stack: np.ndarray, out: np.ndarray | None = None):
        """flmisr_reconstruct_host: host fp32 in, host fp32 out (H2D/D2H inside the call)."""
        lr = np.ascontiguousarray(lr_stack, dtype=np.float32)
        if out is None:
            out = np.empty((self.H, self.W), dtype=np.float32)
        trace = np.zeros((self.n_iter + 1, 6))
        rep = Report(0, 0, 0, 0, 0, trace.ctypes.data_as(C.POINTER(C.c_double)))
        _check(_lib.flmisr_reconstruct_host(self._h, _ptr(lr, self.k * self.lr_h * self.lr_w, what="lr_stack"),
                                            _ptr(out, self._out_numel(), what="hr_out"), C.byref(rep)))
        return out, self._report(rep, trace)

    def debug(self, op: int, lr=None, in0=None, in1=None, out=None):
        sc = (C.c_double * 4)()
        d = self.device
        _check(_lib.flmisr_debug_apply(self._h, op, _ptr(lr, self.k * self.lr_h * self.lr_w, d, "lr"),
                                       _ptr(in0, None, d, "in0"), _ptr(in1, None, d, "in1"), _ptr(out, None, d, "out"), sc))
        return list(sc)


def peer_connect(plan: "Plan", group=None) -> None:
    """Row bands over peer memory (flmisr_peer_export / flmisr_peer_connect): every rank exports the
    IPC handles of its halo buffers and mailbox block, the blobs are all-gathered over the torch
    process group in rank order, and each rank maps its peers'.  Afterwards plan.reconstruct* runs
    the band's whole SCG loop as one persistent kernel synchronised through peer memory."""
    import torch.distributed as dist
    blob = C.create_string_buffer(PEER_BLOB_BYTES)
    st = _lib.flmisr_peer_export(plan._h, C.cast(blob, C.c_void_p))
    err = None if st == OK else (st, last_error())
    # every rank takes part in the gather even if its export failed (an all-zero blob), so no rank is
    # left waiting in the collective; then every rank sees the same failure
    blobs = gather_blobs(bytes(blob.raw) if err is None else bytes(PEER_BLOB_BYTES), dist.get_world_size(group), group)
    if err is not None:
        raise FlmisrError(*err)
    if any(b == bytes(PEER_BLOB_BYTES) for b in blobs):
        raise FlmisrError(ERR_CONFIG, "peer export failed on another rank")
    allb = C.create_string_buffer(b"".join(blobs), len(blobs) * PEER_BLOB_BYTES)
    _check(_lib.flmisr_peer_connect(plan._h, C.cast(allb, C.c_void_p)))


def gather_blobs(blob: bytes, world: int, group=None) -> list:
    """All-gather one fixed-size byte blob per rank over the torch process group (rank order)."""
    import torch.distributed as dist
    out = [None] * world
    dist.all_gather_object(out, blob, group=group)
    if any(not isinstance(b, bytes) or len(b) != len(blob) for b in out):
        raise FlmisrError(-1, "peer blobs of unequal size")
    return out


def reconstruct_virtual_peer(plans, lr_stack, x0=None, out=None):
    """flmisr_reconstruct_virtual_peer: the g bands (Plan(..., virtual=True, rank=h, world=g)) as the
    peer-memory band loop, all in one cooperative launch on one device; returns (hr, report)."""
    import torch
    p0 = plans[0]
    if out is None:
        out = torch.empty((p0.H, p0.W), dtype=torch.float32, device=lr_stack.device)
    arr = (C.c_void_p * len(plans))(*[p._h.value for p in plans])
    trace = np.zeros((p0.n_iter + 1, 6))
    rep = Report(0, 0, 0, 0, 0, trace.ctypes.data_as(C.POINTER(C.c_double)))
    torch.cuda.current_stream(lr_stack.device).synchronize()
    _check(_lib.flmisr_reconstruct_virtual_peer(arr, len(plans), p0._lr_ptr(lr_stack), p0._hr_ptr(x0, "x0"),
                                                p0._hr_ptr(out, "hr_out"), C.byref(rep)))
    return out, p0._report(rep, trace)


def reconstruct_virtual(plans, lr_stack, x0=None, out=None):
    """flmisr_reconstruct_virtual: the g bands of one reconstruction (plans from Plan(..., virtual=True,
    rank=h, world=g)) on one device with copies in place of NCCL; returns (hr, report)."""
    import torch
    p0 = plans[0]
    if out is None:
        out = torch.empty((p0.H, p0.W), dtype=torch.float32, device=lr_stack.device)
    arr = (C.c_void_p * len(plans))(*[p._h.value for p in plans])
    trace = np.zeros((p0.n_iter + 1, 6))
    rep = Report(0, 0, 0, 0, 0, trace.ctypes.data_as(C.POINTER(C.c_double)))
    torch.cuda.current_stream(lr_stack.device).synchronize()
    _check(_lib.flmisr_reconstruct_virtual(arr, len(plans), p0._lr_ptr(lr_stack), p0._hr_ptr(x0, "x0"),
                                           p0._hr_ptr(out, "hr_out"), C.byref(rep)))
    return out, p0._report(rep, trace)


class Pipeline:
    """flmisr_pipeline_*: streamed capture-reconstruct.  submit() enqueues
    H2D -> SCG -> D2H of one view and returns; views overlap up to `depth` in flight.  Host buffers
    (numpy arrays or pinned torch CPU tensors) are referenced until their view completes."""

    def __init__(self, plan: Plan, depth: int = 2, input_u16: bool = False, u16_scale: float = 1.0 / 65535.0):
        self.plan = plan
        self.depth = depth
        self._in_dtype = "uint16" if input_u16 else "float32"
        self._h = C.c_void_p()
        _check(_lib.flmisr_pipeline_create(plan._h, depth, int(input_u16), u16_scale, C.byref(self._h)))
        plan._pipes.add(self)
        self._keep = [None] * depth
        self._n = 0

    def submit(self, lr_host, hr_host=None):
        slot = self._n % self.depth
        p = self.plan
        _check(_lib.flmisr_pipeline_submit(self._h, _ptr(lr_host, p.k * p.lr_h * p.lr_w, None, "lr_host", self._in_dtype),
                                           _ptr(hr_host, p.H * p.W, None, "hr_host")))
        self._keep[slot] = (lr_host, hr_host)
        self._n += 1

    def wait(self) -> dict:
        n = C.c_int64()
        rep = Report(0, 0, 0, 0, 0, None)
        _check(_lib.flmisr_pipeline_wait(self._h, C.byref(n), C.byref(rep)))
        self._keep = [None] * self.depth
        return dict(done=n.value, iters_run=rep.iters_run, accepted=rep.accepted,
                    converged_at=rep.converged_at, failed_stage=rep.failed_stage)

    def destroy(self):
        if self._h:
            if self.plan._h:   # flmisr_destroy(plan) already freed an attached pipeline
                _lib.flmisr_pipeline_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.destroy()
        except Exception:
            pass


# ---- functional names mirroring the C ABI ----
def plan(**kw) -> Plan:
    return Plan(**kw)


def reconstruct(p: Plan, lr_stack, x0=None, out=None, stream=None):
    return p.reconstruct(lr_stack, x0=x0, out=out, stream=stream)


def destroy(p: Plan):
    p.destroy()
