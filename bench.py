#!/usr/bin/env python
"""FL-MISR SCG reconstruction benchmark (BASELINE.json metric: HR projections/sec and SCG iter/s
at 1/2/4/8 B200; % of HBM roofline).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl flmisr|reference] [--config C3]

A step is one whole reconstruction of one HR projection (every SURVEY 8(a) row: ingest, initial
estimate, init value/gradient, n_iter SCG passes of update+curvature and value+gradient with the
on-device scalar logic, output) from an LR stack already resident in HBM.  Workload (default C3):
K=4 LR 2048x2048 -> x2 SR 4096x4096 (16.8 MP HR), 20 SCG passes, synthetic phantom (DESIGN.md
section 4).  L2 (126 MB) is flushed before every timed step by a 512 MiB device write.

--impl reference times the fp64 CPU oracle (oracle/) as it stands on this host on bounded row-band
samples of the same workload (the cpu_baseline leg uses the same samples); under torchrun only rank 0
runs it.
Multi-GPU (torchrun, N > 1): the row bands of ONE projection (north_star; scaling "strong"):
the peer-memory band loop when every rank can map its peers (CUDA IPC, native peer atomics), else the
NCCL transport (reported in "transport_fallback").  Rank 0 checks the partitioned result against its
own single-GPU run ("parity"); every rank prints its identity to stderr and into "ranks"; replicas
(one projection per GPU, scaling "weak") are reported beside it.  --mode replicas times replicas only.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from paper_2108_04315_b200 import synth  # noqa: E402

METRIC = "HR projections/sec and SCG iter/s at 1/2/4/8 B200; % of HBM roofline"
WORKLOADS = {
    "C2": "C2: K=4 LR 1024x1024 -> x2 SR 2048x2048 (4.2 MP HR), 50 SCG passes",
    "C3": "C3: K=4 LR 2048x2048 -> x2 SR 4096x4096 (16.8 MP HR), 20 SCG passes",
    "C4": "C4: K=9 LR 2048x2048 -> x3 SR 6144x6144 (37.7 MP HR), 20 SCG passes",
    "G3": "G3: K=4 LR 2048x2048 at quarter-pixel shifts (a composed kernel per frame; per-phase streaming path) -> x2 4096x4096, 20 SCG passes",
    "C6": "C6: K=4 LR 4096x4096 -> x2 SR 8192x8192 (67.1 MP HR), 20 SCG passes (the paper's largest case)",
}
# The paper's own single-GPU runtime for exactly this workload (BASELINE.md tab:runtime, P:435-437:
# LR 2048^2 -> x2, 20 SCG iterations, 1x GTX 1080: 2.43 s) -- context on other hardware, not a target.
PAPER_1GPU_S = {"C3": 2.43}
# unfused general-geometry path (flmisr_general.cu): algorithmic bytes per HR pixel of the two-kernel phases
# for K = mag^2 frames (LR pixels = HR pixels): residual x,p,y,w 16 + gradient w,x,p,r_old,r_new 20;
# update x,p,r -> x,p 20 + data curvature x,p,y 12
BYTES_GEN_VALUE_GRAD = 36
BYTES_GEN_UPDATE_CURV = 32
# algorithmic HBM bytes per HR pixel per launch
BYTES_VALUE_GRAD = 20   # read x, p, Y, r_old; write r_new
BYTES_UPDATE_CURV = 24  # read x, p, r, Y; write x, p


def env_int(k, d):
    try:
        return int(os.environ.get(k, d))
    except ValueError:
        return d


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d.get("hbm_gbs", 6650.0)), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region (B200_PROFILING.md)."""
    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, dev: int):
        self.dev, self.proc, self.out = dev, None, ""

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                                          "-i", str(self.dev), "-lms", "50"], stdout=subprocess.PIPE,
                                         stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            out, _ = self.proc.communicate(timeout=5)
        except Exception:
            self.proc.kill()
            out = ""
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in out.strip().splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) < 7:
                continue
            try:
                sm.append(float(f[0]))
                mx.append(float(f[1]))
            except ValueError:
                continue
            for n, v in zip(names, f[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


_INPUTS = {}


def make_inputs(cfg: str):
    if cfg not in _INPUTS:
        c = synth.CONFIGS[cfg]
        y, sh, _ = synth.make_stack(c["lr"], c["mag"], seed=c["seed"], shifts=c.get("shifts"))
        _INPUTS[cfg] = (y, sh, c)
    return _INPUTS[cfg]


# ------------------------------------------------------------------------------------------ oracle
# One sampling method for both CPU legs (cpu_baseline and --impl reference): a SAMPLE is one HR row band
# of SAMPLE_ROWS rows of the workload, run by the fp64 oracle once with 0 SCG passes (init: x0, f0,
# r0) and once with 1 pass; t_pass = difference.  A projection is extrapolated as
# (H / SAMPLE_ROWS) x (t_init + n_iter x t_pass).
SAMPLE_ROWS = 256


def host_cpu() -> dict:
    model = None
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    model = ln.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    return {"nproc": os.cpu_count(), "model": model}


def oracle_band_run(cfg: str, band: int, rows: int, n_iter: int) -> float:
    """Seconds of one oracle SCG run (single-threaded fp64 C) on HR rows [band*rows, (band+1)*rows)."""
    from oracle import oracle as orc
    c = synth.CONFIGS[cfg]
    mag = c["mag"]
    lr_rows = rows // mag
    y, sh, _ = make_inputs(cfg)
    yb = np.ascontiguousarray(y[:, band * lr_rows:(band + 1) * lr_rows, :]).astype(np.float64)
    pb = orc.Problem(k=len(sh), lr_h=lr_rows, lr_w=c["lr"], shifts=sh, psf=synth.gaussian_psf(), mag=mag)
    t = time.perf_counter()
    orc.scg(pb, yb, n_iter)
    return time.perf_counter() - t


def oracle_sample(cfg: str, band: int):
    """One sample: (t_init, t_pass) seconds on band `band` of SAMPLE_ROWS rows."""
    t0 = oracle_band_run(cfg, band, SAMPLE_ROWS, 0)
    t1 = oracle_band_run(cfg, band, SAMPLE_ROWS, 1)
    return t0, max(t1 - t0, 1e-9)


def extrapolate(cfg: str, t_init: float, t_pass: float) -> float:
    """Seconds per projection from per-band sample times."""
    c = synth.CONFIGS[cfg]
    H = c["lr"] * c["mag"]
    return (H / SAMPLE_ROWS) * (t_init + c["n_iter"] * t_pass)


def sample_text(cfg: str, n: int) -> str:
    c = synth.CONFIGS[cfg]
    H = c["lr"] * c["mag"]
    return (f"{cfg}: {n} sample(s), each = one HR row band {SAMPLE_ROWS}x{H} (1/{H // SAMPLE_ROWS} of the projection) "
            f"run with 0 and with 1 SCG pass; projection = {H // SAMPLE_ROWS} x (t_init + {c['n_iter']} t_pass), "
            "extrapolated; single-threaded fp64 C oracle")


def cpu_baseline(cfg: str, n_iter_full: int):
    """cpu_baseline leg (rank 0, N = 1): every band of the projection sampled once (bounded: ~5 s for C3)."""
    c = synth.CONFIGS[cfg]
    nb = c["lr"] * c["mag"] // SAMPLE_ROWS
    ts = [oracle_sample(cfg, b) for b in range(nb)]
    t_proj = extrapolate(cfg, statistics.mean(t[0] for t in ts), statistics.mean(t[1] for t in ts))
    return {"value": 1.0 / t_proj, "unit": "proj/s", "cores": 1, "kind": "oracle", "sample": sample_text(cfg, nb),
            "host_cpu": host_cpu(), "s_per_projection": t_proj}


def run_reference(args):
    """--impl reference: the fp64 oracle as it stands, one sample per step (bands in rotation)."""
    rank = env_int("RANK", 0)
    if rank != 0:
        return 0
    cfg = args.config
    c = synth.CONFIGS[cfg]
    H = c["lr"] * c["mag"]
    nb = H // SAMPLE_ROWS
    n_full = c["n_iter"]
    import oracle.oracle as orc
    orc.build()
    for w in range(args.warmup):
        oracle_sample(cfg, w % nb)
    steps = []
    tr0 = time.perf_counter()
    for i in range(args.steps):
        steps.append(oracle_sample(cfg, i % nb))
    wall = time.perf_counter() - tr0
    t_proj = extrapolate(cfg, statistics.mean(t[0] for t in steps), statistics.mean(t[1] for t in steps))
    val = 1.0 / t_proj
    line = {"impl": "reference", "metric": METRIC, "value": val, "unit": "proj/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000 * wall / max(args.steps, 1),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": {"workload": WORKLOADS[cfg], "n_iter": n_full, "l2": "n/a (CPU)"},
            "cpu_baseline": {"value": val, "unit": "proj/s", "cores": 1, "kind": "oracle",
                             "sample": sample_text(cfg, args.steps), "host_cpu": host_cpu(),
                             "s_per_projection": t_proj},
            "e2e": {"value": val, "unit": "proj/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "scg_iters_per_s": n_full * val, "wall_s": wall}
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------------------------------------ GPU arm
def host_ring(y: np.ndarray, n: int, seed: int = 77):
    """n distinct pinned fp32 LR stacks: the workload's stack plus independent seeded detector noise."""
    import torch
    rng = np.random.default_rng(seed)
    out = []
    for j in range(n):
        v = y if j == 0 else (y + rng.standard_normal(y.shape, dtype=np.float32) * np.float32(1 / 255))
        out.append(torch.from_numpy(np.ascontiguousarray(v, dtype=y.dtype)).pin_memory())
    return out


def run_pipeline(flmisr, pl, ring, outs, views: int, dist=None, depth: int = 3, u16_scale=None):
    """Stream `views` views through a flmisr pipeline (host ring in, host images out); returns seconds
    from the first submit to the drained pipeline (one untimed warm-up view first)."""
    pipe = flmisr.Pipeline(pl, depth=depth, input_u16=u16_scale is not None,
                           u16_scale=u16_scale if u16_scale is not None else 1.0)
    pipe.submit(ring[0], outs[0] if outs else None)
    pipe.wait()
    if dist is not None:
        dist.barrier()
    t = time.perf_counter()
    for j in range(views):
        pipe.submit(ring[j % len(ring)], outs[j % len(outs)] if outs else None)
    rep = pipe.wait()
    el = time.perf_counter() - t
    assert rep["done"] == views + 1, rep
    pipe.destroy()
    return el


def run_stream(args):
    """C5: a sequence of C3 views streamed through flmisr_pipeline_*: H2D of
    each view's frames (fp32, or 16-bit detector codes with --u16), the reconstruction, D2H of the HR
    image, overlapped across views.  Reports views/s and the verdict against the acquisition window
    (4 exposures x 3 s per view)."""
    import torch
    import torch.distributed as dist

    from paper_2108_04315_b200 import flmisr
    world, rank, local = env_int("WORLD_SIZE", 1), env_int("RANK", 0), env_int("LOCAL_RANK", 0)
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    cfg = args.config
    y, sh, c = make_inputs(cfg)
    k, lr, mag, n_iter = len(sh), c["lr"], c["mag"], c["n_iter"]
    H = W = lr * mag
    partitioned = world > 1 and args.partition
    kw = dict(k=k, lr_h=lr, lr_w=lr, shifts=sh, psf=synth.gaussian_psf(), mag=mag, n_iter=n_iter, device=local)
    if partitioned:
        kw.update(rank=rank, world=world, nccl_id=flmisr.broadcast_unique_id())
    pl = flmisr.Plan(**kw)
    root = rank == 0 or not partitioned
    scale = None
    ring = host_ring(y, 16)
    if args.u16:   # 16-bit detector codes (value = code / 65535); frames are quantised once on the host
        scale = 1.0 / 65535.0
        ring = [torch.from_numpy(np.clip(np.rint(r.numpy() * 65535.0), 0, 65535).astype(np.uint16)).pin_memory()
                for r in ring]
    outs = [torch.empty((H, W), dtype=torch.float32).pin_memory() for _ in range(args.depth)] if root else None
    views = args.steps
    clk = ClockSampler(local)
    clk.start()
    el = run_pipeline(flmisr, pl, ring, outs, views, dist if world > 1 else None, depth=args.depth, u16_scale=scale)
    clocks = clk.stop()
    if world > 1:
        tt = torch.tensor([el], dtype=torch.float64, device="cuda")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        el = float(tt.item())
    # single-view latency (upload + reconstruct + download, nothing to overlap with)
    lat = []
    for j in range(3):
        lat.append(run_pipeline(flmisr, pl, ring, outs, 1, dist if world > 1 else None, depth=2, u16_scale=scale))
    vps = (1 if partitioned else world) * views / el
    acq_s = 12.0
    line = {"metric": "C5 streamed views/s (H2D + SCG + D2H per view, overlapped)", "value": vps, "unit": "views/s",
            "n_gpus": world, "steps": views, "warmup": 1, "ms_per_step": 1000 * el / views,
            "higher_is_better": True, "scaling": "strong" if partitioned else "weak", "vs_baseline": None,
            "dtype": "f32", "data": "synthetic",
            "config": {"workload": "C5: " + WORKLOADS[cfg] + f"; host ring of {len(ring)} distinct stacks",
                       "input": "uint16 codes (scale 1/65535)" if args.u16 else "fp32", "depth": args.depth,
                       "parallelism": (f"row bands x{world}" if partitioned else f"replicas x{world}")},
            "h2d_bytes_per_view": int(ring[0].numel() * ring[0].element_size()),
            "d2h_bytes_per_view": int(H * W * 4),
            "latency_ms_single_view": 1000 * statistics.median(lat),
            "acquisition_window_s": acq_s,
            "hidden": 1000 * statistics.median(lat) < 1000 * acq_s,
            "clocks": clocks, "gpu_launches": (5 + 2 * n_iter + (1 if args.u16 else 0)) * views}
    if rank == 0:
        print(json.dumps(line), flush=True)
    pl.destroy()
    if world > 1:
        dist.destroy_process_group()
    return 0


# ------------------------------------------------------------------------------- multi-rank helpers
def collective_all(dist, ok: bool, device) -> bool:
    """True on every rank iff `ok` holds on every rank (all-reduce MIN of a flag; gloo or NCCL)."""
    import torch
    t = torch.tensor([1 if ok else 0], dtype=torch.int32, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MIN)
    return bool(t.item())


def broadcast_flag(dist, ok: bool, device, src: int = 0) -> bool:
    import torch
    t = torch.tensor([1 if ok else 0], dtype=torch.int32, device=device)
    dist.broadcast(t, src=src)
    return bool(t.item())


def band_parity(img, ref_img, trace, ref_trace) -> dict:
    """Partitioned result vs the single-GPU run of the same projection (north_star: the 2/4/8-GPU
    result matches the unpartitioned one, no seam).  Pass: identical accept/reject sequence, f trace
    within 1e-6 relative, image within 1e-5 relative L2 (the single-device emulation's bars,
    tests/test_gpu_bands.py)."""
    img = np.asarray(img, np.float64)
    ref = np.asarray(ref_img, np.float64)
    e_img = float(np.linalg.norm(img - ref) / max(np.linalg.norm(ref), 1e-300))
    n = min(len(trace), len(ref_trace))
    f, fr = np.asarray(trace)[:n, 1], np.asarray(ref_trace)[:n, 1]
    e_f = float(np.max(np.abs(f - fr) / np.maximum(np.abs(fr), 1e-300))) if n else 0.0
    same_acc = len(trace) == len(ref_trace) and bool(np.array_equal(np.asarray(trace)[:, 5], np.asarray(ref_trace)[:, 5]))
    ok = same_acc and e_f <= 1e-6 and e_img <= 1e-5
    return {"ok": bool(ok), "image_rel_l2": e_img, "f_trace_max_rel": e_f, "same_accept_sequence": same_acc,
            "against": "single-GPU persistent loop on rank 0, same stack"}


def rank_record(rank, world, local, lo, hi, transport) -> dict:
    """One rank's identity for the JSON line and a stderr line (lets the rank count be verified)."""
    rec = {"rank": rank, "world": world, "local_rank": local, "rows": [lo, hi], "transport": transport,
           "host": os.uname().nodename, "pid": os.getpid()}
    try:
        import torch
        if torch.cuda.is_available():
            pr = torch.cuda.get_device_properties(local)
            rec["device"] = f"{pr.name} ({torch.cuda.get_device_properties(local).pci_bus_id})" \
                if hasattr(pr, "pci_bus_id") else pr.name
            rec["nccl"] = ".".join(map(str, torch.cuda.nccl.version()))
    except Exception as e:   # noqa: BLE001 -- identity only
        rec["device"] = f"unknown ({e})"
    print(f"[bench] rank {rank}/{world} local {local} rows [{lo},{hi}) transport {transport} "
          f"device {rec.get('device')} nccl {rec.get('nccl')}", file=sys.stderr, flush=True)
    return rec


def make_band_plan(flmisr, dist, kw: dict, rank: int, world: int, transport: str, device):
    """A row-band plan of one projection on every rank.  transport 'peer' / 'auto': try the
    peer-memory band loop (CUDA IPC); the decision is collective (a rank that cannot map its peers
    makes every rank use NCCL), and 'auto' falls back to the NCCL transport with the reason reported."""
    pl = flmisr.Plan(**kw, rank=rank, world=world, nccl_id=flmisr.broadcast_unique_id())
    if transport == "nccl":
        return pl, "nccl", None
    err = None
    try:
        flmisr.peer_connect(pl)
    except Exception as e:   # noqa: BLE001 -- any failure means: not this transport
        err = f"rank {rank}: {e}"
    if collective_all(dist, err is None, device):
        return pl, "peer", None
    errs = [None] * world
    dist.all_gather_object(errs, err)
    why = next(e for e in errs if e)
    if transport == "peer":
        raise RuntimeError(f"--transport peer unavailable: {why}")
    pl.destroy()   # a plan that did connect must not be mixed with NCCL ranks: rebuild on NCCL everywhere
    pl = flmisr.Plan(**kw, rank=rank, world=world, nccl_id=flmisr.broadcast_unique_id())
    return pl, "nccl", f"peer transport unavailable ({why}); NCCL halo send/recv + allgather used"


def time_steps(pl, y_d, out_d, flush, s, steps, dist, world, dev):
    """Timed reconstructions: L2 flushed before each, CUDA events around each on the launching stream,
    barrier + synchronize on both sides; returns (max-over-ranks total ms, accepted counts, last report)."""
    import torch
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    accepted, rep = [], None
    for i in range(steps):
        flush.zero_()
        ev[i][0].record(s)
        pl.reconstruct_async(y_d, out_d, stream=s)
        ev[i][1].record(s)
        rep = pl.finish()
        accepted.append(rep["accepted"])
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    tot_ms = sum(a.elapsed_time(b) for a, b in ev)
    if world > 1:
        t = torch.tensor([tot_ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        tot_ms = float(t.item())
    return tot_ms, accepted, rep


def run_flmisr(args):
    import torch
    import torch.distributed as dist

    from paper_2108_04315_b200 import flmisr

    world = env_int("WORLD_SIZE", 1)
    rank = env_int("RANK", 0)
    local = env_int("LOCAL_RANK", 0)
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    cfg = args.config
    y, sh, c = make_inputs(cfg)
    k, lr, mag, n_iter = len(sh), c["lr"], c["mag"], c["n_iter"]
    H = W = lr * mag
    npx = H * W
    dev = torch.device("cuda", local)
    mode = args.mode if args.mode != "auto" else ("partitioned" if world > 1 else "replicas")
    partitioned = world > 1 and mode == "partitioned"
    kw = dict(k=k, lr_h=lr, lr_w=lr, shifts=sh, psf=synth.gaussian_psf(), mag=mag, p_norm=1, l1_eps=1e-3,
              lam=0.05, btv_alpha=0.4, btv_window=3, n_iter=n_iter, device=local)
    transport, fallback = None, None
    if partitioned:   # row bands of ONE projection: halo exchange + consensus sums
        pl, transport, fallback = make_band_plan(flmisr, dist, kw, rank, world, args.transport, dev)
    else:             # one GPU, or replicas: every rank reconstructs its own projection
        pl = flmisr.Plan(**kw)
    y_d = torch.from_numpy(y).to(dev)
    out_d = torch.empty((H, W), dtype=torch.float32, device=dev)
    flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    s = torch.cuda.current_stream(dev)

    if partitioned and transport == "peer":
        # the first peer-loop call is the handshake: a rank whose peer memory does not work makes every
        # band abandon the loop after the barrier timeout (an error, not a hang); then all ranks move
        # to the NCCL transport together (auto) or fail loudly (--transport peer)
        err = None
        try:
            pl.reconstruct(y_d, out=out_d)
            torch.cuda.synchronize()
        except Exception as e:   # noqa: BLE001 -- any failure means: not this transport
            err = f"rank {rank}: {e}"
        if not collective_all(dist, err is None, dev):
            errs = [None] * world
            dist.all_gather_object(errs, err)
            why = next((e for e in errs if e), "a peer rank failed")
            if args.transport == "peer":
                raise RuntimeError(f"peer band loop failed: {why}")
            pl.destroy()
            pl, transport, _ = make_band_plan(flmisr, dist, kw, rank, world, "nccl", dev)
            fallback = f"peer band loop failed on its first call ({why}); NCCL used"
    for _ in range(args.warmup):
        pl.reconstruct(y_d, out=out_d)
    torch.cuda.synchronize()

    # partitioned: rank 0 checks the gathered image and the consensus trace against its own
    # single-GPU run of the same projection; a peer-transport result that disagrees falls back to NCCL
    parity = None
    ref_pl = None
    if partitioned:
        _, rep_p = pl.reconstruct(y_d, out=out_d)
        if rank == 0:
            ref_pl = flmisr.Plan(**kw)
            ref_out, rep_1 = ref_pl.reconstruct(y_d)
            parity = band_parity(out_d.cpu().numpy(), ref_out.cpu().numpy(), rep_p["trace"], rep_1["trace"])
            parity["transport"] = transport
        if not broadcast_flag(dist, parity["ok"] if rank == 0 else True, dev) and transport == "peer" \
                and args.transport == "auto":
            pl.destroy()
            pl, transport, _ = make_band_plan(flmisr, dist, kw, rank, world, "nccl", dev)
            fallback = "peer transport disagreed with the single-GPU run; NCCL used"
            for _ in range(args.warmup):
                pl.reconstruct(y_d, out=out_d)
            _, rep_p = pl.reconstruct(y_d, out=out_d)
            if rank == 0:
                parity = band_parity(out_d.cpu().numpy(), ref_out.cpu().numpy(), rep_p["trace"], rep_1["trace"])
                parity["transport"] = transport
    ranks = None
    if world > 1:
        rec = rank_record(rank, world, local, pl.row_lo if partitioned else 0, pl.row_hi if partitioned else H,
                          transport or "none (replica)")
        ranks = [None] * world
        dist.all_gather_object(ranks, rec)

    pl.profile(1)
    clk = ClockSampler(local)
    clk.start()
    time.sleep(0.2)
    tot_ms, accepted, rep = time_steps(pl, y_d, out_d, flush, s, args.steps, dist, world, dev)
    clocks = clk.stop()
    prof = pl.profile(0)
    ms_per_step = tot_ms / args.steps
    # replicas: every rank finished `steps` projections; partitioned: the ranks shared each projection
    value = (1 if partitioned else world) * args.steps / (tot_ms / 1000.0)

    # e2e through the public host API (flmisr_pipeline_*): every step uploads its
    # LR stack from pinned host memory, reconstructs, and downloads the HR image to pinned host memory;
    # consecutive views overlap (copy engines under the compute).  Views rotate through a ring of
    # distinct stacks.  The serial variant (flmisr_reconstruct_host, no overlap) is reported beside it.
    # rank 0 of a band group downloads the fused image; a replica downloads its own image
    root = rank == 0 or not partitioned
    ring = host_ring(y, 4)
    o_h = [torch.empty((H, W), dtype=torch.float32).pin_memory() for _ in range(3)]
    e2e_steps = max(10, min(2 * args.steps, 100))   # amortises the pipeline fill and drain (first upload, last download)

    def max_over_ranks(x):
        if world > 1:
            tt = torch.tensor([x], dtype=torch.float64, device=dev)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            return float(tt.item())
        return x

    e2e_s = max_over_ranks(run_pipeline(flmisr, pl, ring, o_h if root else None, e2e_steps, dist if world > 1 else None))
    # bytes per step summed over the ranks: every rank uploads the full frames (a band needs all
    # K frames of its rows); the fused image (partitioned) or each replica's image comes back
    e2e = {"value": (1 if partitioned else world) * e2e_steps / e2e_s, "unit": "proj/s",
           "h2d_bytes_per_step": int(y.nbytes) * world,
           "d2h_bytes_per_step": int(npx * 4) * (1 if partitioned else world),
           "api": "flmisr_pipeline_submit/wait (depth 3, fp32 frames, pinned host buffers)"}
    y_np, o_np = ring[0].numpy(), o_h[0].numpy()
    pl.reconstruct_host(y_np, o_np if root else None)
    ser_steps = 5
    if world > 1:
        dist.barrier()
    t = time.perf_counter()
    for _ in range(ser_steps):
        pl.reconstruct_host(y_np, o_np if root else None)
    e2e_serial = {"value": (1 if partitioned else world) * ser_steps / max_over_ranks(time.perf_counter() - t),
                  "unit": "proj/s", "api": "flmisr_reconstruct_host (H2D, reconstruct, D2H in sequence)"}

    peak, peak_src = load_peaks()
    vg = prof["value_grad"]
    uc = prof["update_curv"]
    traffic = None
    tp = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tp) and world == 1:
        with open(tp) as f:
            traffic = json.load(f).get(cfg, {})
    # pixels this rank's kernels stream (its band); the roofline is reported per rank against one GPU's peak
    npx_rank = (pl.row_hi - pl.row_lo) * W if partitioned else npx
    acc_flags = rep["trace"][:, 5]
    n_vg = len(acc_flags)                      # init + every pass
    n_uc = int(acc_flags[:-1].sum())           # pass k updates iff pass k-1 was accepted
    n_acc = int(acc_flags[1:].sum())
    n_rej = n_vg - 1 - n_acc
    if uc["launches"]:   # per-phase kernels: the dominant launch is value+gradient
        vg_ms = vg["ms"] / max(vg["launches"], 1)
        uc_ms = uc["ms"] / max(uc["launches"], 1)
        general = pl.fast_path in (0, 3)
        # the fused general kernels (fast_path 3) move what the streaming kernels move (rho' stays on chip)
        bvg = BYTES_GEN_VALUE_GRAD if pl.fast_path == 0 else BYTES_VALUE_GRAD
        buc = BYTES_GEN_UPDATE_CURV if pl.fast_path == 0 else BYTES_UPDATE_CURV
        roof = {"bound": "hbm", "achieved": bvg * npx_rank / (vg_ms / 1000.0) / 1e9, "peak": peak,
                "unit": "GB/s", "traffic": None if pl.fast_path == 0 else (traffic or {}).get("value_grad"),
                "kernel": ("k_gen3_vg" if pl.fast_path == 3 else "k_gen2_residual + k_gen2_grad") if general
                else "k_vg_stream",
                "algorithmic_bytes_per_launch": bvg * npx_rank, "avg_launch_ms": vg_ms,
                "peak_source": peak_src}
        kernels = {"value_grad": {"avg_ms": vg_ms, "launches": vg["launches"],
                                  "gbs": bvg * npx_rank / (vg_ms / 1000.0) / 1e9},
                   "update_curv": {"avg_ms": uc_ms, "launches": uc["launches"],
                                   "gbs": buc * npx_rank / (uc_ms / 1000.0) / 1e9}}
    else:                # one cooperative kernel runs the whole loop (one GPU, or a band of the peer loop)
        loop_bytes = (BYTES_VALUE_GRAD * n_vg + BYTES_UPDATE_CURV * n_uc) * npx_rank
        loop_ms = vg["ms"] / max(vg["launches"], 1)
        kname = "k_scg_peer_loop" if transport == "peer" else ("k_scg_loop4" if pl.fast_path == 4 else "k_scg_loop")
        # achieved = SURVEY 8(d)'s per-pass byte figures x the passes of this launch (init 20N + 8M,
        # accepted 44N + 12M, rejected 8N + 4M; M = N: one LR sample per HR pixel on the streaming
        # paths) -- the compulsory traffic of the survey's value / gradient / update step order.  The
        # fused kernels move less (value and gradient share one read of x, p, Y: 20 + 24 B/px), so the
        # survey figure can exceed the copy peak; the fused model beside it is the DRAM efficiency and
        # what ncu's `traffic` (dram bytes of the launch) compares with.
        surv = (28 * 1 + 56 * n_acc + 12 * n_rej) * npx_rank
        roof = {"bound": "hbm", "achieved": surv / (loop_ms / 1000.0) / 1e9, "peak": peak, "unit": "GB/s",
                "traffic": (traffic or {}).get("scg_loop"), "kernel": kname,
                "algorithmic_bytes_per_launch": surv, "avg_launch_ms": loop_ms, "peak_source": peak_src,
                "bytes_model": "SURVEY 8(d): init 28 + accepted 56 + rejected 12 B per HR pixel",
                "fused_model": {"bytes_per_launch": loop_bytes, "achieved": loop_bytes / (loop_ms / 1000.0) / 1e9,
                                "frac": loop_bytes / (loop_ms / 1000.0) / 1e9 / peak,
                                "bytes_model": "value+gradient 20 + update+curvature 24 B per HR pixel (DESIGN.md 7.1)"}}
        kernels = {"scg_loop": {"kernel": kname, "avg_ms": loop_ms, "launches": vg["launches"],
                                "value_grad_phases": n_vg, "update_curv_phases": n_uc,
                                "avg_phase_us": 1000 * loop_ms / (n_vg + n_uc),
                                "gbs": loop_bytes / (loop_ms / 1000.0) / 1e9}}
        if world == 1:   # context: the same phases as separate kernels (FLMISR_NO_PERSIST=1), not timed
            os.environ["FLMISR_NO_PERSIST"] = "1"
            try:
                pk = flmisr.Plan(**kw)
            finally:
                del os.environ["FLMISR_NO_PERSIST"]
            for _ in range(2):
                pk.reconstruct(y_d, out=out_d)
            pk.profile(1)
            for _ in range(3):
                flush.zero_()
                pk.reconstruct(y_d, out=out_d)
            pp = pk.profile(0)
            pk.destroy()
            pv = pp["value_grad"]["ms"] / max(pp["value_grad"]["launches"], 1)
            pu = pp["update_curv"]["ms"] / max(pp["update_curv"]["launches"], 1)
            kernels["per_phase_kernels"] = {
                "value_grad": {"avg_ms": pv, "gbs": BYTES_VALUE_GRAD * npx / (pv / 1000.0) / 1e9},
                "update_curv": {"avg_ms": pu, "gbs": BYTES_UPDATE_CURV * npx / (pu / 1000.0) / 1e9},
                "note": "FLMISR_NO_PERSIST=1 (per-phase kernels, deferred reduction), 3 reconstructions, not timed"}
    roof["frac"] = roof["achieved"] / peak
    if partitioned:
        roof["scope"] = f"rank {rank}'s band ({npx_rank} px) against one GPU's peak"
    kernels["setup_finalize_ms_per_step"] = prof["setup_finalize"]["ms"] / max(prof["setup_finalize"]["launches"], 1)
    launches_per_step = 5 + 2 * n_iter if uc["launches"] else 6

    # the paper's non-iterative baseline, multi-image interpolation fusion (tab:runtime row P:432:
    # 0.26 s at 2048^2 on its CPU), through the product entry flmisr_interp_fuse, device-resident
    interpolation = None
    if world == 1:
        ie = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(20)]
        pl.interp_fuse(y_d, out_d, stream=s)
        for a, b in ie:
            flush.zero_()
            a.record(s)
            pl.interp_fuse(y_d, out_d, stream=s)
            b.record(s)
        torch.cuda.synchronize()
        i_ms = statistics.median(a.elapsed_time(b) for a, b in ie)
        interpolation = {"ms": i_ms, "value": 1000.0 / i_ms, "unit": "proj/s",
                         "api": "flmisr_interp_fuse (device buffers, L2 flushed)",
                         "paper_s": {"C2": 0.07, "C3": 0.26, "C6": 2.07}.get(cfg),
                         "paper_note": "tab:runtime P:432, multi-image interpolation on the paper's CPU (context)"}

    # partitioned runs also report replicas (one projection per GPU, no communication)
    replicas = None
    if partitioned:
        rp = ref_pl if ref_pl is not None else flmisr.Plan(**kw)
        for _ in range(2):
            rp.reconstruct(y_d, out=out_d)
        rsteps = max(5, min(args.steps, 20))
        r_ms, _, _ = time_steps(rp, y_d, out_d, flush, s, rsteps, dist, world, dev)
        replicas = {"value": world * rsteps / (r_ms / 1000.0), "unit": "proj/s", "scaling": "weak",
                    "steps": rsteps, "ms_per_step": r_ms / rsteps,
                    "note": "every GPU reconstructs its own projection (no communication)"}
        rp.destroy()
    line = {
        "metric": METRIC, "value": value, "unit": "proj/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
        "scaling": "strong" if partitioned else "weak",
        "vs_baseline": (value * PAPER_1GPU_S[cfg] if world == 1 and cfg in PAPER_1GPU_S else None),
        "vs_baseline_note": (f"value / (1 / {PAPER_1GPU_S[cfg]} s): the paper's own runtime for this workload on "
                             "1x GTX 1080 (BASELINE.md tab:runtime) -- context, not a target"
                             if world == 1 and cfg in PAPER_1GPU_S else None),
        "dtype": "f32", "data": "synthetic",
        "config": {"workload": WORKLOADS[cfg], "n_iter": n_iter, "hr": [H, W], "p_norm": 1, "lambda": 0.05,
                   "btv_alpha": 0.4, "btv_window": 3, "psf": "3x3 Gaussian sigma 0.5",
                   "l2": "flushed before every timed step (512 MiB device write)",
                   "parallelism": "single GPU" if world == 1 else
                   ((f"row bands x{world} (peer-memory band loop)" if transport == "peer" else
                     f"row bands x{world} (NCCL halo + allgather)") if partitioned else f"replicas x{world}")},
        "scg_iters_per_s": value * n_iter,
        "accepted_fraction": float(np.mean(accepted)) / n_iter if n_iter else None,
        "roofline": roof,
        "kernels": kernels,
        "clocks": clocks,
        "e2e": e2e,
        "e2e_serial": e2e_serial,
        "gpu_launches": launches_per_step * args.steps,
    }
    if interpolation is not None:
        line["interpolation"] = interpolation
    if world > 1:
        line["ranks"] = ranks
    if partitioned:
        line["transport"] = transport
        line["transport_fallback"] = fallback
        line["parity"] = parity
        line["replicas"] = replicas
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        from oracle import oracle as orc
        orc.build()
        line["cpu_baseline"] = cpu_baseline(cfg, n_iter)
    if rank == 0:
        print(json.dumps(line), flush=True)
    pl.destroy()
    if world > 1:
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="flmisr", choices=["flmisr", "reference"])
    ap.add_argument("--config", default="C3", choices=["C2", "C3", "C4", "C6", "G3"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--mode", default="auto", choices=["auto", "replicas", "partitioned", "stream"],
                    help="auto (default): one GPU, or N > 1 row bands of ONE projection (north_star's strong "
                         "scaling; replicas reported beside it); replicas: independent projections per rank; "
                         "stream: C5 capture-reconstruct pipeline (host frames in, host images out)")
    ap.add_argument("--transport", default="auto", choices=["auto", "nccl", "peer"],
                    help="partitioned mode: auto (default) = the peer-memory band loop (CUDA IPC over NVLink), "
                         "falling back to NCCL if any rank cannot map its peers or the result disagrees with "
                         "the single-GPU run; nccl = halo send/recv + allgather per phase; peer = no fallback")
    ap.add_argument("--partition", action="store_true", help="stream mode, N > 1: row bands instead of replicas")
    ap.add_argument("--u16", action="store_true", help="stream mode: 16-bit detector codes as input")
    ap.add_argument("--depth", type=int, default=3, help="stream mode: views in flight")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3) if args.impl == "flmisr" else args.warmup
    if args.impl == "reference":
        return run_reference(args)
    if args.mode == "stream":
        return run_stream(args)
    return run_flmisr(args)


if __name__ == "__main__":
    sys.exit(main())
