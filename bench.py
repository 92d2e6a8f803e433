"""Benchmark of the NGF + curvature objective/gradient hot path (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--workload c3]

One step = one objective+gradient evaluation (LevelObjective.__call__) of the
config-3 finest level: synthetic 256^3 CT-shaped pair, 64^3 deformation grid,
NGF tau = rho = 10, alpha = 1, fp32.  `value` is whole-job evaluations/s with
the inputs resident in HBM; `e2e` is the same metric through the numpy-facing
LevelObjective call (H2D of y, D2H of J and the gradient inside the timed
region).  The line also carries the full 4-level 256^3 registration time (the
paper's headline), the fused kernel's roofline against MEASURED_PEAKS.json, the
CPU baseline (the oracle port on this host) and the SM clocks seen.

For N > 1 (torchrun), every rank registers its own pair (config 4: independent
pairs, one per GPU, no data-path collective); timings are max over ranks.
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

METRIC = "256^3 full-registration time (s); obj+grad evals/s; HBM GB/s vs peak"

WORKLOADS = {
    # name: (image n, grid ratio, levels for the full registration)
    "c1": (64, 4, 1),
    "c2": (128, 2, 3),  # ratio 2: 64^3 deformation grid on the finest level (DIR-lab-like)
    "c3": (256, 4, 4),
    "c5": (512, 4, 4),  # z-slab decomposition over the ranks (strong scaling), evaluation only
}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="c3", choices=sorted(WORKLOADS))
    ap.add_argument("--precision", default="f32", choices=["f32", "f64"],
                    help="working dtype (the reference's default precision is f64, multilevel.py:55)")
    ap.add_argument("--no-register", action="store_true", help="skip the full-registration leg")
    ap.add_argument("--cpu-budget", type=float, default=25.0, help="seconds of CPU baseline work")
    ap.add_argument("--streams", type=int, default=8,
                    help="config 4: registrations in flight per GPU (host threads, one CUDA stream each)")
    ap.add_argument("--pairs-pageable", action="store_true",
                    help="config 4: keep the batch's volumes in pageable host memory (default: "
                         "page-locked, as the CLI reads them)")
    ap.add_argument("--pairs", type=int, default=0,
                    help="config 4: also register this many independent pairs, split over the ranks "
                         "(distributed.weak_scaling_pairs), and report pairs/s")
    return ap.parse_args()


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


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
    R, T, _ = ngf.ct_pair(n, seed=seed, dtype=dtype)
    gd = ngf.deformation_grid_for(R.grid, ratio)
    y = ngf.smooth_random_field(gd, seed=2, amplitude_mm=2.0).field.astype(dtype)
    return R, T, gd, y


def cpu_baseline(R, T, gd, y, budget_s: float):
    """The oracle port (numpy restatement of the reference, oracle/) on this host's cores."""
    from oracle import ngf_oracle as O
    cores = os.cpu_count() or 1
    og = O.grid(R.grid.dims, R.grid.spacing, R.grid.origin)
    ogd = O.grid(gd.dims, gd.spacing, gd.origin)
    obj = O.Objective(T.values, R.values, ogd, og, workers=cores)
    t0 = time.perf_counter()
    obj(y.ravel())  # warm (thread pools, page faults)
    first = time.perf_counter() - t0
    reps = max(1, min(5, int(budget_s / max(first, 1e-3)) - 1))
    t0 = time.perf_counter()
    for _ in range(reps):
        obj(y.ravel())
    dt = (time.perf_counter() - t0) / reps
    return {"value": 1.0 / dt, "unit": "evals/s", "cores": cores, "kind": "port",
            "sample": f"{reps} full evaluations of the same {R.grid.dims[0]}^3/{gd.dims[0]}^3 workload "
                      f"(oracle/ngf_oracle.py, workers={cores}, {np.dtype(y.dtype).name}) after 1 warm-up; "
                      f"{dt:.2f} s/eval"}


def run_reference(args):
    ws, rank, _ = dist_env()
    if rank != 0:
        return
    n, ratio, _ = WORKLOADS[args.workload]
    R, T, gd, y = make_inputs(n, ratio, 0, np.float32 if args.precision == "f32" else np.float64)
    from oracle import ngf_oracle as O
    cores = os.cpu_count() or 1
    og = O.grid(R.grid.dims, R.grid.spacing, R.grid.origin)
    ogd = O.grid(gd.dims, gd.spacing, gd.origin)
    obj = O.Objective(T.values, R.values, ogd, og, workers=cores)
    t0 = time.perf_counter()
    obj(y.ravel())
    one = time.perf_counter() - t0
    budget = 150.0
    warm = max(0, min(args.warmup - 1, int(budget / 3 / max(one, 1e-3))))
    steps = max(1, min(args.steps, int(budget / max(one, 1e-3)) - warm))
    for _ in range(warm):
        obj(y.ravel())
    t0 = time.perf_counter()
    for _ in range(steps):
        obj(y.ravel())
    dt = time.perf_counter() - t0
    value = steps / dt
    line = {"metric": METRIC, "value": value, "unit": "evals/s", "n_gpus": args.gpus,
            "steps": steps, "warmup": warm + 1, "ms_per_step": 1000 * dt / steps,
            "higher_is_better": True, "scaling": "strong" if args.workload == "c5" else "weak",
            "vs_baseline": None, "dtype": args.precision, "data": "synthetic", "impl": "reference",
            "config": {"workload": f"{args.workload}: {n}^3 CT-shaped pair, {gd.dims[0]}^3 def grid, "
                                   "one LevelObjective evaluation per step"},
            "cpu_baseline": {"value": value, "unit": "evals/s", "cores": cores, "kind": "port",
                             "sample": f"{steps} timed of {args.steps} requested full evaluations "
                                       f"(bounded to ~{budget:.0f} s of CPU work), workers={cores}"},
            "e2e": {"value": value, "unit": "evals/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def run_ours(args):
    import torch
    import torch.distributed as dist

    import paper_1812_06765_b200 as ngf
    from paper_1812_06765_b200 import _lib
    import ctypes

    ws, rank, local = dist_env()
    if ws > 1:
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        torch.cuda.set_device(0)
    dev_index = torch.cuda.current_device()

    n, ratio, levels = WORKLOADS[args.workload]
    strong = args.workload == "c5"  # one pair split in z-slabs over all ranks
    npdt = np.float32 if args.precision == "f32" else np.float64
    es = np.dtype(npdt).itemsize
    R, T, gd, y = make_inputs(n, ratio, seed=0 if strong else rank, dtype=npdt)
    gi = R.grid
    plan = ngf.build_gather_plan(gd, gi)
    T_dev = torch.from_numpy(T.values).cuda()
    R_dev = torch.from_numpy(R.values).cuda()
    obj = ngf.LevelObjective.from_device(T_dev, R_dev, plan, ngf.NgfParams(10.0, 10.0), 1.0)
    level = obj.level
    zlo, zhi = 0, gi.dims[2]
    evaluator = obj
    if strong:
        from paper_1812_06765_b200.distributed import DeviceSlab, SlabObjective, slab_ranges
        zlo, zhi = slab_ranges(gi.dims[2], gd.dims[2], ws)[rank]
        evaluator = SlabObjective(DeviceSlab(level, zlo, zhi))
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
    N, M = gi.dims[0] * gi.dims[1] * (zhi - zlo), gd.num_points  # this rank's slab
    bytes_kernel = es * (5 * N + 3 * M)     # T + packed reference terms + y
    bytes_eval = es * (5 * N + 6 * M)       # + grad J written (B_eval: 20N + 24M in f32)
    peak, peak_kind = peaks()
    achieved = bytes_kernel / (k_ms / 1000.0) / 1e9
    eval_ms = t_ms / args.steps

    # ---------------- end to end through the numpy-facing LevelObjective -------------------
    # the step's input in page-locked host memory (the contract's e2e: H2D from pinned
    # memory, D2H of the result); LevelObjective's numpy call then DMAs it directly
    from paper_1812_06765_b200 import _device as ngf_dev
    y_host = ngf_dev.pinned_empty((y.size,), y.dtype)
    y_host[...] = y.ravel()
    if strong:
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
        # hold each result across the next call, like the timed loop (the page-locked
        # gradient buffers of torch's host cache reach their steady-state count here)
        J, gh = call(y_host)
    barrier()
    t0 = time.perf_counter()
    ee0 = torch.cuda.Event(enable_timing=True)
    ee1 = torch.cuda.Event(enable_timing=True)
    ee0.record(stream)
    per_call = []
    for _ in range(args.steps):
        tc = time.perf_counter()
        J, gh = call(y_host)
        per_call.append(time.perf_counter() - tc)
    ee1.record(stream)
    if os.environ.get("NGF_BENCH_DEBUG"):
        print("e2e per call (us):", [round(v * 1e6) for v in per_call], file=sys.stderr)
    barrier()
    e2e_s = max_over_ranks(max(time.perf_counter() - t0, ee0.elapsed_time(ee1) / 1000.0))
    e2e = {"value": jobs * args.steps / e2e_s, "unit": "evals/s",
           "h2d_bytes_per_step": int(y_host.nbytes), "d2h_bytes_per_step": int(gh.nbytes + 24),
           "input": "page-locked host y (LevelObjective numpy call)"}
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
               "pairs_per_s": ws / reg_s}
        # the same with the volumes in page-locked host memory, as the CLI reads them
        # (fileio.read_volume into dev.pinned_empty): the uploads become direct DMAs
        from paper_1812_06765_b200 import _device as ngf_dev
        pin = []
        for im in (R, T):
            a = ngf_dev.pinned_empty(im.values.shape, im.values.dtype)
            a[...] = im.values
            pin.append(ngf.Image3(im.grid, a))
        ngf.register(pin[0], pin[1], cfg)
        barrier()
        t0 = time.perf_counter()
        ngf.register(pin[0], pin[1], cfg)
        barrier()
        reg["seconds_pinned_inputs"] = max_over_ranks(time.perf_counter() - t0)
        if args.pairs > 0:
            # config 4: a batch of independent pairs (seeds = pair ids), one process per GPU,
            # no collective; inputs generated on the host before the clock starts
            from paper_1812_06765_b200.distributed import weak_scaling_pairs
            mine = weak_scaling_pairs(args.pairs, ws, rank)
            batch = [make_inputs(n, ratio, seed=1000 + p, dtype=npdt)[:2] for p in mine]
            if not args.pairs_pageable:
                # volumes in page-locked host memory, as the CLI reads them: direct DMAs that
                # concurrent registrations do not serialise on the library's staging buffer
                batch = [tuple(ngf.Image3(im.grid, _pinned_copy(ngf_dev, im.values)) for im in pr)
                         for pr in batch]
            k = max(1, min(args.streams, len(batch)))
            streams = [torch.cuda.Stream() for _ in range(k)]
            errors = []

            per_reg = [[] for _ in range(k)]

            def work(i):
                # registrations in flight on their own stream: the coarse levels leave most
                # of the GPU idle, so concurrent pairs fill it
                try:
                    with torch.cuda.stream(streams[i]):
                        for Rp, Tp in batch[i::k]:
                            tr = time.perf_counter()
                            ngf.register(Rp, Tp, cfg)
                            per_reg[i].append(round(time.perf_counter() - tr, 4))
                        streams[i].synchronize()
                except Exception as e:  # surfaced after the join
                    errors.append(e)

            if k > 1:  # warm-up on every stream (reduction scratch, torch's per-stream block cache)
                for st in streams:
                    with torch.cuda.stream(st):
                        ngf.register(batch[0][0], batch[0][1], cfg)
                    st.synchronize()
            barrier()
            t0 = time.perf_counter()
            if k > 1:
                work_threads = [threading.Thread(target=work, args=(i,)) for i in range(k)]
                for th in work_threads:
                    th.start()
                for th in work_threads:
                    th.join()
                if errors:
                    raise errors[0]
            else:
                for Rp, Tp in batch:
                    ngf.register(Rp, Tp, cfg)
            barrier()
            batch_s = max_over_ranks(time.perf_counter() - t0)
            reg["batch"] = {"pairs": args.pairs, "per_rank": len(mine), "streams": k,
                            "inputs": "pageable host" if args.pairs_pageable else "page-locked host",
                            "seconds": batch_s,
                            "pairs_per_s": args.pairs / batch_s}
            if os.environ.get("NGF_BENCH_DEBUG"):
                print("per registration (s), per stream:", per_reg, file=sys.stderr)

    cpu = None
    if rank == 0 and ws == 1:
        cpu = cpu_baseline(R, T, gd, y, args.cpu_budget)

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
                       "parallelism": (f"z-slabs x{ws} (one pair; NCCL all-reduce of grad D and D)"
                                       if strong else f"replicas x{ws} (one independent pair per GPU)")},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak,
                         "traffic": ncu_traffic(args.workload + ("" if args.precision == "f32" else "_f64")),
                         "kernel": "k_eval_fused", "kernel_ms": k_ms,
                         "bytes_per_launch": bytes_kernel, "peak_kind": peak_kind,
                         "eval_frac": bytes_eval / (eval_ms / 1000.0) / 1e9 / peak,
                         "launch": {"ctas": info[0], "smem_bytes": info[1], "z_chunk": info[2]}},
            "e2e": e2e,
            "gpu_launches": launches,
            "clocks": clk.summary(),
            "full_registration": reg,
            "cpu_baseline": cpu,
        }
        print(json.dumps(line), flush=True)
    if ws > 1:
        dist.destroy_process_group()


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
