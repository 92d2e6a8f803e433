"""Limited-memory BFGS with Armijo backtracking (drop-in for ngfreg.lbfgs).

The control flow is the reference's, decision for decision (lbfgs.py:94-181):
two-loop direction, steepest-descent safeguard, Armijo backtracking with
forward expansion at t == 1, curvature-filtered history with ageing, and the
three relative stopping tests after `min_iterations`.  The vectors live on the
device; the two-loop recursion is one cooperative sm_100a kernel, the history
pair (s, y) and its dot products one fused pass, and the only host round trips
are the scalars the driver branches on (J, slope, s.y, norms, max |g|).
"""

from __future__ import annotations

import ctypes
import math
import os
from dataclasses import dataclass, field

import numpy as np

from . import _device as dev
from ._lib import check, dtype_code, lib

__all__ = ["LbfgsConfig", "StoppingRules", "IterationRecord", "OptimizeTrace",
           "two_loop_direction", "lbfgs_minimize"]


@dataclass(frozen=True)
class LbfgsConfig:
    memory: int = 5
    max_iterations: int = 100
    c1: float = 1e-4
    initial_step: float = 1.0
    step_shrink: float = 0.5
    max_ls_steps: int = 20

    def __post_init__(self):
        if self.memory < 1:
            raise ValueError("memory must be >= 1")
        if not 0 < self.c1 < 1:
            raise ValueError("c1 must be in (0, 1)")
        if not 0 < self.step_shrink < 1:
            raise ValueError("step_shrink must be in (0, 1)")


@dataclass(frozen=True)
class StoppingRules:
    tol_J: float = 1e-4
    tol_grad: float = 1e-3
    tol_step: float = 1e-5
    min_iterations: int = 3

    def __post_init__(self):
        if min(self.tol_J, self.tol_grad, self.tol_step) <= 0:
            raise ValueError("all tolerances must be > 0")


@dataclass
class IterationRecord:
    iteration: int
    J: float
    grad_inf: float
    step: float
    ls_evals: int


@dataclass
class OptimizeTrace:
    records: list = field(default_factory=list)
    stop_reason: str = ""
    line_search_failed: bool = False
    evaluations: int = 0

    @property
    def iterations(self) -> int:
        return len(self.records)


class _Pair:
    __slots__ = ("s", "y", "sy", "yy")

    def __init__(self, s, y, sy, yy):
        self.s, self.y, self.sy, self.yy = s, y, sy, yy


def _two_loop(pairs, g, d, slope_dev):
    m = len(pairs)
    S = (ctypes.c_void_p * max(m, 1))(*[dev.ptr(p.s) for p in pairs])
    Y = (ctypes.c_void_p * max(m, 1))(*[dev.ptr(p.y) for p in pairs])
    rho = (ctypes.c_double * max(m, 1))(*[1.0 / p.sy for p in pairs])
    gamma = pairs[-1].sy / pairs[-1].yy if m else 1.0
    check(lib().ngf_lbfgs_two_loop(dtype_code(g.dtype), S, Y, rho, gamma, m, dev.ptr(g), dev.ptr(d),
                                   g.numel(), dev.ptr(slope_dev), dev.stream()),
          "ngf_lbfgs_two_loop")


def two_loop_direction(history, g):
    """-H g from (s, y) pairs, oldest first (lbfgs.py:68-91).  numpy in -> numpy out."""
    np_out = not dev.is_tensor(g)
    gd = dev.to_device(g).reshape(-1)
    pairs = []
    stats = dev.zeros((5,), "float64")
    for s, y in history:
        sd = dev.to_device(s, dev.np_dtype(gd.dtype)).reshape(-1)
        yd = dev.to_device(y, dev.np_dtype(gd.dtype)).reshape(-1)
        check(lib().ngf_vec_stats(dtype_code(gd.dtype), 0, 0, dev.ptr(sd), dev.ptr(yd), sd.numel(),
                                  dev.ptr(stats), dev.stream()), "ngf_vec_stats")
        st = stats.cpu().numpy()
        pairs.append(_Pair(sd, yd, float(st[1]), float(st[3])))
    d = dev.empty(gd.shape, gd.dtype)
    slope = dev.zeros((1,), "float64")
    _two_loop(pairs, gd, d, slope)
    d = d.reshape(g.shape)
    return dev.to_host(d) if np_out else d


class _HostFunction:
    """Adapter for an arbitrary numpy callable f(x) -> (J, g): vectors stay on the
    device, f sees host copies."""

    def __init__(self, f, shape, dtype):
        self.f, self.shape, self.dtype = f, shape, dtype

    def eval_device(self, x_dev, g_dev, scal_dev):
        J, g = self.f(dev.to_host(x_dev).reshape(self.shape))
        g_dev.copy_(dev.to_device(np.asarray(g, dtype=self.dtype).reshape(-1)))
        scal_dev[0] = float(J)
        scal_dev[1] = float("nan")
        scal_dev[2] = float("nan")
        return scal_dev


class _Solver:
    def __init__(self, f, x0, cfg: LbfgsConfig, stop: StoppingRules):
        self.cfg, self.stop = cfg, stop
        self.np_in = not dev.is_tensor(x0)
        self.shape = tuple(x0.shape)
        if hasattr(f, "eval_device"):
            self.f = f
        else:
            self.f = _HostFunction(f, self.shape, np.asarray(x0).dtype if self.np_in else
                                   dev.np_dtype(x0.dtype))
        x = dev.to_device(x0).reshape(-1).clone()
        self.dt = x.dtype
        self.code = dtype_code(self.dt)
        self.n = x.numel()
        self.bufs = {k: dev.empty((self.n,), self.dt) for k in ("g", "d", "xn", "gn", "xt", "gt")}
        self.x = x
        self.scal = dev.zeros((4,), "float64")   # J, D, S, slope
        self.stats = dev.zeros((5,), "float64")
        self.free_pairs = []
        self.evals = 0
        self.trace_rows = []  # (J, D, S) per evaluation

    # -------------------------------------------------------------- device helpers
    def feval(self, x, g):
        self.evals += 1
        self.f.eval_device(x, g, self.scal[:3])

    def read_scal(self):
        v = self.scal.cpu().numpy()
        return [float(a) for a in v]

    def axpy(self, x, t, d, out):
        check(lib().ngf_vec_axpy_step(self.code, dev.ptr(x), float(t), dev.ptr(d), dev.ptr(out),
                                      self.n, dev.stream()), "ngf_vec_axpy_step")

    def gstats(self, g, s=None):
        check(lib().ngf_vec_stats(self.code, dev.ptr(g), 0, dev.ptr(s), 0, self.n,
                                  dev.ptr(self.stats), dev.stream()), "ngf_vec_stats")
        return [float(a) for a in self.stats.cpu().numpy()]

    def new_pair(self):
        if self.free_pairs:
            return self.free_pairs.pop()
        return _Pair(dev.empty((self.n,), self.dt), dev.empty((self.n,), self.dt), 0.0, 0.0)

    # -------------------------------------------------------------- the reference loop
    def run(self):
        cfg, stop = self.cfg, self.stop
        x, g, d = self.x, self.bufs["g"], self.bufs["d"]
        xn, gn, xt, gt = self.bufs["xn"], self.bufs["gn"], self.bufs["xt"], self.bufs["gt"]
        trace = OptimizeTrace()
        self.feval(x, g)
        J, D0, S0 = self.read_scal()[:3]
        self.trace_rows.append((J, D0, S0))
        st = self.gstats(g, x)
        g0_inf = st[4] if self.n else 0.0
        if g0_inf <= 0.0:
            trace.stop_reason = "stationary start"
            return x, trace
        history = []
        x_scale = max(math.sqrt(st[2]), 1.0)
        rejected = 0
        for it in range(cfg.max_iterations):
            if cfg.max_ls_steps < 1:
                # no trial point may be evaluated: the reference's backtracking loop runs
                # zero times and the line search fails (lbfgs.py:121-132)
                trace.stop_reason = "line search failed"
                trace.line_search_failed = True
                trace.evaluations = self.evals
                return x, trace
            # direction and (optimistically) the first trial point, one host sync
            _two_loop(history, g, d, self.scal[3:4])
            t = cfg.initial_step
            self.axpy(x, t, d, xn)
            self.feval(xn, gn)
            Jn, Dn, Sn, slope = self.read_scal()
            ls_evals = 1
            if slope >= 0:  # safeguard: steepest descent (lbfgs.py:113-116)
                self.evals -= 1  # the optimistic trial above is discarded
                self.free_pairs.extend(history)
                history = []
                _two_loop(history, g, d, self.scal[3:4])
                self.axpy(x, t, d, xn)
                self.feval(xn, gn)
                Jn, Dn, Sn, slope = self.read_scal()
            self.trace_rows.append((Jn, Dn, Sn))
            accepted = False
            while True:
                if math.isfinite(Jn) and Jn <= J + cfg.c1 * t * slope:
                    accepted = True
                    break
                if ls_evals >= cfg.max_ls_steps:
                    break
                t *= cfg.step_shrink
                self.axpy(x, t, d, xn)
                self.feval(xn, gn)
                Jn, Dn, Sn = self.read_scal()[:3]
                self.trace_rows.append((Jn, Dn, Sn))
                ls_evals += 1
            if not accepted:
                trace.stop_reason = "line search failed"
                trace.line_search_failed = True
                trace.evaluations = self.evals
                return x, trace
            if t == cfg.initial_step:
                # forward expansion while Armijo holds and J decreases (lbfgs.py:133-143)
                while ls_evals < cfg.max_ls_steps:
                    t_try = t / cfg.step_shrink
                    self.axpy(x, t_try, d, xt)
                    self.feval(xt, gt)
                    Jt, Dt, St = self.read_scal()[:3]
                    self.trace_rows.append((Jt, Dt, St))
                    ls_evals += 1
                    if math.isfinite(Jt) and Jt <= J + cfg.c1 * t_try * slope and Jt < Jn:
                        t, Jn = t_try, Jt
                        xn, xt = xt, xn
                        gn, gt = gt, gn
                    else:
                        break
            # history pair and stopping statistics in one pass (lbfgs.py:145-164)
            pair = self.new_pair()
            check(lib().ngf_lbfgs_pair(self.code, dev.ptr(xn), dev.ptr(x), dev.ptr(gn), dev.ptr(g),
                                       dev.ptr(pair.s), dev.ptr(pair.y), self.n, dev.ptr(self.stats),
                                       dev.stream()), "ngf_lbfgs_pair")
            sy, ss, yy, g_inf = [float(a) for a in self.stats.cpu().numpy()[:4]]
            pair.sy, pair.yy = sy, yy
            if sy > 1e-10 * math.sqrt(ss) * math.sqrt(yy):
                history.append(pair)
                if len(history) > cfg.memory:
                    self.free_pairs.append(history.pop(0))
                rejected = 0
            else:
                self.free_pairs.append(pair)
                rejected += 1
                if history:
                    self.free_pairs.append(history.pop(0))
                if rejected >= cfg.memory:
                    self.free_pairs.extend(history)
                    history = []
            step_norm = math.sqrt(ss)
            J_prev = J
            x, xn = xn, x
            g, gn = gn, g
            J = float(Jn)
            trace.records.append(IterationRecord(it, J, g_inf, t, ls_evals))
            if it + 1 >= stop.min_iterations:
                if abs(J_prev - J) <= stop.tol_J * max(abs(J_prev), 1e-30):
                    trace.stop_reason = "objective change below tolerance"
                    break
                if g_inf <= stop.tol_grad * g0_inf:
                    trace.stop_reason = "gradient below tolerance"
                    break
                if step_norm <= stop.tol_step * x_scale:
                    trace.stop_reason = "step below tolerance"
                    break
        if not trace.stop_reason:
            trace.stop_reason = "max iterations"
        trace.evaluations = self.evals
        return x, trace


class _NativeCfg(ctypes.Structure):
    _fields_ = [("memory", ctypes.c_int), ("max_iterations", ctypes.c_int), ("max_ls_steps", ctypes.c_int),
                ("min_iterations", ctypes.c_int), ("c1", ctypes.c_double), ("initial_step", ctypes.c_double),
                ("step_shrink", ctypes.c_double), ("tol_J", ctypes.c_double), ("tol_grad", ctypes.c_double),
                ("tol_step", ctypes.c_double)]


class _NativeRes(ctypes.Structure):
    _fields_ = [("iterations", ctypes.c_int), ("evaluations", ctypes.c_int), ("stop", ctypes.c_int),
                ("line_search_failed", ctypes.c_int), ("rows", ctypes.c_int)]


_STOP_REASONS = ("objective change below tolerance", "gradient below tolerance", "step below tolerance",
                 "max iterations", "line search failed", "stationary start")


def _native_minimize(f, x0, cfg: LbfgsConfig, stop: StoppingRules):
    """The driver loop in native code (ngf_lbfgs_run_level) for a level objective: the
    same decisions as _Solver.run, without a Python round trip per vector operation."""
    np_in = not dev.is_tensor(x0)
    shape = tuple(x0.shape)
    x = dev.to_device(x0).reshape(-1).clone()
    n = x.numel()
    c = _NativeCfg(cfg.memory, cfg.max_iterations, cfg.max_ls_steps, stop.min_iterations, cfg.c1,
                   cfg.initial_step, cfg.step_shrink, stop.tol_J, stop.tol_grad, stop.tol_step)
    res = _NativeRes()
    rec = (ctypes.c_double * (4 * max(cfg.max_iterations, 1)))()
    max_rows = 2 + cfg.max_iterations * (cfg.max_ls_steps + 1)
    rows = (ctypes.c_double * (3 * max_rows))()
    check(lib().ngf_lbfgs_run_level(f.level.handle, dtype_code(x.dtype), 1 if f.exact else 0, dev.ptr(x), n,
                                    ctypes.byref(c), ctypes.byref(res), rec, rows, max_rows, dev.stream()),
          "ngf_lbfgs_run_level")
    trace = OptimizeTrace()
    trace.records = [IterationRecord(it, rec[4 * it], rec[4 * it + 1], rec[4 * it + 2], int(rec[4 * it + 3]))
                     for it in range(res.iterations)]
    trace.stop_reason = _STOP_REASONS[res.stop]
    trace.line_search_failed = bool(res.line_search_failed)
    trace.evaluations = res.evaluations
    trace.J_rows = [(rows[3 * k], rows[3 * k + 1], rows[3 * k + 2]) for k in range(min(res.rows, max_rows))]
    f.evals += res.evaluations
    x = x.reshape(shape)
    return (dev.to_host(x) if np_in else x), trace


def lbfgs_minimize(f, x0, cfg: LbfgsConfig = LbfgsConfig(), stop: StoppingRules = StoppingRules()):
    """Minimize f(x) -> (J, grad); returns (best x, OptimizeTrace) (lbfgs.py:94-181).

    `f` may be a LevelObjective (device-resident evaluation; its driver loop runs in
    native code, NGF_PY_LBFGS=1 selects the Python loop) or any numpy callable.
    numpy x0 -> numpy x; a CUDA tensor x0 -> CUDA tensor x.
    """
    if hasattr(f, "level") and hasattr(f, "exact") and not os.environ.get("NGF_PY_LBFGS"):
        return _native_minimize(f, x0, cfg, stop)
    solver = _Solver(f, x0, cfg, stop)
    x, trace = solver.run()
    trace.J_rows = solver.trace_rows
    x = x.reshape(solver.shape)
    return (dev.to_host(x) if solver.np_in else x), trace
