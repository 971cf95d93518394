#!/usr/bin/env python
"""Benchmark of the FEOD hot path on B200 (one JSON line on rank 0).

Workload (default C3 = BASELINE.json configs[2], the binding 60 % roofline
target of SURVEY.md §8(d)): nonlinear diffusion div((1+u^2) grad u) = 1 on a
64^3 perturbed hex mesh, Q3, 4^3 Gauss points, 7,189,057 DOFs, fp64.

A "step" = one pass of the hot path over the workload: r = F(u) (Eq. 1) and
Jv = J(u) v (Eq. 2), i.e. feod_residual + feod_jvp. value = DOF applications
per second over all ranks: 2 N x ranks / step time, in GDOF/s.

Timing: W untimed warm-up steps, then K steps bracketed by a barrier and
cuda.synchronize, CUDA events on the launching stream, max over ranks. The
working set (805 MB metric stream + 115 MB of vectors) exceeds the 126 MB L2,
so no flush is inserted. e2e: the same step through the C-ABI host-buffer
entry point feod_apply_host_batch (pinned host memory, every step's H2D + D2H inside the region).
roofline: the fused JVP kernel (dominant launch), algorithmic bytes per launch
(8 B per DOF per vector read/written + 48 B per quadrature
point of stored metric) / its event-timed duration, vs the measured HBM copy
bandwidth in MEASURED_PEAKS.json. cpu_baseline: the CPU oracle (oracle/), as it
stands, on a bounded element sample of the same workload on this host.

--impl reference: there is no reference implementation to install (the paper
ships no code); per the task's tier rules the reference arm is the oracle,
timed on the host cores on a bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import workloads as W  # noqa: E402

HBM_FALLBACK_GBS = 6650.0   # /opt/skills/guides/B200_PROFILING.md fallback
def _fp64_peaks():
    """DFMA rate measured by tools/peaks.py (profiles/r02_peaks_fp64.json, NVML clock record:
    1965 MHz, no throttle reason) and the nominal 148 SMs x 64 FMA/clk x 2 x clock."""
    try:
        with open(os.path.join(ROOT, "profiles", "r02_peaks_fp64.json")) as f:
            pk = json.load(f)
        return float(pk["fp64_tflops_burst"]), float(pk["fp64_tflops_nominal_at_max_clock"])
    except Exception:
        return 33.0, 37.2


FP64_MEASURED_TFLOPS, FP64_NOMINAL_TFLOPS = _fp64_peaks()


def algorithmic_bytes(w, call):
    """8 B per DOF per vector touched, 48 B/point metric, 8 B/elem rho and g."""
    N, E, q3 = w.n_dofs, w.n_elems, w.q ** 3
    geom = 48 * q3 * E if w.perturbed else 0
    vec = {"residual": 2, "jvp": 3, "vjp": 3, "jvp_res": 4, "design": 2}[call]
    extra = 0
    if w.model == W.HEAT:
        extra += 8 * E
    if call == "design":
        extra += 8 * E
    return 8 * N * vec + geom + extra


def algorithmic_flops(w, call):
    """2 x passes x E x (q(k+1)^3 + q^2(k+1)^2 + q^3(k+1) + 3 q^4) + pointwise x E q^3."""
    k, q, E = w.k, w.q, w.n_elems
    per_pass = q * (k + 1) ** 3 + q ** 2 * (k + 1) ** 2 + q ** 3 * (k + 1) + 3 * q ** 4
    passes = {"residual": 2, "jvp": 3, "vjp": 3, "jvp_res": 3, "design": 2}[call]
    table = {  # pointwise flops per point (perturbed / affine) from SURVEY.md §8(d)
        (W.PLAPLACE, True): {"residual": 45, "jvp": 76}, (W.NLDIFF, True): {"residual": 38, "jvp": 43},
        (W.PLAPLACE, False): {"residual": 16, "jvp": 35}, (W.HEAT, False): {"residual": 12, "jvp": 19, "design": 14},
        (W.NLDIFF, False): {"residual": 12, "jvp": 19},
    }
    pw = table.get((w.model, w.perturbed), {}).get("jvp" if call == "vjp" else call, 20)
    return 2 * passes * E * per_pass + pw * E * q ** 3


def read_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            mp = json.load(f)
        return float(mp["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy)"
    except Exception:
        return HBM_FALLBACK_GBS, "fallback (B200_PROFILING.md)"


def traffic_from_profiles(workload_name):
    p = os.path.join(ROOT, "profiles", "traffic.json")
    try:
        with open(p) as f:
            return json.load(f).get(workload_name)
    except Exception:
        return None


class Clocks:
    """SM clock and throttle reasons sampled DURING the timed region (B200_PROFILING.md clocks line).

    NVML (nvidia-ml-py) polled from a background thread every ~2 ms, so even a 10 ms
    region gets several samples; only samples whose host timestamps fall between
    mark_begin() and mark_end() count. nvidia-smi is the fallback (100 ms cadence)."""

    REASONS = {"hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
               "hw_power_brake_slowdown": 0x80, "sw_power_cap": 0x4}

    def __init__(self, gpu_index):
        self.gpu = gpu_index
        self.samples = []
        self.t_begin = self.t_end = None
        self._stop = False
        self._thr = None
        self.max_mhz = None

    def start(self):
        import threading
        try:
            import pynvml
            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(self.gpu)
            self.max_mhz = float(pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM))
        except Exception:
            self._thr = None
            return

        def run():
            while not self._stop:
                try:
                    mhz = float(pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM))
                    rs = int(pynvml.nvmlDeviceGetCurrentClocksEventReasons(h))
                except Exception:
                    break
                self.samples.append((time.perf_counter(), mhz, rs))
                time.sleep(0.002)
        self._thr = threading.Thread(target=run, daemon=True)
        self._thr.start()

    def mark_begin(self):
        self.t_begin = time.perf_counter()

    def mark_end(self):
        self.t_end = time.perf_counter()

    def stop(self):
        self._stop = True
        if self._thr is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "samples": 0, "reasons": ["nvml unavailable"]}
        self._thr.join(timeout=5)
        inside = [s for s in self.samples if self.t_begin is not None and self.t_begin <= s[0] <= self.t_end]
        reasons = sorted({nm for _, _, rs in inside for nm, bit in self.REASONS.items() if rs & bit})
        mhz = [m for _, m, _ in inside]
        return {"sm_mhz": statistics.median(mhz) if mhz else None, "sm_max_mhz": self.max_mhz,
                "samples": len(inside), "source": "NVML, ~2 ms cadence, samples inside the timed region only",
                "region_s": (self.t_end - self.t_begin) if self.t_begin is not None else None,
                "reasons": reasons}


def _oracle_step(pr, d, el):
    from oracle import fem as F
    t0 = time.perf_counter()
    F._assemble(pr, F._residual_elems(pr, d["u"], el), pr.n_dofs)
    F._assemble(pr, F._jvp_elems(pr, d["u"], d["v"], el), pr.n_dofs)
    return time.perf_counter() - t0


def oracle_sample_size(pr, d, E, target_s):
    """Elements per sample so one oracle residual+JVP takes about target_s seconds."""
    S = 64
    while True:
        t = _oracle_step(pr, d, np.arange(min(S, E)))
        if t > target_s / 4 or S >= E:
            return min(E, max(1, int(S * target_s / max(t, 1e-3))))
        S = min(E, S * 4)


def cpu_oracle_sample(w, d, target_s=15.0, S=None):
    """Oracle residual + JVP on a bounded element sample of w (the first S elements).

    Returns (rate, cores, sample, seconds, fraction): rate = the DOF applications the
    sample accounts for (2 N S / E) / the measured seconds of that sample. Nothing is
    extrapolated in time: the seconds are the sample's own wall time."""
    import oracle as O
    pr = O.Problem.from_workload(w, verts=d["verts"], rho=d.get("rho"))
    cores = len(os.sched_getaffinity(0))
    E = w.n_elems
    if S is None:
        S = oracle_sample_size(pr, d, E, target_s)
    el = np.arange(S)
    t = _oracle_step(pr, d, el)
    frac = S / E
    value = 2 * w.n_dofs * frac / t / 1e9
    sample = (f"oracle residual+JVP (dense element matrices, numpy fp64) on the first {S} of {E} elements "
              f"of {w.name} ({100 * frac:.3f} %, {t:.2f} s measured); rate = 2 N x {frac:.5f} DOF applications / "
              f"that time")
    return value, cores, sample, t, frac


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def run_reference(args, w):
    """The reference arm (tier rules: the CPU oracle, as it stands, on the host cores).

    A step = one oracle residual + JVP over a bounded element sample of the workload,
    sized so the whole --warmup W --steps K run ends within a few minutes. ms_per_step is
    the measured time of one such step (the driver's clock sees exactly that); value is
    the DOF applications the sample accounts for per second."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    d = W.draw(w)
    import oracle as O
    pr = O.Problem.from_workload(w, verts=d["verts"], rho=d.get("rho"))
    per_step = min(10.0, 120.0 / max(1, args.steps + args.warmup))
    S = oracle_sample_size(pr, d, w.n_elems, per_step)
    ts = []
    for s in range(args.warmup + args.steps):
        v, cores, sample, t, frac = cpu_oracle_sample(w, d, S=S)
        if s >= args.warmup:
            ts.append(t)
    t_step = statistics.mean(ts)
    value = 2 * w.n_dofs * frac / t_step / 1e9
    line = {"impl": "reference", "metric": "residual+JVP throughput (GDOF/s, fp64)", "value": value,
            "unit": "GDOF/s", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": t_step * 1e3, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": config_of(w), "extrapolated": False, "sample_fraction": frac,
            "cpu_baseline": {"value": value, "unit": "GDOF/s", "cores": cores, "kind": "oracle", "sample": sample,
                             "cpu_model": cpu_model()},
            "e2e": {"value": value, "unit": "GDOF/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def max_over_ranks(x, world, device=None):
    """Max of a per-rank float over all ranks (the timing rule: max over ranks)."""
    if world <= 1:
        return float(x)
    import torch
    import torch.distributed as dist
    t = torch.tensor([float(x)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def whole_job_rate(units_per_rank, world, seconds):
    """value = units all ranks processed / the max-over-ranks time (weak scaling replicas)."""
    return units_per_rank * world / seconds


def config_of(w):
    return {"workload": f"{w.name}: {W.MODEL_NAMES[w.model]}, {w.n}^3 {'perturbed' if w.perturbed else 'affine'} "
                        f"hexes, Q{w.k}, {w.q}^3 Gauss points (BASELINE.json configs[{int(w.name[1]) - 1}])",
            "n": w.n, "k": w.k, "q": w.q, "dofs": w.n_dofs, "elems": w.n_elems,
            "step": "feod_residual + feod_jvp (2 DOF applications per DOF)",
            "l2": "no flush: working set (stored metric + vectors) exceeds the 126 MB L2" if w.perturbed
                  else "no flush: vectors (>=115 MB) + scratch exceed L2 only partially"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=1000)   # ~0.5 s timed region at C3
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="feod", choices=["feod", "reference"])
    ap.add_argument("--workload", default="C3", choices=list(W.CONFIGS))
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--newton", action="store_true",
                    help="also time the Newton-CG driver (A15: 5 steps x 20 CG from u0 = 0; default on for C4)")
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)
    w = W.CONFIGS[args.workload]
    if args.impl == "reference":
        return run_reference(args, w)

    import torch
    import torch.distributed as dist
    import paper_2506_00746_b200 as fe

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    d = W.draw(w)
    rho = torch.as_tensor(d["rho"]).cuda() if "rho" in d else None
    op = fe.from_workload(w, verts=d["verts"], rho=rho)
    u = torch.as_tensor(d["u"]).cuda()
    v = torch.as_tensor(d["v"]).cuda()
    r = torch.empty_like(u)
    Jv = torch.empty_like(u)
    N = op.n_dofs
    stream = torch.cuda.current_stream()

    def step(prof=None):
        op.residual(u, out=r)
        if prof is not None:
            op.profile_next(*prof)
        op.jvp(u, v, out=Jv)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()

    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    for a, b in ev:   # torch creates the CUDA event lazily: record once so the handle exists
        a.record(stream)
        b.record(stream)
    torch.cuda.synchronize()
    clocks = Clocks(local)
    clocks.start()
    time.sleep(0.05)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    clocks.mark_begin()
    t0.record(stream)
    for s in range(args.steps):
        step(prof=ev[s])
    t1.record(stream)
    torch.cuda.synchronize()
    clocks.mark_end()
    if world > 1:
        dist.barrier()
    ck = clocks.stop()
    ms = t0.elapsed_time(t1)
    jvp_kernel_ms = statistics.mean(a.elapsed_time(b) for a, b in ev)
    ms = max_over_ranks(ms, world, device="cuda")
    ms_per_step = ms / args.steps
    value = whole_job_rate(2 * N, world, ms_per_step * 1e-3) / 1e9

    # per-call breakdown (rank-local, diagnostics)
    def time_call(fn, reps=10):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        fn()
        torch.cuda.synchronize()
        a.record(stream)
        for _ in range(reps):
            fn()
        b.record(stream)
        torch.cuda.synchronize()
        return a.elapsed_time(b) / reps
    t_res = time_call(lambda: op.residual(u, out=r))
    t_jvp = time_call(lambda: op.jvp(u, v, out=Jv))

    def each_call(fn, reps=20):
        """R calls each bracketed by events on the stream -> (median, min) in ms."""
        fn()
        torch.cuda.synchronize()
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(reps)]
        for a_, b_ in evs:
            a_.record(stream)
            fn()
            b_.record(stream)
        torch.cuda.synchronize()
        ts = [a_.elapsed_time(b_) for a_, b_ in evs]
        return statistics.median(ts), min(ts)
    res_med, res_min = each_call(lambda: op.residual(u, out=r))
    jvp_med, jvp_min = each_call(lambda: op.jvp(u, v, out=Jv))
    JTw = torch.empty_like(u)
    JTw_buf = torch.empty_like(u)
    t_vjp = time_call(lambda: op.vjp(u, v, out=JTw))   # NEXT-1 (diagnostic, not in the step)
    # the fused entry point of SURVEY §8(b): r and J v from one dual pass (feod_jvp_res)
    r2 = torch.empty_like(u)
    t_jres = time_call(lambda: op.jvp_res(u, v, out=(r2, JTw_buf)))
    # NEXT-2 stored linearisation: one linearize (F(u) + D's linearisation) then J v from it
    t_lin = time_call(lambda: op.linearize(u, out=r))
    t_jlin = time_call(lambda: op.jvp_lin(v, out=JTw))
    t_diag = time_call(lambda: op.jacobi_diag(out=JTw))
    t_des = t_rg = None
    if w.model == W.HEAT:
        g = torch.empty(op.n_elems, dtype=torch.float64, device=u.device)
        lam = torch.as_tensor(d["lam"]).cuda()   # the recipe's lambda draw
        t_des = time_call(lambda: op.design_grad(u, lam, out=g))
        r3 = torch.empty_like(u)
        t_rg = time_call(lambda: op.res_design_grad(u, lam, out=(r3, g)))   # SURVEY §8(d) "C5 r+g fused"

    # e2e through the C-ABI host-buffer path
    e2e = None
    if not args.no_e2e:
        # a stream of `reps` independent problems through feod_apply_host_batch: two pinned
        # host buffer sets in a ring; every step uploads its u, v and downloads its [r | Jv]
        uh = [torch.as_tensor(d["u"]).pin_memory() for _ in range(2)]
        vh = [torch.as_tensor(d["v"]).pin_memory() for _ in range(2)]
        rj = [torch.empty(2 * N, dtype=torch.float64).pin_memory() for _ in range(2)]   # [r | Jv]
        reps = max(4, min(args.steps, 20))
        ring = lambda lst: [lst[i % 2] for i in range(reps)]
        op.apply_host_batch(4, uh, vh, outs=rj)   # warm-up (staging buffers, streams)
        op.apply_host(4, uh[0], vh[0], out=rj[0])
        if world > 1:
            dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        op.apply_host_batch(4, ring(uh), ring(vh), outs=ring(rj))   # residual + JVP per step
        e1.record(stream)
        torch.cuda.synchronize()
        e_ms = e0.elapsed_time(e1) / reps
        e_ms = max_over_ranks(e_ms, world, device="cuda")
        # the one-problem-at-a-time call for comparison (no overlap across steps)
        e0.record(stream)
        for _ in range(4):
            op.apply_host(4, uh[0], vh[0], out=rj[0])
        e1.record(stream)
        torch.cuda.synchronize()
        single_ms = e0.elapsed_time(e1) / 4
        e2e = {"value": whole_job_rate(2 * N, world, e_ms * 1e-3) / 1e9, "unit": "GDOF/s",
               "h2d_bytes_per_step": 2 * 8 * N, "d2h_bytes_per_step": 2 * 8 * N,
               "ms_per_step": e_ms, "steps": reps,
               "path": "feod_apply_host_batch op 4 (C-ABI, pinned host buffers: per step u, v up and r, Jv down; "
                       "step b+1's uploads overlap step b's operator and downloads)",
               "single_call_ms_per_step": single_ms,
               "single_call_value": whole_job_rate(2 * N, world, single_ms * 1e-3) / 1e9}

    peak, peak_src = read_peaks()
    jvp_bytes = algorithmic_bytes(w, "jvp")
    achieved = jvp_bytes / (jvp_kernel_ms * 1e-3) / 1e9
    traffic = traffic_from_profiles(w.name)
    kname = ("col_kernel<JVP> (one thread per element column, Q1/Q2)" if w.k <= 2 else
             "q6tc_perl_kernel<JVP> + evec_assemble_kernel (FP64 tensor cores, Q6 affine)"
             if w.k == 6 and not w.perturbed else "plane_kernel<JVP>")
    roofline = {"bound": "hbm" if w.perturbed else "alu", "kernel": f"{kname}: fused G-B-D-B^T-G^T, {w.name}",
                "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                "traffic": traffic, "peak_source": peak_src,
                "algorithmic_bytes_per_launch": jvp_bytes, "kernel_ms": jvp_kernel_ms}
    if not w.perturbed:
        fl = algorithmic_flops(w, "jvp")
        ach = fl / (jvp_kernel_ms * 1e-3) / 1e12
        roofline.update({"achieved": ach, "peak": FP64_MEASURED_TFLOPS, "unit": "TFLOP/s",
                         "frac": ach / FP64_MEASURED_TFLOPS, "frac_of_nominal": ach / FP64_NOMINAL_TFLOPS,
                         "peak_nominal": FP64_NOMINAL_TFLOPS,
                         "peak_source": "measured DFMA rate at 1965 MHz, no throttle (profiles/r02_peaks_fp64.json); "
                                        "nominal = 148 SMs x 64 FMA/clk x 2 x 1.965 GHz (reached only by DMMA)",
                         "algorithmic_flops_per_launch": fl})

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        val, cores, sample, t_s, frac = cpu_oracle_sample(w, d)
        cpu = {"value": val, "unit": "GDOF/s", "cores": cores, "kind": "oracle", "sample": sample,
               "seconds": t_s, "sample_fraction": frac, "extrapolated": False, "cpu_model": cpu_model()}

    fl_res, fl_jvp = algorithmic_flops(w, "residual"), algorithmic_flops(w, "jvp")
    by_res, by_jvp = algorithmic_bytes(w, "residual"), algorithmic_bytes(w, "jvp")
    line = {"metric": "residual+JVP throughput (GDOF/s, fp64)", "value": value, "unit": "GDOF/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded workloads/ recipe, SURVEY.md §8(d))", "config": config_of(w),
            "parallelism": f"replicas x{world} (no data-path collective; DESIGN.md §Multi-GPU)",
            "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "clocks": ck,
            "gpu_launches": args.steps * 4,   # per call: the fused operator kernel + the fix-up / assembly kernel
            "calls": {
                "residual": {"us": t_res * 1e3, "us_median": res_med * 1e3, "us_min": res_min * 1e3,
                             "gdof_s": N / (t_res * 1e-3) / 1e9,
                             "hbm_frac": by_res / (t_res * 1e-3) / 1e9 / peak,
                             "fp64_frac": fl_res / (t_res * 1e-3) / 1e12 / FP64_MEASURED_TFLOPS},
                "jvp": {"us": t_jvp * 1e3, "us_median": jvp_med * 1e3, "us_min": jvp_min * 1e3,
                        "gdof_s": N / (t_jvp * 1e-3) / 1e9,
                        "hbm_frac": by_jvp / (t_jvp * 1e-3) / 1e9 / peak,
                        "fp64_frac": fl_jvp / (t_jvp * 1e-3) / 1e12 / FP64_MEASURED_TFLOPS,
                        "fused_kernel_us": jvp_kernel_ms * 1e3},
                "linearize": {"us": t_lin * 1e3, "gdof_s": N / (t_lin * 1e-3) / 1e9},
                "jvp_lin": {"us": t_jlin * 1e3, "gdof_s": N / (t_jlin * 1e-3) / 1e9},
                "jacobi_diag": {"us": t_diag * 1e3},
                "jvp_res": {"us": t_jres * 1e3, "gdof_s": 2 * N / (t_jres * 1e-3) / 1e9,
                            "note": "r and J v from one dual pass (feod_jvp_res); 2 DOF applications per DOF"},
                "vjp": {"us": t_vjp * 1e3, "gdof_s": N / (t_vjp * 1e-3) / 1e9,
                        "hbm_frac": algorithmic_bytes(w, "vjp") / (t_vjp * 1e-3) / 1e9 / peak,
                        "fp64_frac": algorithmic_flops(w, "vjp") / (t_vjp * 1e-3) / 1e12 / FP64_MEASURED_TFLOPS},
            }}
    if (args.newton or w.name == "C4") and world == 1:
        # a10 / SURVEY §8(d) C4 row: total device time of the whole driver, 2 warm-up runs, 3 timed
        u0 = torch.zeros_like(u)
        for _ in range(2):
            op.newton_cg(u0, 5, 20)
        torch.cuda.synchronize()
        tn = []
        for _ in range(3):
            a_, b_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a_.record(stream)
            _, norms = op.newton_cg(u0, 5, 20)
            b_.record(stream)
            torch.cuda.synchronize()
            tn.append(a_.elapsed_time(b_))
        n_jvp, n_res = 5 * 20, 6
        op.set_newton_linearization(True)
        op.newton_cg(u0, 5, 20)
        torch.cuda.synchronize()
        tl = []
        for _ in range(3):
            a_, b_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a_.record(stream)
            _, norms_l = op.newton_cg(u0, 5, 20)
            b_.record(stream)
            torch.cuda.synchronize()
            tl.append(a_.elapsed_time(b_))
        line["newton_cg_stored_linearization"] = {"ms": statistics.median(tl), "ms_min": min(tl), "norms": norms_l,
                                                  "note": "feod_set_newton_linearization(1): feod_linearize per step, "
                                                          "feod_jvp_lin per CG iteration (NEXT-2)"}
        op.set_newton_linearization(2)
        op.newton_cg(u0, 5, 20)
        torch.cuda.synchronize()
        tj = []
        for _ in range(3):
            a_, b_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a_.record(stream)
            _, norms_j = op.newton_cg(u0, 5, 20)
            b_.record(stream)
            torch.cuda.synchronize()
            tj.append(a_.elapsed_time(b_))
        op.set_newton_linearization(0)
        line["newton_pcg_jacobi"] = {"ms": statistics.median(tj), "ms_min": min(tj), "norms": norms_j,
                                     "note": "feod_set_newton_linearization(2): + feod_jacobi_diag per step, "
                                             "Jacobi-preconditioned CG (NEXT-3)"}
        op.set_cg_graphs(False)
        op.newton_cg(u0, 5, 20)
        torch.cuda.synchronize()
        tg = []
        for _ in range(3):
            a_, b_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a_.record(stream)
            op.newton_cg(u0, 5, 20)
            b_.record(stream)
            torch.cuda.synchronize()
            tg.append(a_.elapsed_time(b_))
        op.set_cg_graphs(True)
        line["newton_cg"] = {"ms": statistics.median(tn), "ms_min": min(tn), "jvp_calls": n_jvp, "residual_calls": n_res,
                             "norms": norms, "op_share_ms": (n_jvp * t_jvp + n_res * t_res),
                             "ms_without_graphs": statistics.median(tg),
                             "note": "feod_newton_cg: CG iterations as a replayed CUDA graph (5 launches per iteration, "
                                     "alpha/beta reduced in-kernel), host sync once per Newton step"}
    if world == 1:
        # NEXT-4 (Table-1 analogue): element tangents K_e = B^T J_D B on the FP64 tensor cores,
        # RES (integration-point AD) and ELM (element-level forward AD), on a bounded element range
        nn, Qp = (w.k + 1) ** 3, w.q ** 3
        ne = min(op.n_elems, 16384 if w.k <= 3 else 1024)   # Q6: K_e is 941 KB per element
        Ke = torch.empty((ne, nn, nn), dtype=torch.float64, device=u.device)
        pw = {W.PLAPLACE: 35, W.NLDIFF: 19, W.HEAT: 19}[w.model] * (2 if w.perturbed else 1)   # dual flux flops
        gemm = 2.0 * nn * nn * 3 * Qp
        interp = 2.0 * 4 * Qp * nn
        tab = {}
        per_pass = w.q * (w.k + 1) ** 3 + w.q ** 2 * (w.k + 1) ** 2 + w.q ** 3 * (w.k + 1) + 3 * w.q ** 4
        for elm in (False, True):
            t_em = time_call(lambda: op.element_matrices(u, 0, ne, elm=elm, out=Ke), reps=5)
            if elm:
                # value pass (dense B3 + collocated gradients) once, then per seed column: the
                # tangent through B (forward) and B^T (transposed), and Q dual flux evaluations
                fl = 2.0 * Qp * nn + 2.0 * 3 * Qp * w.q + nn * (2.0 * 2 * per_pass + Qp * pw)
            else:
                fl = gemm + interp + (4 * Qp * pw + 2.0 * 4 * 3 * Qp * nn)
            tab["ELM" if elm else "RES"] = {"ns_per_element": t_em * 1e6 / ne, "kflop_per_element": fl / 1e3,
                                            "tflops": fl * ne / (t_em * 1e-3) / 1e12,
                                            "dual_flux_evaluations_per_point": nn if elm else 4}
        line["element_tangents"] = {"elements": ne, "nd3": nn, **tab,
                                    "elm_over_res_flops": tab["ELM"]["kflop_per_element"] / tab["RES"]["kflop_per_element"],
                                    "elm_over_res_time": tab["ELM"]["ns_per_element"] / tab["RES"]["ns_per_element"],
                                    "elm_over_res_dual_flux_evaluations": nn / 4,
                                    "table1_fwd_elm_over_res_flops_context": {"Tet1": 2.5, "Tet2": 5.4, "Tet3": 9.4},
                                    "note": "feod_element_matrices: RES = 4 dual evaluations of D per point + K_e = M^T N "
                                            "on DMMA m8n8k4 f64; ELM = element-level forward AD, one dual pass of "
                                            "B^T D(B u_e) per seed column (B inside the differentiation loop)"}
    if w.model == W.HEAT and world == 1:
        # NEXT-1: adjoint solve, 50 BiCGStab iterations (2 J^T applications each), rhs = the recipe's lambda draw
        lam_rhs = torch.as_tensor(d["lam"]).cuda()
        op.adjoint_solve(u, lam_rhs, iters=5)
        torch.cuda.synchronize()
        a_, b_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a_.record(stream)
        _, hist = op.adjoint_solve(u, lam_rhs, iters=50)
        b_.record(stream)
        torch.cuda.synchronize()
        line["adjoint_solve"] = {"ms": a_.elapsed_time(b_), "iters": 50, "vjp_calls": 100,
                                 "res_first": hist[0], "res_last": hist[-1],
                                 "note": "feod_adjoint_solve, unpreconditioned BiCGStab on P^T J^T (device time)"}
    if t_rg is not None:
        by = 8 * (2 * N + N) + 16 * w.n_elems + (48 * w.q ** 3 * w.n_elems if w.perturbed else 0)
        fl = 2 * 3 * w.n_elems * (w.q * (w.k + 1) ** 3 + w.q ** 2 * (w.k + 1) ** 2 + w.q ** 3 * (w.k + 1) + 3 * w.q ** 4) \
            + 23 * w.n_elems * w.q ** 3
        line["calls"]["res_design_grad"] = {"us": t_rg * 1e3, "hbm_frac": by / (t_rg * 1e-3) / 1e9 / peak,
                                            "fp64_frac": fl / (t_rg * 1e-3) / 1e12 / FP64_MEASURED_TFLOPS,
                                            "note": "feod_res_design_grad: r and g from one dual pass seeded along rho"}
    if t_des is not None:
        line["calls"]["design_grad"] = {"us": t_des * 1e3, "gdof_s": N / (t_des * 1e-3) / 1e9,
                                        "hbm_frac": algorithmic_bytes(w, "design") / (t_des * 1e-3) / 1e9 / peak,
                                        "fp64_frac": algorithmic_flops(w, "design") / (t_des * 1e-3) / 1e12
                                        / FP64_MEASURED_TFLOPS}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
