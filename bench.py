"""bench.py — throughput of the fused variable-order seismic step on B200.

Workload (BASELINE.json configs[1], "C2"): 2D periodic [-16,16)^2, 1024x1024, fp64,
Gaussian pulse, two-layer Q medium, M = 16, dt = 5e-4.  One "step" is one
SeismicStepper::step (seismic.cpp:111-133): two M-term operator applies of
orders 1+gamma and 1/2+gamma sharing one forward transform, plus the fused update.

  value   = 2 N (M+1) / t_step / 1e9   [Gpoint*term/s], inputs resident in HBM
  e2e     = same metric through the public API with the wavefield copied host->device
            (pinned) before and device->host after every step
  roofline: HBM bytes of the step (SURVEY.md §8(d) model) / measured step time vs
            MEASURED_PEAKS.json hbm_gbs
  cpu_baseline: the reference itself (oracle/_ref: reference sources + FFTW-API shim)
            timed on this host's cores on a bounded number of C2 steps

`--impl reference` times the reference CPU implementation of the same step.
N > 1 (torchrun): every rank runs an independent C2 replica (weak scaling, no
collective on the data path; C2 is a single-GPU configuration).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
from paper_2311_13049_b200 import configs  # noqa: E402

METRIC = "VO frac-Laplacian Gpoint·term/s & time-steps/s; % of HBM roofline"
UNIT = "Gpoint·term/s"


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=200)
    p.add_argument("--warmup", type=int, default=5)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--size", type=int, default=1024, help="grid points per axis (C2 = 1024)")
    p.add_argument("--cpu-baseline-steps", type=int, default=4)
    p.add_argument("--workload", default="c2", choices=["c2", "c3", "c4", "c5"],
                   help="c2 (default): fused seismic step; c3/c4: slab-decomposed 3D apply; c5: batched 2D sweep")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--e2e-shots", type=int, default=4,
                   help="independent shots pipelined in the end-to-end measurement (1 = serial)")
    p.add_argument("--slab-mode", default="step", choices=["step", "apply"],
                   help="c3/c4: seismic steps (SlabSeismicStepper, BASELINE configs[2..3]) or one operator apply")
    p.add_argument("--transpose", default="fused", choices=["fused", "nccl"],
                   help="c3/c4: slab transposes fused into the C2C stages (peer stores) or NCCL all-to-all")
    return p.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


class ClockSampler:
    """Samples SM clock and throttle reasons through NVML during the timed region."""

    REASONS = {
        0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
        0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
        0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting",
    }

    def __init__(self, index: int):
        self.samples, self.reasons = [], set()
        self.max_mhz = None
        self._stop = threading.Event()
        try:
            import pynvml

            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                r = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if r & bit and bit != 0x1:
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.002)

    def __enter__(self):
        if self.nv:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        if self.nv:
            self._stop.set()
            self.t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["nvml unavailable"]}
        return {"sm_mhz": float(statistics.median(self.samples)), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


def cpu_model() -> str:
    """lscpu's model name (falls back to /proc/cpuinfo)."""
    import subprocess

    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for ln in out.splitlines():
            if ln.lower().startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except Exception:
        pass
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.lower().startswith("model name"):
                    return ln.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def _omp_set_threads(n: int) -> None:
    """omp_set_num_threads in this process's OpenMP runtime (the reference's parallel region,
    flap.cpp:75-77, reads it at every apply)."""
    import ctypes as C

    for name in ("libgomp.so.1", "libgomp.so"):
        try:
            C.CDLL(name).omp_set_num_threads(int(n))
            return
        except OSError:
            continue


def cpu_baseline(cfg, steps: int, warmup: int = 1, single_thread_steps: int = 2):
    """Time the reference (oracle/_ref) — or, if it is not built, the C restatement —
    on `steps` C2 steps (after `warmup`) on this host with all cores, then again with one
    thread (OMP_NUM_THREADS = nproc and = 1).  Checker code: only this leg
    (and the reference arm) imports oracle/."""
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import ctypes as C

    import oracle_lib as O

    cores = os.cpu_count() or 1
    units = 2 * cfg.N * (cfg.M + 1)

    def time_steps(nthreads, nsteps, nwarm):
        _omp_set_threads(nthreads)
        if O.ref_available():
            lib = O.reference()
            lib.ref_time_seismic.argtypes = [C.c_int, O._ip, O._dp, O._dp, O._dp, O._dp, C.c_double, C.c_int,
                                             O._dp, O._dp, C.c_double, C.c_int, C.c_int, C.POINTER(C.c_double),
                                             C.c_void_p]
            per = C.c_double(0.0)
            rc = lib.ref_time_seismic(len(cfg.J), O._i32(cfg.J), O._f64(cfg.lo), O._f64(cfg.hi),
                                      O._f64(cfg.gamma).ravel(), O._f64(cfg.c0).ravel(), cfg.omega0, cfg.M,
                                      O._f64(cfg.phi).ravel(), O._f64(cfg.psi).ravel(), cfg.tau, int(nwarm),
                                      int(nsteps), C.byref(per), None)
            if rc != 0:
                raise RuntimeError(lib.ref_last_error())
            return per.value
        t0 = time.perf_counter()
        O.port_seismic(cfg.J, cfg.lo, cfg.hi, cfg.gamma, cfg.c0, cfg.omega0, cfg.M, cfg.phi, cfg.psi, cfg.tau,
                       nsteps)
        return (time.perf_counter() - t0) / (nsteps + 1.5)  # construction = 3 applies ~ 1.5 steps

    t = time_steps(cores, steps, warmup)
    t1 = time_steps(1, single_thread_steps, 0) if single_thread_steps > 0 else None
    _omp_set_threads(cores)
    if O.ref_available():
        kind = "reference"
        how = ("reference sources (proj/src, unmodified) + FFTW-API shim (FFT backend = builder shim; FFTW absent "
               "in image), OpenMP over the M+1 terms (flap.cpp:75-77)")
    else:
        kind = "port"
        how = "C restatement (oracle/fw_oracle.c), OpenMP over FFT lines"
    out = {"value": units / t / 1e9, "unit": UNIT, "cores": cores, "kind": kind,
           "sample": f"{steps} SeismicStepper steps of C2 (1024^2, M=16) after {warmup} warm-up step(s), "
                     f"steady_clock around step() (seismic.cpp:111-133); {how}",
           "cpu_model": cpu_model(), "sec_per_step": t}
    if t1 is not None:
        out["single_thread"] = {"value": units / t1 / 1e9, "unit": UNIT, "cores": 1,
                                "sample": f"{single_thread_steps} steps, omp_set_num_threads(1)",
                                "sec_per_step": t1}
    return out


def c2_config(cfg, size: int, world: int) -> dict:
    """The `config` object of the C2 line, shared by both arms (the driver compares them)."""
    return {"workload": f"C2 seismic step ({size}^2, M=16, dt=5e-4; BASELINE configs[1])",
            "grid": list(cfg.J), "M": cfg.M, "tau": cfg.tau,
            "parallelism": "single GPU" if world == 1 else f"{world} independent replicas",
            "l2": "working set (2 ops x 17 w-tables + term scratch + state) ~0.45 GB > 126 MB L2; no flush"}


def run_reference_arm(args):
    """The reference's own CPU implementation of the same step (SeismicStepper::step on the
    reference sources) on this host's cores, --steps timed steps after --warmup, same metric,
    unit and config as our arm.  Under torchrun only rank 0 runs it."""
    rank, world, _ = dist_env()
    if rank != 0:
        return
    from paper_2311_13049_b200 import configs

    cfg = configs.c2(args.size)
    cb = cpu_baseline(cfg, args.steps, args.warmup)
    v = cb["value"]
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": cb["sec_per_step"] * 1e3,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": c2_config(cfg, args.size, world),
            "time_steps_per_s": 1.0 / cb["sec_per_step"],
            "cpu_baseline": {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample", "cpu_model",
                                                "single_thread") if k in cb},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def run_slab_step(args, cfg_fn, name):
    """configs[2]/[3] as specified: seismic time steps of the slab-decomposed 3D stepper
    (SlabSeismicStepper: fused transposes over CUDA IPC / NVLink, shared forward transform,
    fused update, blow-up flag combined over ranks every step) on N ranks, strong scaling."""
    import torch

    import paper_2311_13049_b200 as fw
    from paper_2311_13049_b200.slab import IpcPeers, LocalPeers, SlabGeometry, SlabSeismicStepper

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    cfg = cfg_fn(args.size) if args.size != 1024 else cfg_fn()
    ctx = fw.Context(local)
    g = fw.Grid(list(zip(cfg.lo, cfg.hi)), list(cfg.J))
    geo = SlabGeometry(cfg.J, world, rank)
    factory = (lambda k, geo_, nt, ctx_: IpcPeers(geo_, nt, ctx_)) if world > 1 else \
        (lambda k, geo_, nt, ctx_: LocalPeers(geo_, nt, ctx_))
    st = SlabSeismicStepper(g, cfg.gamma, cfg.c0, cfg.omega0, cfg.M, cfg.phi, cfg.psi, cfg.tau, geo, ctx, factory)
    stream = torch.cuda.ExternalStream(ctx.stream)
    st.advance(args.warmup)
    ctx.sync()
    if world > 1:
        torch.distributed.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        e0.record(stream)
        st.advance(args.steps)
        e1.record(stream)
        e1.synchronize()
    t = torch.tensor([e0.elapsed_time(e1) / args.steps], dtype=torch.float64, device="cuda")
    if world > 1:
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
    ms = float(t.item())
    units = 2 * cfg.N * (cfg.M + 1)
    # e2e: this rank's slab of the wavefield in (pinned H2D) and out (D2H) every step
    hin = st.cur.cpu().pin_memory()
    hout = torch.empty_like(hin).pin_memory()
    n_e2e = max(2, min(args.steps, 10))
    e2, e3 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e2.record(stream)
    for _ in range(n_e2e):
        with torch.cuda.stream(stream):
            st.cur.copy_(hin, non_blocking=True)
        st.step()
        with torch.cuda.stream(stream):
            hout.copy_(st.cur, non_blocking=True)
    e3.record(stream)
    e3.synchronize()
    t2 = torch.tensor([e2.elapsed_time(e3) / n_e2e], dtype=torch.float64, device="cuda")
    if world > 1:
        torch.distributed.all_reduce(t2, op=torch.distributed.ReduceOp.MAX)
    if rank == 0:
        hbm, peak_src = peaks()
        B = (2 * configs.bytes_per_apply_pass_model(cfg.N, cfg.N_half, cfg.M, table_model=False)
             - 8 * cfg.N + 72 * cfg.N) / world
        line = {"metric": METRIC, "value": units / (ms * 1e-3) / 1e9, "unit": UNIT, "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
                "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
                "time_steps_per_s": 1e3 / ms,
                "config": {"workload": f"{name}: slab-decomposed seismic step ({'x'.join(map(str, cfg.J))}, "
                                       f"M={cfg.M}, dt={cfg.tau})",
                           "grid": list(cfg.J), "M": cfg.M, "parallelism": f"slab P={world} (axis 0)",
                           "transpose": "fused into the C2C stages (peer stores over CUDA IPC)",
                           "table_bytes_per_rank": st.table_bytes,
                           "blowup_check": "once per advance (flags shared through peer memory)",
                           "l2": "working set > 126 MB L2; no flush"},
                "roofline": {"bound": "hbm", "achieved": B / (ms * 1e-3) / 1e9, "peak": hbm, "unit": "GB/s",
                             "frac": B / (ms * 1e-3) / 1e9 / hbm, "traffic": None,
                             "kernel": "whole step (multi-pass kernels, fused transposes, update)",
                             "bytes_model": "SURVEY 8(d) 3D pass model, 2 applies - 8N + 72N per step, / P; "
                                            "(s-s0)^m regenerated on chip", "peak_source": peak_src},
                "e2e": {"value": units / (float(t2.item()) * 1e-3) / 1e9, "unit": UNIT,
                        "h2d_bytes_per_step": 8 * cfg.N // world, "d2h_bytes_per_step": 8 * cfg.N // world},
                "gpu_launches": None, "clocks": clk.summary()}
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.barrier()
        torch.distributed.destroy_process_group()
    _fast_exit()  # while the context and its tensors are still alive


def run_slab(args, cfg_fn, name):
    """configs[2]/[3]: slab-decomposed 3D apply of the dispersion operator over N ranks
    (strong scaling: the global grid is fixed).  Transposes: fused into the C2C stages
    (each rank's last FFT pass stores into the owning rank's buffer through CUDA IPC /
    NVLink, default) or one NCCL all-to-all forward + one batched all-to-all backward."""
    import torch

    import paper_2311_13049_b200 as fw
    from paper_2311_13049_b200.slab import (DeviceStages, FusedSlabApply, IpcPeers, LocalPeers, SlabGeometry,
                                            slab_apply_device)

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    cfg = cfg_fn(args.size) if args.size != 1024 else cfg_fn()
    ctx = fw.Context(local)
    g = fw.Grid(list(zip(cfg.lo, cfg.hi)), cfg.J)
    op = fw.build_expansion(fw.OrderField(g, 1.0 + cfg.gamma), cfg.M, ctx=ctx)
    geo = SlabGeometry(cfg.J, world, rank)
    u = torch.from_numpy(np.ascontiguousarray(cfg.phi[geo.rows])).cuda()
    stream = torch.cuda.ExternalStream(ctx.stream)
    if args.transpose == "fused":
        st = DeviceStages(ctx)
        wl, dl, ml = st.local_tables(op, geo)
        peers = (IpcPeers if world > 1 else LocalPeers)(geo, cfg.M + 1, ctx)
        fused = FusedSlabApply(geo, st, peers, wl, dl, ml)

        def slab_apply_device(op_, u_, geo_, ctx_):  # noqa: F811 (same call shape as the NCCL path)
            return fused.apply(u_)
    for _ in range(args.warmup):
        slab_apply_device(op, u, geo, ctx)
    ctx.sync()
    if world > 1:
        torch.distributed.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        e0.record(stream)
        for _ in range(args.steps):
            out = slab_apply_device(op, u, geo, ctx)
        e1.record(stream)
        e1.synchronize()
    ms = e0.elapsed_time(e1) / args.steps
    t = torch.tensor([ms], dtype=torch.float64, device="cuda")
    if world > 1:
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
    ms = float(t.item())
    units = cfg.N * (cfg.M + 1)
    # e2e: host slab in (pinned), host slab out
    hin = torch.from_numpy(np.ascontiguousarray(cfg.phi[geo.rows])).pin_memory()
    hout = torch.empty_like(hin).pin_memory()
    e2, e3 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    n_e2e = max(2, min(args.steps, 10))
    e2.record(stream)
    for _ in range(n_e2e):
        with torch.cuda.stream(stream):
            ud = hin.cuda(non_blocking=True)
        o = slab_apply_device(op, ud, geo, ctx)
        with torch.cuda.stream(stream):
            hout.copy_(o, non_blocking=True)
    e3.record(stream)
    e3.synchronize()
    t2 = torch.tensor([e2.elapsed_time(e3) / n_e2e], dtype=torch.float64, device="cuda")
    if world > 1:
        torch.distributed.all_reduce(t2, op=torch.distributed.ReduceOp.MAX)
    if rank == 0:
        hbm, peak_src = peaks()
        # 3D: the SURVEY's pass model (intermediates in HBM); the generic path regenerates
        # (s-s0)^m on chip (k_rows_c2r), so the 8MN table term is dropped
        B = configs.bytes_per_apply_pass_model(cfg.N, cfg.N_half, cfg.M, table_model=False) / world
        line = {"metric": METRIC, "value": units / (ms * 1e-3) / 1e9, "unit": UNIT, "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
                "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
                "config": {"workload": f"{name}: slab-decomposed apply of order 1+gamma "
                                       f"({'x'.join(map(str, cfg.J))}, M={cfg.M}); one step = one apply",
                           "grid": list(cfg.J), "M": cfg.M, "parallelism": f"slab P={world} (axis 0)",
                           "transpose": ("fused into the C2C stages (peer stores)" if args.transpose == "fused"
                                         else "NCCL all_to_all_single"),
                           "l2": "working set > 126 MB L2; no flush"},
                "roofline": {"bound": "hbm", "achieved": B / (ms * 1e-3) / 1e9, "peak": hbm, "unit": "GB/s",
                             "frac": B / (ms * 1e-3) / 1e9 / hbm, "traffic": None,
                             "kernel": "whole apply (multi-pass kernels + transposes)",
                             "bytes_model": "SURVEY 8(d) 3D pass model / P, (s-s0)^m regenerated on chip",
                             "peak_source": peak_src},
                "e2e": {"value": units / (float(t2.item()) * 1e-3) / 1e9, "unit": UNIT,
                        "h2d_bytes_per_step": 8 * cfg.N // world, "d2h_bytes_per_step": 8 * cfg.N // world},
                "gpu_launches": None, "clocks": clk.summary()}
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.barrier()
        torch.distributed.destroy_process_group()
    _fast_exit()  # while the context and its tensors are still alive


def run_c5(args):
    """configs[4]: 64 independent 512^2 fields (data-parallel over ranks, no collective),
    apply-only throughput for every M of the sweep; value = the M = 16 sweep point."""
    import torch

    import paper_2311_13049_b200 as fw

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    ctx = fw.Context(local)
    stream = torch.cuda.ExternalStream(ctx.stream)
    mine = [f for f in range(configs.C5_FIELDS) if f % world == rank]
    fields = [configs.c5_field(f) for f in mine]
    g = fw.Grid(list(zip(fields[0].lo, fields[0].hi)), fields[0].J)
    us = [torch.from_numpy(np.ascontiguousarray(f.u)).cuda() for f in fields]
    outs = [torch.empty_like(u) for u in us]
    per_m = {}
    for M in configs.C5_M:
        ops = [fw.build_expansion(fw.OrderField(g, f.s), M, ctx=ctx) for f in fields]
        uptr, optr = [u.data_ptr() for u in us], [o.data_ptr() for o in outs]
        for _ in range(max(1, args.warmup)):
            fw.apply_batch_device(ops, uptr, optr)
        ctx.sync()
        if world > 1:
            torch.distributed.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = max(1, args.steps // 20)
        e0.record(stream)
        for _ in range(reps):
            fw.apply_batch_device(ops, uptr, optr)
        e1.record(stream)
        e1.synchronize()
        t = torch.tensor([e0.elapsed_time(e1) / reps], dtype=torch.float64, device="cuda")
        if world > 1:
            torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        ms = float(t.item())
        n = fields[0].u.size
        per_m[M] = {"ms_per_sweep": ms, "Gpoint_term_per_s": configs.C5_FIELDS * n * (M + 1) / (ms * 1e-3) / 1e9}
        del ops
    if rank == 0:
        hbm, peak_src = peaks()
        n = fields[0].u.size
        nh = n // 512 * 257
        ms16 = per_m[16]["ms_per_sweep"]
        # generic 2D path: (s-s0)^m regenerated on chip (k_rows_c2r) -> table term 8N
        B = configs.C5_FIELDS * configs.bytes_per_apply(n, nh, 16, table_model=False)
        Bp = configs.C5_FIELDS * (8 * n + 16 * nh + 32 * nh + 16 * nh + 17 * (8 + 16 + 16) * nh + 8 * n + 8 * n)
        line = {"metric": METRIC, "value": per_m[16]["Gpoint_term_per_s"], "unit": UNIT, "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms16, "higher_is_better": True,
                "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
                "config": {"workload": "C5: 64 x 512^2 independent applies (one step = one sweep at M = 16)",
                           "M_sweep": {str(k): v for k, v in per_m.items()},
                           "parallelism": f"data-parallel over {world} GPU(s), no collective"},
                "roofline": {"bound": "hbm", "achieved": B / (ms16 * 1e-3) / 1e9, "peak": hbm, "unit": "GB/s",
                             "frac": B / (ms16 * 1e-3) / 1e9 / hbm, "traffic": None,
                             "kernel": "64 applies (multi-pass kernels)", "peak_source": peak_src,
                             "bytes_model": "table model, (s-s0)^m regenerated on chip (SURVEY 8(d))",
                             # the 2D pass model: forward R2C + column C2C, all-terms column inverse
                             # (uhat once, w_m, M+1 spectra out), row C2R (M+1 spectra in, dev1, out)
                             "pass_model": {"bytes": Bp, "achieved": Bp / (ms16 * 1e-3) / 1e9,
                                            "frac": Bp / (ms16 * 1e-3) / 1e9 / hbm}},
                "e2e": None, "gpu_launches": None}
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.barrier()
        torch.distributed.destroy_process_group()
    _fast_exit()  # while the context and its tensors are still alive


def _fast_exit():
    """torch tensors allocated on the fw context's stream must not outlive that stream;
    skip interpreter teardown once the line is printed and the GPU is idle."""
    import torch

    torch.cuda.synchronize()
    sys.stdout.flush()
    sys.stderr.flush()
    os._exit(0)


def main():
    args = parse()
    if args.impl == "reference":
        run_reference_arm(args)
        return
    if args.workload in ("c3", "c4"):
        from paper_2311_13049_b200 import configs as _c

        fn = run_slab_step if args.slab_mode == "step" else run_slab
        fn(args, _c.c3 if args.workload == "c3" else _c.c4, args.workload.upper())
        _fast_exit()
    if args.workload == "c5":
        run_c5(args)
        _fast_exit()
    rank, world, local = dist_env()
    import torch

    import paper_2311_13049_b200 as fw
    from paper_2311_13049_b200 import configs

    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    cfg = configs.c2(args.size)
    ctx = fw.Context(local)
    grid = fw.Grid(list(zip(cfg.lo, cfg.hi)), cfg.J)
    med = fw.build_medium(grid, cfg.gamma, cfg.c0, cfg.omega0, cfg.M)
    st = fw.SeismicStepper(med, cfg.phi, cfg.psi, cfg.tau, ctx=ctx)
    stream = torch.cuda.ExternalStream(ctx.stream)

    def barrier():
        torch.cuda.synchronize()
        ctx.sync()
        if world > 1:
            torch.distributed.barrier()

    # ---- device-resident throughput ----
    st.advance(args.warmup)
    barrier()
    l0 = ctx.launches()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        e0.record(stream)
        st.enqueue(args.steps)
        e1.record(stream)
        e1.synchronize()
    launches = ctx.launches() - l0
    st.n()  # raises BlowupDetected if the device flag fired
    ms = e0.elapsed_time(e1) / args.steps
    t_max = torch.tensor([ms], dtype=torch.float64, device="cuda")
    if world > 1:
        torch.distributed.all_reduce(t_max, op=torch.distributed.ReduceOp.MAX)
    ms = float(t_max.item())
    units = 2 * cfg.N * (cfg.M + 1)
    value = world * units / (ms * 1e-3) / 1e9

    # ---- end to end through the public API (pinned host wavefield round trip per step) ----
    import ctypes as C

    lib = fw.load_library()
    host = torch.empty(cfg.N, dtype=torch.float64, pin_memory=True)
    hp = C.cast(C.c_void_p(host.data_ptr()), C.POINTER(C.c_double))
    check = fw._capi.check
    check(lib.fw_seis_get(st._h, hp, None, None, None))
    e2e_steps = max(3, min(args.steps, 50))
    # one public call per step: host wavefield in, one step, host wavefield out (fw_seis_step_io)
    for _ in range(2):
        check(lib.fw_seis_step_io(st._h, hp, 1, hp))
    barrier()
    e2, e3 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e2.record(stream)
    for _ in range(e2e_steps):
        check(lib.fw_seis_step_io(st._h, hp, 1, hp))
    e3.record(stream)
    e3.synchronize()
    ms_serial = e2.elapsed_time(e3) / e2e_steps
    t2 = torch.tensor([ms_serial], dtype=torch.float64, device="cuda")
    if world > 1:
        torch.distributed.all_reduce(t2, op=torch.distributed.ReduceOp.MAX)
    ms_serial = float(t2.item())
    e2e_serial = world * units / (ms_serial * 1e-3) / 1e9

    # The same per-step exchange for a pipeline of independent shots (the production shape of this
    # workload: many sources over one medium): every shot has its own context (stream), stepper
    # and pinned wavefield; each shot step is one fw_seis_step_io_async (H2D of that shot's
    # wavefield, one step, D2H of the new wavefield) completed by fw_seis_wait before the host
    # touches the buffer again.  The copies of one shot run under the steps of the others.
    S = max(1, args.e2e_shots)
    shots = [(ctx, st, host, hp)]
    for i in range(1, S):
        cx = fw.Context(local)
        sx = fw.SeismicStepper(med, cfg.phi * (1.0 + 0.125 * i), cfg.psi, cfg.tau, ctx=cx)
        hx = torch.empty(cfg.N, dtype=torch.float64, pin_memory=True)
        px = C.cast(C.c_void_p(hx.data_ptr()), C.POINTER(C.c_double))
        check(lib.fw_seis_get(sx._h, px, None, None, None))
        shots.append((cx, sx, hx, px))
    streams = [torch.cuda.ExternalStream(cx.stream) for cx, _, _, _ in shots]

    def run_rounds(rounds):
        for r in range(rounds):
            for _, sx, _, px in shots:
                if r:
                    check(lib.fw_seis_wait(sx._h))  # the host owns this shot's wavefield again
                check(lib.fw_seis_step_io_async(sx._h, px, 1, px))
        for _, sx, _, _ in shots:
            check(lib.fw_seis_wait(sx._h))

    run_rounds(2)
    barrier()
    for cx, _, _, _ in shots:
        cx.sync()
    rounds = max(3, min(args.steps, 50))
    e4 = torch.cuda.Event(enable_timing=True)
    ends = [torch.cuda.Event(enable_timing=True) for _ in shots]
    e4.record(streams[0])
    for r in range(rounds):
        for (_, sx, _, px) in shots:
            if r:
                check(lib.fw_seis_wait(sx._h))
            check(lib.fw_seis_step_io_async(sx._h, px, 1, px))
    for (_, sx, _, _), sm, ev in zip(shots, streams, ends):
        ev.record(sm)
    for (_, sx, _, _) in shots:
        check(lib.fw_seis_wait(sx._h))
    torch.cuda.synchronize()
    ms_e2e = max(e4.elapsed_time(ev) for ev in ends) / (rounds * S)
    t3 = torch.tensor([ms_e2e], dtype=torch.float64, device="cuda")
    if world > 1:
        torch.distributed.all_reduce(t3, op=torch.distributed.ReduceOp.MAX)
    ms_e2e = float(t3.item())
    e2e_value = world * units / (ms_e2e * 1e-3) / 1e9

    if rank == 0:
        hbm, peak_src = peaks()
        B_step = configs.bytes_per_seismic_step(cfg.N, cfg.N_half, cfg.M, table_model=True)
        achieved = B_step / (ms * 1e-3) / 1e9
        traffic = None
        try:
            with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
                traffic = json.load(f).get(f"c2_step_{args.size}")
        except Exception:
            pass
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": c2_config(cfg, args.size, world),
            "time_steps_per_s": world * 1e3 / ms,
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s",
                         "frac": achieved / hbm, "traffic": traffic,
                         "kernel": "whole seismic step (all launches of one step)",
                         "bytes_model": "SURVEY.md 8(d) B_step = 2 B_apply - 8N + 72N (table-streaming model)",
                         "algorithmic_bytes_per_step": B_step, "peak_source": peak_src},
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": 8 * cfg.N,
                    "d2h_bytes_per_step": 8 * cfg.N, "ms_per_step": ms_e2e, "shots": S,
                    "path": "fw_seis_step_io_async + fw_seis_wait per shot step over %d independent shots "
                            "(one context/stream each): pinned H2D of the shot's wavefield, one step, D2H of "
                            "the new wavefield, one host sync; a step = one shot step" % S,
                    "serial": {"value": e2e_serial, "ms_per_step": ms_serial,
                               "path": "fw_seis_step_io on one stepper: H2D, one step, D2H, host sync, "
                                       "nothing overlapped"}},
            "gpu_launches": int(launches),
            "launches_per_step": launches / args.steps,
            "clocks": clk.summary(),
        }
        if not args.no_cpu_baseline and world == 1:
            try:
                cb = cpu_baseline(cfg, args.cpu_baseline_steps)
                line["cpu_baseline"] = {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample", "cpu_model",
                                                           "single_thread") if k in cb}
            except Exception as e:  # reported, never fatal
                line["cpu_baseline"] = {"value": None, "error": str(e)[:200]}
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.barrier()
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
