"""Benchmark: models/sec of a full CALS sweep (BASELINE.json metric) on B200.

Workload (BASELINE.json configs[1]): 200x200x200 synthetic
tensor (generate_synthetic rank 20, noise 0.1, seed 0), 200 models = ranks
1..20 x 10 random inits (build_models seed 1), r_star = 2100 (all admitted),
a full sweep = every model run to retirement with tol = 0 and 5 iterations
(the fixed-iteration sweep of BASELINE.md section 3).  A "step" is one such
sweep.

  value  -- device-resident: tensor + starting factors already in HBM, one
            step = reload the model pool (D2D) + run the device loop to the
            last retirement; CUDA events on the launch stream, L2 flushed
            (256 MiB write) between steps, max over ranks.
  e2e    -- the public API ``paper_2010_04678_b200.run`` with host numpy
            inputs (tensor data in pinned host memory): a fresh DenseTensor
            each step (tensor H2D), model pool H2D, results D2H and the Model
            objects built -- wall clock with device syncs.  Device workspaces
            persist between calls (the driver's engine cache).
  roofline -- the fused MTTKRP (+ Lo slicing + split reduction) at the c2
            shape and W=2100 through cals_mttkrp, CUDA events.  On the INT8
            tensor-core (Ozaki) path: algorithmic INT8 ops (2 x 28 slice
            products x W x prod(dims), unpadded) against the INT8 peak
            measured live by cals_int8_peak_probe, plus the FP64-equivalent
            rate (2*W*prod(dims) per launch, mttkrp.py:72-76) against the live
            DMMA peak (cals_fp64_peak_probe); on the DMMA path the latter only.
  cpu_baseline -- the reference package (baseline/_ref, unmodified) on the
            host cores, rank 0 at N=1: a 1-iteration warm-up run, then the
            full workload's sweep (c2: 200 models x 5 iterations) timed.

Multi-GPU: one process per GPU (torchrun), tensor replicated, no collective
on the data path.  With --gpus N > 1 the default workload is c4: the fixed
500-model 500^3 sweep split into rank-balanced model batches ("scaling":
"strong", widths per rank in ``config``).  ``--config c2`` at N > 1 runs
one c2 batch per rank (weak scaling); ``--config c3`` runs the converging
EEM-shaped sweep with converged-slot refill (r_star = 300).

``--impl reference`` times the reference CPU implementation instead: every
step one full ``cals.run`` of the same workload on all host cores (c4: a
rank-balanced tenth of the sweep, scaled by width -- the full c4 sweep is
~20 TFLOP on the host).
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "models/sec for full CALS sweep (200^3, 200 models, ranks 1-20 x 10, 5 iterations)"

# BASELINE.json configs usable from bench.py.  c2 is the N=1 headline; with
# --gpus N > 1 the default is c4's fixed 500-model sweep split over the ranks
# (strong scaling); c3 is the converging refill sweep.
WORKLOADS = {
    "c2": dict(dims=(200, 200, 200), true_rank=20, ranks=list(range(1, 21)), per_rank=10,
               tol=0.0, iters=5, r_star=2100, shard=False,
               desc="c2: 200x200x200 dense FP64, 200 CP models (ranks 1..20 x 10), tol=0, "
                    "5 iterations per model, r_star=2100"),
    "c3": dict(dims=(250, 251, 21), true_rank=10, ranks=list(range(2, 11)), per_rank=20,
               tol=1e-6, iters=1000, r_star=300, shard=False,
               desc="c3: EEM-shaped 250x251x21, 180 models (ranks 2..10 x 20), tol=1e-6, cap "
                    "1000, r_star=300 (converged-slot refill)"),
    "c4": dict(dims=(500, 500, 500), true_rank=20, ranks=list(range(1, 21)), per_rank=25,
               tol=0.0, iters=5, r_star=None, shard=True,
               desc="c4: 500x500x500 dense FP64, 500 models (ranks 1..20 x 25) split by "
                    "rank-balanced model batches over the GPUs, 5 iterations"),
    # config 5: the tensor itself is sharded on mode 0 (rows split over the
    # ranks, each rank generates only its slab); all-reduce of the partial
    # MTTKRPs of modes 1, 2 and the mode-0 Gramians every iteration
    "c5": dict(dims=(2000, 2000, 1000), true_rank=20, ranks=list(range(1, 21)), per_rank=5,
               tol=0.0, iters=5, r_star=1050, shard=False, mode0=True,
               desc="c5: 2000x2000x1000 dense FP64 (32 GB) sharded on mode 0 over the GPUs "
                    "(per-rank slab generated on the device), 100 models (ranks 1..20 x 5), "
                    "5 iterations, all-reduce of the partial MTTKRPs"),
}


def _env_rank():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))


def _metric(name: str) -> str:
    return METRIC if name == "c2" else \
        f"models/sec for full CALS sweep ({WORKLOADS[name]['desc']})"


def _config(name: str, world: int) -> dict:
    """The ``config`` object -- identical for both arms of the same run."""
    from paper_2010_04678_b200.parallel import shard_widths

    wl = WORKLOADS[name]
    ranks = [r for r in wl["ranks"] for _ in range(wl["per_rank"])]
    c = {"workload": wl["desc"], "dims": list(wl["dims"]),
         "models_total": len(ranks) * (1 if wl["shard"] else world),
         "models_per_gpu": len(ranks) if not wl["shard"] else None,
         "tol": wl["tol"], "max_iterations": wl["iters"],
         "r_star": wl["r_star"],
         "parallelism": (f"model-batch x{world} (rank-balanced snake partition of the fixed "
                         f"sweep), tensor replicated, no collective" if wl["shard"] else
                         f"model-batch x{world} (every rank its own batch), tensor replicated, "
                         f"no collective"),
         "l2": "flushed between steps (256 MiB write)"}
    if wl.get("mode0"):
        from paper_2010_04678_b200.parallel import row_ranges

        c["models_total"] = len(ranks)
        c["models_per_gpu"] = len(ranks)
        c["parallelism"] = (f"mode-0 tensor sharding x{world} (rows {row_ranges(wl['dims'][0], world)}),"
                            f" every rank runs all models on its slab; NCCL all-reduce of the "
                            f"partial MTTKRPs of modes 1, 2 and the mode-0 Gramians per iteration")
        c["data_note"] = ("generate_synthetic's signal factors, noise drawn per 50-row block on "
                          "the device (parallel.synthetic_slab)")
    if wl["shard"]:
        c["widths_per_rank"] = shard_widths(ranks, world)
        c["models_per_rank"] = [len(s) for s in __import__(
            "paper_2010_04678_b200.parallel", fromlist=["x"]).snake_partition(ranks, world)]
        c["r_star"] = "width of the rank's batch"
    return c


# ------------------------------------------------------------------ clocks --
class ClockSampler:
    """SM clock + throttle reasons sampled every 10 ms during the timed region
    (NVML; the recipe's nvidia-smi clocks line is the fallback)."""

    REASONS = {"hw_slowdown": 0x8, "hw_thermal_slowdown": 0x40, "sw_thermal_slowdown": 0x20,
               "sw_power_cap": 0x4}

    def __init__(self, device: int):
        self.device = device
        self.samples = []
        self._stop = threading.Event()
        self._t = None

    def start(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        time.sleep(0.02)
        return self

    def _run(self):
        try:
            import pynvml

            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(self.device)
            mx = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)
            while not self._stop.is_set():
                sm = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
                rs = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
                self.samples.append((float(sm), float(mx), int(rs)))
                self._stop.wait(0.01)
        except Exception:
            q = ("--query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.active")
            while not self._stop.is_set():
                try:
                    out = subprocess.run(["nvidia-smi", "-i", str(self.device), q,
                                          "--format=csv,noheader,nounits"], capture_output=True,
                                         text=True, timeout=5).stdout.strip().split(",")
                    self.samples.append((float(out[0]), float(out[1]), int(out[2].strip(), 16)))
                except Exception:
                    pass
                self._stop.wait(0.1)

    def stop(self) -> dict:
        self._stop.set()
        if self._t:
            self._t.join(timeout=6)
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        reasons = sorted({k for _, _, r in self.samples for k, bit in self.REASONS.items()
                          if r & bit})
        return {"sm_mhz": float(np.median([s[0] for s in self.samples])),
                "sm_max_mhz": max(s[1] for s in self.samples), "reasons": reasons,
                "samples": len(self.samples)}


# --------------------------------------------------------------- reference --
def _reference_module():
    """The unmodified reference package installed in baseline/_ref."""
    path = os.path.join(ROOT, "baseline", "_ref")
    if os.path.isdir(os.path.join(path, "cals")):
        if path not in sys.path:
            sys.path.insert(0, path)
        import cals  # noqa: F401

        return cals, "reference"
    return None, "port"


class _CpuWorkload:
    """The workload's inputs for the host-side arm: the unmodified reference
    (``baseline/_ref``) when installed, else the oracle port."""

    def __init__(self, name: str, world: int = 1):
        from paper_2010_04678_b200.parallel import snake_partition

        self.name = name
        self.wl = wl = WORKLOADS[name]
        self.ref, self.kind = _reference_module()
        if self.ref is not None:
            from cals.io import build_models, generate_synthetic

            self.t = generate_synthetic(wl["dims"], wl["true_rank"], 0.1, seed=0)
            every = build_models(wl["dims"], wl["ranks"], wl["per_rank"], seed=1)
        else:
            from oracle import cals_oracle as O

            self.dims, self.data = O.generate_synthetic(wl["dims"], wl["true_rank"], 0.1, seed=0)
            every = O.build_models(self.dims, wl["ranks"], wl["per_rank"], seed=1)
        rank_of = (lambda m: m.rank) if self.ref is not None else (lambda m: m[1])
        self.total_models = len(every)
        self.total_width = sum(rank_of(m) for m in every)
        self.sampled = False
        if wl["shard"]:
            # c4: the full sweep is ~4 TFLOP per iteration plus a 10.5 GB KRP
            # workspace on the host -- a step is one tenth of it (shard 0 of a
            # 10-way rank-balanced snake partition, every model run its full
            # 5 iterations) and the rate is scaled by the width ratio (MTTKRP
            # cost is linear in W, mttkrp.py:72-76)
            part = snake_partition([rank_of(m) for m in every], 10)[0]
            self.models = [every[i] for i in part]
            self.sampled = True
        else:
            self.models = every
        self.width = sum(rank_of(m) for m in self.models)
        self.r_star = wl["r_star"] or self.width

    def fresh_models(self):
        if self.ref is not None:
            from cals.model import Model

            return [Model(id=m.id, rank=m.rank, factors=[f.copy() for f in m.factors])
                    for m in self.models]
        return [(i, r, [f.copy() for f in fac]) for i, r, fac in self.models]

    def run(self, threads: int, iters: int | None = None) -> float:
        wl = self.wl
        iters = wl["iters"] if iters is None else iters
        models = self.fresh_models()
        if self.ref is not None:
            from cals.als import ConvergenceConfig
            from cals.driver import ExecutionMode, run

            tic = time.perf_counter()
            run(self.t, models, ConvergenceConfig(tol=wl["tol"], max_iterations=iters),
                mode=ExecutionMode.CALS, r_star=self.r_star, threads=threads)
            return time.perf_counter() - tic
        from oracle import cals_oracle as O

        tic = time.perf_counter()
        O.run_cals(self.data, self.dims, models, wl["tol"], iters, self.r_star)
        return time.perf_counter() - tic

    def rate(self, sec: float) -> float:
        """models/s of the whole workload from one timed step."""
        if self.sampled:
            return self.total_models / (sec * self.total_width / self.width)
        return len(self.models) / sec

    def sample_text(self, n_steps: int, sec: float) -> str:
        what = (f"{len(self.models)} of {self.total_models} models (rank-balanced 1/10 share, "
                f"W={self.width} of {self.total_width}), full {self.wl['iters']}-iteration "
                f"sweep, rate scaled by the width ratio" if self.sampled else
                f"the full workload ({len(self.models)} models, "
                f"{'tol ' + str(self.wl['tol']) if self.wl['tol'] > 0 else str(self.wl['iters']) + ' iterations'})")
        return (f"{self.name}: {what}; reference cals.run(mode=CALS, r_star={self.r_star}); "
                f"mean of {n_steps} timed run(s) after a 1-iteration warm-up run, "
                f"{sec:.2f} s per run")


def cpu_sample(name: str, threads: int, steps: int = 2) -> dict:
    """Bounded host-core baseline for the cpu_baseline key (rank 0, N=1)."""
    w = _CpuWorkload(name)
    w.run(threads, iters=1)  # warm-up (first touch of the workspaces), as bench.py:191-195
    secs = [w.run(threads) for _ in range(steps)]
    sec = float(np.mean(secs))
    return {"value": w.rate(sec), "unit": "models/s", "cores": threads, "kind": w.kind,
            "sample": w.sample_text(steps, sec)}


def run_reference_arm(args) -> None:
    """The reference's own CPU implementation, unmodified, through its public
    ``cals.run`` on all host cores: every step is one full sweep of the same
    workload (c2: 200 models x 5 iterations), after ``warmup`` untimed ones."""
    rank, world, _ = _env_rank()
    if rank != 0:
        return
    name = args.config or ("c2" if args.gpus <= 1 else "c4")
    threads = os.cpu_count() or 1
    if WORKLOADS[name].get("mode0"):
        print(json.dumps({"impl": "reference", "unavailable":
                          "c5 needs the 32 GB tensor plus a 33.6 GB Khatri-Rao workspace in host "
                          "memory (SURVEY.md 8(d)); the reference has no sharded path"}),
              flush=True)
        return
    w = _CpuWorkload(name, world)
    w.run(threads, iters=1)
    for _ in range(args.warmup):
        w.run(threads)
    secs = [w.run(threads) for _ in range(args.steps)]
    sec = float(np.mean(secs))
    v = w.rate(sec)
    sample = w.sample_text(args.steps, sec)
    line = {"impl": "reference", "metric": _metric(name), "value": v, "unit": "models/s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": sec * 1e3, "higher_is_better": True,
            "scaling": "strong" if WORKLOADS[name]["shard"] else "weak",
            "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (generate_synthetic noise 0.1 seed 0; build_models seed 1)",
            "config": _config(name, args.gpus),
            "host": {"threads": threads, "impl": "reference CPU path (baseline/_ref, unmodified)"
                     if w.kind == "reference" else "oracle port (reference not installed)",
                     "step_seconds": [round(x, 4) for x in secs]},
            "cpu_baseline": {"value": v, "unit": "models/s", "cores": threads, "kind": w.kind,
                             "sample": sample},
            "e2e": {"value": v, "unit": "models/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# --------------------------------------------------------------- our arm ---
def secondary_sweep(name: str, stream, flush, warmup: int = 1, steps: int = 3) -> dict:
    """A second workload timed beside the headline (default N = 1 run only):
    device-resident sweeps through the same engine path as ``value`` (pool
    re-loaded every step, L2 flushed between steps, CUDA events on the engine
    stream).  Reported under ``secondary`` -- not the headline metric."""
    import torch

    import paper_2010_04678_b200 as cals
    from paper_2010_04678_b200.engine import CalsEngine

    wl = WORKLOADS[name]
    t = cals.generate_synthetic(wl["dims"], wl["true_rank"], 0.1, seed=0)
    models = cals.build_models(wl["dims"], wl["ranks"], wl["per_rank"], seed=1)
    dev_t = t.device()
    eng = CalsEngine(dev_t, wl["r_star"], [m.rank for m in models], trace_capacity=64)
    pool = torch.from_numpy(eng.pack([m.factors for m in models])).cuda()
    sq = t.sqnorm
    iters, launches, times = [], [], []
    for i in range(warmup + steps):
        flush.fill_(float(i))
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        eng.load_pool(pool)
        iters.append(eng.run(wl["tol"], wl["iters"], sq))
        b.record(stream)
        launches.append(eng.last_launches())
        torch.cuda.synchronize()
        if i >= warmup:
            times.append(a.elapsed_time(b))
    res = eng.results(with_pool=False)
    eng.close()
    t.release_device()
    ms = float(np.mean(times))
    return {"metric": _metric(name), "value": len(models) / (ms * 1e-3), "unit": "models/s",
            "ms_per_step": ms, "steps": steps, "warmup": warmup,
            "driver_iterations_per_step": float(np.mean(iters[warmup:])),
            "gpu_launches_per_step": float(np.mean(launches[warmup:])),
            "statuses": {str(k): int(v) for k, v in zip(*np.unique(res.status,
                                                                  return_counts=True))},
            "timing": "device-resident, CUDA events on the engine stream, L2 flushed between "
                      "steps; config " + wl["desc"]}


def main_gpu(args) -> None:
    import ctypes as C

    import torch
    import torch.distributed as dist

    import paper_2010_04678_b200 as cals
    from paper_2010_04678_b200 import _native
    from paper_2010_04678_b200.engine import CalsEngine

    rank, world, local = _env_rank()
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    lib = _native.load()
    stream = torch.cuda.current_stream()
    s = stream.cuda_stream

    name = args.config or ("c2" if world <= 1 else "c4")
    wl = WORKLOADS[name]
    dims = wl["dims"]
    if wl.get("mode0"):
        return main_mode0(args, name, rank, world, local)
    t = cals.generate_synthetic(dims, wl["true_rank"], 0.1, seed=0)
    if wl["shard"]:  # fixed total work split over the ranks (strong scaling)
        from paper_2010_04678_b200.parallel import snake_partition

        every = cals.build_models(dims, wl["ranks"], wl["per_rank"], seed=1)
        models = [every[i] for i in snake_partition([m.rank for m in every], world)[rank]]
        total_models = len(every)
        r_star = max(1, sum(m.rank for m in models))
    else:  # every rank its own batch (weak scaling)
        models = cals.build_models(dims, wl["ranks"], wl["per_rank"], seed=1 + rank)
        total_models = len(models) * world
        r_star = wl["r_star"]
    n_models = len(models)
    dev_t = t.device()
    eng = CalsEngine(dev_t, r_star, [m.rank for m in models], trace_capacity=64)
    pool_host = eng.pack([m.factors for m in models])
    pool_dev = torch.from_numpy(pool_host).cuda()
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
    sq = t.sqnorm

    iters_run, launches_run = [], []

    def step():
        eng.load_pool(pool_dev)
        iters_run.append(eng.run(wl["tol"], wl["iters"], sq))
        launches_run.append(eng.last_launches())

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clocks = ClockSampler(local).start()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(args.steps)]
    torch.cuda.synchronize()
    for i in range(args.steps):
        flush.fill_(float(i))
        ev[i][0].record(stream)
        step()
        ev[i][1].record(stream)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ms = sum(a.elapsed_time(b) for a, b in ev) / args.steps
    clk = clocks.stop()
    res = eng.results(with_pool=False)
    assert (res.status >= 2).all(), "sweep did not complete"
    if wl["tol"] <= 0:
        assert (res.iterations == wl["iters"]).all() and (res.status == 3).all()
    tmax = torch.tensor([ms], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(tmax, op=dist.ReduceOp.MAX)
    ms_max = float(tmax.item())
    value = total_models / (ms_max * 1e-3)
    # our kernels launched inside the timed region, counted by the library for
    # every run (kernel nodes of the captured iteration graph x graph
    # launches + reset / initial plan / move; cals_engine_last_launches)
    gpu_launches = int(sum(launches_run[-args.steps:]))

    # ---- e2e through the public API with host buffers
    from paper_2010_04678_b200.driver import LAST_RUN_PROFILE

    t.pin()  # the step's host input lives in page-locked memory (contract: pinned host buffers)
    e2e_times, phases = [], []
    h2d = t.data.nbytes + pool_host.nbytes
    d2h = pool_host.nbytes + n_models * (4 * 3 + 8 * 3) + 8 * sum(m.rank for m in models)
    n_e2e = max(3, min(args.steps, 10))
    for i in range(args.warmup + n_e2e):
        tt = cals.DenseTensor(dims, t.data)  # fresh tensor: upload inside the timed region
        torch.cuda.synchronize()
        tic = time.perf_counter()
        out = cals.run(tt, models, cals.ConvergenceConfig(tol=wl["tol"],
                                                          max_iterations=wl["iters"]),
                       r_star=r_star)
        torch.cuda.synchronize()
        if i >= args.warmup:
            e2e_times.append(time.perf_counter() - tic)
            phases.append(dict(LAST_RUN_PROFILE))
        tt.release_device()
        assert len(out) == n_models
    e2e_sec = float(np.mean(e2e_times))
    te = torch.tensor([e2e_sec], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
    e2e = {"value": total_models / float(te.item()), "unit": "models/s",
           "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
           "phases_ms": {k: 1e3 * float(np.mean([p[k] for p in phases])) for k in phases[0]},
           "samples_ms": [round(1e3 * x, 3) for x in e2e_times],
           "timing": "wall clock per run() call (mean over the samples), device synchronised "
                     "before and after"}

    # ---- roofline of the fused MTTKRP kernel at the workload's capacity width
    peak = C.c_double()
    _native.call("cals_fp64_peak_probe", s, C.byref(peak))
    peak_i8 = C.c_double()
    _native.call("cals_int8_peak_probe", s, C.byref(peak_i8))
    W = r_star
    fac = [torch.rand((d, W), dtype=torch.float64, device="cuda") for d in dims]
    ptrs = (C.c_void_p * 3)(*[f.data_ptr() for f in fac])
    out_t = torch.empty((max(dims), W), dtype=torch.float64, device="cuda")
    per_mode, kinds, tops = [], [], []
    for n in range(3):
        b = C.c_size_t()
        _native.call("cals_mttkrp_workspace_bytes", dev_t.handle, n, W, C.byref(b))
        kind, ops = C.c_int32(), C.c_double()
        _native.call("cals_mttkrp_kernel_info", dev_t.handle, n, W, C.byref(kind), C.byref(ops))
        kinds.append(int(kind.value))
        tops.append(float(ops.value))
        work = torch.empty(b.value // 8 + 1, dtype=torch.float64, device="cuda")
        args_ = (dev_t.handle, n, W, ptrs, W, out_t.data_ptr(), W, work.data_ptr(), b.value,
                 eng.variant(n)["variant"], s)
        for _ in range(2):
            _native.call("cals_mttkrp", *args_)
        reps = 5
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(reps):
            _native.call("cals_mttkrp", *args_)
        e1.record(stream)
        torch.cuda.synchronize()
        per_mode.append(e0.elapsed_time(e1) / reps)
    flops = 2.0 * W * np.prod(dims)
    fp64_eq = flops / (np.mean(per_mode) * 1e-3) / 1e12
    int8 = all(k == 1 for k in kinds)
    traffic = None
    prof = os.path.join(ROOT, "profiles", "r02_ozaki_ncu.json" if int8 else "r01_mttkrp_ncu.json")
    if os.path.exists(prof):
        try:
            traffic = json.load(open(prof)).get("dram_bytes_per_launch")
        except Exception:
            traffic = None
    if int8:
        # algorithmic INT8 work of one launch: the 28 slice products of the
        # Ozaki scheme over the unpadded contraction, 2 x 28 x W x prod(dims)
        # (the padded tiles the kernel actually issues are reported beside it)
        alg_ops = 2.0 * 28.0 * W * float(np.prod(dims))
        ach = float(np.mean([alg_ops / (t * 1e-3) / 1e12 for t in per_mode]))
        executed = float(np.mean([o / (t * 1e-3) / 1e12 for o, t in zip(tops, per_mode)]))
        roofline = {"bound": "tensor", "achieved": ach, "peak": peak_i8.value, "unit": "TOPS",
                    "frac": ach / peak_i8.value, "traffic": traffic,
                    "kernel": f"mttkrp_ozaki_kernel (INT8 tcgen05, 7x7 Ozaki slices, 28 products) "
                              f"+ Lo slicing + split reduce (cals_mttkrp), W={W}, {name}",
                    "achieved_counts": "algorithmic INT8 ops per launch: 2 x 28 slice products "
                                       "x W x prod(dims) (unpadded)",
                    "executed_tops": executed,
                    "executed_counts": "INT8 ops the kernel issues: 2 x 28 x padded M x W x K "
                                       "tiles per slab (64-row / 128-column / 32-deep tiles)",
                    "peak_source": "cals_int8_peak_probe: tcgen05.mma kind::i8 M128 N256 K32 on "
                                   "all SMs, measured live (MEASURED_PEAKS.json has no INT8 entry)",
                    "fp64_equivalent": {"tflops": fp64_eq, "dmma_peak_tflops": peak.value,
                                        "frac_of_dmma_peak": fp64_eq / peak.value,
                                        "flops_per_launch": flops,
                                        "definition": "2*W*prod(dims) (mttkrp.py:72-76) / time"},
                    "ms_per_launch_by_mode": per_mode}
    else:
        roofline = {"bound": "tensor", "achieved": fp64_eq, "peak": peak.value, "unit": "TFLOP/s",
                    "frac": fp64_eq / peak.value, "traffic": traffic,
                    "kernel": f"mttkrp_dmma_kernel + split_reduce (cals_mttkrp), W={W}, "
                              f"{name} shape",
                    "ms_per_launch_by_mode": per_mode,
                    "peak_source": "cals_fp64_peak_probe: DMMA.8x8x4 all SMs, measured live "
                                   "(MEASURED_PEAKS.json has no FP64 entry)",
                    "flops_per_launch": flops}

    it_mean = float(np.mean(iters_run))
    cfg = _config(name, world)
    details = {"models_this_gpu": n_models, "r_star_this_gpu": r_star,
               "driver_iterations_per_step": it_mean,
               "gpu_launches_per_step": gpu_launches / max(1, args.steps),
               "mttkrp_kernels": {f"mode{n}": ("int8-ozaki" if k == 1 else "fp64-dmma")
                                  for n, k in enumerate(kinds)},
               "tensor_slices": "the INT8 path's tensor slices (a derived format of the "
                                "immutable tensor) are built once per tensor: outside the timed "
                                "steps of `value` (tensor resident), inside every step of `e2e` "
                                "(fresh tensor per run)"}
    if wl["tol"] <= 0:  # reference flop model (driver.py:124-125) over the sweep
        details["sweep_mttkrp_tflops_reference_model"] = 3 * wl["iters"] * 2 * sum(
            m.rank for m in models) * float(np.prod(dims)) * world / (ms_max * 1e-3) / 1e12
    line = {"metric": _metric(name), "value": value, "unit": "models/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_max,
            "higher_is_better": True, "scaling": "strong" if wl["shard"] else "weak",
            "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (generate_synthetic noise 0.1 seed 0; build_models seed "
                    + ("1" if wl["shard"] else "1+rank") + ")",
            "config": cfg, "details": details, "clocks": clk, "e2e": e2e,
            "gpu_launches": gpu_launches, "roofline": roofline}
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_sample(name, os.cpu_count() or 1,
                                          steps=1 if wl["shard"] or wl["tol"] > 0 else 2)
    eng.close()
    if world == 1 and name == "c2" and args.config is None:
        line["secondary"] = {"c3": secondary_sweep("c3", stream, flush)}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def main_mode0(args, name: str, rank: int, world: int, local: int) -> None:
    """Config 5: the tensor sharded on mode 0.  Each rank
    generates its row slab on its GPU, runs every model on it and all-reduces
    the partial MTTKRPs (modes >= 1) and the mode-0 Gramians per driver
    iteration (parallel.drive_mode0_sharded).  `value`: models / s of the
    whole sweep (max over ranks of the device time, CUDA events)."""
    import torch
    import torch.distributed as dist

    import paper_2010_04678_b200 as cals
    from paper_2010_04678_b200.parallel import Mode0Shard, row_ranges, synthetic_slab

    wl = WORKLOADS[name]
    dims = wl["dims"]
    if os.environ.get("CALS_C5_DIMS"):  # down-scaled smoke runs of the c5 harness
        dims = tuple(int(x) for x in os.environ["CALS_C5_DIMS"].split(","))
    stream = torch.cuda.current_stream()
    rows = row_ranges(dims[0], world)[rank]
    tic = time.perf_counter()
    slab, sq = synthetic_slab(dims, rows, wl["true_rank"], 0.1, seed=0, block_rows=50)
    torch.cuda.synchronize()
    t_gen = time.perf_counter() - tic
    models = cals.build_models(dims, wl["ranks"], wl["per_rank"], seed=1)
    W = sum(m.rank for m in models)
    shard = Mode0Shard(slab, rows, dims, models, r_star=W)
    iters_run = []

    def step():
        iters_run.append(shard.sweep(wl["tol"], wl["iters"], sq))

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clocks = ClockSampler(local).start()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(args.steps)]
    for i in range(args.steps):
        ev[i][0].record(stream)
        step()
        ev[i][1].record(stream)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ms = sum(a.elapsed_time(b) for a, b in ev) / args.steps
    clk = clocks.stop()
    tmax = torch.tensor([ms], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(tmax, op=dist.ReduceOp.MAX)
    ms_max = float(tmax.item())
    # e2e: the pool's H2D (starting factors from host memory), the sweep,
    # and the results D2H + gather of the A0 row blocks, wall clock
    host_pool = shard.pool.cpu().pin_memory()
    e2e_times = []
    for _ in range(max(2, min(args.steps, 3))):
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        tic = time.perf_counter()
        shard.pool.copy_(host_pool, non_blocking=True)
        shard.sweep(wl["tol"], wl["iters"], sq)
        out = shard.results()
        torch.cuda.synchronize()
        e2e_times.append(time.perf_counter() - tic)
        assert len(out) == len(models)
    te = torch.tensor([float(np.mean(e2e_times))], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
    flops = 3 * wl["iters"] * 2 * W * float(np.prod(dims))  # driver.py:124-125 model
    line = {"metric": _metric(name), "value": len(models) / (ms_max * 1e-3), "unit": "models/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_max,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic, generated per rank on the device (see config.data_note)",
            "config": _config(name, world), "clocks": clk,
            "details": {"driver_iterations_per_step": float(np.mean(iters_run)),
                        "slab_rows": list(rows), "slab_generation_s": t_gen,
                        "sweep_mttkrp_tflops_reference_model": flops / (ms_max * 1e-3) / 1e12,
                        "allreduce_bytes_per_iteration": 8 * W * (dims[1] + dims[2]) +
                        8 * sum(m.rank ** 2 for m in models)},
            "e2e": {"value": len(models) / float(te.item()), "unit": "models/s",
                    "h2d_bytes_per_step": int(host_pool.numel() * 8),
                    "d2h_bytes_per_step": int(host_pool.numel() * 8),
                    "timing": "wall clock: pool H2D + sweep + results D2H / gather, max over ranks"},
            "gpu_launches": None, "roofline": None}
    if rank == 0:
        print(json.dumps(line), flush=True)
    shard.close()
    if world > 1:
        dist.destroy_process_group()


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--config", default=None, choices=sorted(WORKLOADS),
                    help="default: c2 at --gpus 1, c4 (strong scaling) at --gpus > 1")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference_arm(args)
    else:
        main_gpu(args)


if __name__ == "__main__":
    main()
