#!/usr/bin/env python
"""bench.py -- MSBFM K.u throughput on B200 (BASELINE.json metric).

Workload (BASELINE.json configs[1], largest single-GPU rung): 2D linear
bond-based PD, 4096 x 4096 nodes (2 DOF/node), delta = 3.015 h (M = 3),
micromodulus 9E/(pi t delta^3) with E = t = 1, no constraints, no cracks
(near-surface diagonal correction on 12N-36 rows), fp64, batch of 16 seeded
uniform[-1,1] displacement vectors per step.  One step = one batched
K.u = FastForce::apply + apply_corrections over the 16 vectors.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]

value   : DOF-matvecs/s over the timed steps, inputs resident in HBM
          (4.3 GB per step >> 126 MB L2: no flush needed).
e2e     : the same metric through the public host API pdgpu_matvec_host
          (pinned host u in, host f out, copies inside the timed region).
roofline: the dominant pass (largest share of the step; all three in per_pass),
          algorithmic bytes per launch / its mean CUDA-event duration.
configs : secondary BASELINE numbers -- CG solve times (configs 1, 3, 4) and
          the 3D K.u rate (config 4, 128^3) -- skipped with --no-extra.
cpu_baseline: the reference's own FastForce::apply + apply_corrections
          (oracle/_ref, headers compiled unmodified) on the host cores,
          bounded sample.  --impl reference prints that arm alone.
N > 1 (torchrun): the same 4096^2 x 16 lattice split into row slabs, one
          libpdgpu engine per rank with the library's own NCCL halo exchange
          (strong scaling, BASELINE configs[1]); time = max over ranks.
          --shard vectors instead gives every rank its own batch (replicas).
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

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

N_SIDE = 4096
BATCH = 16
DIM = 2
M = 3
METRIC = "DOF-matvecs/sec of MSBFM K·u (fp64)"
UNIT = "DOF-matvecs/s"


def workload_config(n_gpus: int):
    return {"workload": f"2D MSBFM K·u, {N_SIDE}x{N_SIDE} nodes, batch {BATCH} (BASELINE configs[1] top rung)",
            "grid": [N_SIDE, N_SIDE], "dof_per_node": DIM, "batch": BATCH, "delta_over_h": 3.015, "M": M,
            "E": 1.0, "thickness": 1.0, "corrections": "surface diagonal (12N-36 rows), no cracks",
            "embedding": "periodic P = N per axis + wrap correction (PDGPU_EMBED=padded: P = 2N)", "l2": "inputs 4.3 GB per step > L2, no flush",
            "parallelism": f"{n_gpus} ranks x own batch (replicas, no data-path collective)" if n_gpus > 1
            else "single GPU (N > 1: the same lattice in row slabs, strong scaling)"}


# ----------------------------------------------------------------- clocks --
class ClockSampler:
    """nvidia-smi -lms 100 streamed during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.idx = gpu_index
        self.samples = []
        self.proc = None
        self.thread = None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.idx), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
            return
        self.thread = threading.Thread(target=self._read, daemon=True)
        self.thread.start()
        time.sleep(0.3)  # first sample lands before the timed region

    def _read(self):
        for line in self.proc.stdout:
            vals = [v.strip() for v in line.strip().split(",")]
            if len(vals) >= 6:
                self.samples.append(vals)

    def stop(self):
        if self.proc:
            time.sleep(0.15)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
        if self.thread:
            self.thread.join(timeout=5)
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}

        def num(x):
            try:
                return float(x)
            except ValueError:
                return None

        sm = [v for v in (num(s[0]) for s in self.samples) if v is not None]
        mx = [v for v in (num(s[1]) for s in self.samples) if v is not None]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4) if s[2 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples)}


# ----------------------------------------------------------- peaks / bytes --
def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


def pass_algorithmic_bytes(n_side: int, batch: int, periodic: bool):
    """Algorithmic HBM bytes per launch of each 2D pass (SURVEY.md 8(d) pass
    model, with the transform geometry of the embedding in use):
      K1: read u (8 B per node-component), write the half spectrum
          (16 B x Hx x Ny per component);
      K3: read + write the half spectrum, read the real symbol once per launch
          (n_pairs x Hx x Py doubles);
      K5: read the half spectrum, write f.
    Padded (P = 2N, the reference's PadTransform): Hx = N + 1, Py = 2N --
    80 B/DOF/vector + 48N B symbol.  Periodic (P = N): Hx = N/2 + 1, Py = N --
    48 B/DOF/vector + 12N B symbol."""
    n = n_side * n_side
    hx = (n_side // 2 + 1) if periodic else (n_side + 1)
    py = n_side if periodic else 2 * n_side
    spec = DIM * hx * n_side * 16
    return {"K1_rfft_x": batch * (8 * DIM * n + spec),
            "K3_spectral": batch * 2 * spec + 3 * hx * py * 8,
            "K5_irfft_x": batch * (spec + 8 * DIM * n)}


def pass_algorithmic_bytes_3d(n: int, batch: int, n_pairs: int = 6):
    """3D periodic pass model (P = N on every axis, R2C along x: Hx = N/2 + 1):
    K1 reads u (8 B per node-component) and writes S1 = d*Nz*Hx*Ny complex; K2
    (y) reads S1 and writes S2 = d*Hx*Ny*Nz; K3 (z, symbol, inverse z) reads
    and writes S2 plus the real symbol once per launch (n_pairs*Hx*Ny*Nz
    doubles); K4 reads S2, writes S1; K5 reads S1 and writes f."""
    d = 3
    nodes = n ** 3
    hx = n // 2 + 1
    spec = d * hx * n * n * 16
    field = d * nodes * 8
    return {"K1_rfft_x": batch * (field + spec), "K2_fft_y": batch * 2 * spec,
            "K3_spectral": batch * 2 * spec + n_pairs * hx * n * n * 8, "K4_ifft_y": batch * 2 * spec,
            "K5_irfft_x": batch * (spec + field)}


# ------------------------------------------------------------------ CPU leg --
def _mem_available_bytes():
    try:
        with open("/proc/meminfo") as f:
            for line in f:
                if line.startswith("MemAvailable:"):
                    return int(line.split()[1]) * 1024
    except Exception:
        pass
    return 16 << 30


def cpu_threads_for(n_side):
    # one reference FastForce holds (n_pairs + d + 2) padded complex grids (convolution.hpp:263-266)
    footprint = (3 + DIM + 2) * (2 * n_side) ** 2 * 16 + 4 * DIM * n_side * n_side * 8
    cores = os.cpu_count() or 1
    return max(1, min(cores, int(0.6 * _mem_available_bytes() // footprint))), cores


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


CPU_BUILD = ("reference headers (proj/include/pdfast, unmodified) compiled g++ -O3 -ffp-contract=off against "
             "oracle/fftw_cpu (our radix-2/4 Stockham stand-in for the 10 FFTW3 symbols the reference calls; FFTW3 "
             "is absent from the image and unpinned by the reference)")


def cpu_reference_sample(n_side, steps=3, budget_s=150.0):
    """Time the reference path (oracle/_ref) on host cores: each step one
    vector per thread, independent FastForce instances (convolution.hpp:53-54);
    median over the steps that fit in the wall budget (at least one)."""
    import numpy as np
    from oracle import oracle as orc
    if not orc.ref_available():
        return None
    threads, cores = cpu_threads_for(n_side)
    h = 1.0 / n_side
    r = orc.RefProblem((n_side, n_side), h=h, delta=3.015 * h, M=M, E=1.0, thickness=1.0)
    r.finalize()
    rng = np.random.default_rng(1234)
    u = rng.uniform(-1.0, 1.0, size=(threads, DIM, n_side * n_side))
    times = []
    t_start = time.time()
    for _ in range(steps):
        times.append(r.bench(u, threads))
        if time.time() - t_start > budget_s:
            break
    per_step = statistics.median(times)
    value = threads * DIM * n_side * n_side / per_step
    return {"value": value, "unit": UNIT, "cores": threads, "host_cores": cores, "cpu_model": cpu_model(),
            "kind": "reference",
            "sample": f"{threads} of the {BATCH} vectors per step ({threads} threads x 1 vector, one FastForce each; "
                      f"thread count capped by host memory, 7.5 GB per 4096^2 instance), {len(times)} step(s), "
                      f"median {per_step:.2f} s (all: {', '.join(f'{t:.2f}' for t in times)})",
            "build": CPU_BUILD, "steps_timed": len(times), "s_per_step": per_step}


def cpu_reference_cg_config1():
    """CG on BASELINE config 1 (128^2, clamped delta layers, tol 1e-10) over the
    reference's own mat-vec (FastForce::apply + apply_corrections, oracle/_ref;
    the CG loop itself is the restated Hestenes-Stiefel of SURVEY 8(c): the
    reference has no CG), single host thread."""
    import numpy as np
    from oracle import oracle as orc
    if not orc.ref_available():
        return None
    n = 128
    h = 1.0 / n
    r = orc.RefProblem((n, n), h=h, delta=3.015 * h, M=M, E=1.0, thickness=1.0)
    for lo, hi in clamp_boxes(2, 3.015 * h):
        r.add_constraint(lo, hi, 3)
    r.finalize()
    b = orc.random_field(orc.Rng(1001), 2, n * n)
    t0 = time.perf_counter()
    _, it, rel, _ = r.cg(b, tol=1e-10, maxit=20000)
    return {"grid": [n, n], "tol": 1e-10, "iterations": it, "relres": rel,
            "solve_s": time.perf_counter() - t0, "threads": 1, "kind": "reference mat-vec + restated CG"}


def run_reference_arm(args):
    from paper_2301_11828_b200 import dist as D
    rank, world, _ = D.env()
    if rank != 0:
        return 0
    res = cpu_reference_sample(N_SIDE, steps=max(args.steps, 1), budget_s=args.ref_budget)
    if res is None:
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libpdref.so not built"}))
        return 0
    line = {"metric": METRIC, "value": res["value"], "unit": UNIT, "n_gpus": args.gpus, "steps": res["steps_timed"],
            "warmup": 0, "ms_per_step": res["s_per_step"] * 1e3, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic", "impl": "reference",
            "config": workload_config(1),
            "cpu_baseline": {k: res[k] for k in ("value", "unit", "cores", "host_cores", "cpu_model", "kind", "sample",
                                                 "build")},
            "e2e": {"value": res["value"], "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "note": "reference arm: the reference's own CPU path; warm-up steps skipped (no caches/JIT to warm), "
                    "timed steps capped by a wall budget"}
    print(json.dumps(line))
    return 0


# -------------------------------------------------------- secondary configs --
def clamp_boxes(dim, dl):
    out = []
    for ax in range(dim):
        lo0, hi0 = [0.0] * dim, [1.0] * dim
        hi0[ax] = dl
        lo1, hi1 = [0.0] * dim, [1.0] * dim
        lo1[ax] = 1.0 - dl
        out += [(lo0, hi0), (lo1, hi1)]
    return out


def extra_configs(device, stream):
    """CG solve times (configs 1, 3, 4), the 3D K.u rate (config 4, 128^3 and 256^3), the
    config-2 sweep (512^2 .. 2048^2, batch 16) and the VV step (config 5), device-resident."""
    import torch
    from paper_2301_11828_b200 import FastForce, build_kernel
    out = {}

    def engine(dims, constraints):
        dim = len(dims)
        h = 1.0 / dims[0]
        ff = FastForce(dims, M, build_kernel(dim, h, 3.015 * h, M, 1.0, 1.0), device=device)
        ff.set_geometry(h, [0.0] * dim, 3.015 * h, 1.0)
        for lo, hi, mask, value in constraints:
            ff.add_constraint(lo, hi, mask, 0, value)
        return ff

    def timed(fn):
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        ev0.record(stream)
        r = fn()
        ev1.record(stream)
        torch.cuda.synchronize()
        return ev0.elapsed_time(ev1), r

    g = torch.Generator(device="cuda")
    # config 1: 128^2, clamped delta layers, CG to 1e-10
    dims = (128, 128)
    dl = 3.015 / 128
    ff = engine(dims, [(lo, hi, 3, 0.0) for lo, hi in clamp_boxes(2, dl)])
    b = torch.empty((2, 128 * 128), dtype=torch.float64, device="cuda").uniform_(-1, 1, generator=g.manual_seed(1001))
    x = torch.empty_like(b)
    ff.cg_solve_device(b, x, tol=1e-10, maxit=20000, stream=stream)  # warm
    ms, (it, rel) = timed(lambda: ff.cg_solve_device(b, x, tol=1e-10, maxit=20000, stream=stream))
    out["config1_cg"] = {"grid": [128, 128], "tol": 1e-10, "iterations": it, "relres": rel, "solve_ms": ms}
    ff.cg_operator("direct")  # the same K summed directly (comparison point, not the MSBFM metric)
    ff.cg_solve_device(b, x, tol=1e-10, maxit=20000, stream=stream)
    ms, (it, rel) = timed(lambda: ff.cg_solve_device(b, x, tol=1e-10, maxit=20000, stream=stream))
    out["config1_cg_direct_operator"] = {"iterations": it, "relres": rel, "solve_ms": ms,
                                         "what": "CG with the direct stencil sum of K (pdgpu_set_cg_operator)"}
    ff.close()
    # config 3: 1024^2, centre crack L/2, +-1e-3 on top/bottom layers (u_y), CG to 1e-10
    n = 1024
    dl = 3.015 / n
    cons = [((0.0, 1.0 - dl), (1.0, 1.0), 0b01, 0.0), ((0.0, 1.0 - dl), (1.0, 1.0), 0b10, 1e-3),
            ((0.0, 0.0), (1.0, dl), 0b01, 0.0), ((0.0, 0.0), (1.0, dl), 0b10, -1e-3)]
    ff = engine((n, n), cons)
    bonds = ff.seed_segment((0.25, 0.5), (0.75, 0.5))
    b = torch.zeros((2, n * n), dtype=torch.float64, device="cuda")
    x = torch.empty_like(b)
    ms, (it, rel) = timed(lambda: ff.cg_solve_device(b, x, tol=1e-10, maxit=50000, stream=stream))
    out["config3_cg"] = {"grid": [n, n], "crack_bonds": bonds, "tol": 1e-10, "iterations": it, "relres": rel,
                         "solve_ms": ms}
    ff.cg_operator("direct")
    ms, (it, rel) = timed(lambda: ff.cg_solve_device(b, x, tol=1e-10, maxit=50000, stream=stream))
    out["config3_cg_direct_operator"] = {"iterations": it, "relres": rel, "solve_ms": ms,
                                         "what": "CG with the direct stencil sum of K (pdgpu_set_cg_operator)"}
    ff.close()
    # config 4: 128^3 clamped cube; K.u rate and CG to 1e-9
    n = 128
    dl = 3.015 / n
    ff = engine((n, n, n), [(lo, hi, 7, 0.0) for lo, hi in clamp_boxes(3, dl)])
    u = torch.empty((3, n ** 3), dtype=torch.float64, device="cuda").uniform_(-1, 1, generator=g.manual_seed(4000))
    f = torch.empty_like(u)
    for _ in range(3):
        ff.matvec_device(u, f, 1, stream)
    reps = 20
    ms, _ = timed(lambda: [ff.matvec_device(u, f, 1, stream) for _ in range(reps)])
    out["config4_matvec"] = {"grid": [n, n, n], "value": 3 * n ** 3 / (ms / reps * 1e-3), "unit": UNIT,
                             "ms_per_matvec": ms / reps}
    b = torch.empty((3, n ** 3), dtype=torch.float64, device="cuda").uniform_(-1, 1, generator=g.manual_seed(4001))
    x = torch.empty_like(b)
    ms, (it, rel) = timed(lambda: ff.cg_solve_device(b, x, tol=1e-9, maxit=20000, stream=stream))
    out["config4_cg"] = {"grid": [n, n, n], "tol": 1e-9, "iterations": it, "relres": rel, "solve_ms": ms}
    ff.close()
    del u, f, b, x
    # config 4, 256^3 rung: K.u rate on one GPU
    n = 256
    dl = 3.015 / n
    ff = engine((n, n, n), [(lo, hi, 7, 0.0) for lo, hi in clamp_boxes(3, dl)])
    u = torch.empty((3, n ** 3), dtype=torch.float64, device="cuda").uniform_(-1, 1, generator=g.manual_seed(4002))
    f = torch.empty_like(u)
    for _ in range(3):
        ff.matvec_device(u, f, 1, stream)
    reps = 10
    ms, _ = timed(lambda: [ff.matvec_device(u, f, 1, stream) for _ in range(reps)])
    # per-pass breakdown in a separate run: the event brackets must not sit
    # inside the region the mat-vec rate is taken from
    ff.timing_read()
    ff.timing(True)
    timed(lambda: [ff.matvec_device(u, f, 1, stream) for _ in range(reps)])
    passes = ff.timing_read()
    ff.timing(False)
    peak, peak_src = measured_peaks()
    pb = pass_algorithmic_bytes_3d(n, 1)
    per_pass = {}
    for k, b in pb.items():
        ms_k, n_k = passes.get(k, (0.0, 0))
        avg = ms_k / max(n_k, 1)
        per_pass[k] = {"algorithmic_bytes_per_launch": b, "mean_launch_ms": avg,
                       "achieved_gbs": b / (avg * 1e-3) / 1e9 if avg else None,
                       "frac": b / (avg * 1e-3) / 1e9 / peak if avg else None}
    dom = max(per_pass, key=lambda k: per_pass[k]["mean_launch_ms"])
    tot = sum(pb.values())
    mv_gbs = tot / (ms / reps * 1e-3) / 1e9
    out["config4_matvec_256"] = {
        "grid": [n, n, n], "value": 3 * n ** 3 / (ms / reps * 1e-3), "unit": UNIT, "ms_per_matvec": ms / reps,
        "roofline": {"bound": "hbm", "kernel": dom, "achieved": per_pass[dom]["achieved_gbs"], "peak": peak,
                     "unit": "GB/s", "frac": per_pass[dom]["frac"], "peak_source": peak_src, "per_pass": per_pass,
                     "passes_ms_per_matvec": {k: v[0] / reps for k, v in passes.items()},
                     "matvec": {"algorithmic_bytes": tot, "achieved_gbs": mv_gbs, "frac": mv_gbs / peak,
                                "model": "periodic 3D pass model (bench.pass_algorithmic_bytes_3d), batch 1"}}}
    ff.close()
    del u, f
    # config 2 sweep (512^2 .. 2048^2, batch 16, no constraints); 4096^2 is the headline line
    sweep = {}
    for n in (512, 1024, 2048):
        ff = engine((n, n), [])
        u = torch.empty((BATCH, 2, n * n), dtype=torch.float64, device="cuda").uniform_(
            -1, 1, generator=g.manual_seed(2000 + n))
        f = torch.empty_like(u)
        for _ in range(3):
            ff.matvec_device(u, f, BATCH, stream)
        reps = 10
        ms, _ = timed(lambda: [ff.matvec_device(u, f, BATCH, stream) for _ in range(reps)])
        sweep[f"{n}x{n}"] = {"ms_per_step": ms / reps, "value": BATCH * 2 * n * n / (ms / reps * 1e-3), "unit": UNIT}
        ff.close()
        del u, f
    out["config2_sweep_b16"] = sweep
    # config 5: 2048^2 notch, velocity-driven top/bottom layers, VV with bond breaking (s0 = 1e-3)
    import numpy as np
    n = 2048
    h = 1.0 / n
    dl = 3.015 * h
    K = build_kernel(2, h, dl, M, 1.0, 1.0)
    lam = max(sum(2.0 * np.abs(K[0 if (a, b) == (0, 0) else (1 if a != b else 2)]).sum() for b in range(2))
              for a in range(2))
    dt = 0.8 * 2.0 * (1.0 / lam) ** 0.5  # Gershgorin bound of adr_mass, rho = 1
    ff = FastForce((n, n), M, K, device=device)
    ff.set_geometry(h, [0.0, 0.0], dl, 1.0)
    ff.add_constraint((0.0, 1.0 - dl), (1.0, 1.0), 0b10, 1, 1e-4)
    ff.add_constraint((0.0, 0.0), (1.0, dl), 0b10, 1, -1e-4)
    bonds = ff.seed_segment((0.0, 0.5), (0.25, 0.5))
    ff.sim_init(dt)
    # the full 2000-step run: the tensile wave reaches the notch after ~1150
    # steps and the crack then grows (tools/crack_scan.py: +-1e-4 grows it,
    # +-1e-3 and 1e-4 per step tear the loaded layers off instead)
    steps, chunk = 2000, 100
    hist = []

    def run():
        for _ in range(steps // chunk):
            hist.append(int(ff.sim_step(chunk, 1e-3)))
        return sum(hist)

    ms, broken = timed(run)
    pairs = ff.ledger_pairs()
    xm = ((pairs[:, 0] % n) + (pairs[:, 1] % n)) * 0.5 * h
    ym = ((pairs[:, 0] // n) + (pairs[:, 1] // n)) * 0.5 * h
    mid = np.abs(ym - 0.5) < 0.05
    act = [i for i, c in enumerate(hist) if c]
    out["config5_vv"] = {"grid": [n, n], "notch_bonds": bonds, "dt": dt, "s0": 1e-3, "steps": steps,
                         "ms_per_step": ms / steps, "bonds_broken": broken, "broken_per_100_steps": hist,
                         "ms_per_step_while_breaking": None,
                         "crack_tip_x": float(xm[mid].max()) if mid.any() else None, "notch_tip_x": 0.25,
                         "finite": ff.sim_finite(),
                         "note": "velocity BC +-1e-4 on the top/bottom delta layers; stretch test and CSR "
                                 "append every step; one host read-back per 100 steps (break count)"}
    if act:  # re-time the breaking phase alone: restart and run to the first breaking chunk, then time the rest
        ff.close()
        ff = FastForce((n, n), M, K, device=device)
        ff.set_geometry(h, [0.0, 0.0], dl, 1.0)
        ff.add_constraint((0.0, 1.0 - dl), (1.0, 1.0), 0b10, 1, 1e-4)
        ff.add_constraint((0.0, 0.0), (1.0, dl), 0b10, 1, -1e-4)
        ff.seed_segment((0.0, 0.5), (0.25, 0.5))
        ff.sim_init(dt)
        ff.sim_step(act[0] * chunk, 1e-3)
        rest = steps - act[0] * chunk
        ms2, _ = timed(lambda: ff.sim_step(rest, 1e-3))
        out["config5_vv"]["ms_per_step_while_breaking"] = ms2 / rest
    ff.close()
    return out


# -------------------------------------------------------------------- main --
def run_transpose(args):
    """The all-to-all distributed-FFT arm (SURVEY.md 8e comparison, opt-in:
    --shard transpose): rank r holds rows and half-spectrum columns of the
    BATCH x N^2 lattice (pdgpu_set_transpose), two NCCL all-to-all transposes
    of the spectrum and the ring halo per K.u (csrc/transpose.cu, comm.cpp).
    Timed like the slab arm: barrier + synchronize, CUDA events, max over ranks."""
    import torch
    import torch.distributed as tdist
    from paper_2301_11828_b200 import FastForce, build_kernel
    from paper_2301_11828_b200 import dist as D
    from paper_2301_11828_b200.engine import transpose_splits

    os.environ.setdefault("NCCL_DEBUG", "INFO")
    os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    rank, world, local = D.env()
    torch.cuda.set_device(local)
    D.init("nccl", torch.device("cuda", local))
    h = 1.0 / N_SIDE
    K = build_kernel(DIM, h, 3.015 * h, M, 1.0, 1.0)
    rb, cb = transpose_splits(N_SIDE, N_SIDE, world)
    R = rb[rank + 1] - rb[rank]
    ff = FastForce((N_SIDE, R), M, K, device=local)
    ff.set_geometry(h, [0.0, rb[rank] * h], 3.015 * h, 1.0)
    ff.set_transpose(world, rank, N_SIDE, rb, cb)
    if world > 1:
        uid = [ff.comm_unique_id() if rank == 0 else None]
        if tdist.is_initialized():
            tdist.broadcast_object_list(uid, src=0)
        ff.comm_init(world, rank, uid[0])
    stream = torch.cuda.Stream()
    gen = torch.Generator(device="cuda").manual_seed(D.vector_seed(2000, 0) + rank)
    u = torch.empty((BATCH, DIM, R * N_SIDE), dtype=torch.float64, device="cuda")
    u.uniform_(-1.0, 1.0, generator=gen)
    f = torch.empty_like(u)
    for _ in range(args.warmup):
        ff.matvec_device(u, f, BATCH, stream)
    torch.cuda.synchronize()
    ff.timing_read()
    ff.timing(True)
    launches0 = ff.launch_count()
    clk = ClockSampler(local)
    clk.start()
    D.barrier()
    torch.cuda.synchronize()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    for _ in range(args.steps):
        ff.matvec_device(u, f, BATCH, stream)
    ev1.record(stream)
    torch.cuda.synchronize()
    D.barrier()
    clocks = clk.stop()
    ms_step = D.max_over_ranks(ev0.elapsed_time(ev1), "cuda") / args.steps
    passes = ff.timing_read()
    ff.timing(False)
    assert torch.isfinite(f).all().item(), "non-finite K.u"
    hx = N_SIDE // 2 + 1
    share = BATCH * DIM * hx * (N_SIDE // world) * 16
    line = {"metric": METRIC, "value": BATCH * DIM * N_SIDE * N_SIDE / (ms_step * 1e-3), "unit": UNIT,
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded uniform[-1,1], torch Philox)",
            "config": dict(workload_config(world), parallelism=f"{world} ranks: all-to-all distributed FFT "
                                                               "(two spectrum transposes + ring halo per K.u)"),
            "transpose": {"bytes_sent_per_rank_per_step": 2 * share * (world - 1) / world,
                          "passes_ms_per_step": {k: v[0] / args.steps for k, v in passes.items()}},
            "gpu_launches": ff.launch_count() - launches0, "clocks": clocks}
    if rank == 0:
        print(json.dumps(line), flush=True)
    ff.close()
    D.finalize()


def run_slab(args):
    """Strong scaling of the BATCH x N^2 lattice over the ranks (BASELINE
    configs[1]: "the 4096^2 grid is slab-sharded across 2/4/8 GPUs"): row
    slabs of the halo decomposition (paper_2301_11828_b200/slab.py), each rank
    one libpdgpu engine with the library's NCCL halo exchange (csrc/comm.cpp:
    M rows per interior face per vector, packed and sent on a side stream
    while K1..K5 run).  Timed like the single-GPU line: barrier + synchronize
    on both sides, CUDA events on the launching stream, max over ranks."""
    import torch
    from paper_2301_11828_b200 import build_kernel
    from paper_2301_11828_b200 import dist as D
    from paper_2301_11828_b200.slab import SlabForce

    os.environ.setdefault("NCCL_DEBUG", "INFO")
    os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    rank, world, local = D.env()
    torch.cuda.set_device(local)
    D.init("nccl", torch.device("cuda", local))
    n = N_SIDE * N_SIDE
    h = 1.0 / N_SIDE
    K = build_kernel(DIM, h, 3.015 * h, M, 1.0, 1.0)
    sf = SlabForce((N_SIDE, N_SIDE), M, K, rank=rank, world=world, device=torch.device("cuda", local))
    sf.set_geometry(h, None, 3.015 * h, 1.0)
    ff = sf.eng
    stream = torch.cuda.Stream()
    gen = torch.Generator(device="cuda").manual_seed(D.vector_seed(2000, 0) + rank)
    u = torch.empty((BATCH, DIM, sf.n_owned), dtype=torch.float64, device="cuda")
    u.uniform_(-1.0, 1.0, generator=gen)
    f = torch.empty_like(u)
    with torch.cuda.stream(stream):
        for _ in range(args.warmup):
            sf.matvec(u, f)
    torch.cuda.synchronize()
    ff.timing_read()
    ff.timing(True)
    launches0 = ff.launch_count()
    clk = ClockSampler(local)
    clk.start()
    D.barrier()
    torch.cuda.synchronize()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    with torch.cuda.stream(stream):
        for _ in range(args.steps):
            sf.matvec(u, f)
    ev1.record(stream)
    torch.cuda.synchronize()
    D.barrier()
    clocks = clk.stop()
    ms_step = D.max_over_ranks(ev0.elapsed_time(ev1), "cuda") / args.steps
    launches = ff.launch_count() - launches0
    passes = ff.timing_read()
    ff.timing(False)
    assert torch.isfinite(f).all().item(), "non-finite K.u"
    value = BATCH * DIM * n / (ms_step * 1e-3)
    halo_bytes = (2 * (sf.gl > 0) + 2 * (sf.gh > 0)) * M * N_SIDE * DIM * 8 * BATCH  # sent + received

    # roofline of this rank's slab (its own lattice: Nx x R rows)
    peak, peak_src = measured_peaks()
    periodic = ff.embedding() == 3
    R = sf.R
    hx = (N_SIDE // 2 + 1) if periodic else (N_SIDE + 1)
    py = R if periodic else 2 * R
    spec = DIM * hx * R * 16
    own = DIM * N_SIDE * R * 8
    sym = min(3 * hx * py * 8, ff.symbol_stream_bytes())  # the symbol bytes K3 streams (full table or mirror planes)
    pbytes = {"K1_rfft_x": BATCH * (own + spec), "K3_spectral": BATCH * 2 * spec + sym,
              "K5_irfft_x": BATCH * (spec + own)}
    per_pass = {}
    for k, b in pbytes.items():
        ms_k, n_k = passes.get(k, (0.0, 0))
        avg = ms_k / max(n_k, 1)
        per_pass[k] = {"algorithmic_bytes_per_launch": b, "mean_launch_ms": avg,
                       "achieved_gbs": b / (avg * 1e-3) / 1e9 if avg else None,
                       "frac": b / (avg * 1e-3) / 1e9 / peak if avg else None}
    dom = max(per_pass, key=lambda k: per_pass[k]["mean_launch_ms"])
    halo_ms, halo_n = passes.get("halo_exchange", (0.0, 0))
    roofline = {"bound": "hbm", "kernel": dom, "achieved": per_pass[dom]["achieved_gbs"], "peak": peak,
                "unit": "GB/s", "frac": per_pass[dom]["frac"], "traffic": None, "peak_source": peak_src,
                "rank": rank, "slab_rows": R, "per_pass": per_pass,
                "passes_ms_per_step": {k: v[0] / args.steps for k, v in passes.items()},
                "halo": {"bytes_per_rank_per_step": halo_bytes,
                         "comm_stream_ms_per_step": halo_ms / args.steps if halo_n else 0.0,
                         "gbs": (halo_bytes / (halo_ms / args.steps * 1e-3) / 1e9) if halo_n and halo_ms else None,
                         "overlapped_with": "K1..K5 (K6w waits for it)"}}

    # end to end through the public host API: this rank's owned rows from pinned host memory
    e2e = None
    if not args.no_e2e:
        uh = torch.empty((BATCH, DIM, sf.n_owned), dtype=torch.float64, pin_memory=True)
        uh.copy_(u)
        fh = torch.empty_like(uh, pin_memory=True)
        ff.matvec(uh.numpy(), out=fh.numpy())
        e2e_steps = max(1, min(args.steps, 3))
        D.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(e2e_steps):
            ff.matvec(uh.numpy(), out=fh.numpy())
        torch.cuda.synchronize()
        e2e_s = D.max_over_ranks((time.perf_counter() - t0) / e2e_steps, "cuda")
        nbytes = BATCH * DIM * n * 8
        e2e = {"value": BATCH * DIM * n / e2e_s, "unit": UNIT, "h2d_bytes_per_step": nbytes,
               "d2h_bytes_per_step": nbytes, "steps": e2e_steps, "ms_per_step": e2e_s * 1e3,
               "api": "pdgpu_matvec_host on every rank (its pinned host rows in, host f out; NCCL halo inside)"}
        del uh, fh
    cpu = None
    if rank == 0 and not args.no_cpu:
        try:
            cpu = cpu_reference_sample(N_SIDE, steps=3, budget_s=45.0)
            if cpu:
                cpu = {k: cpu[k] for k in ("value", "unit", "cores", "host_cores", "cpu_model", "kind", "sample",
                                           "build")}
        except Exception as exc:
            cpu = {"error": str(exc)[:200]}
    D.barrier()
    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
                "scaling": "strong", "vs_baseline": None, "dtype": "f64",
                "data": "synthetic (seeded uniform[-1,1], torch Philox)",
                "config": dict(workload_config(world),
                               parallelism=f"{world} row slabs + {M}-row halo (library NCCL send/recv, overlapped "
                                           f"with K1..K5)", halo=sf.halo, transport=sf.transport,
                               engine_rows=sf.L, embedding_bits=ff.embedding()),
                "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e,
                "gpu_launches": launches, "clocks": clocks,
                "nccl": {"nranks": world, "comm": "pdgpu_comm_init (ncclCommInitRank)",
                         "collectives": "grouped ncclSend/ncclRecv of the halo rows per K.u"}}
        print(json.dumps(line))
    ff.close()
    D.finalize()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--n", type=int, default=N_SIDE)
    ap.add_argument("--batch", type=int, default=BATCH)
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-extra", action="store_true", help="skip the secondary configs")
    ap.add_argument("--ref-budget", type=float, default=150.0)
    ap.add_argument("--slab-single", action="store_true",
                    help="run the slab arm (NCCL engine transport, one rank) at N = 1 too")
    ap.add_argument("--shard", default="slab", choices=["vectors", "slab", "transpose"],
                    help="N>1: slab = the one lattice split into row slabs with the M-row NCCL halo exchange "
                         "(strong scaling, BASELINE configs[1], default); vectors = every rank its own batch "
                         "(replicas, weak)")
    args = ap.parse_args()
    globals()["N_SIDE"] = args.n
    globals()["BATCH"] = args.batch
    if args.impl == "reference":
        return run_reference_arm(args)
    from paper_2301_11828_b200 import dist as D0
    if args.shard == "transpose":
        return run_transpose(args)
    if args.shard == "slab" and (D0.env()[1] > 1 or args.slab_single):
        return run_slab(args)

    import torch
    from paper_2301_11828_b200 import FastForce, build_kernel
    from paper_2301_11828_b200 import dist as D

    rank, world, local = D.env()
    torch.cuda.set_device(local)
    D.init("nccl", torch.device("cuda", local))

    n = N_SIDE * N_SIDE
    h = 1.0 / N_SIDE
    K = build_kernel(DIM, h, 3.015 * h, M, 1.0, 1.0)
    ff = FastForce((N_SIDE, N_SIDE), M, K, device=local)
    ff.set_geometry(h, [0.0, 0.0], 3.015 * h, 1.0)

    stream = torch.cuda.Stream()
    lo, _ = D.vector_range(BATCH, rank, world)
    gen = torch.Generator(device="cuda").manual_seed(D.vector_seed(2000, lo))
    u = torch.empty((BATCH, DIM, n), dtype=torch.float64, device="cuda")
    u.uniform_(-1.0, 1.0, generator=gen)
    f = torch.empty_like(u)
    torch.cuda.synchronize()

    def step():
        ff.matvec_device(u, f, BATCH, stream)

    with torch.cuda.stream(stream):
        for _ in range(args.warmup):
            step()
    torch.cuda.synchronize()
    ff.timing_read()  # discard warm-up marks
    ff.timing(True)
    launches0 = ff.launch_count()
    clk = ClockSampler(local)
    clk.start()
    D.barrier()
    torch.cuda.synchronize()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    for _ in range(args.steps):
        step()
    ev1.record(stream)
    torch.cuda.synchronize()
    D.barrier()
    clocks = clk.stop()
    ms_total = D.max_over_ranks(ev0.elapsed_time(ev1), "cuda")
    launches = ff.launch_count() - launches0
    passes = ff.timing_read()
    ff.timing(False)
    ms_step = ms_total / args.steps
    value = world * BATCH * DIM * n / (ms_step * 1e-3)
    assert torch.isfinite(f).all().item(), "non-finite K.u"

    peak, peak_src = measured_peaks()
    periodic = ff.embedding() == 3
    pbytes = pass_algorithmic_bytes(N_SIDE, BATCH, periodic)
    # the symbol bytes K3 actually streams (the model's 3 doubles per frequency of
    # the full table, or the mirror planes over ky in [0, Pl/2]: about half)
    sym_model = 3 * ((N_SIDE // 2 + 1) if periodic else (N_SIDE + 1)) * (N_SIDE if periodic else 2 * N_SIDE) * 8
    sym_stream = min(sym_model, ff.symbol_stream_bytes())
    pbytes["K3_spectral"] += sym_stream - sym_model
    p2 = periodic and N_SIDE == 4096 and not any(os.environ.get(k) for k in ("PDGPU_K1_P2", "PDGPU_K5_P2", "PDGPU_K3"))
    kernels = {"K1_rfft_x": ("k_rfft_rows_p2 (K1: R2C along x, persistent two-group CTA, TMA-landed rows, TMA-stored "
                             "transposed blocks)" if p2 else "k_rfft_rows_duo/pipe (K1: R2C along x, transposed store)"),
               "K3_spectral": ("k_spectral2d_tx (K3: y-FFT + symbol + inverse y-FFT, TMEM park, TMA-landed operands "
                               "and symbol planes)" if p2 else "k_spectral2d_tm/duo (K3: y-FFT + symbol + inverse y-FFT)"),
               "K5_irfft_x": ("k_irfft_rows_p2 (K5: TMA gather + C2R along x + epilogue, persistent two-group CTA)"
                              if p2 else "k_irfft_rows (K5: gather + C2R along x + epilogue)")}
    per_pass = {}
    for k in kernels:
        ms_k, n_k = passes.get(k, (0.0, 0))
        avg_s = (ms_k / max(n_k, 1)) * 1e-3
        gbs = pbytes[k] / avg_s / 1e9 if avg_s > 0 else None
        per_pass[k] = {"algorithmic_bytes_per_launch": pbytes[k], "mean_launch_ms": avg_s * 1e3,
                       "achieved_gbs": gbs, "frac": (gbs / peak) if gbs else None}
    # dominant kernel = the pass with the largest share of the step
    dom = max(per_pass, key=lambda k: per_pass[k]["mean_launch_ms"])
    mv_bytes = sum(pbytes.values())
    mv_gbs = mv_bytes / (ms_step * 1e-3) / 1e9
    traffic = None
    tr_path = os.path.join(ROOT, "profiles", "dram_bytes.json")
    if os.path.exists(tr_path):
        try:
            with open(tr_path) as fh:
                tj = json.load(fh)
            if tj.get("n") == N_SIDE and tj.get("batch") == BATCH and tj.get("periodic") == periodic:
                traffic = tj.get("dram_bytes_per_launch", {}).get(dom)
        except Exception:
            pass
    pd = per_pass[dom]
    roofline = {"bound": "hbm", "kernel": kernels[dom],
                "achieved": pd["achieved_gbs"], "peak": peak, "unit": "GB/s", "frac": pd["frac"],
                "traffic": traffic, "algorithmic_bytes_per_launch": pd["algorithmic_bytes_per_launch"],
                "mean_launch_ms": pd["mean_launch_ms"], "peak_source": peak_src,
                "embedding": "periodic (P = N + wrap correction)" if periodic else "padded (P = 2N)",
                "per_pass": per_pass,
                "matvec": {"algorithmic_bytes_per_step": mv_bytes, "achieved_gbs": mv_gbs, "frac": mv_gbs / peak,
                           "symbol_bytes_per_launch": sym_stream,
                           "model": ("48 B/DOF/vector + the symbol K3 streams (12N B full table, 6N B mirror planes) "
                                     "(periodic)" if periodic
                                     else "SURVEY 8(d): 80 B/DOF/vector + 48N B symbol (padded)")},
                "passes_ms_per_step": {k: v[0] / args.steps for k, v in passes.items()},
                "symbol_mode": ff.symbol_mode()}

    # comparison point: the same apply by direct stencil summation
    direct = None
    if not args.no_extra:
        try:
            fd = torch.empty_like(u)
            with torch.cuda.stream(stream):
                ff.apply_direct_device(u, fd, BATCH, stream)
                ff.apply_device(u, f, BATCH, stream)
            torch.cuda.synchronize()
            rel = float(torch.linalg.norm(fd - f) / torch.linalg.norm(f))
            d0 = torch.cuda.Event(enable_timing=True)
            d1 = torch.cuda.Event(enable_timing=True)
            d0.record(stream)
            for _ in range(args.steps):
                ff.apply_direct_device(u, fd, BATCH, stream)
            d1.record(stream)
            torch.cuda.synchronize()
            dms = d0.elapsed_time(d1) / args.steps
            direct = {"what": "FastForce::apply by direct stencil summation (csrc/direct.cu): SURVEY 8f comparison "
                              "point and on-device cross-check, not the MSBFM metric",
                      "ms_per_step": dms, "value": BATCH * DIM * n / (dms * 1e-3), "unit": UNIT,
                      "rel_diff_vs_fft_apply": rel, "bytes_per_dof_model": 16}
            del fd
        except Exception as exc:
            direct = {"error": str(exc)[:200]}

    # end to end through the public host API (pinned host buffers)
    e2e = None
    if not args.no_e2e:
        uh = torch.empty((BATCH, DIM, n), dtype=torch.float64, pin_memory=True)
        uh.copy_(u)
        fh = torch.empty_like(uh, pin_memory=True)
        uh_np, fh_np = uh.numpy(), fh.numpy()
        ff.matvec(uh_np, out=fh_np)  # warm the staging buffers (not timed)
        e2e_steps = max(1, min(args.steps, 3))
        D.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(e2e_steps):
            ff.matvec(uh_np, out=fh_np)
        torch.cuda.synchronize()
        e2e_s = D.max_over_ranks((time.perf_counter() - t0) / e2e_steps, "cuda")
        nbytes = BATCH * DIM * n * 8
        e2e = {"value": world * BATCH * DIM * n / e2e_s, "unit": UNIT, "h2d_bytes_per_step": nbytes,
               "d2h_bytes_per_step": nbytes, "steps": e2e_steps, "ms_per_step": e2e_s * 1e3,
               "api": "pdgpu_matvec_host (pinned host u -> host f; H2D/compute/D2H pipelined in 1-vector chunks)"}
        del uh, fh
    ff.close()
    del u, f
    torch.cuda.empty_cache()

    extra = None
    if not args.no_extra and world == 1:
        try:
            extra = extra_configs(local, stream)
        except Exception as exc:
            extra = {"error": str(exc)[:300]}
    if direct is not None:
        extra = dict(extra or {}, direct_stencil_4096_b16=direct)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        try:
            cpu = cpu_reference_sample(N_SIDE, steps=3, budget_s=45.0)
            if cpu:
                cpu = {k: cpu[k] for k in ("value", "unit", "cores", "host_cores", "cpu_model", "kind", "sample",
                                           "build")}
                cg = cpu_reference_cg_config1()
                if cg:
                    cpu["config1_cg"] = cg
        except Exception as exc:  # the CPU leg must not kill the GPU number
            cpu = {"error": str(exc)[:200]}

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
                "scaling": "weak" if args.shard == "vectors" else "strong",
                "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded uniform[-1,1], torch Philox)",
                "config": workload_config(world), "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e,
                "gpu_launches": launches, "clocks": clocks, "configs": extra}
        print(json.dumps(line))
    D.finalize()
    return 0


if __name__ == "__main__":
    sys.exit(main())
