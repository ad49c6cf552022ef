#!/usr/bin/env python
"""Benchmark of the hot path: effective conductivity of a 512^3 random-inclusion
RVE (reference RANDOM_BALL_PRESETS["a"] geometry, contrast 100) in all three
load directions, PCG to relative residual 1e-6 (BASELINE.json config 4).

One "step" = the full three-direction homogenization (3 x homogenize():
permute + scale + stats + LP + preconditioner setup + rhs + PCG + flux),
inputs resident in HBM.  Prints ONE JSON line (rank 0).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]

--impl reference times the reference algorithm's CPU implementation (the
numpy oracle port, oracle/etc_oracle.py) on the host cores.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "PCG time-to-solution, 512^3 random-inclusion RVE (contrast 100), x/y/z, rtol 1e-6"


def cfg_tag(args) -> str:
    return " (BASELINE config 4)" if (args.n, args.contrast) == (512, 100.0) else ""


def bench_config(args) -> dict:
    """The workload both arms report (identical keys and values)."""
    n = args.n
    kind = "random-inclusion RVE" if args.field == "balls" else "log-uniform random field"
    return {"workload": f"{n}^3 {kind}, contrast {args.contrast:g}, directions {args.axes}, "
                        f"rtol {args.rtol:g}, {args.precision}"
                        f"{cfg_tag(args) if args.field == 'balls' and args.precision == 'f64' else ''}",
            "n": n, "contrast": args.contrast, "rtol": args.rtol, "directions": args.axes,
            "l2": "inputs larger than L2 (one f64 vector = %.2f GB)" % (8 * n ** 3 / 1e9)}


def metric_for(args) -> str:
    """BASELINE.json's metric for the default workload; the same wording with
    the actual size / contrast / directions / rtol otherwise."""
    if (args.n, args.contrast, args.axes, args.rtol, args.field, args.precision) == (512, 100.0, "xyz", 1e-6, "balls",
                                                                                     "f64"):
        return METRIC
    ax = "/".join(args.axes)
    kind = "random-inclusion RVE" if args.field == "balls" else "log-uniform random field"
    return (f"PCG time-to-solution, {args.n}^3 {kind} (contrast {args.contrast:g}), {ax}, "
            f"rtol {args.rtol:g}" + (", precision f32" if args.precision == "f32" else ""))
KCLASS = ["stencil", "update_fwd2d", "fwd2d", "zsolve", "unused", "inv2d", "setup"]


def bytes_per_cell(wfuse: bool, phases: bool = False, esz: int = 8) -> dict:
    """Algorithmic (compulsory) HBM bytes per cell per launch, f64 (esz 8)
    or the fused float32 solve (esz 4).

    wfuse (single-GPU square planes, the default): the inverse transform
    builds the search direction w = z + beta w_old itself, so the stencil
    reads w instead of z and w_old and writes only q.  phases (the field has
    at most 16 distinct conductivity triples, as every benchmark field does):
    a one-byte phase index replaces the three face arrays."""
    if esz == 4:  # every vector and face in float32; the phase index stays one byte
        return {"stencil": 9 if phases else 20, "update_fwd2d": 16, "fwd2d": 8, "zsolve": 8, "inv2d": 12}
    if wfuse:
        return {
            "stencil": 17 if phases else 40,  # w, idx (or tx, ty, tz) read; q written
            "update_fwd2d": 32,  # r, q read; r, t(=q) written; x+y DCT-II fused per plane
            "fwd2d": 16, "zsolve": 16,
            "inv2d": 24,  # t, w_old read; w written (16 on the first launch of a solve: w = z)
        }
    return {
        # z, w_old, tx, ty, tz read; w_new, q written (p only on the outflow plane)
        "stencil": 56,
        "update_fwd2d": 32,  # r, q read; r, t(=q) written; x+y DCT-II fused per plane
        "fwd2d": 16, "zsolve": 16, "inv2d": 16,
    }


NCU_PREFIX = {"stencil": "k_stencil", "update_fwd2d": "k_fwd", "zsolve": "k_zsolve",
              "inv2d": "k_inv"}


def load_traffic(n: int) -> tuple[dict, str | None]:
    """DRAM bytes per launch (dram__bytes_read.sum + dram__bytes_write.sum)
    of each kernel class from the committed `ncu --set full` capture of the
    default workload (the latest profiles/rNN/ncu_full_512_traffic.json,
    written by profiles/ncu_summary.py); {} for other sizes."""
    caps = sorted((ROOT / "profiles").glob("r[0-9][0-9]/ncu_full_512_traffic.json"))
    if n != 512 or not caps:
        return {}, None
    p = caps[-1]
    d = json.loads(p.read_text())
    out = {}
    for cls, pre in NCU_PREFIX.items():
        for name, v in d.items():
            if name.startswith(pre):
                out[cls] = int(v["dram_bytes"])
    return out, str(p.relative_to(ROOT))


def load_peaks() -> dict:
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        try:
            d = json.loads(p.read_text())
            return {"hbm_gbs": float(d["hbm_gbs"]), "source": "measured"}
        except Exception:
            pass
    return {"hbm_gbs": 6650.0, "source": "fallback"}


class Clocks:
    """nvidia-smi sampler running during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.path = Path(os.environ.get("TMPDIR", "/tmp")) / f"etc_clocks_{os.getpid()}.csv"

    def start(self):
        try:
            self.fh = open(self.path, "w")
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=self.fh, stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.fh.close()
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in self.path.read_text().splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                smax.append(float(f[2]))
            except ValueError:
                continue
            for nm, v in zip(names, f[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        try:
            self.path.unlink()
        except OSError:
            pass
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(smax) if smax else None,
                "samples": len(sm), "reasons": sorted(reasons)}


# ----------------------------------------------------------------------------
# CPU baseline: the oracle port of the reference algorithm (numpy + pocketfft)
# ----------------------------------------------------------------------------

def cpu_sample(n: int, contrast: float, iters: int, workers: int) -> dict:
    """Setup and per-PCG-iteration host time of the reference algorithm at n^3
    (oracle/etc_oracle.py: same stencil, Makhoul DCT via pocketfft, Thomas
    sweep, Alg. 1 vector algebra), z direction."""
    from oracle import etc_oracle as O

    k = O.random_balls(n, 40, 0.05, 0.15, contrast, 11)
    t0 = time.perf_counter()
    s = O.scale(k, 1.0 / n)
    fc = O.faces(s, s, s)
    refs = O.reference_constants(O.stats(fc))
    tab = O.tables(n, n, n, refs)
    b = O.rhs(fc, k.shape, 1.0, 0.0).reshape(-1)
    t_setup = time.perf_counter() - t0
    shape = k.shape
    A = lambda u: O.stencil(fc, u.reshape(shape)).reshape(-1)
    M = lambda r: O.precond(tab, r.reshape(shape), workers).reshape(-1)
    r = b.copy()
    p = np.zeros_like(b)
    z = M(r)
    w = z.copy()
    rho = float(np.dot(r, z))
    times = []
    for _ in range(iters):
        t0 = time.perf_counter()
        q = A(w)
        qw = float(np.dot(q, w))
        _ = 100 * 2.2e-16 * float(np.linalg.norm(q)) * float(np.linalg.norm(w))
        alpha = rho / qw
        p += alpha * w
        r -= alpha * q
        _ = float(np.linalg.norm(r))
        z = M(r)
        rho_new = float(np.dot(r, z))
        w = z + (rho_new / rho) * w
        rho = rho_new
        times.append(time.perf_counter() - t0)
    return {"setup_s": t_setup, "iter_s": min(times), "iters": iters}


def iterations_512() -> dict:
    """Reference iteration counts at 512^3 (tests/golden/solves_512.json, made
    by running the reference here), else None per missing axis."""
    out = {}
    p = ROOT / "tests" / "golden" / "solves_512.json"
    if p.exists():
        for c in json.loads(p.read_text()):
            out[c["axis"]] = int(c["iterations"])
    return out


# ----------------------------------------------------------------------------
# GPU arm
# ----------------------------------------------------------------------------

def run_b200(args, rank, world, local_rank):
    import torch

    import paper_2404_02433_b200 as P

    dev = torch.device("cuda", local_rank)
    torch.cuda.set_device(dev)
    dist = world > 1 or args.slab
    if dist:
        import torch.distributed as td
    n = args.n
    if args.field == "random":
        # a general field (every cell its own conductivity, no phase tables):
        # log-uniform in [1/C, C], isotropic, seeded on the device
        gen = torch.Generator(device=dev)
        gen.manual_seed(11)
        u = torch.rand(n ** 3, dtype=torch.float64, device=dev, generator=gen)
        kk = torch.exp((2.0 * u - 1.0) * float(np.log(args.contrast)))
        field = P.OrthotropicField(P.GridSpec(n, n, n), kk, kk, kk)
    else:
        field = P.gen_random_balls(n, 40, 0.05, 0.15, args.contrast, 11, device=dev)
    axes = args.axes
    if dist:
        from paper_2404_02433_b200 import dist as D

        comm = D.TorchComm()

        def step(fld=field):
            return D.effective_tensor_dist(fld, comm, rtol=args.rtol, axes=axes, device=dev, zsolve=args.zsolve)
    else:
        def step(fld=field):
            return P.effective_tensor(fld, rtol=args.rtol, axes=axes, device=dev, precision=args.precision)

    for _ in range(args.warmup):
        kappa, reps = step()
    torch.cuda.synchronize()
    lib = P._native.lib()
    import ctypes as C

    def handles():
        if dist:
            return [ops._h for ops in D._OPS_CACHE.values()]
        return [P.get_plan(field.grid, dev).handle]

    ms8 = (C.c_double * 8)()
    cnt8 = (C.c_longlong * 8)()

    def prof_read(reset=1):
        tot_ms, tot_cnt = [0.0] * 8, [0] * 8
        for h in handles():
            lib.etc_profile_read(h, ms8, cnt8, reset)
            for i in range(8):
                tot_ms[i] += ms8[i]
                tot_cnt[i] += cnt8[i]
        return tot_ms, tot_cnt

    prof_read()  # reset counters
    # per-kernel device times are taken live over the timed region: CUDA
    # events around every launch on the plan stream (read after the region)
    for h in handles():
        lib.etc_profile(h, 1)

    clocks = Clocks(local_rank)
    if dist:
        td.barrier()
    torch.cuda.synchronize()
    clocks.start()
    stream = torch.cuda.current_stream()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        kappa, reps = step()
    e1.record(stream)
    torch.cuda.synchronize()
    clk = clocks.stop()
    if dist:
        td.barrier()
    ms_total = e0.elapsed_time(e1)
    for h in handles():
        lib.etc_profile(h, 0)
    pms, cnts = prof_read()
    launches = int(sum(cnts))
    if dist:
        t = torch.tensor([ms_total], device=dev)
        td.all_reduce(t, op=td.ReduceOp.MAX)
        ms_total = float(t.item())
    ms_step = ms_total / args.steps
    iters = {a: reps[a].iterations for a in axes}
    total_iters = sum(iters.values())

    kms = [pms[i] / args.steps for i in range(8)]  # per-kernel totals per timed step
    kcnt = [cnts[i] / args.steps for i in range(8)]
    N = n ** 3 // world  # cells per rank per launch
    # z-slab ranks run the same fused kernels (etc_slab_fused: ny / P a power of two >= 2)
    wfuse = (os.environ.get("ETC_WFUSE", "1") != "0" and n >= 128 and n & (n - 1) == 0
             and (not dist or n // world >= 2))
    phases = wfuse and os.environ.get("ETC_PHASES", "1") != "0" and args.field == "balls"  # two phases
    esz = 4 if args.precision == "f32" else 8
    bpc = bytes_per_cell(wfuse, phases, esz)
    if dist and args.zsolve == "spike":
        # compulsory traffic only (re-reads are not algorithmic): k_zsub_ends reads the slab once
        # (8 B/cell; it reads it twice), k_zsub_solve moves t r/w, d' w/r and the pivot table r
        # (40 B/cell; it reads t twice): 24 B/cell per launch on average
        bpc["zsolve"] = 24
    peaks = load_peaks()
    kern = {}
    for i, name in enumerate(KCLASS):
        if kcnt[i] == 0:
            continue
        avg = kms[i] / kcnt[i]
        d = {"ms_total": round(kms[i], 4), "launches": int(round(kcnt[i])), "ms_avg": round(avg, 5)}
        if name in bpc:
            b = bpc[name] * N
            if wfuse and name == "inv2d":  # first launch of each solve writes w = z (16 B/cell)
                b = (2 * esz * N * len(axes) + 3 * esz * N * (kcnt[i] - len(axes))) / kcnt[i]
            gbs = b / (avg * 1e-3) / 1e9
            d.update(bytes_per_launch=int(b), gbs=round(gbs, 1), frac=round(gbs / peaks["hbm_gbs"], 4))
        kern[name] = d
    dom = max((k for k in kern if k in bpc), key=lambda k: kern[k]["ms_total"])
    traffic, tsrc = load_traffic(n) if args.precision == "f64" else ({}, None)
    if not dist:
        for k, v in traffic.items():
            if k in kern:
                kern[k]["dram_bytes_ncu"] = v
    it_kernels = [k for k in ("stencil", "update_fwd2d", "zsolve", "inv2d") if k in kern]
    prof_total = sum(v["ms_total"] for v in kern.values())
    roofline = {
        "bound": "hbm", "kernel": dom, "achieved": kern[dom]["gbs"], "peak": peaks["hbm_gbs"], "unit": "GB/s",
        "frac": kern[dom]["frac"], "traffic": traffic.get(dom) if not dist else None,
        "traffic_source": (tsrc + " (ncu --set full, one launch)") if traffic and not dist else None,
        "peak_source": peaks["source"] + " (MEASURED_PEAKS.json hbm_gbs, copy)",
        "bytes_per_launch": kern[dom]["bytes_per_launch"],
        "share_of_step": round(kern[dom]["ms_total"] / prof_total, 4),
        "iteration_bytes_per_cell": sum(bpc[k] for k in it_kernels),
        "iteration_frac": round(sum(kern[k]["bytes_per_launch"] * kern[k]["launches"] for k in it_kernels) / 1e9
                                / (sum(kern[k]["ms_total"] for k in it_kernels) * 1e-3) / peaks["hbm_gbs"], 4),
    }
    # end-to-end through the public API with host buffers
    e2e = None
    if not args.no_e2e:
        # the step's input lives in pinned host memory (the contract's e2e
        # setup); every step copies it to the device inside the timed region
        kh_t = torch.empty(n ** 3, dtype=torch.float64, pin_memory=True)
        kh_t.copy_(field.kx.reshape(-1).cpu())
        kh = kh_t.numpy()
        hostgrid = field.grid
        torch.cuda.synchronize()
        t_e2e = []
        for it in range(args.steps + 1):
            hf = P.OrthotropicField(hostgrid, kh, kh, kh, validate=False)  # fresh object: re-uploaded
            torch.cuda.synchronize()
            if dist:
                td.barrier()
            t0 = time.perf_counter()
            kap, rp = step(hf)
            torch.cuda.synchronize()
            if dist:
                td.barrier()
            if it > 0:  # first call is a warm-up
                t_e2e.append(time.perf_counter() - t0)
        e2e = {"value": round(statistics.mean(t_e2e), 4), "unit": "s",
               "h2d_bytes_per_step": int(kh.nbytes if not dist else kh.nbytes // world),  # dist: this rank's slab
               "d2h_bytes_per_step": int(sum(8 * (r.iterations + 1) + 8 for r in rp.values())),
               "samples": len(t_e2e),
               "api": "paper_2404_02433_b200.effective_tensor(numpy field in pinned host memory)"}

    # the general-field stencil (stored faces, k_stencil_gt, 40 B/cell): the
    # benchmark field has two phases and runs the phase-table stencil, so a
    # log-uniform field of the same size is solved for a few iterations here
    # and its stencil launches are timed the same way (etc_profile)
    general = None
    if not dist and args.field == "balls" and not args.no_general and args.precision == "f64":
        gen = torch.Generator(device=dev)
        gen.manual_seed(11)
        u = torch.rand(n ** 3, dtype=torch.float64, device=dev, generator=gen)
        kr = torch.exp((2.0 * u - 1.0) * float(np.log(args.contrast)))
        del u
        frand = P.OrthotropicField(P.GridSpec(n, n, n), kr, kr, kr)
        P.homogenize(frand, P.BoundaryConfig(P.Axis.Z, 1.0, 0.0), 1e-30, max_iter=3, device=dev)  # warm-up
        h = P.get_plan(frand.grid, dev).handle
        lib.etc_profile_read(h, ms8, cnt8, 1)
        lib.etc_profile(h, 1)
        P.homogenize(frand, P.BoundaryConfig(P.Axis.Z, 1.0, 0.0), 1e-30, max_iter=20, device=dev)
        torch.cuda.synchronize()
        lib.etc_profile(h, 0)
        lib.etc_profile_read(h, ms8, cnt8, 1)
        if cnt8[0] > 0:
            avg = ms8[0] / cnt8[0]
            gbs = 40 * n ** 3 / (avg * 1e-3) / 1e9
            general = {"workload": f"{n}^3 log-uniform random field in [1/C, C], contrast {args.contrast:g}, z, "
                                   "20 PCG iterations", "kernel": "k_stencil_gt (stored faces, TMA ring)",
                       "launches": int(cnt8[0]), "ms_avg": round(avg, 5), "bytes_per_launch": 40 * n ** 3,
                       "gbs": round(gbs, 1), "frac": round(gbs / peaks["hbm_gbs"], 4)}
        del frand, kr
        P.release_plans()

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        workers = os.cpu_count() or 1
        smp = cpu_sample(args.cpu_n, args.contrast, 2, workers)
        scale = (n / args.cpu_n) ** 3
        val = scale * (len(axes) * smp["setup_s"] + total_iters * smp["iter_s"])
        cpu = {"value": round(val, 2), "unit": "s", "cores": workers, "kind": "port",
               "sample": (f"oracle/etc_oracle.py (numpy + pocketfft, {workers} FFT workers, ufuncs 1 core) "
                          f"at {args.cpu_n}^3: setup {smp['setup_s']:.2f} s, PCG iteration {smp['iter_s']:.2f} s "
                          f"(best of 2); extrapolated x{scale:.0f} cells to {len(axes)} setups + "
                          f"{total_iters} iterations")}

    line = {
        "metric": metric_for(args), "value": round(ms_step / 1e3, 4), "unit": "s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(ms_step, 3), "higher_is_better": False, "scaling": "strong",
        "vs_baseline": None, "dtype": args.precision,
        "data": ("synthetic: random-ball RVE (preset a: 40 balls r 0.05-0.15, seed 11), voxelised on device"
                 if args.field == "balls" else
                 "synthetic: log-uniform random field in [1/C, C] per cell (seed 11), generated on device"),
        "config": bench_config(args),
        "details": {
            "iterations": iters, "ms_per_iter": round(ms_step / max(1, total_iters), 4),
            "kappa_eff": {a: reps[a].kappa_eff for a in axes},
            "parallelism": (f"z-slab x{world} (NCCL halo + pencil all-to-all + all-reduce)" if args.zsolve == "pencil"
                            else f"z-slab x{world} (NCCL halo + spike z-solve all-gather + all-reduce)") if dist
                           else "single",
        },
        "roofline": roofline, "kernels": kern, "general_field_stencil": general, "e2e": e2e, "cpu_baseline": cpu,
        "gpu_launches": launches, "clocks": clk,
    }
    if rank == 0:
        print(json.dumps(line), flush=True)


def plan_iso(plan) -> bool:
    f = plan._keepalive
    return f is not None and f[0] is f[1] and f[1] is f[2]


# ----------------------------------------------------------------------------
# reference arm
# ----------------------------------------------------------------------------

def run_reference(args, rank, world):
    if rank != 0:
        return
    workers = os.cpu_count() or 1
    n = args.n
    from oracle import etc_oracle as O

    k = O.random_balls(n, 40, 0.05, 0.15, args.contrast, 11)
    t0 = time.perf_counter()
    s = O.scale(k, 1.0 / n)
    fc = O.faces(s, s, s)
    refs = O.reference_constants(O.stats(fc))
    tab = O.tables(n, n, n, refs)
    b = O.rhs(fc, k.shape, 1.0, 0.0).reshape(-1)
    t_setup = time.perf_counter() - t0
    shape = k.shape
    r = b.copy()
    p = np.zeros_like(b)
    z = O.precond(tab, r.reshape(shape), workers).reshape(-1)
    w = z.copy()
    rho = float(np.dot(r, z))

    def iteration():
        nonlocal w, rho
        q = O.stencil(fc, w.reshape(shape)).reshape(-1)
        alpha = rho / float(np.dot(q, w))
        p.__iadd__(alpha * w)
        r.__isub__(alpha * q)
        zz = O.precond(tab, r.reshape(shape), workers).reshape(-1)
        rho_new = float(np.dot(r, zz))
        w = zz + (rho_new / rho) * w
        rho = rho_new

    for _ in range(args.warmup):
        iteration()
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        iteration()
        times.append(time.perf_counter() - t0)
    it_s = statistics.mean(times)
    known = iterations_512() if n == 512 else {}
    iters = {a: known.get(a, 48) for a in args.axes}
    total = sum(iters.values())
    value = len(args.axes) * t_setup + total * it_s
    line = {
        "metric": metric_for(args), "value": round(value, 3), "unit": "s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(it_s * 1e3, 3), "higher_is_better": False, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic: random-ball RVE (preset a), host voxeliser",
        "impl": "reference",
        "config": bench_config(args),
        "details": {"iterations": iters, "setup_s": round(t_setup, 3), "iter_s": round(it_s, 4),
                    "iterations_source": "tests/golden/solves_512.json (reference runs); 48 where absent"},
        "cpu_baseline": {"value": round(value, 3), "unit": "s", "cores": workers, "kind": "port",
                         "sample": f"one PCG iteration of the oracle port per step at {n}^3 ({workers} FFT workers, "
                                   f"numpy ufuncs 1 core); value = {len(args.axes)} setups + {total} iterations"},
        "e2e": {"value": round(value, 3), "unit": "s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["b200", "reference"], default="b200")
    ap.add_argument("--n", type=int, default=512)
    ap.add_argument("--contrast", type=float, default=100.0)
    ap.add_argument("--rtol", type=float, default=1e-6)
    ap.add_argument("--axes", default="xyz")
    ap.add_argument("--cpu-n", type=int, default=256)
    ap.add_argument("--field", choices=["balls", "random"], default="balls",
                    help="balls: the BASELINE random-inclusion RVE (two phases: phase-table stencil); "
                         "random: a general log-uniform field (stored-faces stencil, 40 B/cell)")
    ap.add_argument("--precision", choices=["f64", "f32"], default="f64",
                    help="f32: the reference's single-precision study (homogenize(..., precision='f32'))")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-general", action="store_true", help="skip the general-field stencil measurement")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--slab", action="store_true", help="z-slab path even on one rank (exercises NCCL plumbing)")
    ap.add_argument("--zsolve", choices=["pencil", "spike"], default=None,
                    help="z-slab z-solve: pencil all-to-alls, or the substructured spike solve (default for N > 1)")
    args = ap.parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # one process per GPU: relaunch under torchrun (the driver launches it that way itself)
        os.execvp(sys.executable, [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
                                   f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1",
                                   "--master-port", os.environ.get("MASTER_PORT", "29512"), __file__,
                                   *sys.argv[1:]])
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if args.gpus != world:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE {world}: launch one process per GPU")
    if args.precision == "f32" and (world > 1 or args.slab):
        raise SystemExit("--precision f32 runs on single-GPU plans")
    if args.zsolve is None:
        args.zsolve = "spike" if world > 1 else "pencil"
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    if world > 1 or args.slab:
        import torch
        import torch.distributed as td

        if args.slab and "MASTER_ADDR" not in os.environ:
            os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT="29511", RANK="0", WORLD_SIZE="1")
        torch.cuda.set_device(local_rank)
        import datetime

        # a rank that fails or hangs surfaces as a NCCL timeout error (torch's
        # watchdog, async error handling) within minutes instead of a stuck job
        os.environ.setdefault("TORCH_NCCL_ASYNC_ERROR_HANDLING", "3")
        td.init_process_group("nccl", device_id=torch.device("cuda", local_rank),
                              timeout=datetime.timedelta(seconds=int(os.environ.get("ETC_NCCL_TIMEOUT_S", "300"))))
    run_b200(args, rank, world, local_rank)
    if world > 1 or args.slab:
        import torch.distributed as td

        td.destroy_process_group()


if __name__ == "__main__":
    main()
