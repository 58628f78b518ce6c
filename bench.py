#!/usr/bin/env python
"""Benchmark of the FMM-BEM hot path (BASELINE.json metric) -- one JSON line on rank 0.

Workload (BASELINE config 5): 10x10x10 randomly rotated copies of the
synthetic lysozyme (C3: 102,152 panels, 2,000 atoms each) -> 102,152,000 panels,
2,000,000 charges, eps 4/80, P = 10 terms, centroid rule.  A step is one application of
the GMRES operator A = I - f K' (one "FMM evaluation" = one BEM iteration):
upward sweep, M2L, downward sweep, P2P, L2P, all in libfmmbem's kernels, inputs resident
in HBM.  x (409 MB) and the point data (3.3 GB) exceed the 126 MB L2, so no flush is needed.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config c5|c3|...] [--impl reference]
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

FLOPS_PER_INTERACTION = 19.0  # SURVEY 8(d) convention for a K' interaction
METRIC = "FMM-BEM matvec s and P2P Ginteractions/s at 1/2/4/8 B200; % FP32 peak"


def fp32_peak_tflops(sm_count=148, mhz=1965.0):
    """148 SMs x 128 FP32 lanes x 2 flops (FFMA) x max SM clock (B200_PROFILING.md / DESIGN.md)."""
    return sm_count * 128 * 2 * mhz * 1e6 / 1e12


def m2l_rot_flops(P):
    """Algorithmic flops of one rotation-based M2L: 4 fixed-matrix stages of
    sum_n (n+1)^2 FMAs (the Wigner-parity zeros excluded), 4 phase stages of (NC - P) complex
    products (6 flops), the coaxial translation 2 sum_k (P-k)^2 FMAs and 2 degree scalings."""
    NC = P * (P + 1) // 2
    mat = sum((n + 1) ** 2 for n in range(P)) * 2
    coax = 2 * sum((P - k) ** 2 for k in range(P)) * 2
    return 4 * mat + 4 * 6 * (NC - P) + coax + 2 * 2 * NC


def launches_per_matvec(L, P):
    """libfmmbem kernels per A-matvec: P2M, M2M per level (rotation: translate + sum), one M2L,
    L2L per level, the scaled P2P source table (k_scale_src), P2P, L2P (memsets and NCCL kernels
    excluded)."""
    if L < 2:
        return 2
    m2m = 2 if P in (8, 10, 12) else 1
    return 1 + m2m * (L - 2) + 1 + (L - 2) + 1 + 1 + 1


def workload(name):
    from synth import configs
    if name == "c5":
        base = configs.lysozyme(113)
        return configs.array((10, 10, 10), base=base), "array_10x10x10_lysozyme_nu113"
    if name == "c5_small":  # 3x3x3 array (2.76 M panels)
        base = configs.lysozyme(113)
        return configs.array((3, 3, 3), base=base), "array_3x3x3_lysozyme_nu113"
    if name == "c3":
        return configs.lysozyme(113), "lysozyme_nu113"
    if name == "c2":
        return configs.kirkwood(64), "kirkwood_octa64"
    raise SystemExit(f"unknown config {name}")


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled every 200 ms during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu):
        self.gpu = gpu
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if not self.proc:
            return None
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(2)
        except Exception:
            self.proc.kill()
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx = max(mx, float(f[2]))
            except ValueError:
                continue
            for nm, v in zip(names, f[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        if not sm:
            return None
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


def oracle_sample(cfg, rows, x_global):
    """FP64 oracle K' rows (plain direct sums over ALL sources) for a bounded target sample."""
    from oracle import bem, _cdirect
    pan = bem.Panels(cfg["vertices"], cfg["triangles"])
    t0 = time.perf_counter()
    y = bem.apply_kprime(pan, x_global, rows=rows)
    dt = time.perf_counter() - t0
    return y, dt, _cdirect.threads(), pan


def reference_arm(args, rank, world):
    """--impl reference: the FP64 oracle as it stands, on a bounded sample, rank 0 only."""
    if rank != 0:
        return
    cfg, wname = workload(args.config)
    n = len(cfg["triangles"])
    rng = np.random.default_rng(7)
    x = rng.normal(size=n)
    rows_per_step = max(2, int(args.ref_rows))
    for _ in range(args.warmup):
        oracle_sample(cfg, rng.choice(n, rows_per_step, replace=False), x)
    fits = []
    for _ in range(args.steps):  # each step: a small and a full sample -> fixed + per-row terms
        _, d1, cores, _ = oracle_sample(cfg, rng.choice(n, rows_per_step // 2, replace=False), x)
        _, d2, cores, _ = oracle_sample(cfg, rng.choice(n, rows_per_step, replace=False), x)
        per_row = max((d2 - d1) / (rows_per_step - rows_per_step // 2), 1e-12)
        fits.append((max(d2 - per_row * rows_per_step, 0.0), per_row))
    fixed = float(np.mean([f[0] for f in fits]))
    per_row = float(np.mean([f[1] for f in fits]))
    t_full = fixed + per_row * n  # extrapolated full direct matvec
    value = 1.0 / t_full
    sample = (f"{rows_per_step // 2} and {rows_per_step} target rows x {n} sources per step (FP64 direct): "
              f"{fixed:.2f} s fixed + {per_row * 1e3:.1f} ms/row, extrapolated to {n} rows")
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "matvec/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": t_full * 1e3, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": wname, "n_panels": n, "terms": args.terms, "quad_points": 1,
                       "l2_flush": "inputs larger than L2"},
            "cpu_baseline": {"value": value, "unit": "matvec/s", "cores": cores, "kind": "oracle",
                             "sample": sample},
            "e2e": {"value": value, "unit": "matvec/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c5")
    ap.add_argument("--terms", type=int, default=12)
    ap.add_argument("--leaf-points", type=int, default=128)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--ref-rows", type=int, default=64)
    ap.add_argument("--cpu-rows", type=int, default=128, help="oracle sample rows for cpu_baseline/parity")
    ap.add_argument("--no-cpu", action="store_true")
    args = ap.parse_args()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        return reference_arm(args, rank, world)

    import torch
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_1007_4591_b200 import Solver

    cfg, wname = workload(args.config)
    n = len(cfg["triangles"])
    t0 = time.perf_counter()
    if world > 1:  # octree domain decomposition over NCCL; every rank gets the full input
        s = Solver.distributed(cfg, terms=args.terms, leaf_points=args.leaf_points, device=local)
    else:
        s = Solver.from_config(cfg, terms=args.terms, leaf_points=args.leaf_points, device=local)
    torch.cuda.synchronize()
    setup_s = time.perf_counter() - t0
    info = s.tree_info()
    rng = np.random.default_rng(7)
    x_global = rng.normal(size=n)
    x = torch.tensor(s.to_local(x_global), dtype=torch.float32, device=f"cuda:{local}")
    y = torch.empty_like(x)
    stream = torch.cuda.current_stream()

    def step():
        s.matvec(x, "A", out=y)

    for _ in range(max(3, args.warmup)):
        step()
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    clk = ClockSampler(local)
    clk.start()
    phases = {k: [] for k in ("upward", "comm", "m2l", "p2p", "l2p", "total")}
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    for _ in range(args.steps):
        step()
        tm = s.timing()  # per-phase CUDA-event times of this matvec (launch stream)
        for k in phases:
            phases[k].append(tm[k])
    ev1.record(stream)
    torch.cuda.synchronize()
    clocks = clk.stop()
    ms = ev0.elapsed_time(ev1) / args.steps
    if dist:
        t = torch.tensor([ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
        dist.barrier()
    tm = s.timing()
    ph = {k: float(np.mean(v)) for k, v in phases.items()}
    value = 1.0 / (ms * 1e-3)  # matvecs of the whole (fixed) problem per second, all ranks together

    # e2e: through the C ABI with pinned host buffers (H2D x, matvec, D2H y inside the region)
    nl = s.n
    xh = torch.empty(nl, dtype=torch.float32, pin_memory=True)
    xh.copy_(torch.from_numpy(s.to_local(x_global).astype(np.float32)))
    yh = torch.empty(nl, dtype=torch.float32, pin_memory=True)
    xh_np, yh_np = xh.numpy(), yh.numpy()
    for _ in range(2):
        s.matvec_host(xh_np, "A", yh_np)
    e2e_steps = max(2, min(args.steps, 5))
    if dist:
        dist.barrier()
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        s.matvec_host(xh_np, "A", yh_np)
    e2e_s = (time.perf_counter() - t0) / e2e_steps
    if dist:
        t = torch.tensor([e2e_s], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s = float(t.item())

    # BIBEE energy (charge-FMM + reduction), once, outside the timed region
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    bib = s.bibee("cfa")
    bibee_s = time.perf_counter() - t0
    t0 = time.perf_counter()
    s.bibee("cfa")
    bibee_warm_s = time.perf_counter() - t0

    p2p_int = int(tm["p2p_interactions"])
    p2p_s = ph["p2p"] * 1e-3
    if dist:  # job-wide P2P rate: all ranks' interactions over the slowest rank's P2P time
        t = torch.tensor([float(p2p_int)], device="cuda", dtype=torch.float64)
        dist.all_reduce(t)
        p2p_int = int(t.item())
        t = torch.tensor([p2p_s], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        p2p_s = float(t.item())
    p2p_tflops = FLOPS_PER_INTERACTION * p2p_int / p2p_s / 1e12
    peak = fp32_peak_tflops() * world
    m2l_pairs = int(tm["m2l_pairs"])
    P = args.terms
    m2l_flops = m2l_rot_flops(P) * m2l_pairs
    dominant = max(("p2p", "m2l"), key=lambda k: ph[k])
    if dominant == "p2p":
        roof = {"kernel": "k_p2p (near field)", "bound": "alu", "achieved": p2p_tflops, "peak": peak,
                "unit": "TFLOP/s", "frac": p2p_tflops / peak}
    else:
        a = m2l_flops / (ph["m2l"] * 1e-3) / 1e12
        roof = {"kernel": "k_m2l_rot (rotation M2L, O(P^3))", "bound": "alu", "achieved": a, "peak": peak,
                "unit": "TFLOP/s", "frac": a / peak}
    roof["traffic"] = None
    prof = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(prof):
        try:
            tr = json.load(open(prof))
            if tr.get("config") == wname and roof["kernel"].split()[0] in tr:
                roof["traffic"] = tr[roof["kernel"].split()[0]]
        except Exception:
            pass
    # the second-largest kernel, for context (same conventions)
    a_m2l = m2l_flops / (ph["m2l"] * 1e-3) / 1e12 if ph["m2l"] > 0 else 0.0
    roof_m2l = {"kernel": "k_m2l_rot_sync (rotation M2L, O(P^3))", "bound": "alu", "achieved": a_m2l,
                "peak": peak, "unit": "TFLOP/s", "frac": a_m2l / peak, "traffic": None}
    try:
        tr = json.load(open(prof))
        if tr.get("config") == wname and "k_m2l_rot" in tr:
            roof_m2l["traffic"] = tr["k_m2l_rot"]
    except Exception:
        pass

    out = {"metric": METRIC, "value": value, "unit": "matvec/s", "n_gpus": world, "steps": args.steps,
           "warmup": max(3, args.warmup), "ms_per_step": ms, "higher_is_better": True,
           "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
           "config": {"workload": wname, "n_panels": n, "n_charges": len(cfg["charge_q"]), "terms": P,
                      "quad_points": 1, "leaf_points": args.leaf_points, "operator": "A = I - f K'",
                      "tree_levels": info["levels"], "n_leaves": info["n_leaves"],
                      "l2_flush": "inputs larger than L2 (x 409 MB, points 3.3 GB)",
                      "parallelism": "single GPU" if world == 1 else
                      f"octree domain decomposition x{world} (NCCL: all-gather x, LET multipole send/recv)"},
           "matvec_s": ms * 1e-3,
           "phases_ms": ph,
           "p2p_ginteractions_s": p2p_int / p2p_s / 1e9,
           "p2p_interactions": p2p_int,
           "p2p_frac_fp32_peak": p2p_tflops / peak,
           "m2l_pairs": m2l_pairs,
           "setup_s": setup_s,
           "bibee_cfa": {"dG_kcal_mol": bib["dG_kcal"], "first_call_s": bibee_s, "warm_s": bibee_warm_s},
           "roofline": roof, "roofline_m2l": roof_m2l,
           "gpu_launches": args.steps * launches_per_matvec(info["levels"], P),
           "e2e": {"value": 1.0 / e2e_s, "unit": "matvec/s", "h2d_bytes_per_step": 4 * n,
                   "d2h_bytes_per_step": 4 * n},
           "comm_ms": ph["comm"],
           "clocks": clocks}
    if dist:  # per-rank breakdown (load balance of the domain decomposition)
        mine = {"rank": rank, "n_local": s.n, "phases_ms": ph, "p2p_interactions": int(tm["p2p_interactions"]),
                "m2l_pairs": int(tm["m2l_pairs"])}
        allr = [None] * world
        dist.all_gather_object(allr, mine)
        out["per_rank"] = allr
        out["m2l_pairs"] = int(sum(r["m2l_pairs"] for r in allr))
    if rank == 0 and world == 1 and not args.no_cpu:
        # oracle as it stands: t(rows) = fixed setup + rows x per-row direct sum over all sources;
        # two sample sizes give both terms, extrapolated to the full n-row matvec
        rng2 = np.random.default_rng(11)
        r1 = rng2.choice(n, max(1, args.cpu_rows // 4), replace=False)
        rows = rng2.choice(n, args.cpu_rows, replace=False)
        _, dt1, cores, _ = oracle_sample(cfg, r1, x_global)
        y_ref, dt, cores, _ = oracle_sample(cfg, rows, x_global)
        per_row = max((dt - dt1) / (len(rows) - len(r1)), 1e-12)
        fixed = max(dt - per_row * len(rows), 0.0)
        y_loc = y.cpu().numpy().astype(np.float64)
        y_glob = s.to_global(y_loc)
        f = 2.0 * (80.0 - 4.0) / 84.0
        a_ref = x_global[rows] - f * y_ref
        out["parity_sampled_rows"] = {"rows": int(len(rows)),
                                      "rel_l2_A": float(np.linalg.norm(y_glob[rows] - a_ref) / np.linalg.norm(a_ref)),
                                      "rel_l2_Kprime": float(np.linalg.norm((x_global[rows] - y_glob[rows]) / f - y_ref)
                                                             / np.linalg.norm(y_ref))}
        t_full = fixed + per_row * n
        out["cpu_baseline"] = {"value": 1.0 / t_full, "unit": "matvec/s", "cores": cores, "kind": "oracle",
                               "sample": f"FP64 direct K' rows over all {n} sources: {len(r1)} rows in {dt1:.2f} s "
                                         f"and {len(rows)} rows in {dt:.2f} s -> {fixed:.2f} s fixed + "
                                         f"{per_row * 1e3:.1f} ms/row, extrapolated to the full {n}-row matvec"}
    if rank == 0:
        print(json.dumps(out), flush=True)
    if dist:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
