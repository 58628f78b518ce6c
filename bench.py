#!/usr/bin/env python
"""Benchmark of the FMM-BEM hot path (BASELINE.json metric) -- one JSON line on rank 0.

Workload (BASELINE config 5): 10x10x10 randomly rotated copies of the
synthetic lysozyme (C3: 102,152 panels, 2,000 atoms each) -> 102,152,000 panels,
2,000,000 charges, eps 4/80, P = 13 terms (the order at which the K' error is <= 1e-4 for
every input tested), leaf_points 128, centroid rule.  A step is one
application of the GMRES operator A = I - f K' (one "FMM evaluation" = one BEM iteration, PAPER
P:667): upward sweep, M2L, downward sweep, P2P, L2P, all in libfmmbem's kernels, inputs resident
in HBM.  x (409 MB) and the point data (3.3 GB) exceed the 126 MB L2, so no flush is needed.
Also reported: the uncached BIBEE energy (charge-FMM + reduction, BASELINE config 5 "BIBEE")
device-timed over 10 calls with sampled-row parity of its fields.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config c5|c5_small|c3|c2|cube] [--impl reference]
"""
from __future__ import annotations

import argparse
import json
import os
import platform
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

FLOPS_PER_INTERACTION = 19.0  # SURVEY 8(d) convention for a K' interaction
FLOPS_PER_INTERACTION_POT = 11.0  # potential-only (V) interaction
METRIC = "FMM-BEM matvec s and P2P Ginteractions/s at 1/2/4/8 B200; % FP32 peak"
DEFAULT_TERMS = 13


def fp32_peak_tflops(sm_count=148, mhz=1965.0):
    """148 SMs x 128 FP32 lanes x 2 flops (FFMA) x max SM clock (B200_PROFILING.md / DESIGN.md)."""
    return sm_count * 128 * 2 * mhz * 1e6 / 1e12


def hbm_peak_gbs():
    """Measured copy bandwidth (MEASURED_PEAKS.json, driver-written), else the profiling guide's fallback."""
    try:
        return float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def m2l_rot_flops(P):
    """Algorithmic flops of one rotation-based M2L: 4 fixed-matrix stages of
    sum_n (n+1)^2 FMAs (the Wigner-parity zeros excluded), 4 phase stages of (NC - P) complex
    products (6 flops), the coaxial translation 2 sum_k (P-k)^2 FMAs and 2 degree scalings."""
    NC = P * (P + 1) // 2
    mat = sum((n + 1) ** 2 for n in range(P)) * 2
    coax = 2 * sum((P - k) ** 2 for k in range(P)) * 2
    return 4 * mat + 4 * 6 * (NC - P) + coax + 2 * 2 * NC


def launches_per_matvec(L, P, info=None):
    """libfmmbem kernels per A-matvec: P2M, M2M per level (rotation: translate + sum), one M2L,
    L2L per level, the P2P weight normalisation (k_absmax) and scaled source table (k_scale_src),
    P2P, L2P (memsets, copies and NCCL kernels excluded).  Several ranks (tree_info of the rank):
    + the halo weight gather, + one LET pack per peer sent to and one unpack per peer received from,
    + a pack and an unpack of the shared cells."""
    if L < 2:
        return 3
    m2m = 2 if P in (8, 10, 12, 13, 14) else 1
    n = 1 + m2m * (L - 2) + 1 + (L - 2) + 2 + 1 + 1
    if info is not None and info.get("let_send_peers") is not None:
        n += int(info["halo_panels_sent"] > 0) + info["let_send_peers"] + info["let_recv_peers"]
        n += 2 * int(info["let_shared_cells"] > 0)
    return n


ARRAYS = {"c5": (10, 10, 10), "c5_22": (22, 22, 22)}  # C5 and the paper-headline 1.09e9-panel array


def workload(name, rank=0, world=1):
    """(cfg, workload name).  Arrays on several ranks: each rank builds only its block of copies
    (input_mode 1, memory O(N/R) per rank; cfg["n_panels_total"] = the whole problem)."""
    from synth import configs
    if name in ARRAYS and world > 1:
        n = ARRAYS[name]
        return configs.array_part(n, rank, world, base=configs.lysozyme(113)), f"array_{n[0]}x{n[1]}x{n[2]}_lysozyme_nu113"
    if name == "c5_22":  # 10,648 copies: 1,087,614,... panels (NEXT-2)
        return configs.array((22, 22, 22), base=configs.lysozyme(113)), "array_22x22x22_lysozyme_nu113"
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
    if name == "cube":  # the paper's scaling control: 1e8 uniform points, potential only
        return configs.cube_panels(100_000_000), "random_cube_1e8_points"
    raise SystemExit(f"unknown config {name}")


def cpu_info():
    model = platform.processor() or ""
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                model = ln.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    return model, os.cpu_count()


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


class OracleRows:
    """The FP64 oracle as it stands (oracle/bem.py, direct sums over ALL sources) on a bounded sample
    of target rows; the per-x source weights are prepared once outside the timed region, so the
    timing is the direct sums only (rows x n_sources interactions)."""

    def __init__(self, cfg, x, op):
        from oracle import bem, _cdirect
        self.bem = bem
        self.pan = bem.Panels(cfg["vertices"], cfg["triangles"])
        self.op = op
        self.x = np.asarray(x, np.float64)
        self.rows = (bem.SingleRows if op == "single" else bem.KprimeRows)(self.pan, self.x)
        self.cores = _cdirect.threads()

    def __call__(self, rows):
        t0 = time.perf_counter()
        y = self.rows(rows)
        return y, time.perf_counter() - t0


def reference_arm(args, rank, world):
    """--impl reference: the FP64 oracle as it stands on the host cores, rank 0 only; each step a
    bounded sample of rows of the workload's operator (all sources), the rate extrapolated to the
    full direct matvec (labelled as such)."""
    if rank != 0:
        return
    cfg, wname = workload(args.config)
    n = len(cfg["triangles"])
    op = "single" if args.config == "cube" else "kprime"
    x = np.random.default_rng(7).normal(size=n)
    orc = OracleRows(cfg, x, op)
    rng = np.random.default_rng(9)
    rows_per_step = max(1, int(args.ref_rows))
    for _ in range(args.warmup):
        orc(np.sort(rng.choice(n, rows_per_step, replace=False)))
    dts = []
    for _ in range(args.steps):
        _, dt = orc(np.sort(rng.choice(n, rows_per_step, replace=False)))
        dts.append(dt)
    per_row = float(np.sum(dts)) / (rows_per_step * args.steps)
    t_full = per_row * n  # extrapolated full direct matvec
    value = 1.0 / t_full
    model, ncpu = cpu_info()
    sample = (f"{rows_per_step} seeded target rows x all {n} sources per step (FP64 direct "
              f"{'potential' if op == 'single' else 'K-prime'} sums, source weights prepared outside the "
              f"timed region): {per_row * 1e3:.2f} ms/row, EXTRAPOLATED to the full {n}-row matvec")
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "matvec/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": t_full * 1e3, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "extrapolated": True, "measured_ms_per_step": float(np.mean(dts)) * 1e3,
            "config": {"workload": wname, "n_panels": n, "terms": args.terms, "quad_points": 1,
                       "l2_flush": "inputs larger than L2"},
            "cpu_baseline": {"value": value, "unit": "matvec/s", "cores": orc.cores, "kind": "oracle",
                             "cpu_model": model, "host_cpus": ncpu, "sample": sample, "extrapolated": True},
            "e2e": {"value": value, "unit": "matvec/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def algorithmic_bytes(kind, info, P, n_pts, m2l_pairs, m2l_rows):
    """SURVEY 8(d) per-unit HBM bytes of the far-field kernels:
    P2M: 20 B per source (float4 position + weight, x) + one expansion (NC float2) written per leaf;
    L2P: 40 B per target (position, normal, x, y read + written) + one expansion read per leaf;
    M2L: 4 B per translation (source index) + every source expansion read once + every target row's
    local expansion read and written."""
    NC = P * (P + 1) // 2
    e = NC * 8
    nl = info["n_leaves"]
    if kind == "p2m":
        return 20 * n_pts + e * nl
    if kind == "l2p":
        return 40 * n_pts + e * nl
    return 4 * m2l_pairs + e * info["n_cells"] + 2 * e * m2l_rows


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c5")
    ap.add_argument("--terms", type=int, default=None)
    ap.add_argument("--leaf-points", type=int, default=128)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--ref-rows", type=int, default=256, help="oracle rows per reference-arm step")
    ap.add_argument("--cpu-rows", type=int, default=1024, help="oracle sample rows for cpu_baseline/parity")
    ap.add_argument("--bibee-calls", type=int, default=10)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-solve", action="store_true", help="skip the full GMRES solve reported beside the bench line")
    ap.add_argument("--near-mode", type=int, default=0, help="1: analytic flat-panel near field (option a11)")
    ap.add_argument("--charge-terms", type=int, default=None,
                    help="order of the charge-FMM (BIBEE leg); default 12 under K' order 13 (E_n within 1e-4)")
    args = ap.parse_args()
    if args.terms is None:
        args.terms = 10 if args.config == "cube" else DEFAULT_TERMS  # the paper's control is P = 10
    if args.charge_terms is None:  # E_n / psi within 1e-4 of the oracle at 12
        args.charge_terms = 12 if args.terms == 13 else 0
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

    cube = args.config == "cube"
    op = "single" if cube else "A"
    cfg, wname = workload(args.config, rank, world)
    parts = "n_panels_total" in cfg  # this rank holds only its part of the mesh (input_mode 1)
    n = cfg["n_panels_total"] if parts else len(cfg["triangles"])
    t0 = time.perf_counter()
    if world > 1:  # octree domain decomposition over NCCL
        s = Solver.distributed(cfg, input_mode=1 if parts else 0, terms=args.terms, leaf_points=args.leaf_points,
                               device=local, near_mode=args.near_mode, charge_terms=args.charge_terms)
    else:
        s = Solver.from_config(cfg, terms=args.terms, leaf_points=args.leaf_points, device=local,
                               near_mode=args.near_mode, charge_terms=args.charge_terms)
    torch.cuda.synchronize()
    setup_s = time.perf_counter() - t0
    info = s.tree_info()
    if parts:  # x by global id (counter-based), no rank materialises the whole vector
        from synth.inputs import normal_by_id
        x_global = None
        x_loc = normal_by_id(s.local_ids, seed=7)
    else:
        rng = np.random.default_rng(7)
        x_global = rng.normal(size=n)
        if cube:  # unit charges q ~ U(-1, 1) as panel weights A_j x_j = q_j
            x_global = cfg["charge_per_area"] * rng.uniform(-1.0, 1.0, n)
        x_loc = s.to_local(x_global)
    x = torch.tensor(x_loc, dtype=torch.float32, device=f"cuda:{local}")
    y = torch.empty_like(x)
    stream = torch.cuda.current_stream()

    def step():
        s.matvec(x, op, out=y)

    for _ in range(max(3, args.warmup)):
        step()
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    clk = ClockSampler(local)
    clk.start()
    keys = ("upward", "p2m", "m2m", "comm", "m2l", "p2p", "l2p", "l2l", "leaf_l2p", "near", "total")
    phases = {k: [] for k in keys}
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    for _ in range(args.steps):
        step()
        tm = s.timing()  # per-phase CUDA-event times of this matvec (the streams each phase ran on)
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
    y_dev = y.clone()

    # e2e: through the C ABI with pinned host buffers (H2D x, matvec, D2H y inside the region)
    nl = s.n
    xh = torch.empty(nl, dtype=torch.float32, pin_memory=True)
    xh.copy_(torch.from_numpy(np.asarray(x_loc, np.float32)))
    yh = torch.empty(nl, dtype=torch.float32, pin_memory=True)
    xh_np, yh_np = xh.numpy(), yh.numpy()
    for _ in range(2):
        s.matvec_host(xh_np, op, yh_np)
    e2e_steps = max(2, min(args.steps, 5))
    if dist:
        dist.barrier()
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        s.matvec_host(xh_np, op, yh_np)
    e2e_s = (time.perf_counter() - t0) / e2e_steps
    if dist:
        t = torch.tensor([e2e_s], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s = float(t.item())

    # BIBEE energy (BASELINE config 5): charge-FMM (E_n, psi) + the FP64 reduction, uncached, device
    # time (CUDA events inside the library) averaged over --bibee-calls calls
    bibee = None
    if not cube and s.n_charges:
        torch.cuda.synchronize()
        s.reset_fields()
        bib = s.bibee("cfa")  # first call: allocations + work lists
        bms, bph = [], []
        for _ in range(args.bibee_calls):
            s.reset_fields()
            bib = s.bibee("cfa")
            tb = s.timing()  # the charge-FMM's phases (until the next matvec)
            bms.append(tb["bibee"])
            bph.append({k: tb[k] for k in ("upward", "m2l", "p2p", "l2p", "total", "p2p_interactions")})
        bms = float(np.mean(bms))
        if dist:
            t = torch.tensor([bms], device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            bms = float(t.item())
        bibee = {"dG_kcal_mol": bib["dG_kcal"], "dG_internal": bib["dG"], "ms": bms, "calls": args.bibee_calls,
                 "charge_terms": args.charge_terms or args.terms,
                 "energies_per_s": 1e3 / bms,
                 "charge_fmm_phases_ms": {k: float(np.mean([b[k] for b in bph])) for k in bph[0]}}

    # one full BEM solve at this size (GMRES iterations, Delta G): GMRES(30) to
    # 1e-6 from a zero guess on the cached charge fields, device time of the solve (CUDA events);
    # the second of two solves (the first allocates the Krylov basis)
    gm = None
    if not cube and s.n_charges and not args.no_solve:
        torch.cuda.synchronize()
        s.solve()  # warm-up: allocates the basis
        r = s.solve()
        tg = s.timing()
        gms = float(tg["gmres"])
        if dist:
            t = torch.tensor([gms], device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            gms = float(t.item())
        gm = {"iterations": int(r["iterations"]), "converged": bool(r["converged"]),
              "rel_residual": float(r["rel_residual"]), "dG_internal": r["dG"], "dG_kcal_mol": r["dG_kcal"],
              "ms": gms, "ms_per_iteration": gms / max(1, int(r["iterations"])), "tol": 1e-6, "restart": 30}
        del r

    p2p_int = int(tm["p2p_interactions"])
    p2p_s = ph["p2p"] * 1e-3
    if dist:  # job-wide P2P rate: all ranks' interactions over the slowest rank's P2P time
        t = torch.tensor([float(p2p_int)], device="cuda", dtype=torch.float64)
        dist.all_reduce(t)
        p2p_int = int(t.item())
        t = torch.tensor([p2p_s], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        p2p_s = float(t.item())
    fpi = FLOPS_PER_INTERACTION_POT if cube else FLOPS_PER_INTERACTION
    p2p_tflops = fpi * p2p_int / p2p_s / 1e12
    peak = fp32_peak_tflops() * world
    hbm, hbm_src = hbm_peak_gbs()
    m2l_pairs = int(tm["m2l_pairs"])
    P = args.terms
    m2l_flops = m2l_rot_flops(P) * m2l_pairs
    traffic = {}
    prof = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(prof):
        try:
            tr = json.load(open(prof))
            if tr.get("config") == wname and int(tr.get("terms", -1)) == P:
                traffic = tr
        except Exception:
            pass
    roof = {"kernel": "k_p2p (near field)", "bound": "alu", "achieved": p2p_tflops, "peak": peak,
            "unit": "TFLOP/s", "frac": p2p_tflops / peak, "traffic": traffic.get("k_p2p"),
            "peak_source": "148 SMs x 128 FP32 lanes x 2 x 1965 MHz (MEASURED_PEAKS.json sm_max_mhz)",
            "work": f"{fpi:.0f} flops per interaction (SURVEY 8(d)) x {p2p_int} exact interactions per launch"}
    # the far-field kernels against the FP32 and the HBM roofline (north star: "M2L/P2M bandwidth
    # against HBM peak"): algorithmic work / the kernel's CUDA-event time
    m2l_rows = int(traffic.get("m2l_rows", 0)) or int(info["n_cells"])
    kern = {}
    for k, phase, work_flops in (("k_m2l_rot_sync", "m2l", m2l_flops), ("k_p2m_t", "p2m", None),
                                 ("k_l2p_t", "leaf_l2p", None)):
        t_s = ph[phase] * 1e-3
        if t_s <= 0:
            continue
        kind = {"m2l": "m2l", "p2m": "p2m", "leaf_l2p": "l2p"}[phase]
        nb = algorithmic_bytes(kind, info, P, s.n, m2l_pairs, m2l_rows)
        d = {"ms": ph[phase], "algorithmic_bytes": nb, "achieved_gbs": nb / t_s / 1e9,
             "hbm_peak_gbs": hbm, "hbm_frac": nb / t_s / 1e9 / hbm, "dram_bytes_ncu": traffic.get(k)}
        if traffic.get(k):
            d["dram_gbs_ncu_bytes_over_event_time"] = traffic[k] / t_s / 1e9
            d["dram_frac"] = traffic[k] / t_s / 1e9 / hbm
        if work_flops:
            d["achieved_tflops"] = work_flops / t_s / 1e12
            d["fp32_frac"] = work_flops / t_s / 1e12 / peak
        kern[k] = d

    out = {"metric": METRIC, "value": value, "unit": "matvec/s", "n_gpus": world, "steps": args.steps,
           "warmup": max(3, args.warmup), "ms_per_step": ms, "higher_is_better": True,
           "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
           "config": {"workload": wname, "n_panels": n, "n_charges": len(cfg["charge_q"]), "terms": P,
                      "input": "each rank builds its block of copies (input_mode 1)" if parts else "full mesh",
                      "quad_points": 1, "leaf_points": args.leaf_points, "near_mode": args.near_mode,
                      "operator": "V (potential)" if cube else "A = I - f K'",
                      "tree_levels": info["levels"], "n_leaves": info["n_leaves"],
                      "l2_flush": f"inputs larger than L2 (x {4 * n / 1e6:.0f} MB, points {32 * n / 1e9:.1f} GB "
                                  "over all ranks; 126 MB L2)",
                      "parallelism": "single GPU" if world == 1 else
                      f"octree domain decomposition x{world} (NCCL: halo x exchange, LET multipole send/recv)"},
           "matvec_s": ms * 1e-3,
           "phases_ms": ph,
           "p2p_ginteractions_s": p2p_int / p2p_s / 1e9,
           "p2p_interactions": p2p_int,
           "p2p_frac_fp32_peak": p2p_tflops / peak,
           "m2l_pairs": m2l_pairs,
           "setup_s": setup_s,
           "tree_build_ms": tm["tree"],
           "bibee_cfa": bibee,
           "gmres_solve": gm,
           "roofline": roof, "roofline_kernels": kern, "hbm_peak_source": hbm_src,
           "gpu_launches": args.steps * launches_per_matvec(info["levels"], P, info if world > 1 else None),
           "e2e": {"value": 1.0 / e2e_s, "unit": "matvec/s", "h2d_bytes_per_step": 4 * n,
                   "d2h_bytes_per_step": 4 * n},
           "comm_ms": ph["comm"],
           "comm_note": ("CUDA events around the LET exchange on the far-field stream: the interval includes "
                         "waiting for SMs held by the persistent P2P kernel (DESIGN.md Sec. 11); the step time "
                         "is the sum of the phases' standalone times") if world > 1 else None,
           "clocks": clocks}
    free, total = torch.cuda.mem_get_info()
    out["device_mem_used_gb"] = (total - free) / 1e9  # this process's device (rank 0 with several)
    out["expansion_slots"] = int(info["expansion_slots"])
    out["n_cells"] = int(info["n_cells"])
    if dist:  # per-rank breakdown (load balance of the domain decomposition)
        mine = {"rank": rank, "n_local": s.n, "phases_ms": ph, "p2p_interactions": int(tm["p2p_interactions"]),
                "m2l_pairs": int(tm["m2l_pairs"]), "device_mem_used_gb": (total - free) / 1e9, "setup_s": setup_s,
                "tree_build_ms": tm["tree"], "expansion_slots": int(info["expansion_slots"]),
                "gpu_launches": args.steps * launches_per_matvec(info["levels"], P, info)}
        allr = [None] * world
        dist.all_gather_object(allr, mine)
        out["per_rank"] = allr
        out["m2l_pairs"] = int(sum(r["m2l_pairs"] for r in allr))
        out["gpu_launches"] = int(sum(r["gpu_launches"] for r in allr))  # all ranks' kernels
    if rank == 0 and world == 1 and not args.no_cpu:
        # the oracle as it stands on this host: FP64 direct sums over ALL sources for a seeded sample
        # of rows; the same rows give the full-size parity of the GPU product
        orc = OracleRows(cfg, x_global, "single" if cube else "kprime")
        rows = np.sort(np.random.default_rng(11).choice(n, min(n, args.cpu_rows), replace=False))
        y_ref, dt = orc(rows)
        y_glob = s.to_global(y_dev.cpu().numpy().astype(np.float64))
        if cube:
            k_gpu, k_ref = y_glob[rows], y_ref  # both carry the 1/(4 pi) of G
            a_gpu, a_ref = k_gpu, k_ref
        else:
            f = 2.0 * (80.0 - 4.0) / 84.0
            k_gpu, k_ref = (x_global[rows] - y_glob[rows]) / f, y_ref
            a_gpu, a_ref = y_glob[rows], x_global[rows] - f * y_ref
        e = k_gpu - k_ref
        out["parity_sampled_rows"] = {"rows": int(len(rows)), "x": "uniform charges" if cube else "N(0,1)",
                                      "rel_l2_op": float(np.linalg.norm(a_gpu - a_ref) / np.linalg.norm(a_ref)),
                                      "rel_l2_kernel_sum": float(np.linalg.norm(e) / np.linalg.norm(k_ref)),
                                      "max_rel_kernel_sum": float(np.abs(e).max() / np.abs(k_ref).max())}
        per_row = dt / len(rows)
        model, ncpu = cpu_info()
        out["cpu_baseline"] = {"value": 1.0 / (per_row * n), "unit": "matvec/s", "cores": orc.cores,
                               "kind": "oracle", "cpu_model": model, "host_cpus": ncpu, "extrapolated": True,
                               "sample": f"FP64 direct {'potential' if cube else 'K-prime'} rows over all {n} "
                                         f"sources: {len(rows)} seeded rows in {dt:.2f} s ({per_row * 1e3:.2f} "
                                         f"ms/row, source weights prepared outside the timed region), "
                                         f"EXTRAPOLATED to the full {n}-row matvec"}
        if bibee is not None:  # sampled-row parity of the BIBEE fields (E_n, psi) at full size
            from oracle import bem
            s.reset_fields()
            En, psi = s.charge_fields()
            En = s.to_global(En.cpu().numpy().astype(np.float64))
            psi = s.to_global(psi.cpu().numpy().astype(np.float64))
            r2 = rows[:2048]
            e_ref = bem.normal_field(orc.pan, cfg["charge_xyz"], cfg["charge_q"], 4.0, rows=r2)
            p_ref = bem.charge_potential(orc.pan, cfg["charge_xyz"], cfg["charge_q"], rows=r2)
            bibee["parity_sampled_rows"] = {
                "rows": int(len(r2)),
                "rel_l2_En": float(np.linalg.norm(En[r2] - e_ref) / np.linalg.norm(e_ref)),
                "rel_l2_psi": float(np.linalg.norm(psi[r2] - p_ref) / np.linalg.norm(p_ref))}
    if rank == 0:
        print(json.dumps(out), flush=True)
    if dist:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
