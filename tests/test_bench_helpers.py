"""bench.py's launch count pinned by measurement: the ncu launch list of the bench command
(`profiles/r2_final_launches_bench_c5.csv`, every kernel the process launched, in launch order) shows
exactly launches_per_matvec(L, P) of the library's kernels per device-path A-matvec at C5 (leaf level
8, P = 13) -- the count the bench line reports as gpu_launches / steps."""
import csv
import importlib.util
import os
import re

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _bench():
    spec = importlib.util.spec_from_file_location("bench_mod", os.path.join(ROOT, "bench.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


def _launch_sequence(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
    hdr = rows[hi]
    ix = {h: i for i, h in enumerate(hdr)}
    seen, seq = set(), []
    for r in rows[hi + 1:]:
        if len(r) < len(hdr) or r[ix["ID"]] in seen:
            continue
        seen.add(r[ix["ID"]])
        m = re.search(r"\b(k_[a-z0-9_]+)", r[ix["Kernel Name"]])
        seq.append(m.group(1) if m else "lib:" + r[ix["Kernel Name"]][:40])
    return seq


def test_launches_per_matvec_equals_the_ncu_launch_list():
    b = _bench()
    seq = _launch_sequence(os.path.join(ROOT, "profiles", "r2_final_launches_bench_c5.csv"))
    ours = [k for k in seq if k.startswith("k_")]
    starts = [i for i, k in enumerate(ours) if k == "k_p2m_t"]
    groups = [ours[a:b] for a, b in zip(starts, starts[1:])]
    # device-path matvecs: one P2M, one M2L, one P2P, no setup (work-item) kernels in between
    steady = [g for g in groups if g.count("k_p2m_t") == 1 and g.count("k_m2l_rot_sync") == 1 and "k_absmax" in g
              and g.count("k_p2p") == 1 and "k_item_count" not in g]
    assert len(steady) >= 3
    want = b.launches_per_matvec(8, 13)
    assert all(len(g) == want for g in steady), [len(g) for g in steady]
    assert want == 24


def test_p2p_flop_convention():
    # FADD/FMUL = 1, FFMA = 2, MUFU.RSQ = 1 -> 19 flops per K' interaction
    assert _bench().FLOPS_PER_INTERACTION == 19
