"""bench.py's counting conventions (DESIGN.md Sec. 5 / 11), checked on the CPU: the algorithmic
flops per M2L translation and per P2P interaction, and the kernel launches per matvec."""
import importlib.util
import os

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _bench():
    spec = importlib.util.spec_from_file_location("bench_mod", os.path.join(ROOT, "bench.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


def test_m2l_flops_per_translation():
    b = _bench()
    P = 12
    nc = P * (P + 1) // 2
    mat = 4 * 2 * sum((n + 1) ** 2 for n in range(P))   # four fixed-matrix stages, 2 flops per FMA
    coax = 2 * 2 * sum((P - k) ** 2 for k in range(P))  # (re, im) FMAs of the coaxial translation
    phases = 4 * 6 * (nc - P)                          # complex products for m > 0
    assert b.m2l_rot_flops(P) == mat + coax + phases + 4 * nc == 9696


def test_launches_per_matvec_c5():
    b = _bench()
    # leaf level 8: P2M, 6 x (M2M rotate + sum), M2L, 6 L2L, P2P weight max + source table, P2P, L2P
    assert b.launches_per_matvec(8, 13) == 1 + 2 * 6 + 1 + 6 + 2 + 1 + 1 == 24
    assert b.launches_per_matvec(1, 13) == 3  # no far field: weight max + source table + P2P


def test_p2p_flop_convention():
    assert _bench().FLOPS_PER_INTERACTION == 19
