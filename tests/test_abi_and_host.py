"""CPU tests of the C-ABI library: it loads, exports every symbol include/propring.h declares, and its
host control plane (pr_alloc_*) is bit-exact against the oracle (SURVEY §4 tier T1)."""

import math
import os
import re

import numpy as np
import pytest

import paper_2111_08272_b200 as pr
from paper_2111_08272_b200 import _lib
from oracle import allocation as A

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared_symbols():
    txt = open(os.path.join(ROOT, "include", "propring.h")).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(pr_[a-z0-9_]+)\s*\(", txt)) - {"pr_exchange_fn"})


def test_library_exports_every_declared_symbol():
    syms = _declared_symbols()
    assert len(syms) >= 25
    for s in syms:
        assert hasattr(_lib.LIB, s), s
        assert s in _lib.SIGNATURES, f"binding lacks {s}"
    assert pr.version() == 10100


def test_library_is_built_for_sm100a():
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_strerror_codes():
    for code in range(0, -13, -1):
        assert _lib.LIB.pr_strerror(code)


def _oracle_view(a):
    return {"w": a.w, "n": a.n, "len": a.len, "off": a.off, "S": a.S, "B": a.B}


def _lib_view(v):
    return {k: v[k] for k in ("w", "n", "len", "off", "S", "B")}


@pytest.mark.parametrize("N,ratios,C,g", [
    (1000, [1, 3], 4, 25), (50000, [1, 2], 3, 128), (51200, [1, 1, 1, 1], 64, 16),
    (50000, [1, 1, 1, 1, 2, 2, 4, 4], 64, 16), (50000, [4, 1, 1, 1, 2, 2, 4, 4], 64, 16),
    (50000, [1, 1, 1, 2, 2, 4, 4], 256, 4), (1281167, [1.0, 2.5, 0.7, 3.3], 1000, 3)])
def test_init_configs_bit_exact(N, ratios, C, g):
    o = A.alloc_init(N, ratios, C=C, g=g)
    l = pr.alloc_init(N, ratios, C=C, g=g).view()
    assert _lib_view(l) == _oracle_view(o)


def test_init_errors_match():
    with pytest.raises(pr.PropringError) as e:
        pr.alloc_init(100, [1, 1, 1], C=2)
    assert e.value.code == pr.PR_ERR_INFEASIBLE_FLOOR
    with pytest.raises(pr.PropringError) as e:
        pr.alloc_init(10, [1, 1], C=20)
    assert e.value.code == pr.PR_ERR_DATASET_TOO_SMALL
    for bad in ([1, -1], [1, float("nan")], [1, float("inf")]):
        with pytest.raises(pr.PropringError) as e:
            pr.alloc_init(10, bad, C=2)
        assert e.value.code == pr.PR_ERR_INVALID
    with pytest.raises(pr.PropringError):
        pr.alloc_init(10, [1.5, 1], C=0)


def test_random_init_and_trajectories_bit_exact():
    """10^4 random (N, P, ratios, C, g, floor) and controller sequences: identical integers."""
    rng = np.random.Generator(np.random.PCG64(2024))
    n_cases = 0
    for case in range(10000):
        P = int(rng.integers(1, 17))
        floor = int(rng.integers(0, 3))
        C = int(rng.integers(max(P * floor, 1), 4 * P + 60))
        g = int(rng.integers(1, 9))
        N = int(g * C * rng.integers(1, 40) + rng.integers(0, 1000))
        kind = case % 3
        ratios = (rng.integers(1, 9, P).astype(float) if kind == 0 else rng.uniform(0.05, 5.0, P))
        try:
            o = A.alloc_init(N, list(ratios), C=C, g=g, floor=floor)
        except (A.InfeasibleFloor, A.DatasetTooSmall, ValueError):
            with pytest.raises(pr.PropringError):
                pr.alloc_init(N, list(ratios), C=C, g=g, floor=floor)
            continue
        l = pr.alloc_init(N, list(ratios), C=C, g=g, floor=floor)
        assert _lib_view(l.view()) == _oracle_view(o), (N, ratios, C, g, floor)
        if case % 10:
            continue
        for ep in range(6):
            mode = rng.integers(0, 4)
            if mode == 0:
                t = rng.uniform(0.1, 10.0, P)
            elif mode == 1:
                t = np.full(P, 2.5)                                  # ties
            elif mode == 2:
                t = np.array(o.w, dtype=float) * rng.uniform(0.5, 2.0, P)   # linear costs
            else:
                t = rng.uniform(0.1, 10.0, P)
                t[rng.integers(0, P)] = [0.0, -1.0, float("nan"), float("inf")][ep % 4]
            try:
                ch_o = A.alloc_update(o, list(t))
                err_o = None
            except A.ZeroTiming:
                err_o = pr.PR_ERR_ZERO_TIMING
            if err_o is None:
                ch_l = l.update(list(t))
                assert ch_l == ch_o
            else:
                with pytest.raises(pr.PropringError) as e:
                    l.update(list(t))
                assert e.value.code == err_o
            v = l.view()
            assert _lib_view(v) == _oracle_view(o) and v["frozen"] == o.frozen and v["epoch"] == o.epoch
            assert v["hist_len"] == len(o.history)
        n_cases += 1
    assert n_cases > 300


def test_controller_spec_examples_via_library():
    a = pr.alloc_init(10 ** 6, [10, 10], C=20)
    a.update([2.0, 1.0])
    assert a.view()["w"] == [7, 13]
    a = pr.alloc_init(10 ** 6, [10, 10, 10], C=30)
    a.update([1.0, 2.0, 5.0])
    assert a.view()["w"] == [18, 9, 3]


def test_policy_and_ema_match_oracle():
    rng = np.random.Generator(np.random.PCG64(77))
    for _ in range(200):
        P = int(rng.integers(2, 9))
        o = A.alloc_init(10 ** 6, [1] * P, C=64)
        l = pr.alloc_init(10 ** 6, [1] * P, C=64)
        al = float(rng.choice([1.0, 0.5, 0.3]))
        o.ema_alpha, o.never_freeze, o.window, o.tol = al, True, 3, 0
        l.set_policy(window=3, tol=0, never_freeze=True, ema_alpha=al)
        for _ in range(5):
            t = list(rng.uniform(0.5, 3.0, P))
            A.alloc_update(o, t)
            l.update(t)
            assert l.view()["w"] == o.w
    with pytest.raises(pr.PropringError):
        l.set_policy(window=1)


def test_save_load_roundtrip_resumes_identically():
    a = pr.alloc_init(51200, [1, 1, 1, 1], C=64, g=16)
    a.set_policy(ema_alpha=0.5, never_freeze=True)
    a.update([2.0, 2.0, 1.0, 1.0])
    b = pr.Alloc.load(a.save())
    assert b.view() == a.view()
    assert [b.history(k) for k in range(2)] == [a.history(k) for k in range(2)]
    for t in ([2.0, 2.1, 1.0, 0.9], [1.0, 1.0, 1.0, 1.0]):
        a.update(t)
        b.update(t)
        assert a.view() == b.view()
    with pytest.raises(pr.PropringError):
        pr.Alloc.load(b"garbage" * 20)


def test_load_rejects_corrupt_checkpoints():
    """pr_alloc_load validates what pr_alloc_init / set_policy would refuse: a corrupt buffer
    must come back as PR_ERR_INVALID, never as a division by zero (C or g = 0), an overflow, or a throw."""
    import struct

    a = pr.alloc_init(51200, [1, 1, 1, 1], C=64, g=16)
    a.update([2.0, 2.0, 1.0, 1.0])
    good = bytearray(a.save())
    assert pr.Alloc.load(bytes(good)).view() == a.view()
    # SaveHeader: magic@0 version@8 P@12 N@16 C@24 g@32 floor@40 epoch@48 frozen@56 has_tprev@60
    #             policy{window@64 never_freeze@68 tol@72 ema@80 model@88 fit_window@92} hist_len@96;
    #             w[P] @104, hist[hist_len][P], t_prev[P], t_hist[hist_len-1][P]
    def patched(off, fmt, val):
        b = bytearray(good)
        struct.pack_into(fmt, b, off, val)
        return bytes(b)

    bad = [patched(24, "<q", 0), patched(32, "<q", 0), patched(16, "<q", 1 << 41), patched(16, "<q", 100),
           patched(40, "<q", 17), patched(48, "<q", -1), patched(56, "<i", 7), patched(64, "<i", 1),
           patched(72, "<q", -1), patched(80, "<d", 0.0), patched(80, "<d", float("nan")),
           patched(88, "<i", 7), patched(92, "<i", 1), patched(92, "<i", 65), patched(60, "<i", 0),
           patched(96, "<q", 1 << 60), patched(96, "<q", 0), patched(96, "<q", 3),
           patched(104, "<q", 17),                     # current w no longer sums to C
           patched(104 + 8 * 4, "<q", -1),             # a history vector with a negative entry
           patched(len(good) - 40, "<d", -1.0),        # a non-positive EMA time (t_prev)
           patched(len(good) - 8, "<d", float("nan")), # a non-finite recorded t (t_hist)
           bytes(good[:-1]), bytes(good) + b"\0"]
    for b in bad:
        with pytest.raises(pr.PropringError):
            pr.Alloc.load(b)


def test_frozen_update_is_noop():
    a = pr.alloc_init(10 ** 6, [10, 10], C=20)
    cost = [1e-3, 2e-3]
    for _ in range(5):
        w = a.view()["w"]
        a.update([w[0] * cost[0], w[1] * cost[1]])
    v = a.view()
    assert v["frozen"] and v["w"] == [13, 7]
    assert a.update([1.0, 100.0]) is False and a.view() == v


def test_header_is_plain_c():
    """The boundary is a C ABI: include/propring.h compiles as C99 (no C++ or torch types)."""
    import shutil
    import subprocess

    cc = shutil.which("gcc") or shutil.which("cc")
    if cc is None:
        import pytest

        pytest.skip("no C compiler")
    hdr = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "include", "propring.h")
    r = subprocess.run([cc, "-fsyntax-only", "-std=c99", "-Wall", "-Werror", "-x", "c", hdr], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr


def test_affine_model_trajectories_bit_exact():
    """PR_ALLOC_MODEL_AFFINE (DESIGN.md §3 #49): 2,000 random controller trajectories — affine, linear and
    noisy step costs, ties, zero-timing rejections, checkpoint/restore mid-run — give the same integers,
    history and frozen flag as the oracle's definition."""
    rng = np.random.Generator(np.random.PCG64(4949))
    for case in range(2000):
        P = int(rng.integers(1, 9))
        floor = int(rng.integers(1, 3))
        C = int(rng.integers(P * floor, 6 * P + 40))
        g = int(rng.integers(1, 5))
        N = g * C * int(rng.integers(1, 20))
        window = int(rng.integers(2, 4))
        fit_window = int(rng.integers(2, 10))
        never = bool(rng.integers(0, 2))
        o = A.alloc_init(N, [1.0] * P, C=C, g=g, floor=floor)
        o.model, o.fit_window, o.window, o.never_freeze = "affine", fit_window, window, never
        l = pr.alloc_init(N, [1.0] * P, C=C, g=g, floor=floor)
        l.set_policy(window=window, never_freeze=never, model=pr.ALLOC_MODEL_AFFINE, fit_window=fit_window)
        fixed = rng.uniform(0.0, 3.0, P) * rng.integers(0, 2)
        per = rng.uniform(0.05, 2.0, P)
        for ep in range(8):
            kind = int(rng.integers(0, 5))
            w = np.array(o.w, dtype=float)
            if kind == 0:
                t = fixed + per * w                                   # affine, noise-free
            elif kind == 1:
                t = (fixed + per * w) * rng.uniform(0.9, 1.1, P)      # noisy (fits may fall back)
            elif kind == 2:
                t = per * w                                           # linear (the paper's model)
            elif kind == 3:
                t = np.full(P, 1.5)                                   # ties
            else:
                t = rng.uniform(0.1, 5.0, P)
                if ep % 3 == 0:
                    t[int(rng.integers(0, P))] = [0.0, float("nan")][ep % 2]
            try:
                ch_o = A.alloc_update(o, list(t))
                err = None
            except A.ZeroTiming:
                err = pr.PR_ERR_ZERO_TIMING
            if err is None:
                assert l.update(list(t)) == ch_o
            else:
                with pytest.raises(pr.PropringError) as e:
                    l.update(list(t))
                assert e.value.code == err
            v = l.view()
            assert v["w"] == o.w and v["frozen"] == o.frozen and v["hist_len"] == len(o.history), (case, ep)
            if ep == 4:                                               # checkpoint / restore mid-trajectory
                l = pr.Alloc.load(l.save())
                assert l.view() == v


def test_binding_constants_match_the_header():
    """Every PR_ALGO_* / PR_COMM_FLAG_* / PR_ERR_* / PR_DTYPE_* #define in include/propring.h has the same value
    in the Python binding (the binding only marshals: a drifted constant would select another kernel)."""
    txt = open(os.path.join(ROOT, "include", "propring.h")).read()
    defs = dict(re.findall(r"#define\s+(PR_(?:ALGO|COMM_FLAG|ERR|DTYPE)_[A-Z0-9_]+)\s+(-?\d+)", txt))
    assert len(defs) >= 15
    for name, val in defs.items():
        py = name[3:]                       # PR_ALGO_RING -> ALGO_RING
        alt = name                          # some error codes keep the PR_ prefix in the binding
        got = getattr(pr, py, getattr(pr, alt, None))
        assert got is not None, f"binding lacks {name}"
        assert int(got) == int(val), (name, got, val)
