"""CPU checks of bench.py's host logic (no GPU): the batch rule per scaling mode, the config both arms
print, the mix-ceiling parser, and the oracle leg's allocation matching the timed arm's."""

import importlib
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def _bench():
    return importlib.import_module("bench")


def test_weak_and_strong_batch_rule():
    b = _bench()
    for n in (1, 2, 4, 8):
        assert b.units_for(n) == 64 * n and b.units_for(n, strong=True) == 64
        cw, cs = b.bench_config(n), b.bench_config(n, strong=True)
        assert cw["global_batch"] == 1024 * n and cs["global_batch"] == 1024
        assert cw["step"] == f"one epoch (S={50_000 // (1024 * n)} aggregations)"
        assert cw["parallelism"] == f"dp{n}"
    assert b.bench_config(1) == b.bench_config(1, strong=True)   # N = 1: the two modes coincide


def test_oracle_leg_allocation_matches_timed_arm():
    from oracle import allocation as OA

    b = _bench()
    for n in (1, 2, 8):
        a = OA.alloc_init(b.N_DATA, [1] * n, C=b.units_for(n), g=b.G_UNIT)
        assert a.n == [1024] * n and a.S == 50_000 // (1024 * n)


def test_mix_ceiling_parser(tmp_path, monkeypatch):
    b = _bench()
    prof = tmp_path / "profiles"
    prof.mkdir()
    (prof / "round1_k2_mix_ceiling.txt").write_text(
        "widen u1 grid 4xSM                 best   81.92 us mean   82.34 us   5529.6 GB/s (best)\n"
        "copy 151MB->151MB grid 4xSM        best   63.49 us mean   64.33 us   4756.6 GB/s (best)\n")
    monkeypatch.setattr(b, "ROOT", str(tmp_path))
    assert b.mix_ceiling() == 5529.6
    (prof / "round1_k2_mix_ceiling.txt").unlink()
    assert b.mix_ceiling() is None
