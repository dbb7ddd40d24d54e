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
    """Default = strong scaling (SURVEY §8(d) Scaling row: fixed global batch 1,024 for every N)."""
    b = _bench()
    for n in (1, 2, 4, 8):
        assert b.units_for(n) == 64 and b.units_for(n, strong=False) == 64 * n
        cs, cw = b.bench_config(n), b.bench_config(n, strong=False)
        assert cw["global_batch"] == 1024 * n and cs["global_batch"] == 1024
        assert cw["step"] == f"one epoch (S={50_000 // (1024 * n)} aggregations)"
        assert cs["step"] == "one epoch (S=48 aggregations)" and cs["scaling"] == "strong"
        assert cw["parallelism"] == f"dp{n}"
        v = b.bench_config(n, workload="vgg16")
        assert v["global_batch"] == 1024 and v["step"] == "one epoch (S=50 aggregations)"
        assert "138,357,544" in v["workload"]
    c1s, c1w = b.bench_config(1), b.bench_config(1, strong=False)
    c1s.pop("scaling"), c1w.pop("scaling")
    assert c1s == c1w                                              # N = 1: the two modes coincide


def test_self_launch_command(monkeypatch):
    """--gpus N > 1 without WORLD_SIZE re-runs bench.py under torch.distributed.run (127.0.0.1)."""
    b = _bench()
    seen = {}
    monkeypatch.setattr(b.subprocess, "call", lambda cmd: seen.setdefault("cmd", cmd) and 0)
    a = b.parse(["--gpus", "4", "--steps", "2"])
    b.self_launch(a, ["--gpus", "4", "--steps", "2"])
    cmd = seen["cmd"]
    assert cmd[1:4] == ["-m", "torch.distributed.run", "--nnodes=1"] and "--nproc-per-node=4" in cmd
    assert cmd[cmd.index("--master-addr") + 1] == "127.0.0.1" and cmd[-3:] == ["--gpus", "4", "--steps", "2"][-3:]


def test_reference_arm_does_not_load_the_product():
    """The oracle arm builds torchvision's ResNet-18 directly: importing bench + running its setup must not
    load libpropring.so (VERDICT r1 "What's weak" #1)."""
    import subprocess

    code = ("import sys; sys.argv=['bench.py']; import bench; bench.cpu_reference_setup(1); "
            "import os; maps=open('/proc/self/maps').read(); print('LOADED' if 'libpropring' in maps else 'CLEAN'); "
            "print('MOD' if any(m.startswith('paper_2111_08272_b200') for m in sys.modules) else 'NOMOD')")
    out = subprocess.run([sys.executable, "-c", code], cwd=ROOT, capture_output=True, text=True, timeout=300).stdout
    assert "CLEAN" in out and "NOMOD" in out, out


def test_oracle_leg_allocation_matches_timed_arm():
    from oracle import allocation as OA

    b = _bench()
    for n in (1, 2, 8):
        a = OA.alloc_init(b.N_DATA, [1] * n, C=b.units_for(n, strong=False), g=b.G_UNIT)
        assert a.n == [1024] * n and a.S == 50_000 // (1024 * n)
        s = OA.alloc_init(b.N_DATA, [1] * n, C=b.units_for(n), g=b.G_UNIT)
        assert sum(s.n) == 1024 and s.S == 48


def test_mix_ceiling_parser(tmp_path, monkeypatch):
    """The K2 ceiling is the best 1:2 widen line of the ImageNet-size mix probe (the plain copy lines and
    the mean columns are not it)."""
    b = _bench()
    prof = tmp_path / "profiles"
    prof.mkdir()
    (prof / "round2_k2_mix_probe_imagenet.txt").write_text(
        "clean  widen stg grid 4xSM            best   1239.0 us mean   1241.3 us   5971.4 GB/s best   5960.7 GB/s mean\n"
        "clean  copy 1:1 grid 8xSM             best    792.6 us mean    805.5 us   6223.4 GB/s best   6123.3 GB/s mean\n"
        "dirty  widen tma-store grid 3xSM      best   1183.7 us mean   1186.1 us   6250.3 GB/s best   6237.7 GB/s mean\n")
    monkeypatch.setattr(b, "ROOT", str(tmp_path))
    assert b.mix_ceiling() == 6250.3
    (prof / "round2_k2_mix_probe_imagenet.txt").unlink()
    assert b.mix_ceiling() is None
