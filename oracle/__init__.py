"""CPU ORACLE for arXiv 2111.08272 — TEST INFRASTRUCTURE ONLY.

Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s `cpu_baseline` / `--impl reference` legs may
import, call, link or execute anything under `oracle/`.  The product path
(`paper_2111_08272_b200/`) never imports it and has no CPU fallback.  The oracle shares no code,
header, table or constant generator with the CUDA path; the only common module is `synth/`, which
draws seeded inputs and holds none of the method's arithmetic.

Plain, slow, obviously-correct implementations, fp64 unless a definition fixes another precision.
Citation keys: P:n = /root/reference/PAPER.md line n; S:n = /root/reference/SPEC.md line n;
SURVEY §8(c) #k = the k-th "silent/ambiguous point" reading adopted in DESIGN.md §3.

Parts:
  apportion.py   O1  largest-remainder (Hamilton) rounding
  allocation.py  O2  static allocation init, O8 self-adaptive controller,
                     Eq. 9 / Eq. 22 closed form and the Appendix linear system
  permutation.py O3  per-epoch permutation (Philox4x32-10 Feistel cycle walk),
                 O4  shard indices                                           P:69, P:145 (shuffle: silent)
  gather.py      O5  step-batch row gather with u8 -> f32/bf16 affine
  wavg.py        O6  sample-count-weighted average (Eq. 1) + ring-order emulation
  linmodel.py    O7  logistic-regression closed form, SGD trajectory
  epoch_model.py O9  epoch-time model and the Σspeed-balanced bound

Pins (what each part is checked against, other than itself) are listed in DESIGN.md §4 and tested in
tests/test_oracle_*.py.  Parts without an external pin say "parity unpinned" in their header.
"""
