#!/bin/bash
# Everything that cannot be measured on a one-GPU box, for the first call that gets > 1 GPU.
# Output -> gpurun_out/mg_*.  Usage: bash tools/multigpu_first_run.sh [max GPUs, default 8]
G=${1:-8}
mkdir -p gpurun_out
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
nvidia-smi topo -m > gpurun_out/mg_topo.txt 2>&1
for P in 2 4 8; do
  [ $P -gt $G ] && break
  # C5: K3 (ring) vs NCCL premul-sum / scale+sum, 1 MiB .. 1 GiB, fp32 + bf16, parity on samples
  timeout 1200 $TR --nproc-per-node $P --master-port $((29600 + P)) tools/ar_sweep.py --max-mib 1024 \
      > gpurun_out/mg_ar_sweep_p$P.jsonl 2> gpurun_out/mg_ar_sweep_p$P.err
  # the bench at N = P, without and with N1 overlap
  timeout 1200 $TR --nproc-per-node $P --master-port $((29610 + P)) bench.py --gpus $P --steps 5 --warmup 3 \
      > gpurun_out/mg_bench_p$P.json 2> gpurun_out/mg_bench_p$P.err
  timeout 1200 $TR --nproc-per-node $P --master-port $((29620 + P)) bench.py --gpus $P --steps 5 --warmup 3 --overlap \
      --no-cpu-baseline > gpurun_out/mg_bench_overlap_p$P.json 2> gpurun_out/mg_bench_overlap_p$P.err
  timeout 1200 $TR --nproc-per-node $P --master-port $((29660 + P)) bench.py --gpus $P --steps 5 --warmup 3 --weak \
      --no-cpu-baseline --no-vgg > gpurun_out/mg_bench_weak_p$P.json 2> gpurun_out/mg_bench_weak_p$P.err
  # TMA bulk-store data path vs 16-byte STG over real NVLink (co-located proxy: 5-8 % slower)
  timeout 900 $TR --nproc-per-node $P --master-port $((29670 + P)) tools/ar_sweep.py --max-mib 256 --bulk \
      > gpurun_out/mg_ar_sweep_bulk_p$P.jsonl 2> gpurun_out/mg_ar_sweep_bulk_p$P.err
  # L2 prefetch of the own gradient before the flag waits (co-located proxy: 13 % slower per channel)
  timeout 900 $TR --nproc-per-node $P --master-port $((29690 + P)) tools/ar_sweep.py --max-mib 256 --l2pf \
      > gpurun_out/mg_ar_sweep_l2pf_p$P.jsonl 2> gpurun_out/mg_ar_sweep_l2pf_p$P.err
  # pull two-shot (peer loads instead of pushes; co-located proxy: 1.6-2.3x the ring per channel)
  timeout 900 $TR --nproc-per-node $P --master-port $((29710 + P)) tools/ar_sweep.py --max-mib 1024 --algo 6 \
      > gpurun_out/mg_ar_sweep_pull_p$P.jsonl 2> gpurun_out/mg_ar_sweep_pull_p$P.err
  # the same with its source tiles TMA-staged in shared memory (deeper queue for remote reads)
  PR_AR_SWEEP_PULL_TMA=1 timeout 900 $TR --nproc-per-node $P --master-port $((29730 + P)) tools/ar_sweep.py --max-mib 1024 --algo 6 \
      > gpurun_out/mg_ar_sweep_pull_tma_p$P.jsonl 2> gpurun_out/mg_ar_sweep_pull_tma_p$P.err
  # NVLS (in-switch reduction), where the box can create a multicast object
  timeout 900 $TR --nproc-per-node $P --master-port $((29680 + P)) tools/ar_sweep.py --max-mib 1024 --algo 5 \
      > gpurun_out/mg_ar_sweep_nvls_p$P.jsonl 2> gpurun_out/mg_ar_sweep_nvls_p$P.err
done
# ring channel count (CTAs per rank) at the largest P: 16 is the co-located optimum, NVLink may want more
for ch in 16 24 32 48 64; do
  timeout 900 $TR --nproc-per-node $G --master-port $((29650 + ch)) tools/ar_sweep.py --max-mib 256 --channels $ch \
      > gpurun_out/mg_ar_sweep_ch${ch}_p$G.jsonl 2> gpurun_out/mg_ar_sweep_ch${ch}_p$G.err
done
# ring slicing A/B on NVLink: G slices per phase (min_slice_bytes) vs slot-sized slices
for ms in 65536 262144; do
  timeout 900 $TR --nproc-per-node $G --master-port $((29700 + ms / 65536)) tools/ar_sweep.py --max-mib 256 --min-slice $ms \
      > gpurun_out/mg_ar_sweep_ms${ms}_p$G.jsonl 2> gpurun_out/mg_ar_sweep_ms${ms}_p$G.err
done
# AUTO (one-shot / LL / two-shot / ring by size) at the largest P
timeout 1200 $TR --nproc-per-node $G --master-port 29630 tools/ar_sweep.py --max-mib 64 --algo 2 \
    > gpurun_out/mg_ar_sweep_auto_p$G.jsonl 2> gpurun_out/mg_ar_sweep_auto_p$G.err
# emulated heterogeneity one rank per GPU (C4 scenarios need 8)
[ $G -ge 8 ] && timeout 1800 $TR --nproc-per-node 8 --master-port 29640 experiments.py --scenario c4 \
    > gpurun_out/mg_c4.jsonl 2> gpurun_out/mg_c4.err
[ $G -ge 8 ] && timeout 1800 $TR --nproc-per-node 8 --master-port 29642 experiments.py --scenario c4 --spin sample \
    --model affine > gpurun_out/mg_c4_affine.jsonl 2> gpurun_out/mg_c4_affine.err
[ $G -ge 4 ] && timeout 1800 $TR --nproc-per-node 4 --master-port 29641 experiments.py --scenario c3 \
    > gpurun_out/mg_c3.jsonl 2> gpurun_out/mg_c3.err
ls -la gpurun_out/mg_*
