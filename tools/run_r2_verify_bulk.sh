#!/bin/bash
# After the K2 bulk-store kernel: GPU parity suite, ncu captures of the bulk kernel at both epoch sizes,
# the default bench line, and the bench command's launch list.
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_gpu2.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu2.log
NCU="ncu --clock-control none --set full --import-source on"
$NCU -k regex:gather_hwc_bulk -s 2 -c 1 -f -o gpurun_out/prof3_gather_bulk python tools/profile_kernels.py gather_epoch_hwc_bulk 3 > gpurun_out/ncu3_g.log 2>&1
$NCU -k regex:gather_hwc_bulk -s 2 -c 1 -f -o gpurun_out/prof3_gather_bulk_imagenet python tools/profile_kernels.py gather_imagenet_epoch_hwc_bulk 3 > gpurun_out/ncu3_gi.log 2>&1
timeout 1200 python bench.py > gpurun_out/bench2.json 2> gpurun_out/bench2.err
BENCH="bench.py --steps 1 --warmup 1 --e2e-epochs 0 --no-cpu-baseline --no-colocated --no-vgg"
timeout 1500 ncu --clock-control none --metrics gpu__time_duration.sum --csv --log-file gpurun_out/launches3.csv python $BENCH > gpurun_out/ncu3_bench.log 2>&1
tail -3 gpurun_out/pytest_gpu2.log; tail -3 gpurun_out/bench2.err; head -c 400 gpurun_out/bench2.json
