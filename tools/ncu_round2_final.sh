#!/bin/bash
# Launch list (gpu__time_duration per launch) of the bench's headline command with the final round-2 code.
#   python tools/summarize_ncu.py round2_final gpurun_out/k1c_refill.ncu-rep --launches gpurun_out/launches2f.csv
mkdir -p gpurun_out
BENCH="bench.py --steps 1 --warmup 1 --e2e-epochs 0 --no-cpu-baseline --no-colocated --no-vgg"
timeout 2400 ncu --clock-control none --metrics gpu__time_duration.sum --csv --log-file gpurun_out/launches2f.csv python $BENCH > gpurun_out/ncu2f_bench.log 2>&1
echo "ncu exit $?"; ls -la gpurun_out/launches2f.csv; tail -n 2 gpurun_out/ncu2f_bench.log | cut -c1-200
