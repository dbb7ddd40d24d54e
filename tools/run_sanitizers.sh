#!/bin/bash
# compute-sanitizer (memcheck, racecheck, synccheck) over tools/sanitize_workload.py.
mkdir -p gpurun_out
for tool in memcheck synccheck racecheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_workload.py > gpurun_out/san_$tool.log 2>&1
  echo "$tool exit $?" >> gpurun_out/san_$tool.log
  tail -4 gpurun_out/san_$tool.log
done
