#!/bin/bash
# Affine controller in the linear regime (C3, VGG-16) and on the add-slow-worker pair; bench colocated leg.
mkdir -p gpurun_out
out=gpurun_out/hetero_r2_affine2.jsonl
: > $out
for sc in c4-add-base c4-add; do
  for model in proportional affine; do
    echo "== $sc $model" >&2
    timeout 900 python experiments.py --virtual --scenario $sc --epochs 8 --spin sample --model $model \
      | sed "s/^{/{\"run\": \"$sc-$model\", \"spin_mode\": \"sample\", /" >> $out
  done
done
echo "== c3 affine" >&2
timeout 1500 python experiments.py --virtual --scenario c3 --epochs 4 --spin t1 --model affine \
  | sed "s/^{/{\"run\": \"c3-affine\", \"spin_mode\": \"t1\", /" >> $out
timeout 900 python bench.py --steps 3 --warmup 3 --no-vgg --no-cpu-baseline --e2e-epochs 1 > gpurun_out/bench_coloc.json 2> gpurun_out/bench_coloc.err
python -c "import json; d=json.load(open('gpurun_out/bench_coloc.json')); print(json.dumps(d['allreduce_colocated']['vgg16_C3_P4']))"
