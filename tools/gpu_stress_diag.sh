#!/bin/bash
cd "$(dirname "$0")/.."
O=gpurun_out; mkdir -p $O
for rep in 1 2 3; do
  for a in "" "--no-direct" "--bucket-mb 256"; do
    timeout 600 python bench.py --gpus 2 --config stress --steps 5 --warmup 3 --no-extras --no-parity $a 2>/dev/null | grep '^{' | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('rep$rep [$a]', d['value'], d['ms_per_step'])" >> $O/stress_diag.log
  done
done
