#!/bin/bash
# the 2048-key stress set at N=2: direct gradient reads vs staged
cd "$(dirname "$0")/.."
O=gpurun_out; mkdir -p $O
for a in "" "--no-direct" "--no-zero"; do
  timeout 600 python bench.py --gpus 2 --config stress --steps 3 --warmup 2 --no-extras --no-parity $a 2>/dev/null | grep '^{' | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('$a', d['value'], d['ms_per_step'])" >> $O/stress_ab.log
done
timeout 600 python bench.py --gpus 2 --config resnet50 --no-extras --no-parity 2>/dev/null | grep '^{' | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('resnet50', d['value'], d['ms_per_step'])" >> $O/stress_ab.log
