#!/bin/bash
cd "$(dirname "$0")/.."
O=gpurun_out; mkdir -p $O
for n in 1 2 4; do for b in 64 128 256; do
  timeout 600 python bench.py --gpus $n --config stress --bucket-mb $b --steps 3 --warmup 3 --no-extras --no-parity 2>/dev/null | grep '^{' | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('N=$n bucket=$b', d['value'], d['ms_per_step'], d['buckets'])" >> $O/stress_256.log
done; done
