#!/bin/bash
cd "$(dirname "$0")/.."
O=gpurun_out; mkdir -p $O
for rep in 1 2 3; do
  timeout 600 python bench.py --gpus 2 --config stress --steps 5 --warmup 3 --no-extras --no-parity 2>/dev/null | grep '^{' | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('N=2 stress', d['value'], d['ms_per_step'], d['clocks'])" >> $O/stress_rep.log
  CSB_P2P_PIECE=0 timeout 600 python bench.py --gpus 2 --config stress --steps 5 --warmup 3 --no-extras --no-parity 2>/dev/null | grep '^{' | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('N=2 stress piece0', d['value'], d['ms_per_step'])" >> $O/stress_rep.log
done
