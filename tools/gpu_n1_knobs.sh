#!/bin/bash
# N=1 streaming-kernel knobs: groups per thread (CSB_SGD_U) x resident CTAs per SM
cd "$(dirname "$0")/.."
O=gpurun_out; mkdir -p $O
for rep in 1 2; do
for cfg in "CSB_SGD_U=1 CSB_STREAM_CTAS_PER_SM=3" "CSB_SGD_U=2 CSB_STREAM_CTAS_PER_SM=2" "CSB_SGD_U=2 CSB_STREAM_CTAS_PER_SM=3" "CSB_SGD_U=1 CSB_STREAM_CTAS_PER_SM=2" "CSB_SGD_U=1 CSB_STREAM_CTAS_PER_SM=4"; do
  env $cfg timeout 300 python bench.py --no-parity --steps 50 --warmup 5 2>/dev/null | grep '^{' | python -c "import sys,json; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$cfg', d['value'], d['ms_per_step'], r['frac'], r['avg_launch_us'])" >> $O/knobs_n1.log
done; done
