#!/bin/bash
# fused peer kernel with direct reads: piece size x grid at N=2 and N=4
cd "$(dirname "$0")/.."
O=gpurun_out; mkdir -p $O
for n in 2 4; do
  for cfg in "CSB_P2P_PIECE=4096" "CSB_P2P_PIECE=2048" "CSB_P2P_PIECE=8192" "CSB_P2P_PIECE=1024" "CSB_P2P_CTAS=128" "CSB_P2P_CTAS=296" "CSB_P2P_FENCE=0 CSB_P2P_PIECE=4096"; do
    env $cfg timeout 300 python bench.py --gpus $n --no-extras --no-parity --steps 30 2>/dev/null | grep '^{' | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('N=$n $cfg', d['value'], d['ms_per_step'])" >> $O/p2p_sweep2.log
  done
done
