#!/bin/bash
cd "$(dirname "$0")/.."
O=gpurun_out; mkdir -p $O
for cfg in "X=1" "CSB_P2P_CTAS=296" "CSB_P2P_CTAS=96" "CSB_P2P_COOP=0"; do
  env $cfg timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29901 tools/p2pbench.py --mb 4 16 64 2>/dev/null | grep '^{' | python -c "
import sys, json
d = json.loads(sys.stdin.read())
print('$cfg', {k: (v['p2p_us'], v['p2p_busbw'], v['p2p_fused_sgd_shard_us']) for k, v in d['results'].items()})" >> $O/small.log
done
