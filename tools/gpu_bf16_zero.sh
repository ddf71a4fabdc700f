#!/bin/bash
cd "$(dirname "$0")/.."
O=gpurun_out; mkdir -p $O
for n in 2 4; do for v in "" "--replicated"; do
  timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $((29820+n)) tools/p2ptrace.py --keyset resnet152 --dtype bf16 --bucket-mb 128 $v 2>/dev/null | grep '^{' >> $O/bf16_zero.log
done; done
