#!/bin/bash
# round-2 final, 4 GPUs: bench lines at N=2/4, the stress set after the
# direct-read search fix, real ResNet-50 training (KvStore vs DDP vs local)
cd "$(dirname "$0")/.."
O=gpurun_out; mkdir -p $O
for n in 2 4; do
  timeout 600 python tools/dbg/dump_run.py 550 bench.py --gpus $n > $O/fm_b$n.log 2> $O/fm_b$n.err; echo "rc=$?" >> $O/fm_b$n.err
done
for n in 1 2 4; do
  timeout 900 python bench.py --gpus $n --config stress --steps 3 --warmup 3 --no-extras 2> /dev/null | grep '^{' | sed "s/^/N=$n cfg=stress /" >> $O/fm_stress.txt
done
port=29600
for N in 1 4; do for impl in local kv ddp; do
  port=$((port+1))
  timeout 600 python -m torch.distributed.run --nproc-per-node $N --master-addr 127.0.0.1 --master-port $port tools/train_resnet50.py --impl $impl >> $O/fm_train.txt 2> $O/fm_train_err_${impl}_$N.log
done; done
