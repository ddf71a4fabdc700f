#!/bin/bash
# round-2 final (4 GPUs): multi-GPU suite, bench at N=2/4 with every leg, every config at N=2/4
cd "$(dirname "$0")/.."
O=gpurun_out; mkdir -p $O
timeout 1200 python -m pytest tests/test_nccl_multigpu.py -q -p no:cacheprovider > $O/h_tests_mg.log 2>&1; echo "rc=$?" >> $O/h_tests_mg.log
for n in 2 4; do
  timeout 600 python tools/dbg/dump_run.py 550 bench.py --gpus $n > $O/h_b$n.log 2> $O/h_b$n.err; echo "rc=$?" >> $O/h_b$n.err
done
timeout 600 python bench.py --impl reference --gpus 4 --steps 5 --warmup 2 > $O/h_ref4.log 2>&1
for n in 2 4; do for cfg in resnet50 alexnet resnet152 inception_v3 uniform16 stress; do
  steps=20; [ $cfg = stress ] && steps=3
  timeout 900 python bench.py --gpus $n --config $cfg --steps $steps --warmup 3 --no-extras 2> /dev/null | grep '^{' | sed "s/^/N=$n cfg=$cfg /" >> $O/h_configs.txt
done; done
