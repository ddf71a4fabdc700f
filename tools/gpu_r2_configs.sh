#!/bin/bash
# every config through bench.py (headline + parity) at N = 1, 2, 4
cd "$(dirname "$0")/.."
O=gpurun_out; mkdir -p $O
for N in 1 2 4; do for cfg in resnet50 alexnet resnet152 inception_v3 uniform16 stress; do
  steps=20; [ $cfg = stress ] && steps=3
  timeout 900 python bench.py --gpus $N --config $cfg --steps $steps --warmup 3 --no-extras 2> $O/cfg_err_${cfg}_$N.log | grep '^{' | sed "s/^/N=$N cfg=$cfg /" >> $O/r2_config_sweep.txt
done; done
