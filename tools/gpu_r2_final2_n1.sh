#!/bin/bash
# round-2 final (one GPU): smoke, -m gpu, N=1 bench + reference arm, every config at N=1
cd "$(dirname "$0")/.."
O=gpurun_out; mkdir -p $O
timeout 200 python tools/dbg/dump_run.py 150 __graft_entry__.py smoke > $O/g_smoke.log 2>&1; echo "rc=$?" >> $O/g_smoke.log
timeout 1500 python -m pytest tests -q -m gpu -p no:cacheprovider > $O/g_tests.log 2>&1; echo "rc=$?" >> $O/g_tests.log
timeout 600 python bench.py > $O/g_b1.log 2> $O/g_b1.err; echo "rc=$?" >> $O/g_b1.err
timeout 600 python bench.py --impl reference > $O/g_ref1.log 2>&1; echo "rc=$?" >> $O/g_ref1.log
for cfg in resnet50 alexnet resnet152 inception_v3 uniform16 stress; do
  steps=20; [ $cfg = stress ] && steps=3
  timeout 900 python bench.py --config $cfg --steps $steps --warmup 3 --no-extras 2> /dev/null | grep '^{' | sed "s/^/N=1 cfg=$cfg /" >> $O/g_configs_n1.txt
done
