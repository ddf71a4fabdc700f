#!/bin/bash
cd "$(dirname "$0")/.."
O=gpurun_out; mkdir -p $O
timeout 600 python -m pytest tests/test_nccl_multigpu.py -q -p no:cacheprovider -k "direct or funnel" > $O/fdm.log 2>&1; echo "rc=$?" >> $O/fdm.log
for n in 2 4; do for a in "" "--no-direct"; do
  timeout 300 python bench.py --gpus $n --mode funnel --no-extras $a 2>/dev/null | grep '^{' | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('N=$n funnel [$a]', d['value'], d['ms_per_step'], d['parity']['bit_exact_vs_restatement'])" >> $O/fdm.log
done; done
