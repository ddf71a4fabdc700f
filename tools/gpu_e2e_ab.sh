#!/bin/bash
# e2e double-buffer A/B on one box: N=1 and N=4
cd "$(dirname "$0")/.."
O=gpurun_out; mkdir -p $O
for rep in 1 2; do for v in 1 0; do for n in 1 4; do
  CSB_E2E_DBUF=$v timeout 600 python bench.py --gpus $n --no-parity 2>/dev/null | grep '^{' | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('N=$n DBUF=$v', d['e2e']['value'], d['e2e']['ms_per_step'])" >> $O/e2e_ab.log
done; done; done
