#!/bin/bash
cd "$(dirname "$0")/.."
O=gpurun_out; mkdir -p $O
CSB_P2P_DYN=1 timeout 600 python -m pytest tests/test_peer_local_gpu.py -q -p no:cacheprovider -x -k "zero or direct" > $O/dyn2_tests.log 2>&1; echo "rc=$?" >> $O/dyn2_tests.log
for rep in 1 2 3; do for v in 0 1; do for n in 2 4; do
  CSB_P2P_DYN=$v timeout 300 python bench.py --gpus $n --no-extras --no-parity --steps 50 2>/dev/null | grep '^{' | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('N=$n DYN=$v', d['value'], d['ms_per_step'])" >> $O/dyn2_ab.log
done; done; done
