#!/bin/bash
# one GPU: kernel parity tests after a walker change, then N=1 bench A/B (PDL on/off), 3 runs each
cd "$(dirname "$0")/.."
O=gpurun_out; mkdir -p $O
timeout 900 python -m pytest tests/test_kernels_gpu.py tests/test_single_rank_gpu.py tests/test_configs_gpu.py tests/test_kvstore_gpu.py -q -p no:cacheprovider -x > $O/ab_tests.log 2>&1; echo "rc=$?" >> $O/ab_tests.log
for i in 1 2 3; do
  for v in 1 0; do
    CSB_PDL=$v timeout 300 python bench.py --no-parity --steps 50 --warmup 5 2>/dev/null | grep '^{' | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('PDL=$v', d['value'], d['ms_per_step'], d['roofline']['frac'], d['roofline']['avg_launch_us'])" >> $O/ab_n1.log
  done
done
