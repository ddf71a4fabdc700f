#!/bin/bash
cd "$(dirname "$0")/.."
O=gpurun_out; mkdir -p $O
timeout 600 python -m pytest tests/test_single_rank_gpu.py -q -p no:cacheprovider > $O/e2e_tests.log 2>&1; echo "rc=$?" >> $O/e2e_tests.log
timeout 600 python bench.py > $O/e2e_b1.log 2>&1
timeout 600 python bench.py --gpus 4 > $O/e2e_b4.log 2>&1
