#!/bin/bash
cd "$(dirname "$0")/.."
O=gpurun_out; mkdir -p $O
for i in 1 2 3; do
  (cd headtree && timeout 300 python -m pytest tests/test_kvstore_gpu.py -q -p no:cacheprovider -k aggregation_correctness 2>&1 | tail -2) >> $O/agg_head.log
  timeout 300 python -m pytest tests/test_kvstore_gpu.py -q -p no:cacheprovider -k aggregation_correctness 2>&1 | tail -2 >> $O/agg_cur.log
  CSB_ENGINE_SPIN_US=0 timeout 300 python -m pytest tests/test_kvstore_gpu.py -q -p no:cacheprovider -k aggregation_correctness 2>&1 | tail -2 >> $O/agg_cur_nospin.log
done
