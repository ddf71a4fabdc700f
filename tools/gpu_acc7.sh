#!/bin/bash
cd "$(dirname "$0")/.."
O=gpurun_out; mkdir -p $O
for i in 1 2 3 4 5 6; do
  timeout 300 python -m pytest tests/test_metrics_gpu.py -q -p no:cacheprovider -k "acceptance_7 or gauges or overlaps" 2>&1 | tail -1 >> $O/acc7.log
done
timeout 600 python -m pytest tests/test_metrics_gpu.py tests/test_kvstore_gpu.py -q -p no:cacheprovider 2>&1 | tail -1 >> $O/acc7.log
