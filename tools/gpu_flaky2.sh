#!/bin/bash
cd "$(dirname "$0")/.."
O=gpurun_out; mkdir -p $O
for i in 1 2 3; do
  timeout 900 python -m pytest tests -q -m gpu -p no:cacheprovider > $O/flaky2_$i.log 2>&1
  tail -1 $O/flaky2_$i.log >> $O/flaky2.log
done
