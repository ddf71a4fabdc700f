#!/bin/bash
# the -m gpu suite several times in a row (flakiness hunt), smoke between runs
cd "$(dirname "$0")/.."
O=gpurun_out; mkdir -p $O
for i in 1 2 3 4; do
  timeout 900 python -m pytest tests -q -m gpu -p no:cacheprovider 2>&1 | tail -4 >> $O/flaky.log
  echo "---" >> $O/flaky.log
done
