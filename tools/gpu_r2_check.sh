#!/bin/bash
# one GPU: smoke, the -m gpu suite, a flakiness loop, N=1 bench + host profile
cd "$(dirname "$0")/.."
O=gpurun_out; mkdir -p $O
timeout 200 python tools/dbg/dump_run.py 150 __graft_entry__.py smoke > $O/c_smoke.log 2>&1; echo "rc=$?" >> $O/c_smoke.log
timeout 1500 python -m pytest tests -q -m gpu -p no:cacheprovider > $O/c_tests.log 2>&1; echo "rc=$?" >> $O/c_tests.log
for i in 1 2 3 4 5 6; do
  timeout 300 python -m pytest tests/test_kvstore_gpu.py tests/test_metrics_gpu.py -q -p no:cacheprovider -k "aggregation or concom or gauges" 2>&1 | tail -1 >> $O/c_loop.log
done
timeout 600 python tools/dbg/dump_run.py 500 bench.py > $O/c_b1.log 2> $O/c_b1.err; echo "rc=$?" >> $O/c_b1.err
CSB_HOST_PROFILE=1 timeout 300 python tools/dbg/dump_run.py 200 bench.py --no-extras --no-parity > $O/c_hostprof.log 2>&1
