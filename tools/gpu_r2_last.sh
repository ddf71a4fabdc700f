#!/bin/bash
# last check after the final code change: smoke + the -m gpu suite + N=1 bench
cd "$(dirname "$0")/.."
O=gpurun_out; mkdir -p $O
timeout 200 python tools/dbg/dump_run.py 150 __graft_entry__.py smoke > $O/l_smoke.log 2>&1; echo "rc=$?" >> $O/l_smoke.log
timeout 1500 python -m pytest tests -q -m gpu -p no:cacheprovider > $O/l_tests.log 2>&1; echo "rc=$?" >> $O/l_tests.log
timeout 600 python bench.py > $O/l_b1.log 2> $O/l_b1.err; echo "rc=$?" >> $O/l_b1.err
