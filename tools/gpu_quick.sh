#!/bin/bash
# quick re-measure: N=1 full bench + host profile, N=4 full bench
cd "$(dirname "$0")/.."
O=gpurun_out; mkdir -p $O
timeout 600 python bench.py > $O/q_n1.log 2> $O/q_n1.err; echo "rc=$?" >> $O/q_n1.err
CSB_HOST_PROFILE=1 timeout 300 python bench.py --no-extras --no-parity > $O/q_hostprof_n1.log 2>&1
[ "${1:-1}" -gt 1 ] && timeout 600 python bench.py --gpus $1 > $O/q_n$1.log 2> $O/q_n$1.err
exit 0
