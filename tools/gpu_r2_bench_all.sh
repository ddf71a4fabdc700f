#!/bin/bash
# full bench lines at N=1/2/4 (schedules, busbw legs), host dispatch profile at
# N=1, small-bucket allreduce latency at N=4
cd "$(dirname "$0")/.."
O=gpurun_out; mkdir -p $O
timeout 600 python bench.py > $O/b_n1.log 2> $O/b_n1.err; echo "rc=$?" >> $O/b_n1.err
CSB_HOST_PROFILE=1 timeout 300 python bench.py --no-extras --no-parity > $O/hostprof_n1.log 2>&1
for n in 2 4; do
  timeout 600 python bench.py --gpus $n > $O/b_n$n.log 2> $O/b_n$n.err; echo "rc=$?" >> $O/b_n$n.err
done
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29533 \
  tools/p2pbench.py --mb 0.25 1 4 16 > $O/p2pbench_small_n4.log 2>&1
