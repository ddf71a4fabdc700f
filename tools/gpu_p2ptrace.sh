#!/bin/bash
cd "$(dirname "$0")/.."
O=gpurun_out; mkdir -p $O
for n in 2 4; do for v in "" "--staged" "--replicated"; do
  timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $((29800+n)) tools/p2ptrace.py $v 2>/dev/null | grep '^{' >> $O/p2ptrace.log
done; done
timeout 300 python -m pytest tests/test_peer_local_gpu.py -q -p no:cacheprovider -x -k "zero or direct" > $O/p2ptrace_tests.log 2>&1; echo "rc=$?" >> $O/p2ptrace_tests.log
