#!/bin/bash
# dynamic ZeRO-1 all-gather (CSB_P2P_DYN=1): parity (colocated + 2/4 GPUs), A/B bench, phase trace
cd "$(dirname "$0")/.."
O=gpurun_out; mkdir -p $O
CSB_P2P_DYN=1 timeout 600 python -m pytest tests/test_peer_local_gpu.py tests/test_configs_gpu.py -q -p no:cacheprovider -x -k "zero or direct or c2 or c5 or torch or stress" > $O/dyn_tests.log 2>&1; echo "rc=$?" >> $O/dyn_tests.log
CSB_P2P_DYN=1 timeout 900 python -m pytest tests/test_nccl_multigpu.py -q -p no:cacheprovider -x -k "zero or p2p_fused or direct or torch or stress" > $O/dyn_tests_mg.log 2>&1; echo "rc=$?" >> $O/dyn_tests_mg.log
for rep in 1 2; do for v in 0 1; do for n in 2 4; do
  CSB_P2P_DYN=$v timeout 300 python bench.py --gpus $n --no-extras --no-parity --steps 30 2>/dev/null | grep '^{' | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('N=$n DYN=$v', d['value'], d['ms_per_step'])" >> $O/dyn_ab.log
done; done; done
for n in 2 4; do
  CSB_P2P_DYN=1 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $((29810+n)) tools/p2ptrace.py 2>/dev/null | grep '^{' >> $O/dyn_trace.log
done
