#!/bin/bash
# ConCom over the peer-memory kernel: colocated + config tests on one GPU,
# the multi-GPU suite, AlexNet (C3) at N=2/4 p2p vs NCCL, full bench at N=4
cd "$(dirname "$0")/.."
O=gpurun_out; mkdir -p $O
timeout 900 python -m pytest tests/test_peer_local_gpu.py tests/test_configs_gpu.py tests/test_kvstore_gpu.py -q -p no:cacheprovider -x > $O/cc_tests1.log 2>&1; echo "rc=$?" >> $O/cc_tests1.log
timeout 1200 python -m pytest tests/test_nccl_multigpu.py -q -p no:cacheprovider > $O/cc_tests_mg.log 2>&1; echo "rc=$?" >> $O/cc_tests_mg.log
for n in 2 4; do for c in p2p nccl; do
  timeout 300 python bench.py --gpus $n --config alexnet --comm $c --no-extras 2>/dev/null | grep '^{' | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('N=$n $c', d['value'], d['ms_per_step'], d['parity']['bit_exact_vs_restatement'], d['parity']['max_rel_err_vs_f64'])" >> $O/cc_alexnet.log
done; done
timeout 600 python tools/dbg/dump_run.py 550 bench.py --gpus 4 > $O/cc_b4.log 2> $O/cc_b4.err; echo "rc=$?" >> $O/cc_b4.err
