#!/bin/bash
# 4 GPUs: the multi-GPU test suite (NCCL, fused peer kernels incl. direct
# gradient reads over CUDA IPC), bench at N=2/4 with every extra, A/B of
# direct vs staged gradients, the reference arm at N=4
cd "$(dirname "$0")/.."
O=gpurun_out; mkdir -p $O
timeout 1200 python -m pytest tests/test_nccl_multigpu.py -q -p no:cacheprovider > $O/m_tests.log 2>&1; echo "rc=$?" >> $O/m_tests.log
for n in 2 4; do
  timeout 600 python tools/dbg/dump_run.py 550 bench.py --gpus $n > $O/m_b$n.log 2> $O/m_b$n.err; echo "rc=$?" >> $O/m_b$n.err
  timeout 300 python bench.py --gpus $n --no-extras --no-parity --no-direct > $O/m_b${n}_staged.log 2>&1
done
timeout 600 python bench.py --impl reference --gpus 4 --steps 5 --warmup 2 > $O/m_ref4.log 2>&1
