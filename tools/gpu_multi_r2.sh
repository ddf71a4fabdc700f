#!/bin/bash
# Round-2 multi-GPU pass (gpurun --gpus 4): NCCL/peer parity tests at 2 and 4
# ranks, the bench at N=2/4 (self-launched), the reference arm at N=4, A/B of
# the in-kernel pack and the interleaved piece map, and the busbw sweep.
cd "$(dirname "$0")/.."
O=gpurun_out
timeout 900 python -m pytest tests/test_nccl_multigpu.py -x -q -p no:cacheprovider > $O/mg_tests.log 2>&1; echo "rc=$?" >> $O/mg_tests.log
for n in 2 4; do
  timeout 600 python bench.py --gpus $n > $O/bench_n$n.log 2> $O/bench_n$n.err; echo "rc=$?" >> $O/bench_n$n.err
done
timeout 600 python bench.py --impl reference --gpus 4 --steps 5 --warmup 2 > $O/bench_ref_n4.log 2>&1
for v in "CSB_P2P_FUSE_PACK=0" "CSB_P2P_PIECE=4096" "CSB_P2P_PIECE=16384" "CSB_P2P_FUSE_PACK=1"; do
  env $v timeout 300 python bench.py --gpus 4 --no-extras --no-parity >> $O/bench_n4_ab.log 2>&1; echo "^ $v" >> $O/bench_n4_ab.log
done
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29533 \
  tools/p2pbench.py --mb 16 64 256 > $O/p2pbench_n4.log 2>&1
