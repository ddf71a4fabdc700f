#!/bin/bash
# piece-size sweep of the fused peer kernels at N=2 and N=4, NVLink probe
# (SM loads/stores vs copy engines), busbw at N=4 with the new default
cd "$(dirname "$0")/.."
O=gpurun_out; mkdir -p $O
for n in 2 4; do
  for pc in 1024 2048 4096 8192 16384; do
    echo "== N=$n piece=$pc" >> $O/piece.log
    CSB_P2P_PIECE=$pc timeout 300 python bench.py --gpus $n --no-extras --no-parity 2>/dev/null | grep '^{' | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'])" >> $O/piece.log 2>&1
  done
done
timeout 300 tools/bin/nvlink_probe 4 100 1 > $O/nvlink_probe_ce_n4.txt 2>&1
timeout 300 tools/bin/nvlink_probe 2 100 1 > $O/nvlink_probe_ce_n2.txt 2>&1
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29533 \
  tools/p2pbench.py --mb 16 64 256 > $O/p2pbench_n4_piece4096.log 2>&1
