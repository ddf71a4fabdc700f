#!/bin/bash
# N=2 regression hunt: current defaults vs knobs vs the round-1 tree (r1tree/)
cd "$(dirname "$0")/.."
O=gpurun_out; mkdir -p $O
run() { echo "== $*" >> $O/n2ab.log; env "$@" timeout 300 python bench.py --gpus 2 --no-extras --no-parity 2>/dev/null | grep '^{' | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'])" >> $O/n2ab.log 2>&1; }
run X=1
run CSB_P2P_FUSE_PACK=0
run CSB_P2P_PIECE=4096
run CSB_P2P_COOP=0
run CSB_P2P_CTAS=296
echo "== --no-zero" >> $O/n2ab.log; timeout 300 python bench.py --gpus 2 --no-extras --no-parity --no-zero 2>/dev/null | grep '^{' | cut -c1-200 >> $O/n2ab.log
echo "== r1tree" >> $O/n2ab.log; (cd r1tree && timeout 300 python -m torch.distributed.run --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29611 bench.py --gpus 2 --no-extras 2>/dev/null | grep '^{' | cut -c1-250) >> $O/n2ab.log
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 \
  tools/p2pbench.py --mb 16 64 100 > $O/p2pbench_n2.log 2>&1
(cd r1tree && timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29534 \
  tools/p2pbench.py --mb 16 64 100 > ../$O/p2pbench_n2_r1.log 2>&1)
