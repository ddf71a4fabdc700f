#!/bin/bash
# minimum pieces per CTA (CSB_P2P_KMIN) on the stress set and the plain allreduce sizes
cd "$(dirname "$0")/.."
O=gpurun_out; mkdir -p $O
for k in 1 2; do
  for n in 2 4; do
    CSB_P2P_KMIN=$k timeout 600 python bench.py --gpus $n --config stress --steps 3 --warmup 2 --no-extras --no-parity 2>/dev/null | grep '^{' | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('KMIN=$k N=$n stress', d['value'], d['ms_per_step'])" >> $O/kmin.log
  done
  for n in 2 4; do
    CSB_P2P_KMIN=$k timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $((29700+n+k)) tools/p2pbench.py --mb 16 64 256 2>/dev/null | grep '^{' | sed "s/^/KMIN=$k N=$n /" >> $O/kmin.log
  done
done
