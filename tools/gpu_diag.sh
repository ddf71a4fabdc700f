#!/bin/bash
cd "$(dirname "$0")/.."
O=gpurun_out; mkdir -p $O
nvidia-smi > $O/d_smi.txt 2>&1
timeout 200 python tools/dbg/dump_run.py 150 __graft_entry__.py smoke > $O/d_smoke.log 2>&1; echo "rc=$?" >> $O/d_smoke.log
timeout 200 python tools/dbg/dump_run.py 120 bench.py --no-extras --no-parity --steps 5 --warmup 3 > $O/d_b1.log 2>&1; echo "rc=$?" >> $O/d_b1.log
CSB_ENGINE_SPIN_US=0 timeout 200 python tools/dbg/dump_run.py 120 bench.py --no-extras --no-parity --steps 5 --warmup 3 > $O/d_b1_nospin.log 2>&1; echo "rc=$?" >> $O/d_b1_nospin.log
