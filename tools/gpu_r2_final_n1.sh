#!/bin/bash
# round-2 final, one GPU: smoke, -m gpu, N=1 bench (ours + reference arm),
# ncu launch list + full capture of the N=1 kernel (each after a plain run exited 0)
cd "$(dirname "$0")/.."
O=gpurun_out; mkdir -p $O
timeout 200 python tools/dbg/dump_run.py 150 __graft_entry__.py smoke > $O/f_smoke.log 2>&1; echo "rc=$?" >> $O/f_smoke.log
timeout 1500 python -m pytest tests -q -m gpu -p no:cacheprovider > $O/f_tests.log 2>&1; echo "rc=$?" >> $O/f_tests.log
timeout 600 python bench.py > $O/f_b1.log 2> $O/f_b1.err; echo "rc=$?" >> $O/f_b1.err
timeout 600 python bench.py --impl reference > $O/f_ref1.log 2>&1; echo "rc=$?" >> $O/f_ref1.log
timeout 300 python bench.py --no-extras --no-parity --steps 5 --warmup 3 > $O/f_ncu_pre.log 2>&1 || exit 1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/r2f_launches_n1.csv \
    python bench.py --no-extras --no-parity --steps 5 --warmup 3 > $O/f_ncu_launch.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:pack_sgd_tab_kernel -s 4 -c 1 -o $O/r2f_pack_sgd_tab_kernel \
    python bench.py --no-extras --no-parity --steps 5 --warmup 3 > $O/f_ncu_full.log 2>&1
