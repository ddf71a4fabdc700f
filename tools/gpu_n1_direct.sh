#!/bin/bash
cd "$(dirname "$0")/.."
O=gpurun_out; mkdir -p $O
timeout 600 python -m pytest tests/test_single_rank_gpu.py tests/test_kvstore_gpu.py tests/test_peer_local_gpu.py -q -p no:cacheprovider > $O/nd_tests.log 2>&1; echo "rc=$?" >> $O/nd_tests.log
timeout 600 python bench.py > $O/nd_b1.log 2> $O/nd_b1.err; echo "rc=$?" >> $O/nd_b1.err
timeout 300 python bench.py --no-extras --no-parity --no-direct > $O/nd_b1_staged.log 2>&1
timeout 300 python bench.py --no-extras --no-parity --steps 5 --warmup 3 > $O/nd_ncu_pre.log 2>&1 || exit 1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:pack_sgd_tab_kernel -s 4 -c 1 -o $O/r2g_pack_sgd_tab_kernel \
    python bench.py --no-extras --no-parity --steps 5 --warmup 3 > $O/nd_ncu_full.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/r2g_launches_n1.csv \
    python bench.py --no-extras --no-parity --steps 5 --warmup 3 > $O/nd_ncu_launch.log 2>&1
