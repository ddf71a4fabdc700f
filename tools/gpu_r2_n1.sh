#!/bin/bash
# Round-2 one-GPU pass: smoke, the full -m gpu suite, the N=1 bench (ours and
# the reference arm), then the ncu launch list and one full capture of the
# top kernel -- each ncu run only after the same command exited 0 without ncu.
cd "$(dirname "$0")/.."
O=gpurun_out; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,temperature.gpu --format=csv > $O/r2_gpu.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/r2_smoke.log 2>&1; echo "rc=$?" >> $O/r2_smoke.log
timeout 1500 python -m pytest tests -q -m gpu -p no:cacheprovider -x > $O/r2_tests.log 2>&1; echo "rc=$?" >> $O/r2_tests.log
timeout 600 python bench.py > $O/r2_bench_n1.log 2> $O/r2_bench_n1.err; echo "rc=$?" >> $O/r2_bench_n1.err
timeout 600 python bench.py --impl reference > $O/r2_ref_n1.log 2>&1; echo "rc=$?" >> $O/r2_ref_n1.log
timeout 300 python bench.py --no-extras --no-parity --steps 5 --warmup 3 > $O/r2_ncu_pre.log 2>&1 || exit 1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/r2_launches_n1.csv \
    python bench.py --no-extras --no-parity --steps 5 --warmup 3 > $O/r2_ncu_launch.log 2>&1
for k in pack_sgd_tab_kernel; do
timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -s 4 -c 1 -o $O/r2_$k \
    python bench.py --no-extras --no-parity --steps 5 --warmup 3 > $O/r2_ncu_$k.log 2>&1
done
