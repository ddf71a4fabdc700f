# ncu evidence for the N=1 bench kernels (run only after the same bench command exits 0 without ncu)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python bench.py --no-extras --steps 5 --warmup 3 > gpurun_out/ncu_pre.log 2>&1 || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r1b_launches.csv \
    python bench.py --no-extras --steps 5 --warmup 3 > gpurun_out/ncu_launch.log 2>&1
for k in sgd_tab_kernel pack_tab_kernel; do
ncu --set full --clock-control none --import-source on -k regex:$k -s 4 -c 1 -o gpurun_out/r1b_$k \
    python bench.py --no-extras --steps 5 --warmup 3 > gpurun_out/ncu_$k.log 2>&1
done
