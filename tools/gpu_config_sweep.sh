# bench.py headline for every config at N = 1, 2, 4 (the per-config table in DESIGN.md)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_nccl_multigpu.py -k "p2p_fused" -x -q > gpurun_out/sweep_tests.log 2>&1; echo rc=$? >> gpurun_out/sweep_tests.log
port=29900
for N in 1 2 4; do for cfg in resnet50 alexnet resnet152 inception_v3 uniform16 stress; do
port=$((port+1)); steps=20; [ $cfg = stress ] && steps=3
timeout 900 python -m torch.distributed.run --nproc-per-node $N --master-addr 127.0.0.1 --master-port $port bench.py --gpus $N --config $cfg --steps $steps --warmup 3 --no-extras 2>gpurun_out/sweep_err_${cfg}_$N.log | grep '^{' | sed "s/^/N=$N cfg=$cfg /" >> gpurun_out/config_sweep.txt
done; done
