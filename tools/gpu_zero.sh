# ZeRO-1: multi-GPU parity + bench with/without at N=2,4
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_nccl_multigpu.py -k "p2p_fused or torch" -x -q > gpurun_out/zero_tests.log 2>&1; echo rc=$? >> gpurun_out/zero_tests.log
port=29700
for N in 2 4; do for z in "" "--zero"; do for v in "" "--grad-views"; do port=$((port+1))
timeout 600 python -m torch.distributed.run --nproc-per-node $N --master-addr 127.0.0.1 --master-port $port bench.py --gpus $N --steps 50 --warmup 10 --no-extras $z $v 2>/dev/null | grep '^{' | sed "s/^/N=$N zero=$z views=$v /" >> gpurun_out/zero_bench.txt
done; done; done
