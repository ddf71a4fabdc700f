# bucket views: GPU tests + bench with/without views at N=1,2,4
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_kvstore_gpu.py -k "views or train_steps" tests/test_torch_dp_gpu.py -x -q > gpurun_out/views_tests.log 2>&1; echo rc=$? >> gpurun_out/views_tests.log
port=29800
for N in 1 2 4; do for v in "" "--grad-views"; do
port=$((port+1))
timeout 600 python -m torch.distributed.run --nproc-per-node $N --master-addr 127.0.0.1 --master-port $port bench.py --gpus $N --steps 50 --warmup 10 $v 2>/dev/null | grep '^{' | sed "s/^/N=$N views=$v /" >> gpurun_out/views_bench.txt
done; done
