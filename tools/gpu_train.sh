# real ResNet-50 steps: kv vs local vs ddp at N=1 and N=4, after the producer tests
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_torch_dp_gpu.py tests/test_nccl_multigpu.py -k "torch" -x -q > gpurun_out/train_tests.log 2>&1; echo "rc=$?" >> gpurun_out/train_tests.log
port=29600
for N in 1 4; do for impl in local kv ddp; do
port=$((port+1))
timeout 600 python -m torch.distributed.run --nproc-per-node $N --master-addr 127.0.0.1 --master-port $port tools/train_resnet50.py --impl $impl >> gpurun_out/train.txt 2>gpurun_out/train_err_${impl}_$N.log
done; done
port=$((port+1))
timeout 600 python -m torch.distributed.run --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $port tools/train_resnet50.py --impl kv --comm nccl >> gpurun_out/train.txt 2>gpurun_out/train_err_kvnccl_4.log
