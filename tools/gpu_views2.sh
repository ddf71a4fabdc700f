# bucket views in tests + real ResNet-50 at N=4 + bench extras line
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_torch_dp_gpu.py -x -q > gpurun_out/views2_tests.log 2>&1; echo rc=$? >> gpurun_out/views2_tests.log
port=29850
for v in "" "--bucket-views"; do for impl in kv local; do port=$((port+1))
timeout 600 python -m torch.distributed.run --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $port tools/train_resnet50.py --impl $impl $v 2>/dev/null | grep '^{' >> gpurun_out/views2_train.txt
done; done
port=$((port+1))
timeout 600 python -m torch.distributed.run --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $port bench.py --gpus 4 > gpurun_out/views2_bench4.log 2>&1
