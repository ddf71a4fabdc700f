# full GPU pass: GPU tests, bench at N=1 (all extras) and N=2/4, reference arm at N=1
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 1200 python -m pytest tests -x -q -m gpu > gpurun_out/full_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/full_tests.log
timeout 600 python bench.py > gpurun_out/full_bench_n1.log 2>&1
for N in ${NS:-2 4}; do
timeout 600 python -m torch.distributed.run --nproc-per-node $N --master-addr 127.0.0.1 --master-port $((29950+N)) bench.py --gpus $N > gpurun_out/full_bench_n$N.log 2>&1
done
timeout 600 python bench.py --impl reference > gpurun_out/full_ref_n1.log 2>&1
# real ResNet-50 through the KvStore (replicated / ZeRO-1) vs DDP at N=4
port=29990
for opt in "--impl kv" "--impl kv --zero" "--impl ddp" "--impl local"; do port=$((port+1))
timeout 600 python -m torch.distributed.run --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $port tools/train_resnet50.py $opt 2>/dev/null | grep '^{' >> gpurun_out/full_train4.txt
done
