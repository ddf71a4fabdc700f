# DepCha fused (ZeRO-1) step vs bucket size at N = 2, 4
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
port=29700
for N in 2 4; do for mb in 25 34 50 100; do port=$((port+1))
timeout 600 python -m torch.distributed.run --nproc-per-node $N --master-addr 127.0.0.1 --master-port $port bench.py --gpus $N --steps 100 --warmup 10 --no-extras --bucket-mb $mb 2>/dev/null | grep '^{' | sed "s/^/N=$N mb=$mb /" >> gpurun_out/bucket_sweep.txt
done; done
