# DepCha fused (ZeRO-1) step vs bucket size at N ranks
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
N=${1:-2}; port=29700
for mb in 34 50 100; do port=$((port+1))
timeout 600 python -m torch.distributed.run --nproc-per-node $N --master-addr 127.0.0.1 --master-port $port bench.py --gpus $N --steps 100 --warmup 10 --no-extras --bucket-mb $mb 2>/dev/null | grep '^{' | sed "s/^/N=$N mb=$mb /" >> gpurun_out/bucket_sweep.txt
done
