# one shared stream vs separate pack/comm/update streams (bench headline)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
port=29600
for N in 1 2 4; do for l in 0 1; do for rep in 1 2; do port=$((port+1))
CSB_KV_LANES=$l timeout 600 python -m torch.distributed.run --nproc-per-node $N --master-addr 127.0.0.1 --master-port $port bench.py --gpus $N --steps 100 --warmup 10 --no-extras 2>/dev/null | grep '^{' | sed "s/^/N=$N lanes1=$l /" >> gpurun_out/lanes.txt
done; done; done
