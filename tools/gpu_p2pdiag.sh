# bench.py with extras at N=4 for nccl vs p2p (kernel split + host profile)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
port=29900
for comm in nccl p2p; do
port=$((port+1))
CSB_HOST_PROFILE=1 timeout 300 python -m torch.distributed.run --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $port bench.py --gpus 4 --steps 100 --warmup 20 --comm $comm --bucket-mb 50 > gpurun_out/diag_$comm.log 2>&1
done
