# allreduce bus bandwidth vs bucket size at N ranks: NCCL, peer-memory kernel, NVLS kernel
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
N=${1:-4}
timeout 600 python -m torch.distributed.run --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29777 tools/p2pbench.py --mb 16 64 256 1024 --iters 10 2>&1 | grep '^{' > gpurun_out/busbw_n$N.json
