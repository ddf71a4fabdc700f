# peer-memory / NVLS allreduce variants at 4 ranks (scratch experiment script)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 240 python -m torch.distributed.run --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29711 tools/p2pbench.py --mb 25 50 100 2>&1 | grep '^{' > gpurun_out/push.json
COMMS="p2p nvls nccl" MBS="50 100" bash tools/gpu_commsweep.sh 4
