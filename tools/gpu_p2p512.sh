# peer-memory allreduce variants at 4 ranks (scratch experiment script)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 400 python -m pytest tests/test_nccl_multigpu.py -x -q -k "p2p or nvls" > gpurun_out/push_tests.log 2>&1; echo tests=$?
CSB_P2P_PUSH=0 timeout 240 python -m torch.distributed.run --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29711 tools/p2pbench.py --mb 25 50 100 2>&1 | grep '^{' > gpurun_out/push.json
bash tools/gpu_commsweep.sh 4
