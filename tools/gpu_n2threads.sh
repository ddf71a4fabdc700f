# 2-GPU reduce phase on all 512 threads: parity + p2pbench + bench
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_nccl_multigpu.py -k "p2p_fused or zero or torch" -x -q > gpurun_out/n2t_tests.log 2>&1; echo rc=$? >> gpurun_out/n2t_tests.log
timeout 300 python -m torch.distributed.run --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29951 tools/p2pbench.py --mb 1 25 100 --iters 30 2>&1 | grep "^{" > gpurun_out/n2t_p2p.json
timeout 300 python -m torch.distributed.run --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29952 bench.py --gpus 2 --steps 100 --warmup 10 --no-extras 2>/dev/null | grep '^{' > gpurun_out/n2t_bench.json
