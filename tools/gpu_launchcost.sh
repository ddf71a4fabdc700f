# fused-kernel fixed cost: cooperative vs plain launch, explicit fence vs release store only
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
port=29800
for cfg in "1 1" "0 1" "1 0" "0 0"; do set -- $cfg; port=$((port+1))
CSB_P2P_COOP=$1 CSB_P2P_FENCE=$2 timeout 300 python -m torch.distributed.run --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $port tools/p2pbench.py --mb 0.25 4 25 --iters 50 2>&1 | grep "^{" | sed "s/^/coop=$1 fence=$2 /" >> gpurun_out/launchcost.txt
port=$((port+1))
CSB_P2P_COOP=$1 CSB_P2P_FENCE=$2 timeout 300 python -m torch.distributed.run --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $port bench.py --gpus 4 --steps 100 --warmup 10 --no-extras --bucket-mb 25 2>/dev/null | grep '^{' | sed "s/^/coop=$1 fence=$2 bench25 /" >> gpurun_out/launchcost.txt
done
timeout 600 python -m pytest tests/test_nccl_multigpu.py -k "p2p_fused" -x -q > gpurun_out/lc_tests.log 2>&1; echo rc=$? >> gpurun_out/lc_tests.log
