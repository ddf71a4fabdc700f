# bench.py headline at N ranks for each collective engine and bucket size
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
N=${1:-4}; port=29800
for comm in ${COMMS:-nccl p2p}; do for mb in ${MBS:-25 50 100}; do for rep in 1 2; do
port=$((port+1))
timeout 240 python -m torch.distributed.run --nproc-per-node $N --master-addr 127.0.0.1 --master-port $port bench.py --gpus $N --steps 200 --warmup 20 --no-extras --comm $comm --bucket-mb $mb 2>/dev/null | grep '^{' | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$comm', $mb, $rep, d['value'], d['ms_per_step'], d.get('clocks',{}).get('sm_mhz'))" >> gpurun_out/commsweep_n$N.txt
done; done; done
