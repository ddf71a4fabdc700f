# bf16 gradient sets: bucket size and ZeRO-1 vs replicated update at N = 2, 4
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
port=29720
for N in 2 4; do for cfg in resnet152 inception_v3; do for opt in "--bucket-mb 25" "--bucket-mb 128" "--bucket-mb 128 --no-zero"; do port=$((port+1))
timeout 300 python -m torch.distributed.run --nproc-per-node $N --master-addr 127.0.0.1 --master-port $port bench.py --gpus $N --config $cfg --steps 50 --warmup 5 --no-extras $opt 2>/dev/null | grep '^{' | sed "s/^/N=$N $cfg $opt /" >> gpurun_out/bf16_sweep.txt
done; done; done
