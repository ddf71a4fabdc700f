# kv p2p on real ResNet-50 at N=4: fused-kernel grid size x bucket size
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
port=29700
for c in 32 64 148; do for mb in 10 25 50; do
port=$((port+1))
CSB_P2P_CTAS=$c timeout 600 python -m torch.distributed.run --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $port tools/train_resnet50.py --impl kv --bucket-mb $mb 2>/dev/null | grep '^{' | sed "s/^/ctas=$c /" >> gpurun_out/train_sweep.txt
done; done
for mb in 10 50; do port=$((port+1))
timeout 600 python -m torch.distributed.run --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $port tools/train_resnet50.py --impl ddp --bucket-mb $mb 2>/dev/null | grep '^{' >> gpurun_out/train_sweep.txt
done
