# round-end verification: smoke, GPU suite, bench at N=1/2/4, reference arm
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/final_smoke.log 2>&1
timeout 1000 python -m pytest tests -q -m gpu > gpurun_out/final_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/final_tests.log
timeout 400 python bench.py > gpurun_out/final_bench_n1.log 2>&1
for N in 2 4; do
timeout 400 python -m torch.distributed.run --nproc-per-node $N --master-addr 127.0.0.1 --master-port $((29960+N)) bench.py --gpus $N > gpurun_out/final_bench_n$N.log 2>&1
done
timeout 300 python bench.py --impl reference > gpurun_out/final_ref_n1.log 2>&1
