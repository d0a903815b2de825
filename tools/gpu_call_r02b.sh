# round-2 functional check of bench.py's N > 1 path on real CUDA (2 ranks on the pool's one GPU:
# NOT a measurement -- the ranks share the GPU), plus smoke()
set -x
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_r02.txt 2>&1; tail -2 gpurun_out/smoke_r02.txt
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 20 --warmup 3 > gpurun_out/bench_n2_functional_r02.json 2> gpurun_out/bench_n2_functional_r02.err
echo rc=$?
tail -c 1500 gpurun_out/bench_n2_functional_r02.json
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29534 bench.py --impl reference --gpus 2 --steps 3 --warmup 3 > gpurun_out/bench_n2_ref_r02.json 2>&1
echo rc=$?
cat gpurun_out/bench_n2_ref_r02.json | tail -2
