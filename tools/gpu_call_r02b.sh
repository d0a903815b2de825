set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw,power.limit --format=csv
(time timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/gputest_r02n.log 2>&1) 2> gpurun_out/gputest_r02n.time
tail -3 gpurun_out/gputest_r02n.log
timeout 900 python bench.py > gpurun_out/bench_r02n.json 2> gpurun_out/bench_r02n.err
tail -c 300 gpurun_out/bench_r02n.json
python -c "import ast,__graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke_r02n.log 2>&1; tail -1 gpurun_out/smoke_r02n.log
