# Round-end evidence capture (one gpurun call): bench line, reference arm,
# ncu launch list of the bench command, and ncu --set full of the main kernels.
set -x
timeout 900 python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err
timeout 300 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-extra --no-cpu > gpurun_out/ncu_launch.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_map -s 3 -c 1 -o gpurun_out/prof_tanh_bf16_c2 python tools/profile_targets.py tanh_bf16 > gpurun_out/ncu1.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:'k_gemm_tILi9' -s 2 -c 1 -o gpurun_out/prof_gemm_cell python tools/gemm_one.py 6400 4096 1024 cell > gpurun_out/ncu2.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:'k_gemm_tILin1ELi2'  -s 2 -c 1 -o gpurun_out/prof_gemm_pair python tools/gemm_one.py 16384 16384 4096 none > gpurun_out/ncu3.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_lstm_cell -s 3 -c 1 -o gpurun_out/prof_cell python tools/profile_targets.py lstm_cell > gpurun_out/ncu4.log 2>&1
ls -la gpurun_out
