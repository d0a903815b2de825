# round-2 dev call: new isolated-tie test, kernel mutants, full F32 derived sweep
set -x
timeout 600 python -m pytest tests/test_gpu_parity.py -k "ties or lstm_cell" -x -q -p no:cacheprovider > gpurun_out/gputest_r02j.log 2>&1
tail -2 gpurun_out/gputest_r02j.log
timeout 2400 python tools/kernel_mutants.py run > gpurun_out/kernel_mutants_r02.txt 2>&1
tail -30 gpurun_out/kernel_mutants_r02.txt
timeout 1800 python tools/f32_derived_sweep.py > gpurun_out/f32_derived_sweep_r02.txt 2>&1
cat gpurun_out/f32_derived_sweep_r02.txt
