set -x
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_exhaustive_f32.py tests/test_gpu_gemm.py -x -q -p no:cacheprovider > gpurun_out/gputest_r02w.log 2>&1
tail -2 gpurun_out/gputest_r02w.log
timeout 3000 python tools/kernel_mutants.py run > gpurun_out/kernel_mutants_r02b.txt 2>&1
tail -30 gpurun_out/kernel_mutants_r02b.txt
timeout 1800 python tools/f32_derived_sweep.py > gpurun_out/f32_derived_sweep_r02b.txt 2>&1
cat gpurun_out/f32_derived_sweep_r02b.txt
