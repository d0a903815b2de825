set -x
timeout 600 python -m pytest tests/test_gpu_gemm.py -k tiny -q -s -p no:cacheprovider > gpurun_out/gputest_r02m.log 2>&1
grep -E "ties|passed|failed" gpurun_out/gputest_r02m.log | tail -6
(time timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/gputest_r02n.log 2>&1) 2> gpurun_out/gputest_r02n.time
tail -2 gpurun_out/gputest_r02n.log
