set -x
timeout 1200 python -m pytest tests/test_gpu_large.py -q -p no:cacheprovider > gpurun_out/gputest_r02t.log 2>&1
tail -3 gpurun_out/gputest_r02t.log
