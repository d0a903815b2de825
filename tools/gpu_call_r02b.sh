# round-2 dev call: staged-ring cell parity, first-wave prefetch A/B, then the round capture
set -x
KT_CELL_KERNEL=1 timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_guards.py tests/test_gpu_large.py -k "cell" -x -q -p no:cacheprovider > gpurun_out/gputest_r02f_k1.log 2>&1
tail -2 gpurun_out/gputest_r02f_k1.log
for rep in 1 2; do for pf in 1 0; do
  echo "{\"variant\": \"KT_CELL_PF=$pf\"}" >> gpurun_out/ab_r02f.jsonl
  KT_CELL_PF=$pf timeout 300 python tools/ab_stream.py c4_lstm_gates:lstm_cell >> gpurun_out/ab_r02f.jsonl 2>> gpurun_out/ab_r02f.err
done; done
TAG=r02a bash tools/gpu_round_capture.sh
