set -x
R=$GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py -k "fused or ties" -x -q -p no:cacheprovider > gpurun_out/gputest_r02r.log 2>&1
tail -2 gpurun_out/gputest_r02r.log
for rep in 1 2; do for v in default d2m4 d4m4 d4m3 b2m4 b4m3 c3; do
  unset KT_LIB; [ $v != default ] && export KT_LIB=$R/abtmp/lib_$v.so
  echo "{\"variant\": \"$v\"}" >> gpurun_out/ab_r02r.jsonl
  timeout 400 python tools/ab_stream.py c5_ffn_2p30:kgelu_swish_bf16 c5_ffn_2p30:kgelu_bwd_bf16 c4_lstm_gates:lstm_cell >> gpurun_out/ab_r02r.jsonl 2>> gpurun_out/ab_r02r.err
done; done
