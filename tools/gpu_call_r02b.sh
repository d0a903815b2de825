# round-2 dev call: backward / 64-interval unroll A/B, parity of the build
set -x
R=$GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_bwd.py tests/test_gpu_guards.py -x -q -p no:cacheprovider > gpurun_out/gputest_r02i.log 2>&1
tail -2 gpurun_out/gputest_r02i.log
L="c5_ffn_2p30:kgelu_bwd_bf16 c2_bf16_2p24:ktanh64_bf16"
for rep in 1 2; do for v in default b1 b4 b4m4 t64u4 t64u1; do
  unset KT_LIB; [ $v != default ] && export KT_LIB=$R/abtmp/lib_$v.so
  echo "{\"variant\": \"$v\"}" >> gpurun_out/ab_r02i.jsonl
  timeout 400 python tools/ab_stream.py $L >> gpurun_out/ab_r02i.jsonl 2>> gpurun_out/ab_r02i.err
done; done
