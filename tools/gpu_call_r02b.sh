# round-2 dev call: parity of the per-kernel unroll build, then unroll A/B
set -x
R=$GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_guards.py tests/test_gpu_exhaustive_f32.py tests/test_gpu_f32_tables.py -x -q -p no:cacheprovider > gpurun_out/gputest_r02h.log 2>&1
tail -2 gpurun_out/gputest_r02h.log
L="c5_ffn_2p30:kgelu_bf16 c5_ffn_2p30:kgelu_swish_bf16 c3_f32_2p28:ktanh_f32 c3_f32_2p28:ktanh_f32_via_bf16"
for rep in 1 2; do for v in default g8 f8 d1m8 g2; do
  unset KT_LIB; [ $v != default ] && export KT_LIB=$R/abtmp/lib_$v.so
  echo "{\"variant\": \"$v\"}" >> gpurun_out/ab_r02h.jsonl
  timeout 400 python tools/ab_stream.py $L >> gpurun_out/ab_r02h.jsonl 2>> gpurun_out/ab_r02h.err
done; done
