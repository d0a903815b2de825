# round-2: K-GELU threads per CTA A/B (+ parity of the default build)
set -x
R=$GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py -k "gelu or ties or sizes or in_place or exhaustive" -x -q -p no:cacheprovider > gpurun_out/gputest_r02o.log 2>&1
tail -2 gpurun_out/gputest_r02o.log
for rep in 1 2; do for v in default tpb256 tpb64; do
  unset KT_LIB; [ $v != default ] && export KT_LIB=$R/abtmp/lib_$v.so
  echo "{\"variant\": \"$v\"}" >> gpurun_out/ab_r02o.jsonl
  timeout 400 python tools/ab_stream.py c5_ffn_2p30:kgelu_bf16 >> gpurun_out/ab_r02o.jsonl 2>> gpurun_out/ab_r02o.err
done; done
