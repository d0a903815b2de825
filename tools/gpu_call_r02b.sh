# round-2: GEMM epilogue tie screen (parity + A/B against the exact-always epilogue)
set -x
R=$GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_parity.py -k "gemm or ties or exhaustive_bf16" -x -q -p no:cacheprovider > gpurun_out/gputest_r02l.log 2>&1
tail -2 gpurun_out/gputest_r02l.log
for rep in 1 2; do for v in default gexact; do
  unset KT_LIB; [ $v != default ] && export KT_LIB=$R/abtmp/lib_$v.so
  echo "{\"variant\": \"$v\"}" >> gpurun_out/ab_r02l.jsonl
  timeout 600 python tools/ab_stream.py gemm:gelu gemm:swish gemm: >> gpurun_out/ab_r02l.jsonl 2>> gpurun_out/ab_r02l.err
done; done
