# round-2 dev call: K-GELU occupancy / unroll A/B
set -x
R=$GRAFT_REPO_ROOT
L="c5_ffn_2p30:kgelu_bf16 c3_f32_2p28:ktanh_f32"
for rep in 1 2; do for v in default m5 g3 g3m5 g6; do
  unset KT_LIB; [ $v != default ] && export KT_LIB=$R/abtmp/lib_$v.so
  echo "{\"variant\": \"$v\"}" >> gpurun_out/ab_r02k.jsonl
  timeout 400 python tools/ab_stream.py $L >> gpurun_out/ab_r02k.jsonl 2>> gpurun_out/ab_r02k.err
done; done
