set -x
R=$GRAFT_REPO_ROOT
for rep in 1 2; do for v in default ct128 ct128m9 ct128m10 ct64m18; do
  unset KT_LIB; [ $v != default ] && export KT_LIB=$R/abtmp/lib_$v.so
  echo "{\"variant\": \"$v\"}" >> gpurun_out/ab_r02s.jsonl
  timeout 400 python tools/ab_stream.py c4_lstm_gates:lstm_cell >> gpurun_out/ab_r02s.jsonl 2>> gpurun_out/ab_r02s.err
done; done
