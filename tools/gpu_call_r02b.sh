# round-2 dev call: cell parity (all cell kernels), A/B of variants, ncu of GELU / cell
set -x
R=$GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_guards.py tests/test_gpu_large.py -k "cell or ties or binding or exhaustive_bf16" -x -q -p no:cacheprovider > gpurun_out/gputest_r02d.log 2>&1
tail -2 gpurun_out/gputest_r02d.log
KT_CELL_KERNEL=1 timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_guards.py -k "cell" -x -q -p no:cacheprovider > gpurun_out/gputest_r02d_k1.log 2>&1
tail -2 gpurun_out/gputest_r02d_k1.log
for rep in 1 2; do
for v in default tieser tie2 minb6 tie1; do
  if [ $v = default ]; then unset KT_LIB; else export KT_LIB=$R/abtmp/lib_$v.so; fi
  timeout 300 python tools/ab_stream.py c5_ffn_2p30:kgelu_bf16 c5_ffn_2p30:kswish_bf16 >> gpurun_out/ab_r02d.jsonl 2>> gpurun_out/ab_r02d.err
done
done
unset KT_LIB
for v in default cf1 cf4 k1 k0 default; do
  unset KT_LIB KT_CELL_KERNEL
  case $v in k1) export KT_CELL_KERNEL=1;; k0) export KT_CELL_KERNEL=0;; default) ;; *) export KT_LIB=$R/abtmp/lib_$v.so;; esac
  echo "{\"variant\": \"$v\"}" >> gpurun_out/ab_r02d.jsonl
  timeout 300 python tools/ab_stream.py c4_lstm_gates:lstm_cell >> gpurun_out/ab_r02d.jsonl 2>> gpurun_out/ab_r02d.err
done
unset KT_LIB KT_CELL_KERNEL
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_map -s 3 -c 1 -o gpurun_out/prof_gelu_c5_r02 python tools/profile_targets.py gelu > gpurun_out/ncu_a.log 2>&1
KT_LIB=$R/abtmp/lib_tie2.so timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_map -s 3 -c 1 -o gpurun_out/prof_gelu_c5_tie2_r02 python tools/profile_targets.py gelu > gpurun_out/ncu_b.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_lstm_cell -s 3 -c 1 -o gpurun_out/prof_cell_flat_r02 python tools/profile_targets.py lstm_cell > gpurun_out/ncu_c.log 2>&1
KT_CELL_KERNEL=0 timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_lstm_cell -s 3 -c 1 -o gpurun_out/prof_cell_reg_r02 python tools/profile_targets.py lstm_cell > gpurun_out/ncu_d.log 2>&1
ls gpurun_out
