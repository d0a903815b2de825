# Round evidence capture in one gpurun call (round 2):
#   GPU test suite, bench line (c5 headline) + reference arm, ncu launch list of
#   the bench command, range-replay DRAM traffic per bench line, ncu --set full
#   of the headline kernel and the LSTM cell.  Outputs land in gpurun_out/;
#   the judged summaries are copied to profiles/ by hand.
set -x
R=$GRAFT_REPO_ROOT
TAG=${TAG:-r02}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw,power.limit --format=csv
if [ "${SKIP_TESTS:-0}" != 1 ]; then
  (time timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -s > gpurun_out/gputest_$TAG.log 2>&1) 2> gpurun_out/gputest_$TAG.time
  tail -3 gpurun_out/gputest_$TAG.log
fi
timeout 900 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
tail -c 400 gpurun_out/bench_$TAG.json
timeout 300 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/bench_reference_$TAG.json 2> gpurun_out/bench_reference_$TAG.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 2 --warmup 3 --no-extra --no-cpu > gpurun_out/ncu_launch_$TAG.log 2>&1
if [ "${SKIP_RANGE:-0}" != 1 ]; then
RT="--replay-mode range --csv --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum"
for spec in "c5_ffn_2p30 kgelu_bf16 4" "c5_ffn_2p30 kswish_bf16 4" "c5_ffn_2p30 kgelu_swish_bf16 4" "c3_f32_2p28 ktanh_f32 8" "c2_bf16_2p24 ktanh_bf16 64" "c4_lstm_gates lstm 64"; do
  set -- $spec
  timeout 600 ncu $RT python tools/range_traffic.py $1 $2 $3 > gpurun_out/range_${1}_${2}_$TAG.csv 2> gpurun_out/range_${1}_${2}_$TAG.err
done
fi
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_map -s 3 -c 1 -o gpurun_out/prof_kgelu_c5_$TAG python tools/profile_targets.py gelu > gpurun_out/ncu_full1_$TAG.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_lstm_cell -s 3 -c 1 -o gpurun_out/prof_klstm_cell_c4_$TAG python tools/profile_targets.py lstm_cell > gpurun_out/ncu_full2_$TAG.log 2>&1
ls -la gpurun_out | tail -30
