# round-2 dev call: compute-sanitizer over every entry point (incl. tie fix-up and the staged cell ring)
set -x
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck racecheck synccheck initcheck; do
  timeout 900 $CS --tool $tool --error-exitcode 9 python tools/sanitize_smoke.py > gpurun_out/sanitize_${tool}_r02.txt 2>&1; echo "$tool rc=$?" >> gpurun_out/sanitize_r02.txt
  KT_CELL_KERNEL=1 timeout 900 $CS --tool $tool --error-exitcode 9 python tools/sanitize_smoke.py > gpurun_out/sanitize_${tool}_ring_r02.txt 2>&1; echo "$tool (KT_CELL_KERNEL=1) rc=$?" >> gpurun_out/sanitize_r02.txt
done
cat gpurun_out/sanitize_r02.txt
