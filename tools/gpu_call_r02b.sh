# round-2: headline repeatability (three default bench runs back to back on one box)
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw,power.limit,temperature.gpu --format=csv
for k in 1 2 3; do
  timeout 600 python bench.py --no-extra > gpurun_out/bench_rep${k}_r02.json 2> gpurun_out/bench_rep${k}_r02.err
  python -c "import json;d=json.loads(open('gpurun_out/bench_rep${k}_r02.json').read().strip().splitlines()[-1]);print('rep $k', d['value'], d['roofline']['frac'], d['clocks'])"
done
