set -x
for c in c1 c2 c3 c4; do
  timeout 600 python bench.py --config $c --no-extra --steps 50 > gpurun_out/bench_cfg_$c.json 2> gpurun_out/bench_cfg_$c.err; echo "$c rc=$?"
  python -c "import json;d=json.loads(open('gpurun_out/bench_cfg_$c.json').read().strip().splitlines()[-1]);print('$c', d['value'], d['roofline']['frac'], d['roofline']['traffic'], d['e2e']['value'], d['config']['l2'])"
done
