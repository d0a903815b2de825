# round-2: headline with every element of the shard checked against the oracle
set -x
timeout 900 python bench.py --no-extra --full-check > gpurun_out/bench_fullcheck_r02.json 2> gpurun_out/bench_fullcheck_r02.err
python -c "import json;d=json.loads(open('gpurun_out/bench_fullcheck_r02.json').read().strip().splitlines()[-1]);print(d['value'], d['roofline']['frac'], d['per_rank'], d['cpu_baseline']['check'])"
tail -3 gpurun_out/bench_fullcheck_r02.err
