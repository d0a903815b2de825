set -x
timeout 900 python -m pytest tests/test_bench_contract.py -q -p no:cacheprovider > gpurun_out/gputest_r02x.log 2>&1
tail -2 gpurun_out/gputest_r02x.log
timeout 900 python bench.py --no-extra --full-check > gpurun_out/bench_fullcheck_r02b.json 2> gpurun_out/bench_fullcheck_r02b.err
python -c "import json;d=json.loads(open('gpurun_out/bench_fullcheck_r02b.json').read().strip().splitlines()[-1]);print(d['value'], d['roofline']['frac'], d['per_rank'], d['clocks'])"
