# R = 6 default for E = 36: full GPU suite, then the 2D workloads
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/gpu_tests.log
tail -2 gpurun_out/gpu_tests.log
for spec in "cfg2 197" "testC 17" "cfg1 17"; do
  set -- $spec
  timeout 900 python bench.py --config $1 --steps $2 --warmup 3 --no-cpu-baseline --sweep 0 --extra "" > gpurun_out/bench_$1.json 2> gpurun_out/bench_$1.err
  python -c "import json; d=json.loads(open('gpurun_out/bench_$1.json').read().strip().splitlines()[-1]); r=d['roofline']; print('$1', d['value'], d['e2e']['value'], r['achieved'], r['frac'], r.get('share_of_step'))"
done
timeout 600 python bench.py --config cfg2 --bc 1 --no-cpu-baseline --sweep 0 --extra "" > gpurun_out/bench_cfg2_mirror.json 2>/dev/null; python -c "import json; d=json.loads(open('gpurun_out/bench_cfg2_mirror.json').read().strip().splitlines()[-1]); print('mirror', d['value'])"
