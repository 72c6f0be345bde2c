mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -x -q -k "3d or cfg4 or cfg5 or testD or 3D or ras or graph" > gpurun_out/gpu_tests_3d.log 2>&1; echo "tests rc=$?" >> gpurun_out/gpu_tests_3d.log
tail -3 gpurun_out/gpu_tests_3d.log
RAS3_VARIANTS=cl2p:3,cl2t:3 timeout 300 python tools/ras3_probe.py 512 3
for spec in "cfg5 7" "cfg4 17"; do
  set -- $spec
  timeout 900 python bench.py --config $1 --steps $2 --warmup 3 --no-cpu-baseline --sweep 0 --extra "" > gpurun_out/bench_$1.json 2> gpurun_out/bench_$1.err
  python -c "import json,sys; d=json.loads(open('gpurun_out/bench_$1.json').read().strip().splitlines()[-1]); r=d['roofline']; print('$1', d['value'], d.get('e2e',{}).get('value'), r['achieved'], r['frac'], r.get('share_of_step'))"
done
