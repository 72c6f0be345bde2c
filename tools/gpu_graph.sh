# f1 graph path (dt on the device): full GPU suite, then graph vs host-loop step rates
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/gpu_tests.log
tail -3 gpurun_out/gpu_tests.log
for spec in "cfg1 17" "cfg2 47" "cfg4 7" "testC 7" "cfg5 3"; do
  set -- $spec
  for g in 1 0; do
    PFC_GRAPH=$g timeout 900 python bench.py --config $1 --steps $2 --warmup 3 --no-cpu-baseline --sweep 0 --extra "" > gpurun_out/bench_g${g}_$1.json 2> gpurun_out/bench_g${g}_$1.err
    python -c "import json,sys; d=json.loads(open('gpurun_out/bench_g${g}_$1.json').read().strip().splitlines()[-1]); print('$1 graph=$g', d['value'], d.get('e2e',{}).get('value'), d.get('gpu_launches'), d.get('newton_its'), d.get('gmres_its'))"
  done
done
