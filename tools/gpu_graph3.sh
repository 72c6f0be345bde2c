mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_graph.py -x -q 2>&1 | tail -2
for rep in 1 2; do
for spec in "cfg5 3" "cfg4 7"; do
  set -- $spec
  for g in 1 0; do
    PFC_GRAPH=$g timeout 900 python bench.py --config $1 --steps $2 --warmup 3 --no-cpu-baseline --sweep 0 --extra "" > gpurun_out/bench_g${g}_$1.json 2> gpurun_out/bench_g${g}_$1.err
    python -c "import json,sys; d=json.loads(open('gpurun_out/bench_g${g}_$1.json').read().strip().splitlines()[-1]); print('$1 graph=$g', d['value'], d.get('e2e',{}).get('value'), d['kernel_classes']['ras']['ms']/d['kernel_classes']['ras']['launches'])"
  done
done
done
