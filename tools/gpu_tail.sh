mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_graph.py tests/test_gpu_parity.py -x -q -k "cfg1 or cfg2 or graph or device_resident or host_pointer" 2>&1 | tail -2
for spec in "cfg2 47" "cfg1 17"; do
  set -- $spec
  for t in 1 0; do
    PFC_TAIL_TILE=$t timeout 900 python bench.py --config $1 --steps $2 --warmup 3 --no-cpu-baseline --sweep 0 --extra "" > gpurun_out/bench_t${t}_$1.json 2> gpurun_out/bench_t${t}_$1.err
    python -c "import json,sys; d=json.loads(open('gpurun_out/bench_t${t}_$1.json').read().strip().splitlines()[-1]); k=d['kernel_classes']['orth']; print('$1 tile=$t', d['value'], d.get('e2e',{}).get('value'), 'orth us/launch', round(1e3*k['ms']/k['launches'],2))"
  done
done
