mkdir -p gpurun_out
for t in 1 0; do PFC_RAS2_TMEM=$t timeout 300 python tools/kernel_probe.py ras2d 10 2>&1 | grep "2d  *ras"; done
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_graph.py -x -q -k "ras or cfg1 or cfg2 or cfg3 or graph or variant or testC" 2>&1 | tail -2
for spec in "cfg2 47" "cfg1 17" "testC 7"; do
  set -- $spec
  for t in 1 0; do
    PFC_RAS2_TMEM=$t timeout 900 python bench.py --config $1 --steps $2 --warmup 3 --no-cpu-baseline --sweep 0 --extra "" > gpurun_out/bench_m${t}_$1.json 2> gpurun_out/bench_m${t}_$1.err
    python -c "import json,sys; d=json.loads(open('gpurun_out/bench_m${t}_$1.json').read().strip().splitlines()[-1]); k=d['kernel_classes']['ras']; print('$1 tmem=$t', d['value'], 'ras us', round(1e3*k['ms']/k['launches'],1), d['roofline']['frac'])"
  done
done
