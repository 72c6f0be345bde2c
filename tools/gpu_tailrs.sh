for rs in 1 2 4 16; do
  PFC_TAIL_RS=$rs timeout 600 python bench.py --config cfg1 --steps 17 --warmup 3 --no-cpu-baseline --sweep 0 --extra "" > gpurun_out/b_rs$rs.json 2>/dev/null
  python -c "import json; d=json.loads(open('gpurun_out/b_rs$rs.json').read().strip().splitlines()[-1]); k=d['kernel_classes']['orth']; print('cfg1 rs=$rs', d['value'], 'orth us', round(1e3*k['ms']/k['launches'],2))"
done
