# 2D column kernel: R = 6 rows per thread (8 warps, 255 registers) vs R = 4 (12 warps)
mkdir -p gpurun_out
for r in 4 6 4 6; do
  echo "== R=$r"; PFC_RAS2_ROWS=$r timeout 300 python tools/kernel_probe.py ras2d 20 2>&1 | grep "2d  *ras"
done
PFC_RAS2_ROWS=6 timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "ras_apply_parity or cfg2 or testC or cfg3" 2>&1 | tail -2
for r in 4 6; do
  echo "== bench cfg2 R=$r"; PFC_RAS2_ROWS=$r timeout 600 python bench.py --config cfg2 --steps 47 --warmup 3 --no-cpu-baseline --sweep 0 --extra "" 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['value'], d['roofline']['achieved'], d['roofline']['share_of_step'], d['counts'])"
  echo "== bench testC R=$r"; PFC_RAS2_ROWS=$r timeout 600 python bench.py --config testC --steps 7 --warmup 3 --no-cpu-baseline --sweep 0 --extra "" 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['value'], d['roofline']['achieved'], d['roofline']['share_of_step'], d['counts'])"
done
