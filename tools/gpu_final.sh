# End-of-round evidence: GPU tests, smoke, default bench + ncu (gpu_evidence.sh), then the other
# configurations and the NEXT-row variants (no CPU baseline on those lines)
bash tools/gpu_evidence.sh > gpurun_out/evidence.log 2>&1
for spec in "cfg1 20" "cfg3 10" "cfg4 20" "cfg5 3"; do
  set -- $spec
  timeout 900 python bench.py --config $1 --steps $2 --warmup 3 --no-cpu-baseline > gpurun_out/bench_$1.json 2> gpurun_out/bench_$1.err; echo "$1 rc=$?"
done
timeout 600 python bench.py --bc 1 --no-cpu-baseline > gpurun_out/bench_cfg2_mirror.json 2>/dev/null; echo "mirror rc=$?"
timeout 600 python bench.py --mobility 1 --no-cpu-baseline > gpurun_out/bench_cfg2_mobility.json 2>/dev/null; echo "mobility rc=$?"
timeout 600 python bench.py --ras-variant 2 --no-cpu-baseline > gpurun_out/bench_cfg2_right_ras.json 2>/dev/null; echo "right-ras rc=$?"
