# NEXT-row measurements on the cfg2 shape (no CPU baseline: the oracle's dense local LU at
# 1296 unknowns per box would take hours)
mkdir -p gpurun_out
timeout 600 python bench.py --bc 1 --no-cpu-baseline > gpurun_out/bench_cfg2_mirror.json 2> gpurun_out/bench_cfg2_mirror.err; echo "mirror rc=$?"
timeout 600 python bench.py --bc 1 --mobility 1 --no-cpu-baseline > gpurun_out/bench_cfg2_mirror_mob.json 2> gpurun_out/bench_cfg2_mirror_mob.err; echo "mirror mob rc=$?"
timeout 900 python bench.py --lu --ilu-reuse 1 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_cfg2_lu.json 2> gpurun_out/bench_cfg2_lu.err; echo "lu rc=$?"
