# round-2 session-5 evidence at HEAD: full GPU suite, smoke, default bench (cfg5 headline + other
# configs + sweeps + CPU baseline), the oracle arm, ncu launch list of the default bench's
# host-loop pass, ncu --set full of the 3D stencils at 512^3
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/gpu_tests.log
tail -2 gpurun_out/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
tail -2 gpurun_out/smoke.log
timeout 1500 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --sweep 0 --extra "" > gpurun_out/ncu_launch.log 2>&1; echo "ncu launch rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:stencil3d -c 2 -o gpurun_out/prof_st3d_s5 -f python tools/kernel_probe.py st3d 1 > gpurun_out/ncu_st3d.log 2>&1; echo "ncu st3d rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:ras3d_cl2t -c 1 -o gpurun_out/prof_cl2t_s5 -f python tools/kernel_probe.py ras3d 1 > gpurun_out/ncu_cl2t.log 2>&1; echo "ncu cl2t rc=$?"
