set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 300 python tools/kernel_probe.py st3d 20 > gpurun_out/st3_probe.log 2>&1
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1; echo "ncu1 rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:ras2d_col -c 1 -o gpurun_out/prof_ras2d_col -f python tools/kernel_probe.py ras2d 2 > gpurun_out/ncu_ras2d.log 2>&1; echo "ncu2 rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:stencil3d --launch-skip 2 -c 2 -o gpurun_out/prof_st3d -f python tools/kernel_probe.py st3d 2 > gpurun_out/ncu_st3d.log 2>&1; echo "ncu3 rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:stencil2d_kernel --launch-skip 2 -c 2 -o gpurun_out/prof_st2d_big -f python tools/kernel_probe.py st2dbig 2 > gpurun_out/ncu_st2d.log 2>&1; echo "ncu5 rc=$?"
timeout 300 python tools/kernel_probe.py st2dsz 20 > gpurun_out/st2_probe.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:ras3d_col -c 1 -o gpurun_out/prof_ras3d_col -f python tools/kernel_probe.py ras3d 2 > gpurun_out/ncu_ras3d.log 2>&1; echo "ncu4 rc=$?"
