# round-2 session-3 baseline: full GPU suite + smoke at HEAD, the 3D stencil probe, ncu --set full
# of the 3D residual kernel at 512^3
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/gpu_tests.log
tail -2 gpurun_out/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
tail -2 gpurun_out/smoke.log
timeout 300 python tools/kernel_probe.py st3d 20 2>&1 | grep "3d "
timeout 600 ncu --set full --clock-control none --import-source on -k regex:stencil3d -c 2 -o gpurun_out/prof_st3d -f python tools/kernel_probe.py st3d 1 > gpurun_out/ncu_st3d.log 2>&1; echo "ncu st3d rc=$?"
