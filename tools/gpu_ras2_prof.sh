# 2D column kernel: per-phase cycles (diagnostic build) and an ncu --set full capture on cfg2
mkdir -p gpurun_out
timeout 300 python tools/ras_phase_probe.py cfg2
timeout 300 python tools/ras_phase_probe.py cfg1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:ras2d_col -c 1 -o gpurun_out/prof_ras2 -f python tools/kernel_probe.py ras2d 1 > gpurun_out/ncu_ras2.log 2>&1; echo "ncu rc=$?"
