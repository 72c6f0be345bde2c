# 2D stencil check: parity tests that touch 2D operators and steps, then HBM-size timing
mkdir -p gpurun_out
python -c "from paper_1703_01202_b200 import build as B; B.build()" || exit 1
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "residual_jacobian or config_ics or cfg1 or cfg2 or device_resident or host_pointer or constant" > gpurun_out/st2_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/st2_tests.log
tail -3 gpurun_out/st2_tests.log
timeout 300 python tools/kernel_probe.py st2dbig 10 2>&1 | grep "n=  10"
timeout 300 python tools/kernel_probe.py all 10 2>&1 | grep "2d .*n=  10"
if [ "$1" = "ncu" ]; then
timeout 600 ncu --set full --clock-control none --import-source on -k regex:stencil2d --launch-skip 2 -c 2 -o gpurun_out/prof_st2d_big -f python tools/kernel_probe.py st2dbig 2 > gpurun_out/ncu_st2d.log 2>&1; echo "ncu rc=$?"
fi
