# 3D stencil check: parity of the operator tests, then isolated timing of J v / residual at 512^3
mkdir -p gpurun_out
python -c "from paper_1703_01202_b200 import build as B; B.build()" || exit 1
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "residual_jacobian or config_ics or 512cubed or cfg4" > gpurun_out/st3_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/st3_tests.log
tail -3 gpurun_out/st3_tests.log
timeout 300 python tools/kernel_probe.py jv3d 20 > gpurun_out/st3_probe.log 2>&1
timeout 300 python tools/kernel_probe.py res3d 20 >> gpurun_out/st3_probe.log 2>&1
cat gpurun_out/st3_probe.log | grep -v warm
if [ "$1" = "ncu" ]; then
timeout 600 ncu --set full --clock-control none --import-source on -k regex:stencil3d -c 1 -o gpurun_out/prof_st3d_v2 -f python tools/kernel_probe.py jv3d 2 > gpurun_out/ncu_st3d.log 2>&1; echo "ncu rc=$?"
fi
