# 2D RAS check: parity tests touching RAS / steps, per-phase cycles, timing on the cfg2 shape
mkdir -p gpurun_out
python -c "from paper_1703_01202_b200 import build as B; B.build()" || exit 1
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "ras or schwarz or cfg1 or cfg2 or device_resident" > gpurun_out/ras2d_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/ras2d_tests.log
tail -3 gpurun_out/ras2d_tests.log
bash tools/gpu_rasprobe.sh 2>&1 | tail -10
timeout 300 python tools/kernel_probe.py ras2d 20 2>&1 | grep "n=  20"
