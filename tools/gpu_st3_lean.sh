# producer-free 3D stencils (s in place): parity, then timing against the producer kernels
mkdir -p gpurun_out
python -c "from paper_1703_01202_b200 import build as B; B.build()" || exit 1
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "residual_jacobian or 512 or config_ics or cfg4_3d" 2>&1 | tail -3
for prod in 0 1; do
  echo "== PFC_ST3_PROD=$prod"
  PFC_ST3_PROD=$prod timeout 300 python tools/kernel_probe.py st3d 20 2>&1 | grep "3d "
done
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
