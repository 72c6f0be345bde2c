# two-phase work plan of the 3D stencils: parity subset, then timing against the chunk-only plan
mkdir -p gpurun_out
python -c "from paper_1703_01202_b200 import build as B; B.build()" || exit 1
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "residual_jacobian or 512 or config_ics or cfg4_3d" 2>&1 | tail -3
ST3_VARIANTS="old:-DST3_TWO_PHASE=0" bash tools/gpu_st3_variants.sh
