# per-phase cycle counts of the 2D RAS column kernel (diagnostic build of ras2d.cu only)
mkdir -p gpurun_out
python -c "from paper_1703_01202_b200 import build as B; B.build()" || exit 1
PFC_VARIANT_SOURCES=ras2d.cu PFC_LIB_NAME=libpfc_rasprof.so PFC_EXTRA_NVCC_FLAGS=-DPFC_RAS_PROFILE python -c "from paper_1703_01202_b200 import build as B; B.build(force=True)" > /dev/null 2>&1 || echo "build failed"
python tools/ras_phase_probe.py cfg2
