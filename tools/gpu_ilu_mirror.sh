# mirror walls with the factor-based subdomain solves: the ILU / Neumann GPU suites
mkdir -p gpurun_out
python -c "from paper_1703_01202_b200 import build as B; B.build()" || exit 1
timeout 1700 python -m pytest tests/test_gpu_ilu.py tests/test_gpu_neumann.py -x -q 2>&1 | tail -15
