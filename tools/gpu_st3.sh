timeout 300 python tools/kernel_probe.py st3d 20 2>&1 | grep "3d "
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "residual_jacobian or 512 or config_ics or cfg4" 2>&1 | tail -1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
