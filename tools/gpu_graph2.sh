timeout 900 python -m pytest tests/test_gpu_graph.py -x -q -s 2>&1 | grep -v "^\s*$" | tail -12
PFC_GRAPH=1 PFC_GRAPH_VERBOSE=1 timeout 600 python bench.py --config cfg2 --steps 47 --warmup 3 --no-cpu-baseline --sweep 0 --extra "" 2>&1 >/dev/null | grep "pfc graph"
