# round-2 session-3 evidence: default bench (cfg5 headline + other configs + sweeps + CPU
# baseline), the oracle arm, ncu launch list of the default bench's host-loop pass
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --sweep 0 --extra "" > gpurun_out/ncu_launch.log 2>&1; echo "ncu launch rc=$?"
