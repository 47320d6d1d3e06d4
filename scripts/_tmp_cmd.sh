mkdir -p gpurun_out
for W in cfg5 cfg4 cfg2; do timeout 300 python bench.py --workload $W --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_${W}_r1J.log 2>&1; echo "bench $W rc=$?"; done
