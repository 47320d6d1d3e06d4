mkdir -p gpurun_out
GS_TRACE_LEVELS=1 timeout 120 python bench.py --workload cfg2 --steps 1 --warmup 3 --no-cpu-baseline 2>&1 | grep -E "^iter|^level" | tail -60 > gpurun_out/trace_cfg2.log; echo "trace rc=$?"
timeout 900 python -m pytest tests -m gpu -q --timeout 600 -p no:cacheprovider -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log | cut -c1-300
for W in cfg2 cfg1 cfg4 cfg5; do timeout 300 python bench.py --workload $W --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/bench_${W}_r1D.log 2>&1; echo "bench $W rc=$?"; done
