mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke.log
timeout 900 python -m pytest tests -m gpu -q --timeout 300 -p no:cacheprovider -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/pytest_gpu.log | cut -c1-300
for W in cfg2 cfg4; do timeout 300 python bench.py --workload $W --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/bench_${W}_r1O.log 2>&1; echo "bench $W rc=$?"; done
