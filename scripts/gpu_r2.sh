# Usage (under gpurun): bash scripts/gpu_r2.sh <tag> [pytest -k expr]: smoke, gpu tests, cfg4/cfg5/cfg2 bench
TAG=${1:-a}; K=${2:-}
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/smoke_$TAG.log | cut -c1-300
if [ -n "$K" ]; then
timeout 1500 python -m pytest tests -m gpu -x -q --timeout 600 -p no:cacheprovider -k "$K" > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?"
else
timeout 1500 python -m pytest tests -m gpu -q --timeout 600 -p no:cacheprovider > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?"
fi
tail -15 gpurun_out/pytest_gpu_$TAG.log | cut -c1-300
for W in cfg4 cfg5 cfg2 cfg3; do timeout 600 python bench.py --workload $W --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_${W}_$TAG.log 2>&1; echo "bench $W rc=$?"; python scripts/bench_summary.py gpurun_out/bench_${W}_$TAG.log; tail -2 gpurun_out/bench_${W}_$TAG.log | grep -v "^{" | cut -c1-300; done
