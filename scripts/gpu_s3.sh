# Usage (under gpurun): bash scripts/gpu_s3.sh <tag>: smoke, full gpu tests, default bench, cfg5/cfg2 bench
TAG=${1:-s3}
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke_$TAG.log
timeout 1500 python -m pytest tests -m gpu -q --timeout 600 -p no:cacheprovider > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/pytest_gpu_$TAG.log | cut -c1-300
timeout 600 python bench.py > gpurun_out/bench_default_$TAG.log 2>&1; echo "bench default rc=$?"; python scripts/bench_summary.py gpurun_out/bench_default_$TAG.log
for W in cfg2 cfg5; do timeout 300 python bench.py --workload $W --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_${W}_$TAG.log 2>&1; echo "bench $W rc=$?"; python scripts/bench_summary.py gpurun_out/bench_${W}_$TAG.log; done
