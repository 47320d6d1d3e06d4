# Usage (under gpurun): bash scripts/gpu_r2r.sh <tag>: full gpu tests, smoke, default bench + tune/track/mspp lines
TAG=${1:-r}
mkdir -p gpurun_out
timeout 240 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke_$TAG.log
timeout 1200 python -m pytest tests -m gpu -q -x --timeout 180 -p no:cacheprovider > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu_$TAG.log | cut -c1-300
timeout 300 python bench.py --no-cpu-baseline > gpurun_out/bench_default_$TAG.log 2>&1; echo "bench default rc=$?"; python scripts/bench_summary.py gpurun_out/bench_default_$TAG.log
for W in tune track mspp; do timeout 300 python bench.py --workload $W --steps 5 --warmup 2 > gpurun_out/bench_${W}_$TAG.log 2>&1; echo "bench $W rc=$?"; tail -1 gpurun_out/bench_${W}_$TAG.log | cut -c1-400; done
