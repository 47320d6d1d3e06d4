# Usage (under gpurun): bash scripts/gpu_r2c.sh <tag>: smoke, full gpu tests, the default bench
# line (with the CPU baseline), the reference arm with defaults, cfg5/cfg2/cfg3 lines
TAG=${1:-c}
mkdir -p gpurun_out
nproc; lscpu | grep "Model name"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke_$TAG.log
timeout 1500 python -m pytest tests -m gpu -q --timeout 600 -p no:cacheprovider > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu_$TAG.log | cut -c1-300
T0=$(date +%s); timeout 900 python bench.py > gpurun_out/bench_default_$TAG.log 2>&1; RC=$?; echo "bench default rc=$RC wall $(( $(date +%s) - T0 )) s"; python scripts/bench_summary.py gpurun_out/bench_default_$TAG.log; tail -1 gpurun_out/bench_default_$TAG.log | cut -c1-200
T0=$(date +%s); timeout 1200 python bench.py --impl reference > gpurun_out/bench_ref_$TAG.log 2>&1; RC=$?; echo "bench ref rc=$RC wall $(( $(date +%s) - T0 )) s"; tail -2 gpurun_out/bench_ref_$TAG.log | cut -c1-400
for W in cfg5 cfg2 cfg3; do timeout 600 python bench.py --workload $W --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_${W}_$TAG.log 2>&1; echo "bench $W rc=$?"; python scripts/bench_summary.py gpurun_out/bench_${W}_$TAG.log; done
