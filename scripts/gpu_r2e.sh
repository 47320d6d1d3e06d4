# Usage (under gpurun): bash scripts/gpu_r2e.sh <tag>: gpu tests, cfg5/cfg3/cfg4 bench, cfg5 launch list
TAG=${1:-e}
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x --timeout 180 -p no:cacheprovider > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/pytest_gpu_$TAG.log | cut -c1-400
for W in cfg5 cfg3 cfg4 cfg2 cfg1; do timeout 300 python bench.py --workload $W --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_${W}_$TAG.log 2>&1; echo "bench $W rc=$?"; python scripts/bench_summary.py gpurun_out/bench_${W}_$TAG.log; tail -1 gpurun_out/bench_${W}_$TAG.log | grep -v "^{" | cut -c1-300; done
CMD="python bench.py --workload cfg5 --steps 3 --warmup 1 --no-cpu-baseline --profile-device"
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg5_$TAG.csv $CMD > gpurun_out/ncu_l_cfg5.log 2>&1; echo "ncu launches cfg5 rc=$?"
python scripts/launch_summary.py gpurun_out/launches_cfg5_$TAG.csv 2>/dev/null | head -16
