# Usage (under gpurun): bash scripts/gpu_round.sh <tag> [workloads...]
# tests + smoke + bench per workload + ncu launch list of the first workload
TAG=${1:-r1}; shift; WL=${@:-cfg2}
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
timeout 1500 python -m pytest tests -m gpu -q --timeout 600 -p no:cacheprovider -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
for W in $WL; do
  timeout 900 python bench.py --workload $W --steps 20 --warmup 3 --cpu-budget 3 > gpurun_out/bench_${W}_${TAG}.log 2>&1; echo "bench $W rc=$?"
done
W1=$(echo $WL | cut -d' ' -f1)
CMD="python bench.py --workload $W1 --steps 3 --warmup 1 --no-cpu-baseline"
$CMD > gpurun_out/plain_$W1.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${W1}_${TAG}.csv $CMD > gpurun_out/ncu_$W1.log 2>&1; echo "ncu rc=$?"
tail -3 gpurun_out/smoke.log; tail -15 gpurun_out/pytest_gpu.log | cut -c1-300
