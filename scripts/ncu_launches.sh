# Usage (under gpurun): bash scripts/ncu_launches.sh <workload> [tag]
W=${1:-cfg2}; TAG=${2:-r1}
mkdir -p gpurun_out
CMD="python bench.py --workload $W --steps 3 --warmup 1 --no-cpu-baseline"
$CMD > gpurun_out/plain_$W.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${W}_${TAG}.csv $CMD > gpurun_out/ncu_$W.log 2>&1
echo "rc=$?"
tail -2 gpurun_out/plain_$W.log | cut -c1-300
