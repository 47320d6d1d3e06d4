# Usage (under gpurun): bash scripts/gpu_r2d.sh <tag>: default bench line + reference arm
# (defaults), ncu K2/K7 captures with traffic, launch lists (cfg4 default, cfg5, cfg3)
TAG=${1:-d}
mkdir -p gpurun_out
nproc
T0=$(date +%s); timeout 900 python bench.py > gpurun_out/bench_default_$TAG.log 2>&1; RC=$?; echo "bench default rc=$RC wall $(( $(date +%s) - T0 )) s"; python scripts/bench_summary.py gpurun_out/bench_default_$TAG.log
T0=$(date +%s); timeout 1500 python bench.py --impl reference > gpurun_out/bench_ref_$TAG.log 2>&1; RC=$?; echo "bench ref rc=$RC wall $(( $(date +%s) - T0 )) s"; tail -1 gpurun_out/bench_ref_$TAG.log | cut -c1-300
bash scripts/gpu_prof.sh $TAG
for W in cfg4 cfg5 cfg3; do
  CMD="python bench.py --workload $W --steps 3 --warmup 1 --no-cpu-baseline --profile-device"
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${W}_$TAG.csv $CMD > gpurun_out/ncu_l_$W.log 2>&1; echo "ncu launches $W rc=$?"
  python scripts/launch_summary.py gpurun_out/launches_${W}_$TAG.csv | head -12
done
