mkdir -p gpurun_out
for W in cfg5 cfg3; do
python bench.py --workload $W --steps 1 --warmup 1 --no-cpu-baseline > /dev/null 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${W}_r1O.csv python bench.py --workload $W --steps 1 --warmup 1 --no-cpu-baseline > /dev/null 2>&1; echo "ncu $W rc=$?"
done
