mkdir -p gpurun_out
python bench.py --workload cfg3 --steps 1 --warmup 1 --no-cpu-baseline > /dev/null 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg3_r1G.csv python bench.py --workload cfg3 --steps 1 --warmup 1 --no-cpu-baseline > /dev/null 2>&1; echo "ncu3 rc=$?"
GS_TRACE_LEVELS=1 python bench.py --workload cfg3 --steps 1 --warmup 1 --no-cpu-baseline 2>&1 | grep "^iter" | tail -8
