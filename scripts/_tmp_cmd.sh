mkdir -p gpurun_out
CMD="python bench.py --workload cfg2 --steps 2 --warmup 1 --no-cpu-baseline"
$CMD > gpurun_out/plain_a.log 2>&1 && ncu --set full --clock-control none --import-source on --sampling-interval 0 -k regex:k_resident -s 2 -c 1 -o gpurun_out/prof_cfg2_resident_r1h $CMD > gpurun_out/ncu_a.log 2>&1; echo "ncu a rc=$?"
CMD3="python bench.py --workload cfg3 --steps 1 --warmup 1 --no-cpu-baseline"
$CMD3 > gpurun_out/plain_b.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg3_r1h.csv $CMD3 > gpurun_out/ncu_b.log 2>&1; echo "ncu b rc=$?"
