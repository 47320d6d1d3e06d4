mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
python bench.py --workload cfg2 --steps 20 --warmup 3 --cpu-budget 2 > gpurun_out/bench_cfg2_r1j.log 2>&1; echo "bench rc=$?"
CMD="python bench.py --workload cfg2 --steps 2 --warmup 1 --no-cpu-baseline"
$CMD > gpurun_out/plain_a.log 2>&1 && ncu --set full --clock-control none --import-source on --warp-sampling-interval 0 -k regex:k_resident -s 2 -c 1 -o gpurun_out/prof_cfg2_resident_r1j $CMD > gpurun_out/ncu_a.log 2>&1; echo "ncu a rc=$?"
$CMD > gpurun_out/plain_b.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg2_r1j.csv $CMD > gpurun_out/ncu_b.log 2>&1; echo "ncu b rc=$?"
