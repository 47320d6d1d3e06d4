mkdir -p gpurun_out
for W in cfg2 cfg4; do timeout 300 python bench.py --workload $W --input u8 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_${W}_u8_r1L.log 2>&1; echo "bench $W rc=$?"; tail -2 gpurun_out/bench_${W}_u8_r1L.log | cut -c1-300; done
