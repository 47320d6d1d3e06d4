# Usage (under gpurun): bash scripts/gpu_r2f.sh <tag>: global-path parity subset, cfg5 bench,
# launch list, ncu capture of the first component sweep of cfg5
TAG=${1:-f}
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x --timeout 180 -p no:cacheprovider -k "injection or global or cfg5 or fuzz or dist" > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu_$TAG.log | cut -c1-400
timeout 300 python bench.py --workload cfg5 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_cfg5_$TAG.log 2>&1; echo "bench rc=$?"; python scripts/bench_summary.py gpurun_out/bench_cfg5_$TAG.log
CMD="python bench.py --workload cfg5 --steps 3 --warmup 1 --no-cpu-baseline --profile-device"
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg5_$TAG.csv $CMD > gpurun_out/ncu_l_cfg5.log 2>&1; echo "ncu launches cfg5 rc=$?"
python scripts/launch_summary.py gpurun_out/launches_cfg5_$TAG.csv 2>/dev/null | head -24
timeout 400 bash scripts/ncu_capture.sh cfg5 k_sweep_comp $TAG 0 --profile-device > /dev/null 2>&1; echo "ncu full rc=$?"
python scripts/ncu_raw_summary.py gpurun_out/prof_cfg5_k_sweep_comp_$TAG.raw.csv
head -40 gpurun_out/prof_cfg5_k_sweep_comp_$TAG.hot.txt
