# Usage (under gpurun): bash scripts/gpu_final.sh <tag>: tests, smoke, every bench line, the
# default command's ncu launch list and the full captures of the kernels the DESIGN cites.
TAG=${1:-r1f}
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke_$TAG.log
timeout 900 python -m pytest tests -m gpu -q --timeout 600 -p no:cacheprovider > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pytest_gpu_$TAG.log
timeout 600 python bench.py > gpurun_out/bench_default_$TAG.log 2>&1; echo "bench default rc=$?"
timeout 600 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/bench_ref_$TAG.log 2>&1; echo "bench ref rc=$?"
for W in cfg1 cfg3 cfg4 cfg5; do timeout 900 python bench.py --workload $W --steps 20 --warmup 3 --cpu-budget 5 > gpurun_out/bench_${W}_$TAG.log 2>&1; echo "bench $W rc=$?"; done
for W in cfg2 cfg4; do timeout 900 python bench.py --workload $W --input u8 --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/bench_${W}u8_$TAG.log 2>&1; echo "bench $W u8 rc=$?"; done
timeout 600 python bench.py --workload tune --steps 5 --warmup 2 > gpurun_out/bench_tune_$TAG.log 2>&1; echo "bench tune rc=$?"
timeout 600 python bench.py --workload track --steps 5 --warmup 2 > gpurun_out/bench_track_$TAG.log 2>&1; echo "bench track rc=$?"
CMD="python bench.py --steps 3 --warmup 1 --no-cpu-baseline"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg2_$TAG.csv $CMD > gpurun_out/ncu_l_cfg2.log 2>&1; echo "ncu launches cfg2 rc=$?"
CMD="python bench.py --workload cfg5 --steps 2 --warmup 1 --no-cpu-baseline"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg5_$TAG.csv $CMD > gpurun_out/ncu_l_cfg5.log 2>&1; echo "ncu launches cfg5 rc=$?"
bash scripts/ncu_capture.sh cfg2 k_resident $TAG 2
bash scripts/ncu_capture.sh cfg2 k_bin_priv $TAG 2
bash scripts/ncu_capture.sh cfg4 k_bin_priv $TAG 2
bash scripts/ncu_capture.sh cfg4 k_bounds_box $TAG 2
bash scripts/ncu_capture.sh cfg5 k_bin_priv $TAG 2
bash scripts/ncu_capture.sh cfg5 k_sweep_cluster $TAG 1
bash scripts/ncu_capture.sh tune k_silhouette $TAG 2
bash scripts/ncu_capture.sh track k_track $TAG 1
rm -f gpurun_out/*.ncu-rep
for f in gpurun_out/bench_*_$TAG.log; do python scripts/bench_summary.py $f 2>/dev/null; done
