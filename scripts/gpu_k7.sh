# Usage (under gpurun): bash scripts/gpu_k7.sh <tag>: label-path parity subset, cfg4 bench, K7 capture
TAG=${1:-k7}
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x --timeout 240 -p no:cacheprovider -k "cfg4 or frame or u8 or render or ragged or misaligned or graph or mspp" > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_$TAG.log | cut -c1-300
timeout 300 python bench.py --workload cfg4 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_cfg4_$TAG.log 2>&1; echo "bench rc=$?"; python scripts/bench_summary.py gpurun_out/bench_cfg4_$TAG.log
timeout 400 bash scripts/ncu_capture.sh cfg4 k_label $TAG 1 --profile-device > /dev/null 2>&1; echo "ncu rc=$?"
python scripts/ncu_raw_summary.py gpurun_out/prof_cfg4_k_label_$TAG.raw.csv | grep -E "duration|dram__bytes|issue|warps_active|stall"
