# Usage (under gpurun): bash scripts/gpu_r2_final.sh <tag>: the round's evidence in one call --
# smoke, the full GPU suite, every bench line (default cfg4 with the CPU baseline, the
# reference arm, cfg2/3/5, tune/track/mspp), launch lists (cfg4 default, cfg5, cfg3) and the
# ncu --set full captures of K2 (cfg4, cfg5), K7 (cfg4) and the component sweep (cfg5), with
# K2's DRAM traffic recorded in profiles/traffic.json for this kernel-source hash.
TAG=${1:-fin}
mkdir -p gpurun_out
nproc; grep -m1 "model name" /proc/cpuinfo
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke_$TAG.log
timeout 1500 python -m pytest tests -m gpu -q --timeout 300 -p no:cacheprovider > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu_$TAG.log | cut -c1-300
T0=$(date +%s); timeout 900 python bench.py > gpurun_out/bench_default_$TAG.log 2>&1; echo "bench default rc=$? wall $(( $(date +%s) - T0 )) s"; python scripts/bench_summary.py gpurun_out/bench_default_$TAG.log
T0=$(date +%s); timeout 1500 python bench.py --impl reference > gpurun_out/bench_ref_$TAG.log 2>&1; echo "bench ref rc=$? wall $(( $(date +%s) - T0 )) s"; tail -1 gpurun_out/bench_ref_$TAG.log | cut -c1-300
for W in cfg2 cfg3 cfg5; do timeout 900 python bench.py --workload $W --steps 20 --warmup 3 --cpu-budget 5 > gpurun_out/bench_${W}_$TAG.log 2>&1; echo "bench $W rc=$?"; python scripts/bench_summary.py gpurun_out/bench_${W}_$TAG.log; done
for W in tune track mspp mspp5; do timeout 600 python bench.py --workload $W --steps 5 --warmup 2 > gpurun_out/bench_${W}_$TAG.log 2>&1; echo "bench $W rc=$?"; tail -1 gpurun_out/bench_${W}_$TAG.log | cut -c1-200; done
for W in cfg4 cfg5 cfg3; do
  CMD="python bench.py --workload $W --steps 3 --warmup 1 --no-cpu-baseline --profile-device"
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${W}_$TAG.csv $CMD > gpurun_out/ncu_l_$W.log 2>&1; echo "ncu launches $W rc=$?"
  python scripts/launch_summary.py gpurun_out/launches_${W}_$TAG.csv > gpurun_out/launches_${W}_$TAG.txt; head -14 gpurun_out/launches_${W}_$TAG.txt
done
for W in cfg4 cfg5; do
  bash scripts/ncu_capture.sh $W k_bin $TAG 1 --profile-device > /dev/null 2>&1; echo "ncu $W k_bin rc=$?"
  python scripts/ncu_traffic.py gpurun_out/prof_${W}_k_bin_${TAG}.raw.csv $W k_bin prof_${W}_k_bin_${TAG}
done
bash scripts/ncu_capture.sh cfg4 k_label $TAG 1 --profile-device > /dev/null 2>&1; echo "ncu cfg4 k_label rc=$?"
bash scripts/ncu_capture.sh cfg5 k_sweep_comp $TAG 0 --profile-device > /dev/null 2>&1; echo "ncu cfg5 k_sweep_comp rc=$?"
{
  for K in cfg4_k_bin cfg5_k_bin cfg4_k_label cfg5_k_sweep_comp; do
    python scripts/ncu_raw_summary.py gpurun_out/prof_${K}_${TAG}.raw.csv
    echo '```'; python scripts/ncu_sass_ops.py gpurun_out/prof_${K}_${TAG}.src.csv.gz 25; echo '```'; echo
  done
} > gpurun_out/ncu_kernels_$TAG.md 2>&1
cp profiles/traffic.json gpurun_out/traffic_$TAG.json
rm -f gpurun_out/*.ncu-rep
