nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/convprim scripts/microbench/convprim.cu && /tmp/convprim > gpurun_out/convprim_$1.txt 2>&1; cat gpurun_out/convprim_$1.txt
# Usage (under gpurun): bash scripts/gpu_prof.sh <tag>: bench lines + ncu full captures of the
# binning and label kernels (cfg4, cfg5) with their traffic recorded in profiles/traffic.json
TAG=${1:-p}
mkdir -p gpurun_out
for W in cfg4 cfg5; do timeout 600 python bench.py --workload $W --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_${W}_$TAG.log 2>&1; echo "bench $W rc=$?"; python scripts/bench_summary.py gpurun_out/bench_${W}_$TAG.log; done
for W in cfg4 cfg5; do
  bash scripts/ncu_capture.sh $W k_bin $TAG 1 --profile-device > /dev/null 2>&1; echo "ncu $W k_bin rc=$?"
  python scripts/ncu_traffic.py gpurun_out/prof_${W}_k_bin_${TAG}.raw.csv $W k_bin prof_${W}_k_bin_${TAG}
  python scripts/ncu_raw_summary.py gpurun_out/prof_${W}_k_bin_${TAG}.raw.csv
  head -25 gpurun_out/prof_${W}_k_bin_${TAG}.hot.txt
done
bash scripts/ncu_capture.sh cfg4 k_label $TAG 1 --profile-device > /dev/null 2>&1; echo "ncu cfg4 k_label rc=$?"
python scripts/ncu_raw_summary.py gpurun_out/prof_cfg4_k_label_${TAG}.raw.csv
cp profiles/traffic.json gpurun_out/traffic_$TAG.json
