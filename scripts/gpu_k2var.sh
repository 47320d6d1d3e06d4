# Usage (under gpurun): bash scripts/gpu_k2var.sh <tag> [variant dirs under build/]: K2 variants
# (the in-tree library first, then each build/<v>/libgridshift_cuda.so swapped in): parity
# subset, cfg4/cfg5 bench lines, K2 ncu capture per variant.
TAG=${1:-k}; shift
mkdir -p gpurun_out
LIB=paper_2206_02200_b200/_lib/libgridshift_cuda.so
cp $LIB /tmp/lib_base.so
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q --timeout 600 -p no:cacheprovider -k "vector or build_bit_exact or cfg4_frames or batched or f32 or run_parity or x_path or ragged or cfg5_full" > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_$TAG.log | cut -c1-300
for V in base "$@"; do
  if [ $V != base ]; then cp build/$V/libgridshift_cuda.so $LIB; fi
  for W in cfg4 cfg5; do timeout 600 python bench.py --workload $W --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_${W}_${TAG}_$V.log 2>&1; echo "bench $V $W rc=$?"; python scripts/bench_summary.py gpurun_out/bench_${W}_${TAG}_$V.log; done
  bash scripts/ncu_capture.sh cfg4 k_bin ${TAG}_$V 1 --profile-device > /dev/null 2>&1
  python scripts/ncu_raw_summary.py gpurun_out/prof_cfg4_k_bin_${TAG}_$V.raw.csv | grep -E "duration|dram__bytes|issue_active|inst_executed|warps_active"
  python scripts/ncu_sass_ops.py gpurun_out/prof_cfg4_k_bin_${TAG}_$V.src.csv.gz 12
done
cp /tmp/lib_base.so $LIB
