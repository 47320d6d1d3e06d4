# Usage (under gpurun): bash scripts/gpu_sanitize.sh <tag>: compute-sanitizer memcheck /
# racecheck / synccheck over the small cases of scripts/sanitize_cases.py
TAG=${1:-s}
mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
for C in k2dense k2hash cluster flow single resident; do
  for T in memcheck racecheck synccheck; do
    timeout 900 $CS --tool $T --print-limit 20 python scripts/sanitize_cases.py $C > gpurun_out/san_${TAG}_${C}_${T}.log 2>&1
    echo "$C $T rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|case .* ok' gpurun_out/san_${TAG}_${C}_${T}.log | tr '\n' ' ')"
  done
done
