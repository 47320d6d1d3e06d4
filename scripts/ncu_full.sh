# Usage (under gpurun): bash scripts/ncu_full.sh <workload> <kernel-regex> <tag> [skip] [count]
W=${1:-cfg2}; K=${2:-k_resident}; TAG=${3:-r1}; SKIP=${4:-2}; CNT=${5:-1}
mkdir -p gpurun_out
CMD="python bench.py --workload $W --steps 2 --warmup 1 --no-cpu-baseline"
$CMD > gpurun_out/plain_full_$W.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:$K -s $SKIP -c $CNT \
    -o gpurun_out/prof_${W}_${K}_${TAG} $CMD > gpurun_out/ncu_full_${W}_${K}.log 2>&1
echo "ncu rc=$?"
