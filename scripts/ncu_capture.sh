# Usage (under gpurun): bash scripts/ncu_capture.sh <workload> <kernel-regex> <tag> [skip] [extra bench args]
# One ncu --set full capture, exported on the box to raw/source CSV (the .ncu-rep is kept only
# when small: gpurun brings back at most 64 MiB).
W=${1:-cfg2}; K=${2:-k_resident}; TAG=${3:-r1}; SKIP=${4:-2}; shift 4; EXTRA="$@"
mkdir -p gpurun_out
CMD="python bench.py --workload $W --steps 2 --warmup 1 --no-cpu-baseline $EXTRA"
OUT=gpurun_out/prof_${W}_${K}_${TAG}
$CMD > gpurun_out/plain_full_$W.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:$K -s $SKIP -c 1 \
    -o $OUT $CMD > gpurun_out/ncu_full_${W}_${K}.log 2>&1
echo "ncu $W $K rc=$?"
ncu -i $OUT.ncu-rep --page raw --csv > $OUT.raw.csv 2>/dev/null
ncu -i $OUT.ncu-rep --page source --csv --print-source=cuda,sass > $OUT.src.csv 2>/dev/null
ncu -i $OUT.ncu-rep --page details --csv > $OUT.details.csv 2>/dev/null
python scripts/ncu_hot_lines.py $OUT.src.csv 40 > $OUT.hot.txt 2>&1
gzip -f $OUT.src.csv
[ $(stat -c %s $OUT.ncu-rep) -gt 15000000 ] && rm -f $OUT.ncu-rep
ls -la gpurun_out | tail -5
