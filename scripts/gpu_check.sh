# Usage (under gpurun): bash scripts/gpu_check.sh [pytest-args...]
mkdir -p gpurun_out
nvidia-smi -L
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
timeout 1500 python -m pytest tests -m gpu -q --timeout 600 -p no:cacheprovider "$@" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
timeout 600 python bench.py --steps 20 --warmup 3 --cpu-budget 3 > gpurun_out/bench.log 2>&1; echo "bench rc=$?"
tail -3 gpurun_out/smoke.log; tail -40 gpurun_out/pytest_gpu.log | cut -c1-300; tail -3 gpurun_out/bench.log | cut -c1-600
