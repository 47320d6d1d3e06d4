bash scripts/gpu_round.sh r1f cfg2 cfg4 cfg1 cfg3
