bash scripts/gpu_round.sh r1d cfg2 cfg4 cfg1
bash scripts/ncu_full.sh cfg2 k_resident r1d 2 1
bash scripts/ncu_full.sh cfg2 k_bin_priv r1d 2 1
