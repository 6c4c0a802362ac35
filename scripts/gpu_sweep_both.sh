bash scripts/gpu_band_sweep.sh
bash scripts/gpu_nvs_sweep.sh
