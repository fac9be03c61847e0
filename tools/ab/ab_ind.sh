# Dense-missing mode (indicator MMAs, k_pm_ind) vs the list walk, by missing rate;
# then the GPU parity suites with the indicator mode forced everywhere.
for m in list ind; do echo "== missing sweep config 2, mode $m"; GKB_MISS_MODE=$m python tools/missing_perf.py 2 0.0 0.005 0.01 0.02 0.05 0.1; done
for m in list ind; do echo "== config 4, mode $m"; GKB_MISS_MODE=$m python tools/missing_perf.py 4 0.01; done
GKB_MISS_MODE=ind timeout 1500 python -m pytest tests/test_gpu_geno.py tests/test_gpu_missing.py tests/test_gpu_fullsize.py tests/test_gpu_parity_full.py tests/test_gpu_gkl.py tests/test_subspace.py tests/test_regress.py -q -m gpu -k "not golden" 2>&1 | tail -15
timeout 1500 python -m pytest tests/test_gpu_missing.py -q -m gpu 2>&1 | tail -3
