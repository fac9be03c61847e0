for i in 1 2 3 4; do timeout 600 python -m pytest tests/test_gpu_spmd.py -q -m gpu 2>&1 | tail -1; done
timeout 900 python -m pytest tests/test_gpu_single_layout.py -q -m gpu --durations=5 2>&1 | tail -25
GKB_LAYOUTS=1 timeout 1500 python -m pytest tests/test_gpu_geno.py tests/test_gpu_fullsize.py tests/test_gpu_gkl.py tests/test_gpu_parity_full.py tests/test_subspace.py tests/test_regress.py tests/test_gpu_missing.py -q -m gpu 2>&1 | tail -8
