# dense-missing kernel: fully unrolled full ranges (libgkb.so) vs generic loop (libgkb_base.so, HEAD)
L=$PWD/paper_1808_03374_b200
for i in 1 2; do for v in base ""; do echo "== ${v:-new}"; GKB_MISS_MODE=ind GKB_LIB=$L/libgkb${v:+_$v}.so python tools/missing_perf.py 2 0.05; GKB_MISS_MODE=ind GKB_LIB=$L/libgkb${v:+_$v}.so python tools/missing_perf.py 4 0.05; done; done
GKB_MISS_MODE=ind timeout 900 python -m pytest tests/test_gpu_geno.py tests/test_gpu_missing.py -q -m gpu 2>&1 | tail -2
