# A/B: main kernels staging digits / coefficients / missing lists by bulk
# copies on an mbarrier (balanced list walk (libgkb.so) vs per-row halves (libgkb_base.so, HEAD)
# register copies (libgkb_base.so). Config 4 and config 2, alternating.
L=$PWD/paper_1808_03374_b200
for i in 1 2 3; do
  for v in base ""; do
    echo "== c4 ${v:-new}"; GKB_LIB=$L/libgkb${v:+_$v}.so python tools/sweep_kt.py --one 4 20
    echo "== c2 ${v:-new}"; GKB_LIB=$L/libgkb${v:+_$v}.so python tools/sweep_kt.py --one 2 100
  done
done
timeout 900 python -m pytest tests/test_gpu_geno.py tests/test_gpu_fullsize.py tests/test_gpu_missing.py -x -q -m gpu 2>&1 | tail -3
for v in base ""; do echo "== missing ${v:-new}"; GKB_MISS_MODE=list GKB_LIB=$PWD/paper_1808_03374_b200/libgkb${v:+_$v}.so python tools/missing_perf.py 2 0.005 0.01 0.02; done
