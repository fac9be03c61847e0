# A/B of the dense-missing (indicator-MMA) kernels, forced: working tree vs HEAD
L=$PWD/paper_1808_03374_b200
for i in 1 2 3; do for c in ${CONFIGS:-2 4}; do for v in base ""; do
  GKB_MISS_MODE=ind GKB_LIB=$L/libgkb${v:+_$v}.so python tools/step_ab.py $c 20
done; done; done
