# whole-solve A/B: libgkb.so (working tree) vs libgkb_base.so (HEAD), alternating
L=$PWD/paper_1808_03374_b200
for c in ${CONFIGS:-2 1}; do for i in 1 2 3; do for v in base ""; do
  GKB_LIB=$L/libgkb${v:+_$v}.so python tools/svdl_ab.py $c ${REPS:-7}
done; done; done
