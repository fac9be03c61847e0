# A/B of the product finish (k2_reduce_seq / unrolled k1_reduce): working tree
# (libgkb.so) vs HEAD (libgkb_base.so), alternating, configs 4 and 2
L=$PWD/paper_1808_03374_b200
for i in 1 2 3; do for c in ${CONFIGS:-4 2}; do for v in base ""; do
  GKB_LIB=$L/libgkb${v:+_$v}.so python tools/step_ab.py $c 20
done; done; done
