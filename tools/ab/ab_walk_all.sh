# A/B of the uniform list walks: working tree (libgkb.so) vs HEAD
# (libgkb_base.so): two-layout products, single-layout K2, block pairs
L=$PWD/paper_1808_03374_b200
for i in 1 2; do for v in base ""; do
  GKB_LIB=$L/libgkb${v:+_$v}.so python tools/step_ab.py 2 20
  GKB_LAYOUTS=1 GKB_LIB=$L/libgkb${v:+_$v}.so python tools/step_ab.py 2 20
  GKB_LAYOUTS=1 GKB_LIB=$L/libgkb${v:+_$v}.so python tools/step_ab.py 4 10
  GKB_LIB=$L/libgkb${v:+_$v}.so python tools/block_ab.py 4 5
done; done
