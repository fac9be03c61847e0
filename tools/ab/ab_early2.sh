# block products with early staging (libgkb.so) vs before (libgkb_base.so)
L=$PWD/paper_1808_03374_b200
for v in base "" base ""; do echo "== ${v:-new}"; GKB_LIB=$L/libgkb${v:+_$v}.so python tools/block_timing.py; done
