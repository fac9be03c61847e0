# fully unrolled column-range width: 14 tiles (libgkb.so) vs 12 / 16 / 18 (libgkb_fNN.so)
L=$PWD/paper_1808_03374_b200
for i in 1 2; do
  for v in "" f12 f16 f18; do
    for c in 4 2; do echo "== c$c ${v:-f14}"; GKB_LIB=$L/libgkb${v:+_$v}.so python tools/sweep_kt.py --one $c 20; done
  done
done
