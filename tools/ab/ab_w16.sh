# A/B: HEAD (libgkb_base.so) vs the multi-half main kernel at 8 warps (libgkb.so)
# and 16 warps per CTA (libgkb_w16.so): per-product main-kernel times.
L=$PWD/paper_1808_03374_b200
for i in 1 2; do
  for c in 2 3; do
    for v in base "" w16; do
      lib=$L/libgkb${v:+_$v}.so
      echo "cfg $c ${v:-new8}"; GKB_LIB=$lib python tools/sweep_kt.py --one $c 50
    done
  done
done
GKB_LIB=$L/libgkb_w16.so timeout 600 python -m pytest tests -x -q -m gpu 2>&1 | tail -2
timeout 600 python -m pytest tests -x -q -m gpu 2>&1 | tail -2
