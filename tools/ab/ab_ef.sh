# A/B: HEAD (libgkb_base.so) vs ctl staging fix only (libgkb_noef.so) vs ctl fix
# + evict-first layout loads (libgkb.so): main-kernel times and config-2 solve.
L=$PWD/paper_1808_03374_b200
for i in 1 2; do
  for v in base noef ""; do
    lib=$L/libgkb${v:+_$v}.so
    echo "== ${v:-new}"; GKB_LIB=$lib python tools/sweep_kt.py --one 2 50
    GKB_LIB=$lib python tools/svdl_run.py 2
  done
done
for v in base ""; do
  echo "== cfg3 ${v:-new}"; GKB_LIB=$L/libgkb${v:+_$v}.so python tools/sweep_kt.py --one 3 20
done
timeout 600 python -m pytest tests -x -q -m gpu 2>&1 | tail -2
