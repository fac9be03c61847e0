# A/B: main kernel with the coefficient/list staging completed before the loop
# (GKB_EARLY_STAGE=1, libgkb.so) vs after it (libgkb_base.so).
L=$PWD/paper_1808_03374_b200
for i in 1 2 3; do
  for v in base ""; do
    echo "== ${v:-new}"; GKB_LIB=$L/libgkb${v:+_$v}.so python tools/sweep_kt.py --one 2 50
  done
done
for v in base ""; do
  echo "== svdl ${v:-new}"; GKB_LIB=$L/libgkb${v:+_$v}.so python tools/svdl_run.py 2
  echo "== cfg3 ${v:-new}"; GKB_LIB=$L/libgkb${v:+_$v}.so python tools/sweep_kt.py --one 3 20
done
timeout 600 python -m pytest tests -x -q -m gpu 2>&1 | tail -2
