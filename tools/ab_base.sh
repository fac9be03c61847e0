# A/B: current build vs paper_1808_03374_b200/libgkb_base.so (per-product main-kernel times)
for i in 1 2; do
  for c in 2 3 1; do
    echo "cfg $c base"; GKB_LIB=$PWD/paper_1808_03374_b200/libgkb_base.so python tools/sweep_kt.py --one $c 50
    echo "cfg $c new";  python tools/sweep_kt.py --one $c 50
  done
done
timeout 600 python -m pytest tests -x -q -m gpu 2>&1 | tail -2
