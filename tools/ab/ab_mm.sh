# A/B: K1 missing sums from the lists (default) vs the missing-indicator MMA
for i in 1 2; do
  for c in 2 3; do
    echo "cfg $c base";  python tools/sweep_kt.py --one $c 50
    echo "cfg $c mm3";   GKB_LIB=$PWD/paper_1808_03374_b200/libgkb_mm3.so python tools/sweep_kt.py --one $c 50
    echo "cfg $c mm4";   GKB_LIB=$PWD/paper_1808_03374_b200/libgkb_mm4.so python tools/sweep_kt.py --one $c 50
  done
done
GKB_LIB=$PWD/paper_1808_03374_b200/libgkb_mm4.so timeout 600 python -m pytest tests -x -q -m gpu 2>&1 | tail -2
