# A/B: register pipeline (default) vs cp.async ring (GKB_RING build)
for i in 1 2; do
  for c in 2 3 1; do
    echo "cfg $c base"; GKB_LIB=$PWD/paper_1808_03374_b200/libgkb_base.so python tools/sweep_kt.py --one $c 50
    echo "cfg $c ring"; GKB_LIB=$PWD/paper_1808_03374_b200/libgkb_ring.so python tools/sweep_kt.py --one $c 50
  done
done
GKB_LIB=$PWD/paper_1808_03374_b200/libgkb_ring.so timeout 600 python -m pytest tests -x -q -m gpu 2>&1 | tail -2
