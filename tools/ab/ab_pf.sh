# A/B: L2 bulk prefetch distance (GKB_L2PF builds) vs base
for i in 1 2; do
  for c in 2 3; do
    echo "cfg $c base"; GKB_LIB=$PWD/paper_1808_03374_b200/libgkb_base.so python tools/sweep_kt.py --one $c 50
    for v in 4 6 8; do
      echo "cfg $c pf$v"; GKB_LIB=$PWD/paper_1808_03374_b200/libgkb_pf$v.so python tools/sweep_kt.py --one $c 50
    done
  done
done
