# A/B: main-loop geometry variants (strips per warp, prefetch depth, CTAs/SM)
for i in 1 2; do
  for c in 2 3; do
    echo "cfg $c base"; GKB_LIB=$PWD/paper_1808_03374_b200/libgkb_base.so python tools/sweep_kt.py --one $c 50
    for v in 145 135 126 233; do
      echo "cfg $c v$v"; GKB_LIB=$PWD/paper_1808_03374_b200/libgkb_v$v.so python tools/sweep_kt.py --one $c 50
    done
  done
done
