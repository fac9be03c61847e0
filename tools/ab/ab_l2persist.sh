# L2 persisting window over the left basis (GKB_L2_PERSIST=1) vs none, alternating
for c in 2 3; do for i in 1 2; do
  python tools/svdl_ab.py $c ${REPS:-5}
  GKB_L2_PERSIST=1 python tools/svdl_ab.py $c ${REPS:-5} | sed 's/}/, "l2_persist": 1}/'
done; done
