# A/B: programmatic dependent launch on (default) vs off (GKB_NO_PDL=1)
for i in 1 2; do
  for cfg in 2 1; do
    echo "PDL on";  python tools/prof_kernels.py $cfg 100
    echo "PDL off"; GKB_NO_PDL=1 python tools/prof_kernels.py $cfg 100
  done
done
