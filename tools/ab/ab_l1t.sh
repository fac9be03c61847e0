# A/B of the single-layout adjoint: strip-pair k32 loop at 2 CTAs/SM (libgkb.so)
# and at 3 CTAs/SM with spills (libgkb_m3.so) vs the per-strip k16 loop (libgkb_base.so, HEAD)
L=$PWD/paper_1808_03374_b200
for i in 1 2; do
  for v in base m3 ""; do
    for c in 4 2; do echo "== c$c ${v:-new}"; GKB_LAYOUTS=1 GKB_LIB=$L/libgkb${v:+_$v}.so python tools/sweep_kt.py --one $c 20; done
  done
done
GKB_LAYOUTS=1 timeout 900 python -m pytest tests/test_gpu_single_layout.py tests/test_gpu_geno.py -q -m gpu 2>&1 | tail -2
