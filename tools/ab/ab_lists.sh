# A/B: byte-delta missing-list runs walked one run per lane (libgkb.so) vs
# 16-bit indices walked in halves (libgkb_base.so, HEAD). Configs 4, 2, and
# config 2 at 5% missing; then the parity tests on the new build.
L=$PWD/paper_1808_03374_b200
for i in 1 2 3; do
  for v in base ""; do
    echo "== c4 ${v:-new}"; GKB_LIB=$L/libgkb${v:+_$v}.so python tools/sweep_kt.py --one 4 20
    echo "== c2 ${v:-new}"; GKB_LIB=$L/libgkb${v:+_$v}.so python tools/sweep_kt.py --one 2 100
  done
done
for v in base ""; do echo "== missing sweep ${v:-new}"; GKB_LIB=$L/libgkb${v:+_$v}.so python tools/missing_perf.py 2 0.0 0.01 0.05 0.1; done
for v in base ""; do echo "== block ${v:-new}"; GKB_LIB=$L/libgkb${v:+_$v}.so python tools/block_timing.py; done
timeout 1500 python -m pytest tests -x -q -m gpu -k "not golden" 2>&1 | tail -3
