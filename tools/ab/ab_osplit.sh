# omega-test split (default) vs separate ctl launches (GKB_NO_OMEGA_SPLIT=1): config-2 solve
timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -3
for i in 1 2 3; do
  echo "== split"; python tools/svdl_run.py 2
  echo "== nosplit"; GKB_NO_OMEGA_SPLIT=1 python tools/svdl_run.py 2
done
echo "== cfg3 split"; python tools/svdl_run.py 3
echo "== cfg3 nosplit"; GKB_NO_OMEGA_SPLIT=1 python tools/svdl_run.py 3
