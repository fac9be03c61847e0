for c in 2 4; do timeout 600 python tools/tc_timing.py $c; done
timeout 1800 python -m pytest tests -m gpu -q -k "not golden" 2>&1 | tail -4
