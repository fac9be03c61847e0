# host-input adjoint: range groups 1 (serial) vs 2 / 3 / 4 (pipelined)
for gr in 1 2 3 4; do echo "groups $gr"; GKB_HOSTIN_GROUPS=$gr python tools/e2e_breakdown.py 2>/dev/null | head -2; done
timeout 600 python -m pytest tests -x -q -m gpu 2>&1 | tail -2
