# fused right tail: parity first (bitwise vs unfused / host step), then whole-solve A/B
timeout 900 python -m pytest tests/test_gpu_gkl.py -q -m gpu -x -k "fused_right_tail or device_step_control or speculative" 2>&1 | tail -15
CONFIGS="2 1" REPS=7 bash tools/ab/ab_solve.sh 2>&1
GKB_VERBOSE=1 python tools/svdl_run.py 2 2>&1 | tail -3
