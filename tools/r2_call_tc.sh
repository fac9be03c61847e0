timeout 600 python -m pytest tests/test_gpu_geno.py -q -m gpu -x -k "tc_block" 2>&1 | tail -30
