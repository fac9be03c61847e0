GKB_TC_BLOCK=1 timeout 1800 python -m pytest tests -m gpu -q -k "not golden" 2>&1 | tail -4
timeout 600 python -m pytest tests/test_gpu_geno.py -m gpu -q -k "tc_block or block_products" 2>&1 | tail -2
GKB_TC_BLOCK=1 python tools/tc_timing.py 4 > gpurun_out/tc_timing_c4.json 2>&1; cat gpurun_out/tc_timing_c4.json
