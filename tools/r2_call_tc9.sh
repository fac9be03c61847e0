timeout 600 python -m pytest tests/test_gpu_geno.py -q -m gpu -k "tc_block" 2>&1 | tail -3
timeout 600 python tools/tc_timing.py 4 2>&1 | tail -2
python tools/tc_prof.py 4 16 > gpurun_out/tcprof_plain.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:k_pm_blk_tc -s 1 -c 1 -o gpurun_out/tc_blk2 python tools/tc_prof.py 4 16 > gpurun_out/tcprof_ncu.log 2>&1; echo ncu rc=$?
