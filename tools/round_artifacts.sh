set -e
python tools/prof_kernels.py 2 3
ncu --set full --clock-control none --import-source on -k regex:"k_pm_main" -c 4 -o gpurun_out/r1g_pm python tools/prof_kernels.py 2 1 > gpurun_out/r1g_ncu.log 2>&1
python tools/ncu_summary.py gpurun_out/r1g_pm.ncu-rep profiles/r1g_ncu_full_config2.json
bash tools/bench_round.sh
python tools/trace_svdl.py 2 gpurun_out/trace_svdl_r1g.json > /dev/null 2>&1
