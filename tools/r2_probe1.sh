set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv
nproc; free -g
timeout 600 python tools/bench_config.py 4 10 > gpurun_out/r2p_c4.json 2> gpurun_out/r2p_c4.err
timeout 300 python tools/sweep_kt.py 4 10 10 14 20 28 40 > gpurun_out/r2p_sweep4.log 2>&1
timeout 600 python tools/bench_config.py 3 10 > gpurun_out/r2p_c3.json 2> gpurun_out/r2p_c3.err
cat gpurun_out/r2p_c4.json gpurun_out/r2p_sweep4.log gpurun_out/r2p_c3.json
