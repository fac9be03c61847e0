L=$PWD/paper_1808_03374_b200
for v in base ""; do echo "== block ${v:-new}"; GKB_LIB=$L/libgkb${v:+_$v}.so python tools/block_timing.py; done
GKB_BENCH_HOST_COMM=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29517 bench.py --gpus 2 --config 3 --steps 5 --warmup 3 --no-cpu > gpurun_out/bench_hc2.json 2> gpurun_out/bench_hc2.err; echo "hc2 rc=$?"
cat gpurun_out/bench_hc2.json; tail -5 gpurun_out/bench_hc2.err
timeout 2400 python -m pytest tests -m gpu -q -k "not golden" --durations=10 > gpurun_out/pytest_r2f.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/pytest_r2f.log
