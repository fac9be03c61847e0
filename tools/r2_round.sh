# Round-2 artefacts for one tag: GPU tests, bench lines (config 4 headline,
# reference arm, configs 3 and 2 beside it), solve timelines, then the ncu
# captures (launch list of the bench command, --set full of the main kernels).
# Usage (on the GPU box): bash tools/r2_round.sh TAG
TAG=${1:-r2}
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_${TAG}.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/pytest_gpu_${TAG}.log
timeout 900 python bench.py > gpurun_out/bench_${TAG}.json 2> gpurun_out/bench_${TAG}.err; echo "bench rc=$?"
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref_${TAG}.json 2> gpurun_out/bench_ref_${TAG}.err; echo "ref rc=$?"
timeout 900 python bench.py --config 3 --no-cpu > gpurun_out/bench_c3_${TAG}.json 2> gpurun_out/bench_c3_${TAG}.err; echo "c3 rc=$?"
timeout 900 python bench.py --config 2 --no-cpu > gpurun_out/bench_c2_${TAG}.json 2> gpurun_out/bench_c2_${TAG}.err; echo "c2 rc=$?"
timeout 600 python tools/trace_svdl.py 2 gpurun_out/trace_svdl_c2_${TAG}.json > gpurun_out/trace_c2_${TAG}.log 2>&1
timeout 600 python tools/trace_svdl.py 4 gpurun_out/trace_svdl_c4_${TAG}.json > gpurun_out/trace_c4_${TAG}.log 2>&1
python bench.py --steps 2 --warmup 3 --no-cpu --no-ingest --no-widen > gpurun_out/plain_launch_${TAG}.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches_${TAG}.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu --no-ingest --no-widen > gpurun_out/ncu_launch_${TAG}.log 2>&1; echo "launch list rc=$?"
python tools/prof_kernels.py 4 2 > gpurun_out/ncu_plain_${TAG}.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_pm_main -s 2 -c 2 \
    -o gpurun_out/${TAG}_pm_c4 python tools/prof_kernels.py 4 2 > gpurun_out/ncu_${TAG}.log 2>&1; echo "ncu rc=$?"
tail -c 3000 gpurun_out/bench_${TAG}.json; echo; tail -c 800 gpurun_out/bench_ref_${TAG}.json
