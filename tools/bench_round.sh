# Bench line, reference arm and launch list for one tag (TAG env, default r1h).
set -e
TAG=${TAG:-r1h}
python bench.py --steps 20 --warmup 3 > gpurun_out/bench_${TAG}.json 2> gpurun_out/bench_${TAG}.err
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref_${TAG}.json 2> gpurun_out/bench_ref_${TAG}.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_${TAG}.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-ingest > gpurun_out/ncu_${TAG}.log 2>&1
tail -c 2500 gpurun_out/bench_${TAG}.json; echo; tail -c 600 gpurun_out/bench_ref_${TAG}.json
