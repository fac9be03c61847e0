set -e
python bench.py --steps 20 --warmup 3 > gpurun_out/bench_r1g.json 2> gpurun_out/bench_r1g.err
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref_r1g.json 2> gpurun_out/bench_ref_r1g.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_r1g.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-ingest > gpurun_out/ncu_r1g.log 2>&1
tail -c 2500 gpurun_out/bench_r1g.json; echo; tail -c 600 gpurun_out/bench_ref_r1g.json
