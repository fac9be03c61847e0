for L in 2 1; do for c in 4 3 2; do echo "== config $c layouts $L"; GKB_LAYOUTS=$L python tools/sweep_kt.py --one $c 20; done; done
timeout 1200 python tools/c5_shard.py 5 120 > gpurun_out/c5_shard_r2.json 2> gpurun_out/c5_shard_r2.err; echo "c5 rc=$?"; cat gpurun_out/c5_shard_r2.json; tail -3 gpurun_out/c5_shard_r2.err
