# usage: bash tools/r2_ncu.sh CFG TAG -- ncu --set full of both main kernels on config CFG
CFG=${1:-4}; TAG=${2:-r2}
python tools/prof_kernels.py $CFG 2 > gpurun_out/ncu_plain_$TAG.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_pm_main -s 2 -c 2 \
    -o gpurun_out/${TAG}_pm_c$CFG python tools/prof_kernels.py $CFG 2 > gpurun_out/ncu_$TAG.log 2>&1
echo "ncu rc=$?"; tail -3 gpurun_out/ncu_$TAG.log
