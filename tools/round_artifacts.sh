# Round artefacts for one tag (default r1h): GPU tests, ncu capture of both
# main kernels, bench line + reference arm + launch list, solve timeline.
# Usage (on the GPU box): bash tools/round_artifacts.sh [TAG]
set -e
TAG=${1:-r1h}
mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_${TAG}.log 2>&1 || { tail -30 gpurun_out/pytest_gpu_${TAG}.log; exit 1; }
tail -3 gpurun_out/pytest_gpu_${TAG}.log
python tools/prof_kernels.py 2 3
ncu --set full --clock-control none --import-source on -k regex:"k_pm_main" -c 4 -o gpurun_out/${TAG}_pm python tools/prof_kernels.py 2 1 > gpurun_out/${TAG}_ncu.log 2>&1
python tools/ncu_summary.py gpurun_out/${TAG}_pm.ncu-rep profiles/${TAG}_ncu_full_config2.json
TAG=${TAG} bash tools/bench_round.sh
python tools/trace_svdl.py 2 gpurun_out/trace_svdl_${TAG}.json > /dev/null 2>&1
