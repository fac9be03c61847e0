# usage: bash tools/r2_tests.sh TAG [pytest args...]
TAG=${1:-r2}; shift
timeout 2400 python -m pytest "$@" > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?"
tail -30 gpurun_out/pytest_$TAG.log
