# usage: bash tools/r2_sanitize.sh TOOL TAG  -- one compute-sanitizer tool per call
TOOL=${1:-memcheck}; TAG=${2:-r2}
EXTRA=""
[ "$TOOL" = memcheck ] && EXTRA="--leak-check no"
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/san_plain_$TAG.log 2>&1 || { echo "plain smoke failed"; exit 1; }
timeout 1500 compute-sanitizer --tool $TOOL $EXTRA --print-limit 50 --error-exitcode 9 \
  python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/san_${TOOL}_smoke_$TAG.log 2>&1
echo "smoke under $TOOL rc=$?"
tail -5 gpurun_out/san_${TOOL}_smoke_$TAG.log
timeout 1500 compute-sanitizer --tool $TOOL $EXTRA --print-limit 50 --error-exitcode 9 \
  python -m pytest tests/test_gpu_geno.py -m gpu -q -x -k "apply_and_adjoint or sharded or pinned or block_products or edge_rows" > gpurun_out/san_${TOOL}_geno_$TAG.log 2>&1
echo "geno tests under $TOOL rc=$?"
tail -5 gpurun_out/san_${TOOL}_geno_$TAG.log
