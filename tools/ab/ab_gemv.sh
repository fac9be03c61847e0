# gemv_t / gemv_n row-chunk counts (microbench, len 10000 / 100000 / 500000)
for b in 296 148 96 64 44 32; do
  echo "== blocks $b"; GKB_GT_BLOCKS=$b GKB_GN_BLOCKS=$b ./tools/microbench/basis_bench | grep "ncols  50\|ncols  25\|^len"
done
