cd tools/microbench
for v in 0 1; do for nk in "16 32" "16 64" "16 128" "80 64" "96 128" "8 64"; do timeout 30 ./tc05 $nk $v; done; done
