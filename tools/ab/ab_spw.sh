set -x
for i in 1 2; do
python tools/prof_kernels.py 2 50
GKB_LIB=$PWD/paper_1808_03374_b200/libgkb_spw4.so python tools/prof_kernels.py 2 50
python tools/prof_kernels.py 1 50
GKB_LIB=$PWD/paper_1808_03374_b200/libgkb_spw4.so python tools/prof_kernels.py 1 50
done
GKB_LIB=$PWD/paper_1808_03374_b200/libgkb_spw4.so timeout 600 python -m pytest tests -x -q -m gpu 2>&1 | tail -3
