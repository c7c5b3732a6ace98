bash tools/gpu_vv.sh vv3 "bitwise or solve_exact or coronal or multirank"
bash tools/gpu_vv_perf.sh vvp2
