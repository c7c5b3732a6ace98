#!/bin/bash
# Quick performance loop (no tests): bench lines for the variants + one ncu --set full of pass A.
# usage: bash tools/gpu_perf.sh TAG
TAG=${1:-perf}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$TAG.log 2>&1
B="python bench.py --steps 3 --warmup 3 --maxit 300 --no-cpu-baseline --no-e2e"
for v in "--path 1" "--path 1 --pdl 0" "--path 1 --kernel-timing 0" "--path 1 --pdl 0 --kernel-timing 0"; do
  echo "== $v" >> gpurun_out/perf_$TAG.txt
  timeout 300 $B $v >> gpurun_out/perf_$TAG.txt 2>&1
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_wave|k_update" -s 4 -c 3 -o gpurun_out/prof_perf_$TAG \
    python bench.py --steps 1 --warmup 0 --maxit 8 --no-cpu-baseline --no-e2e --path 3 > gpurun_out/ncu_perf_$TAG.log 2>&1
