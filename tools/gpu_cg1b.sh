#!/bin/bash
TAG=${1:-cg1b}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$TAG.log 2>&1
B="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e"
for v in "--path 4" "--path 1 --force-comm --maxit 100 --steps 1" "--path 4 --force-comm --maxit 100 --steps 1" "--path 1 --force-comm" "--path 4 --force-comm"; do
  rm -f gpurun_out/bench_${TAG}_tmp.json
  NCCL_DEBUG=WARN timeout 150 $B $v > gpurun_out/bench_${TAG}_tmp.json 2>> gpurun_out/bench_$TAG.err
  echo "rc=$? $v" >> gpurun_out/bench_$TAG.txt
  python -c "import json; d=json.load(open('gpurun_out/bench_${TAG}_tmp.json')); print('$v', round(d['value'],1), d['config']['iters_per_solve'], round(d['ms_per_step'],2), round(d['roofline']['avg_launch_ms']*1e3,1), d['per_kernel'])" >> gpurun_out/bench_$TAG.txt 2>&1
done
cat gpurun_out/bench_$TAG.txt
