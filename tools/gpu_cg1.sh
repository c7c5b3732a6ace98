#!/bin/bash
# single-reduction path: parity tests, bench lines (path 1 vs 4, plain and with a one-rank NCCL communicator)
TAG=${1:-cg1}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$TAG.log 2>&1
timeout 900 python -m pytest tests/test_gpu_cg1.py -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_cg1_$TAG.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_cg1_$TAG.log
tail -15 gpurun_out/pytest_cg1_$TAG.log
B="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e"
for v in "--path 1" "--path 4" "--path 1 --force-comm" "--path 4 --force-comm"; do
  timeout 300 $B $v > gpurun_out/bench_${TAG}_tmp.json 2>> gpurun_out/bench_$TAG.err
  python -c "import json; d=json.load(open('gpurun_out/bench_${TAG}_tmp.json')); print('$v', round(d['value'],1), d['config']['iters_per_solve'], round(d['roofline']['avg_launch_ms']*1e3,1), d['per_kernel'])" | tee -a gpurun_out/bench_$TAG.txt
done
