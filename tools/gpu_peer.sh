#!/bin/bash
TAG=${1:-peer}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$TAG.log 2>&1
timeout 900 python -m pytest tests/test_gpu_peer.py -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_peer_$TAG.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_peer_$TAG.log
tail -30 gpurun_out/pytest_peer_$TAG.log | cut -c1-300
B="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --kernel-timing 0"
for v in "--path 1" "--path 1 --force-comm" "--path 1 --force-comm --comm peer" "--path 4 --force-comm --comm peer"; do
  rm -f gpurun_out/bench_${TAG}_tmp.json
  timeout 200 $B $v > gpurun_out/bench_${TAG}_tmp.json 2>> gpurun_out/bench_$TAG.err
  echo "rc=$? $v" >> gpurun_out/bench_$TAG.txt
  python -c "import json; d=json.load(open('gpurun_out/bench_${TAG}_tmp.json')); print('$v', round(d['value'],1), d['config']['iters_per_solve'], round(d['ms_per_step'],2), d['config']['parallelism'])" >> gpurun_out/bench_$TAG.txt 2>&1
done
cat gpurun_out/bench_$TAG.txt
