#!/bin/bash
# quick: build, a subset of GPU tests, perf variants + ncu.  usage: bash tools/gpu_quick.sh TAG "pytest -k expr"
TAG=${1:-q}
K=${2:-"solve_parity or loop_modes or edge_cases"}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$TAG.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k "$K" > gpurun_out/pytest_quick_$TAG.log 2>&1
bash tools/gpu_perf.sh $TAG
