#!/bin/bash
# vector viscosity round trip: build, GPU parity tests of the vector operator, sanitizer on a small solve
TAG=${1:-vv}
K=${2:-""}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$TAG.log 2>&1
if [ -n "$K" ]; then
  timeout 1200 python -m pytest tests/test_gpu_vv.py -m gpu -q -x -p no:cacheprovider -k "$K" > gpurun_out/pytest_vv_$TAG.log 2>&1
else
  timeout 1200 python -m pytest tests/test_gpu_vv.py -m gpu -q -p no:cacheprovider > gpurun_out/pytest_vv_$TAG.log 2>&1
fi
echo "pytest exit $?" >> gpurun_out/pytest_vv_$TAG.log
tail -30 gpurun_out/pytest_vv_$TAG.log
