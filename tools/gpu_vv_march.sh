#!/bin/bash
# plane-marching TMA vector operator (vv_march.cu): parity, bench A/B against the two phases, ncu --set full
TAG=${1:-vvm}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$TAG.log 2>&1
timeout 900 python -m pytest tests/test_gpu_vv.py -x -q -k "march" > gpurun_out/pytest_march_$TAG.log 2>&1
tail -3 gpurun_out/pytest_march_$TAG.log
timeout 600 python bench.py --operator vv --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_vv_$TAG.json 2> gpurun_out/bench_vv_$TAG.err
cat gpurun_out/bench_vv_$TAG.json
MASPCG_VV_MARCH=0 timeout 600 python bench.py --operator vv --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_vv2ph_$TAG.json 2> gpurun_out/bench_vv2ph_$TAG.err
cat gpurun_out/bench_vv2ph_$TAG.json
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_vv_march" -s 3 -c 1 \
    -o gpurun_out/prof_vvm_$TAG python bench.py --operator vv --steps 1 --warmup 0 --maxit 6 --no-cpu-baseline --no-e2e > gpurun_out/ncu_full_vvm_$TAG.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_vv.py -x -q > gpurun_out/pytest_vv_$TAG.log 2>&1
tail -3 gpurun_out/pytest_vv_$TAG.log
