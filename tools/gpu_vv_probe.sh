#!/bin/bash
# vv march timing probe (+ optional ncu of the arithmetic-only mode and the full kernel)
TAG=${1:-p}
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_vv.py -x -q -k "march" > gpurun_out/pytest_march_$TAG.log 2>&1
tail -2 gpurun_out/pytest_march_$TAG.log
timeout 600 python tools/vv_march_probe.py c3v > gpurun_out/probe_$TAG.txt 2>&1; cat gpurun_out/probe_$TAG.txt
MASPCG_VV_MARCH_DEBUG=2 timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_vv_march" -s 5 -c 1 \
    -o gpurun_out/prof_arith_$TAG python tools/vv_march_probe.py c3v > gpurun_out/ncu_arith_$TAG.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_vv_march" -s 5 -c 1 \
    -o gpurun_out/prof_full_$TAG python tools/vv_march_probe.py c3v > gpurun_out/ncu_full_$TAG.log 2>&1
