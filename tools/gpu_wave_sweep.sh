#!/bin/bash
# wave kernel tile sweep: rebuild with different kWaveTile values and time path 3
mkdir -p gpurun_out
for T in 1024 2048; do
  sed -i "s/^constexpr int kWaveTile = [0-9]*;/constexpr int kWaveTile = $T;/" paper_2303_03398_b200/csrc/wave.cuh
  python -m paper_2303_03398_b200.build --force > /dev/null 2>&1
  echo "== tile $T" >> gpurun_out/sweep.txt
  timeout 300 python bench.py --steps 3 --warmup 3 --maxit 300 --no-cpu-baseline --no-e2e --path 3 >> gpurun_out/sweep.txt 2>&1
done
