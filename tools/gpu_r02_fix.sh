#!/bin/bash
# after the aniso peer shift fix and the vectorized assembly: peer + parity + aniso tests, the assembly launch
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_fix.log 2>&1
timeout 1800 python -m pytest tests/test_gpu_peer.py tests/test_gpu_parity.py tests/test_gpu_multirank.py tests/test_gpu_aniso.py tests/test_gpu_nccl.py -x -q > gpurun_out/pytest_fix.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_fix.log
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"k_assemble|k_face_coeffs|k_finalize_D" --csv --log-file gpurun_out/ncu_assemble.csv \
    python bench.py --steps 1 --warmup 0 --maxit 4 --no-cpu-baseline --no-e2e --from-fields --config c5 > /dev/null 2>&1
timeout 900 python bench.py --config c5 --from-fields --steps 20 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_c5_fields.json 2> gpurun_out/bench_c5.err
