#!/bin/bash
# Round-2 check: the whole -m gpu suite (golden fixtures included), smoke, default bench line (c3), the ncu
# launch list of a short run and ncu --set full of the three loop kernels (refreshes profiles/ncu_stencil_path1.json)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_chk.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_chk.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu_chk.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_chk.log 2>&1; echo "smoke exit $?" >> gpurun_out/smoke_chk.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_chk.json 2> gpurun_out/bench_chk.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_chk.csv \
    python bench.py --steps 1 --warmup 0 --maxit 30 --no-cpu-baseline --no-e2e > gpurun_out/ncu_launch_chk.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_matvec_vec2|k_update_vec2|k_pupdate_vec2" -s 4 -c 3 \
    -o gpurun_out/prof_default_chk python bench.py --steps 1 --warmup 0 --maxit 8 --no-cpu-baseline --no-e2e > gpurun_out/ncu_full_chk.log 2>&1
