#!/bin/bash
# the other BASELINE.json configurations at N = 1 (c4 weak-scaling slab, c5 warm-started time loop, c2)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python bench.py --config c5 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_c5_$1.json 2> gpurun_out/bench_c5_$1.err
timeout 900 python bench.py --config c4 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_c4_$1.json 2> gpurun_out/bench_c4_$1.err
timeout 600 python bench.py --config c2 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_c2_$1.json 2> gpurun_out/bench_c2_$1.err
timeout 600 python bench.py --config c1 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_c1_$1.json 2> gpurun_out/bench_c1_$1.err

timeout 600 python bench.py --config c3 --from-fields --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_c3ff_$1.json 2> gpurun_out/bench_c3ff_$1.err
