mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 600 compute-sanitizer --tool memcheck --print-limit 5 python bench.py --config c1 --steps 1 --warmup 0 --maxit 3 --no-cpu-baseline --no-e2e > gpurun_out/sanit.txt 2>&1
timeout 900 compute-sanitizer --tool memcheck --print-limit 5 python bench.py --config c3 --steps 1 --warmup 0 --maxit 2 --no-cpu-baseline --no-e2e >> gpurun_out/sanit.txt 2>&1
bash tools/gpu_perf.sh p4
