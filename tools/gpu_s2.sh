mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_s2.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_s2.log 2>&1; echo "smoke exit $?" >> gpurun_out/smoke_s2.log
timeout 900 python bench.py > gpurun_out/bench_s2.json 2> gpurun_out/bench_s2.err
