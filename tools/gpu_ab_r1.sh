#!/bin/bash
# Same-box A/B of the round-1 tree (ab_r1/, git archive 724b4d6, untracked) against the current tree:
# the default c3 bench line and the P=8 slab, alternating.
mkdir -p gpurun_out
rm -f gpurun_out/ab_r1.txt
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_ab.log 2>&1
(cd ab_r1 && python -c "import __graft_entry__ as g; g.build()") >> gpurun_out/build_ab.log 2>&1
out=gpurun_out/ab_r1.txt
for rep in 1 2 3; do
  for tree in ab_r1 .; do
    (cd $tree && timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e) > gpurun_out/ab_tmp.json 2>> gpurun_out/ab.err
    python -c "import json; d=json.load(open('gpurun_out/ab_tmp.json')); r=d['roofline']; print('$tree', 'c3', round(d['value'],1), 'it/s stencil', round(r['avg_launch_ms']*1e3,1), 'us', d['per_kernel']['update_GBps'], d['per_kernel']['p_update_GBps'], d['clocks']['sm_mhz'])" >> $out
  done
done
for rep in 1 2; do
  for tree in ab_r1 .; do
    for v in "" "--force-comm" "--force-comm --comm peer"; do
      (cd $tree && timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --kernel-timing 0 --maxit 400 --shape 150,300,75 $v) > gpurun_out/ab_tmp.json 2>> gpurun_out/ab.err
      python -c "import json; d=json.load(open('gpurun_out/ab_tmp.json')); print('$tree', 'P8slab', '$v', round(1e6/d['value'],2), 'us/it', d['clocks']['sm_mhz'])" >> $out
    done
  done
done
# chunked vector-viscosity matvec: parity and bench (default chunked vs MASPCG_VV_CHUNK=0)
timeout 900 python -m pytest tests/test_gpu_vv.py -x -q > gpurun_out/pytest_vv_chunk.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_vv_chunk.log
for rep in 1 2; do
  for ch in "" 0; do
    env MASPCG_VV_CHUNK=$ch timeout 600 python bench.py --operator vv --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/vv_tmp.json 2>> gpurun_out/ab.err
    python -c "import json; d=json.load(open('gpurun_out/vv_tmp.json')); r=d['roofline']; print('vv chunk=$ch', round(d['value'],1), 'it/s matvec', round(r['avg_launch_ms']*1e3,1), 'us frac', r['frac'], d['clocks']['sm_mhz'])" >> gpurun_out/ab_r1.txt
  done
done
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"k_vv" -s 200 -c 60 --csv --log-file gpurun_out/ncu_vv_chunk.csv python bench.py --operator vv --steps 1 --warmup 0 --maxit 8 --no-cpu-baseline --no-e2e > /dev/null 2>&1
