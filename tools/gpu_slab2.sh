#!/bin/bash
# P=8 / P=4 slab after the kernel-entry restructure (loads before scalars, acq_rel tickets), with the
# persisting L2 set-aside for the residency plan; plus parity subset
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_s2.log 2>&1
python -c "
import ctypes, torch
cu = ctypes.CDLL('libcudart.so') if False else None
p = torch.cuda.get_device_properties(0); print('L2', p.L2_cache_size)
" > gpurun_out/slab2.txt 2>&1
B="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --kernel-timing 0 --maxit 400"
run() {  # label, env, shape, extra
  env $2 timeout 200 $B --shape $3 $4 > gpurun_out/s2_tmp.json 2>> gpurun_out/s2.err
  python -c "import json; d=json.load(open('gpurun_out/s2_tmp.json')); print('$3', '$1', '$4', round(d['value'],1), 'us/it', round(1e6/d['value'],2))" >> gpurun_out/slab2.txt
}
for rep in 1 2; do
for sh in 150,300,75 150,300,150; do
  run off "MASPCG_L2_MASK=0" $sh ""
  run auto "X=1" $sh ""
  run auto-nopersist "MASPCG_L2_PERSIST=0" $sh ""
  run budget0.6 "MASPCG_L2_BUDGET=0.6" $sh ""
  run DPRX+Tfirst "MASPCG_L2_MASK=0xC55" $sh ""
done
done
for v in "--force-comm" "--force-comm --comm peer"; do
  run off "MASPCG_L2_MASK=0" 150,300,75 "$v"
  run auto "X=1" 150,300,75 "$v"
  run auto-ipdl1 "MASPCG_INTERIOR_PDL=1" 150,300,75 "$v"
done
run off "MASPCG_L2_MASK=0" 150,300,600 ""
run auto "X=1" 150,300,600 ""
MASPCG_L2_MASK=0xC55 timeout 600 ncu --cache-control none --clock-control none -k regex:"k_matvec_vec2|k_update_vec2|k_pupdate_vec2" -s 60 -c 6 \
    --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct \
    --csv --log-file gpurun_out/ncu_slab2_keep.csv python bench.py --steps 1 --warmup 0 --maxit 40 --shape 150,300,75 --no-cpu-baseline --no-e2e --kernel-timing 0 > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_multirank.py tests/test_gpu_peer.py tests/test_gpu_nccl.py -x -q > gpurun_out/pytest_s2.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_s2.log
