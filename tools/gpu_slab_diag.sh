#!/bin/bash
# Where the P=8 slab iteration goes: size sweep (overhead intercept), per-kernel event times, and ncu
# DRAM bytes per kernel with/without the L2 residency plan (--cache-control none: cross-kernel reuse)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_diag.log 2>&1
B="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --maxit 400"
out=gpurun_out/slab_diag.txt
for sh in 150,300,10 150,300,20 150,300,40 150,300,75 150,300,150; do
  for kt in 0 1; do
    MASPCG_L2_MASK=0 timeout 200 $B --kernel-timing $kt --shape $sh > gpurun_out/d_tmp.json 2>> gpurun_out/diag.err
    python - >> $out <<PY
import json; d=json.load(open('gpurun_out/d_tmp.json')); pk=d['per_kernel']; rf=d['roofline']
print('$sh', 'kt=$kt', round(1e6/d['value'],2), 'us/it', 'stencil_ms', rf['avg_launch_ms'], 'upd GB/s', pk['update_GBps'], 'pupd GB/s', pk['p_update_GBps'], 'kern share', pk['kernels_share_of_step'])
PY
  done
done
for m in 0 0xC15; do
  MASPCG_L2_MASK=$m timeout 600 ncu --cache-control none --clock-control none -k regex:"k_matvec_vec2|k_update_vec2|k_pupdate_vec2" -s 60 -c 9 \
    --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct \
    --csv --log-file gpurun_out/ncu_slab_l2_$m.csv python bench.py --steps 1 --warmup 0 --maxit 40 --shape 150,300,75 --no-cpu-baseline --no-e2e --kernel-timing 0 > /dev/null 2>&1
done
python -c "import torch; p=torch.cuda.get_device_properties(0); print('l2', p.L2_cache_size, 'persist max', getattr(p,'persisting_l2_cache_max_size',None))" >> $out 2>&1
