#!/bin/bash
# chunked vector-viscosity matvec, live: default (ring from 0.45 L2) vs explicit rings vs off
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_vc.log 2>&1
out=gpurun_out/vvchunk.txt
rm -f $out
run() {  # label, env
  env $2 timeout 600 python bench.py --operator vv --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/vv_tmp.json 2>> gpurun_out/vc.err
  python -c "import json; d=json.load(open('gpurun_out/vv_tmp.json')); r=d['roofline']; print('$1', round(d['value'],1), 'it/s matvec', round(r['avg_launch_ms']*1e3,1), 'us frac', round(r['frac'],3), d['clocks']['sm_mhz'])" >> $out
}
for rep in 1 2; do
  run default "X=1"
  run off "MASPCG_VV_CHUNK=0"
  run ring57 "MASPCG_VV_CHUNK=57"
  run ring30 "MASPCG_VV_CHUNK=30"
  run ring80 "MASPCG_VV_CHUNK=80"
done
timeout 600 ncu --cache-control none --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:"k_vv" -s 200 -c 60 --csv --log-file gpurun_out/ncu_vv_chunk_nocc.csv python bench.py --operator vv --steps 1 --warmup 0 --maxit 8 --no-cpu-baseline --no-e2e > /dev/null 2>&1
