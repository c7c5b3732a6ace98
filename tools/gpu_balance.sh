python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
B="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --kernel-timing 0 --maxit 400"
for rep in 1 2; do
for sh in 150,300,75 150,300,600; do
  for e in 0 1; do
    MASPCG_GRID_BALANCE=$e timeout 200 $B --shape $sh > gpurun_out/bal_tmp.json 2>> gpurun_out/bal.err
    python -c "import json; d=json.load(open('gpurun_out/bal_tmp.json')); print('$sh bal=$e', round(d['value'],1), 'us/it', round(1e6/d['value'],2), d['clocks']['sm_mhz'])"
  done
done
done
