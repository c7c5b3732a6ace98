#!/bin/bash
# synccheck / racecheck after the warp-reconvergence fixes
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
out=gpurun_out/sanit_r02c.txt; rm -f $out
S="python bench.py --steps 1 --warmup 0 --maxit 3 --no-cpu-baseline --no-e2e --kernel-timing 0"
for tool in synccheck racecheck; do
  for v in "--config c1" "--config c2" "--operator aniso --config c1a" "--operator vv --config c2v --device-loop 0" "--operator vv --config c2v" "--config c1 --force-comm --comm peer"; do
    echo "== $tool $v" >> $out
    timeout 900 compute-sanitizer --tool $tool --print-limit 2 $S $v > gpurun_out/san_tmp.txt 2>&1
    grep -E "ERROR SUMMARY|RACECHECK SUMMARY|Barrier error|failed|Error:" gpurun_out/san_tmp.txt | head -3 >> $out
    grep -m2 -E "^=========     at " gpurun_out/san_tmp.txt >> $out
  done
done
cat $out
