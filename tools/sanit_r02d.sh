#!/bin/bash
# synccheck: is programmatic dependent launch what the tool flags?
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
out=gpurun_out/sanit_r02d.txt; rm -f $out
S="python bench.py --steps 1 --warmup 0 --maxit 3 --no-cpu-baseline --no-e2e --kernel-timing 0"
for v in "--config c1 --pdl 0" "--config c1 --pdl 0 --l2-keep 0" "--config c1 --l2-keep 0" "--operator vv --config c2v --pdl 0" "--config c2 --pdl 0" "--operator aniso --config c1a --pdl 0" "--config c1 --force-comm --comm peer --pdl 0"; do
  echo "== synccheck $v" >> $out
  timeout 900 compute-sanitizer --tool synccheck --print-limit 2 $S $v > gpurun_out/san_tmp.txt 2>&1
  grep -E "ERROR SUMMARY|Barrier error|failed" gpurun_out/san_tmp.txt | head -2 >> $out
  grep -m1 -E "^=========     at " gpurun_out/san_tmp.txt >> $out
done
cat $out
