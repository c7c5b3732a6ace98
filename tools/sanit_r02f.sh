#!/bin/bash
# synccheck / racecheck with the host loop (--device-loop 0): the conditional-WHILE body is what
# synccheck flags (tools/sanit/repro.cu), so the kernels are checked on the host-chunk path
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
out=gpurun_out/sanit_r02f.txt; rm -f $out
S="python bench.py --steps 1 --warmup 0 --maxit 3 --no-cpu-baseline --no-e2e --kernel-timing 0 --device-loop 0"
for tool in synccheck racecheck; do
for v in "--config c1" "--config c2" "--operator vv --config c2v" "--operator aniso --config c1a" "--config c1 --force-comm --comm peer" "--config c1 --path 4"; do
  echo "== $tool $v" >> $out
  timeout 1200 compute-sanitizer --tool $tool --print-limit 2 $S $v > gpurun_out/san_tmp.txt 2>&1
  echo "rc $?" >> $out
  grep -E "ERROR SUMMARY|Barrier error|hazard|failed|Error|error" gpurun_out/san_tmp.txt | head -3 >> $out
  grep -m1 -E "^=========     at " gpurun_out/san_tmp.txt >> $out
done; done
cat $out
