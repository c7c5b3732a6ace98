#!/bin/bash
# sanitizer follow-up: the same runs with the device loop off, and the full messages of the failing ones
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
out=gpurun_out/sanit_r02b.txt; rm -f $out
S="python bench.py --steps 1 --warmup 0 --maxit 3 --no-cpu-baseline --no-e2e --kernel-timing 0"
for tool in racecheck synccheck; do
  for v in "--config c2 --device-loop 0" "--operator aniso --config c1a --device-loop 0" "--operator vv --config c2v --device-loop 0" "--config c1 --force-comm --comm peer --device-loop 0"; do
    echo "== $tool $v" >> $out
    timeout 900 compute-sanitizer --tool $tool --print-limit 5 $S $v 2>&1 | grep -E "ERROR SUMMARY|RACECHECK SUMMARY|Error|error|Barrier" | head -5 >> $out
  done
done
echo "== full: racecheck --config c2 (device loop on)" >> $out
timeout 900 compute-sanitizer --tool racecheck --print-limit 3 $S --config c2 2>&1 | tail -25 >> $out
echo "== full: synccheck --config c1 (device loop on)" >> $out
timeout 900 compute-sanitizer --tool synccheck --print-limit 2 $S --config c1 2>&1 | head -40 >> $out
echo "== full: synccheck aniso c1a (device loop off)" >> $out
timeout 900 compute-sanitizer --tool synccheck --print-limit 2 $S --operator aniso --config c1a --device-loop 0 2>&1 | head -40 >> $out
