#!/bin/bash
# minimal synccheck reproducer (tools/sanit/repro.cu): plain launches, a captured graph, a WHILE graph
mkdir -p gpurun_out; out=gpurun_out/sanit_r02e.txt; rm -f $out
cd tools/sanit
for m in "0 0" "1 0" "2 0" "2 1"; do
  echo "== repro $m" >> ../../$out
  timeout 300 compute-sanitizer --tool synccheck --print-limit 2 ./repro $m > tmp.txt 2>&1
  grep -E "ERROR SUMMARY|Barrier|mode|at " tmp.txt | head -4 >> ../../$out
done
cat ../../$out
