#!/bin/bash
# L2-residency experiment: narrow fused lanes (SDV_FILL lowers the fused-path
# threshold) whose RK workspace (~13.4 MB per vector at 512^2) stays in the
# 126 MB L2, replayed as CUDA graphs. Prints HVP/s per (lanes, block width).
out=${1:-gpurun_out/l2_probe.txt}
: > $out
for lanes in 1 2 4; do
  echo "== fused lanes=$lanes (SDV_FILL=64)" >> $out
  SDV_FILL=64 SDV_LANES=$lanes SDV_GRAPH_MAX=16 python tools/small_block.py 3 4,6,8,12,16 >> $out 2>&1
done
echo "== default small-block path" >> $out
python tools/small_block.py 3 4,8 >> $out 2>&1
