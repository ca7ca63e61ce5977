#!/bin/bash
# ncu --set full of the two collision passes of one vapr_cost_grad (config 4,
# 43-bit, sparse), their per-SASS-instruction source pages (the self pass is
# launch 0, the world pass launch 1) and the summary; map the SASS to source
# lines here with scripts/sass_line_map.py and the same build's cubin.
set -u
O=gpurun_out/p1
mkdir -p $O
python scripts/run_mode.py 43bit sparse > /dev/null && ncu --set full --import-source on --clock-control none \
  -k regex:collision_kernel -c 2 -o $O/coll -f python scripts/run_mode.py 43bit sparse > $O/ncu.log 2>&1
for L in 0 1; do
  ncu -i $O/coll.ncu-rep --page source --csv -k regex:collision --launch-skip $L --launch-count 1 \
      --print-source sass > $O/sass$L.csv 2>/dev/null
done
python scripts/ncu_summary.py $O/coll.ncu-rep > $O/summary.txt 2>&1
ncu -i $O/coll.ncu-rep --page raw --csv > $O/raw.csv 2>/dev/null
ls -la $O
