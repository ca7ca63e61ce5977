#!/bin/bash
# ncu --set full of the FK, aggregation and BK kernels of one vapr_cost_grad
# (config 4, 43-bit, sparse) and their per-SASS-instruction source pages (map
# them to source lines here with scripts/sass_line_map.py).
set -u
O=gpurun_out/p2
mkdir -p $O
python scripts/run_mode.py 43bit sparse > /dev/null && ncu --set full --import-source on --clock-control none \
  -k 'regex:fk_kernel|aggregate|bk_kernel' -c 3 -o $O/st -f python scripts/run_mode.py 43bit sparse > $O/ncu.log 2>&1
for k in fk_kernel aggregate bk_kernel; do
  ncu -i $O/st.ncu-rep --page source --csv -k regex:$k --launch-count 1 --print-source sass > $O/sass_$k.csv 2>/dev/null
done
python scripts/ncu_summary.py $O/st.ncu-rep > $O/summary.txt 2>&1
ls -la $O
