#!/bin/bash
# A/B of library variants on the GPU box: for each VAPR_SO (space-separated in
# $VARIANTS; "default" = the in-tree libvapr.so): the bench step's per-stage
# times, then an ncu launch list of one step (per-pass collision durations).
O=gpurun_out/ab
mkdir -p $O
for v in ${VARIANTS:-default}; do
  if [ "$v" = default ]; then unset VAPR_SO; else export VAPR_SO=paper_2310_07854_b200/variants/libvapr_$v.so; fi
  for rep in 1 2; do
  timeout 300 python bench.py --no-formats --no-iko --no-to --no-e2e --no-cpu ${QB} > $O/bench_$v.json 2> $O/bench_$v.err
  python -c "
import json;d=json.loads(open('$O/bench_$v.json').read().strip().splitlines()[-1]);r=d['roofline']
print('$v', 'ms', round(d['ms_per_step'],4), 'kernel_ms', r['kernel_ms'])"
  done
  if [ -n "$NCU" ]; then
  ncu --metrics gpu__time_duration.sum --clock-control none -k regex:collision_kernel --csv \
      --log-file $O/launch_$v.csv python scripts/run_mode.py ${MODE:-43bit sparse} 2 > /dev/null 2>&1
  python - <<PY
import csv
rows=list(csv.reader(open('$O/launch_$v.csv')))
h=next(i for i,r in enumerate(rows) if 'Kernel Name' in r); H=rows[h]
print('$v', 'collision launches us:', [round(float(r[H.index('Metric Value')].replace(',',''))/1e3,1) for r in rows[h+1:] if len(r)>5])
PY
  fi
done
