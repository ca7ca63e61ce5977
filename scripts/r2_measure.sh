#!/bin/bash
# Round-2 measurement session (one gpurun call): GPU suite + smoke, the bench
# line and the oracle arm, an ncu launch list of the bench step, full ncu
# captures of the step's kernels (sparse and dense 43-bit, fused), small-batch
# latency.  Outputs under gpurun_out/r2/.
set -u
O=gpurun_out/r2
mkdir -p $O
python -m pytest tests -m gpu -q > $O/gpu_tests.txt 2>&1; tail -1 $O/gpu_tests.txt
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke.txt 2>&1; tail -1 $O/smoke.txt
python bench.py > $O/bench.json 2> $O/bench.err; tail -c 200 $O/bench.json
python bench.py --impl reference --steps 3 --warmup 1 > $O/bench_ref.json 2> $O/bench_ref.err
python scripts/time_tiles.py > $O/small_latency.txt 2>&1
python scripts/time_small.py > $O/small_stages.txt 2>&1
B="bench.py --steps 2 --warmup 1 --no-formats --no-iko --no-to --no-e2e --no-cpu --no-graph"
python $B > /dev/null 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file $O/launches_bench.csv python $B > $O/ncu_list.log 2>&1
K='regex:fk_kernel|collision_kernel|traj_reduce|aggregate|bk_kernel'
for m in sparse dense; do
  python scripts/run_mode.py 43bit $m > /dev/null && ncu --set full --import-source on --clock-control none \
      -k "$K" -c 6 -o $O/step_${m}43 -f python scripts/run_mode.py 43bit $m > $O/ncu_${m}.log 2>&1
done
python scripts/run_mode.py 43bit fused > /dev/null && ncu --set full --import-source on --clock-control none \
    -k "$K" -c 2 -o $O/step_fused43 -f python scripts/run_mode.py 43bit fused > $O/ncu_fused.log 2>&1
python scripts/run_mode.py fp32 sparse > /dev/null && ncu --set full --clock-control none \
    -k "$K" -c 6 -o $O/step_sparse32 -f python scripts/run_mode.py fp32 sparse > $O/ncu_sparse32.log 2>&1
ls $O
# summaries on the box (the reports themselves exceed gpurun's copy-back cap)
for r in $O/*.ncu-rep; do
  b=${r%.ncu-rep}
  python scripts/ncu_summary.py $r > $b.summary.txt 2>&1
  ncu -i $r --page raw --csv > $b.raw.csv 2>/dev/null
done
# the collision passes' per-SASS-instruction source pages (self = launch 0,
# world = launch 1 of the collision kernels), mapped to source lines here
# with scripts/sass_line_map.py and the same build's cubin
for L in 0 1; do
  ncu -i $O/step_sparse43.ncu-rep --page source --csv -k regex:collision --launch-skip $L --launch-count 1 \
      --print-source sass > $O/sass_collision_$L.csv 2>/dev/null
done
rm -f $O/step_dense43.ncu-rep $O/step_sparse32.ncu-rep $O/step_fused43.ncu-rep
du -sh $O
