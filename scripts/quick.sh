#!/bin/bash
# Iteration loop on the GPU box: collision-related GPU parity tests, then the
# bench step (no format legs) with its per-stage kernel times.
O=gpurun_out/q
mkdir -p $O
T=${QT:-"tests/test_gpu_parity.py tests/test_gpu_sparse.py tests/test_gpu_fused.py tests/test_gpu_tiles.py tests/test_gpu_robots.py"}
if [ "${QT}" != "none" ]; then
  timeout 900 python -m pytest $T -m gpu -x -q > $O/tests.txt 2>&1; tail -2 $O/tests.txt
fi
timeout 300 python bench.py --no-formats --no-iko --no-to --no-e2e --no-cpu ${QB} > $O/bench.json 2> $O/bench.err
python -c "
import json;d=json.loads(open('$O/bench.json').read().strip().splitlines()[-1]);r=d['roofline']
print('ms', round(d['ms_per_step'],4), 'kernel_ms', r['kernel_ms'], 'frac', round(r['frac'],4))"
