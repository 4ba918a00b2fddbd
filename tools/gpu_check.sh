#!/bin/bash
# one gpurun call: gpu tests, smoke, bench (JSON line)
OUT=gpurun_out/${TAG:-check}
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $OUT/gpu.txt
if [ -z "$NO_TESTS" ]; then
  timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider ${PYTEST_ARGS} > $OUT/pytest_gpu.log 2>&1
  tail -3 $OUT/pytest_gpu.log
  python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; cat $OUT/smoke.log
fi
timeout 900 python bench.py ${BENCH_ARGS} > $OUT/bench.json 2> $OUT/bench.err
python -c "
import json; d=json.load(open('$OUT/bench.json')); print('ms/step', d['ms_per_step'], {k: round(v['ms_per_step'],2) for k,v in d.get('per_precision',{}).items()})"
