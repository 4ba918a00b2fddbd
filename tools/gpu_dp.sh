#!/bin/bash
# DP kernel iteration: DP parity subset + quick timing of all presets
OUT=gpurun_out/${TAG:-dp}
mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -p no:cacheprovider -k "${PYK:-DP and not 1024 and not 512}" > $OUT/pytest.log 2>&1
tail -3 $OUT/pytest.log
for P in ${PRESETS:-DP SPDP HPSP}; do
  timeout 600 python bench.py --precision $P --steps ${STEPS:-5} --warmup 3 --modes "" --slab-sweep "" --no-e2e --no-cpu-baseline ${ARGS} > $OUT/bench_$P.json 2> $OUT/bench_$P.err
  python -c "import json,sys; d=json.load(open('$OUT/bench_$P.json')); print('$P', round(d['ms_per_step'],2), 'ms/step', round(d['value']/1e9,3), 'Gpt/s')" || tail -5 $OUT/bench_$P.err
done
