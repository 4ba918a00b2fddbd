#!/bin/bash
# quick per-preset timing at 512^3 (no e2e / cpu baseline), optional smoke
OUT=gpurun_out/${TAG:-qb}
mkdir -p $OUT
[ -n "$SMOKE" ] && python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; cat $OUT/smoke.log 2>/dev/null
for P in ${PRESETS:-DP SPDP HPSP}; do
  timeout 600 python bench.py --precision $P --steps ${STEPS:-5} --warmup 3 --modes "" --slab-sweep "" --no-e2e --no-cpu-baseline ${ARGS} > $OUT/bench_$P.json 2> $OUT/bench_$P.err
  python -c "import json,sys; d=json.load(open('$OUT/bench_$P.json')); print('$P', round(d['ms_per_step'],2), 'ms/step', round(d['value']/1e9,3), 'Gpt/s')" || tail -5 $OUT/bench_$P.err
done
