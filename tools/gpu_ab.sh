#!/bin/bash
# A/B: bench each variant library (MPFD_B200_LIB) at 512^3, all presets
OUT=gpurun_out/${TAG:-ab}
mkdir -p $OUT
for v in ${VARIANTS}; do
  L=paper_2505_20911_b200/libmpfd_b200_$v.so
  [ "$v" = base ] && L=paper_2505_20911_b200/libmpfd_b200.so
  MPFD_B200_LIB=$PWD/$L timeout 600 python bench.py --no-e2e --no-cpu-baseline ${BENCH_ARGS} > $OUT/bench_$v.json 2> $OUT/bench_$v.err
  python -c "
import json; d=json.load(open('$OUT/bench_$v.json')); print('$v', {k: round(v['ms_per_step'],2) for k,v in d.get('per_precision',{}).items()})" || tail -3 $OUT/bench_$v.err
done
