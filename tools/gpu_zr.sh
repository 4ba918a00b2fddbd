#!/bin/bash
# A/B of z-range policies: per preset at 512^3 and the HPSP slab sweep
OUT=gpurun_out/${TAG:-zr}
mkdir -p $OUT
for rep in 1 2; do
for v in ${VARIANTS:-base zr0}; do
  L=paper_2505_20911_b200/libmpfd_b200_$v.so
  [ "$v" = base ] && L=paper_2505_20911_b200/libmpfd_b200.so
  MPFD_B200_LIB=$PWD/$L timeout 600 python bench.py --precision DP --modes "SPDP,HPSP" --steps 5 --no-e2e --no-cpu-baseline --no-memory-table --slab-sweep "${SWEEP:-4,8}" > $OUT/bench_${v}.json 2> $OUT/bench_${v}.err
  python -c "
import json; d=json.load(open('$OUT/bench_${v}.json'))
print('$v', {k: round(v['ms_per_step'],2) for k,v in d['per_precision'].items()}, {k:(round(v.get('ms_per_step',0),2)) for k,v in d.get('slab_sweep',{}).items() if k!='note'})" || tail -3 $OUT/bench_${v}.err
done
done
