#!/bin/bash
# ncu --set full captures of the fused kernel per preset, reports kept
# (source-level attribution is read here with `ncu -i ... --page source`)
OUT=gpurun_out/${TAG:-prof}
mkdir -p $OUT
for P in ${NCU_PRESETS:-DP HPSP}; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:${KREGEX:-k_fused} -s ${NCU_SKIP:-3} -c 1 \
     -o $OUT/prof_$P python bench.py --grid ${NCU_N:-256} --precision $P --steps 1 --warmup 3 --modes "" --no-e2e --no-cpu-baseline > $OUT/ncu_$P.log 2>&1
done
ls -la $OUT
