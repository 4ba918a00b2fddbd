#!/bin/bash
# bench + ncu --set full per preset; exports raw and cuda,sass source pages
# (gzipped) on the box, drops the .ncu-rep (64 MiB copy-back limit)
OUT=gpurun_out/${TAG:-prof}
mkdir -p $OUT
if [ -z "$NO_BENCH" ]; then
  timeout 900 python bench.py ${BENCH_ARGS:---no-e2e --no-cpu-baseline} > $OUT/bench.json 2> $OUT/bench.err
  cat $OUT/bench.json
fi
for P in ${NCU_PRESETS:-DP SPDP HPSP}; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:${KREGEX:-k_fused} -s ${NCU_SKIP:-3} -c ${NCU_COUNT:-3} \
     -o $OUT/prof_$P python bench.py --grid ${NCU_N:-256} --precision $P --steps 1 --warmup 3 --modes "" --slab-sweep "" --no-e2e --no-cpu-baseline > $OUT/ncu_$P.log 2>&1
  ncu -i $OUT/prof_$P.ncu-rep --page raw --csv > $OUT/raw_$P.csv 2>/dev/null
  ncu -i $OUT/prof_$P.ncu-rep --page source --csv --print-source cuda,sass > $OUT/src_$P.csv 2>/dev/null
  gzip -f $OUT/src_$P.csv
  rm -f $OUT/prof_$P.ncu-rep
done
ls -la $OUT
