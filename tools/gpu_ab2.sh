#!/bin/bash
# A/B timing of variant libraries (MPFD_B200_LIB) per preset at 512^3, then
# optionally one ncu --set full source capture (NCU_VAR, NCU_PRESET, 256^3)
OUT=gpurun_out/${TAG:-ab2}
mkdir -p $OUT
for rep in ${REPS:-1 2}; do
for v in ${VARIANTS:-base}; do
  L=paper_2505_20911_b200/libmpfd_b200_$v.so
  [ "$v" = base ] && L=paper_2505_20911_b200/libmpfd_b200.so
  for P in ${PRESETS:-HPSP}; do
    MPFD_B200_LIB=$PWD/$L timeout 600 python bench.py --precision $P --steps ${STEPS:-5} --warmup 3 --modes "" --slab-sweep "" --no-e2e --no-cpu-baseline > $OUT/bench_${v}_$P.json 2> $OUT/bench_${v}_$P.err
    python -c "import json; d=json.load(open('$OUT/bench_${v}_$P.json')); print('$v $P', round(d['ms_per_step'],2))" || tail -3 $OUT/bench_${v}_$P.err
  done
done
done
if [ -n "$NCU_VAR" ]; then
  v=$NCU_VAR; P=${NCU_PRESET:-HPSP}
  L=paper_2505_20911_b200/libmpfd_b200_$v.so
  [ "$v" = base ] && L=paper_2505_20911_b200/libmpfd_b200.so
  MPFD_B200_LIB=$PWD/$L timeout 600 ncu --set full --clock-control none --import-source on -k regex:${KREGEX:-k_fused} -s 3 -c 1 \
     -o $OUT/prof_${v}_$P python bench.py --grid ${NCU_N:-256} --precision $P --steps 1 --warmup 3 --modes "" --slab-sweep "" --no-e2e --no-cpu-baseline > $OUT/ncu_${v}_$P.log 2>&1
  ncu -i $OUT/prof_${v}_$P.ncu-rep --page raw --csv > $OUT/raw_${v}_$P.csv 2>/dev/null
  ncu -i $OUT/prof_${v}_$P.ncu-rep --page source --csv --print-source cuda,sass > $OUT/src_${v}_$P.csv 2>/dev/null
  gzip -f $OUT/src_${v}_$P.csv
  rm -f $OUT/prof_${v}_$P.ncu-rep
fi
