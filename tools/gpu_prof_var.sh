#!/bin/bash
# ncu --set full of the fused kernel for each variant library (MPFD_B200_LIB),
# one preset; raw + cuda,sass source pages exported on the box
OUT=gpurun_out/${TAG:-pv}
mkdir -p $OUT
P=${PRESET:-DP}
for v in ${VARIANTS}; do
  L=paper_2505_20911_b200/libmpfd_b200_$v.so
  [ "$v" = base ] && L=paper_2505_20911_b200/libmpfd_b200.so
  MPFD_B200_LIB=$PWD/$L timeout 600 python bench.py --precision $P --steps ${STEPS:-4} --warmup 3 --modes "" --slab-sweep "" --no-e2e --no-cpu-baseline > $OUT/bench_$v.json 2> $OUT/bench_$v.err
  python -c "import json; d=json.load(open('$OUT/bench_$v.json')); print('$v', round(d['ms_per_step'],2))" || tail -3 $OUT/bench_$v.err
  [ -n "$NO_NCU" ] && continue
  MPFD_B200_LIB=$PWD/$L timeout 600 ncu --set full --clock-control none --import-source on -k regex:${KREGEX:-k_fused} -s 3 -c 1 \
     -o $OUT/prof_$v python bench.py --grid ${NCU_N:-256} --precision $P --steps 1 --warmup 3 --modes "" --slab-sweep "" --no-e2e --no-cpu-baseline > $OUT/ncu_$v.log 2>&1
  ncu -i $OUT/prof_$v.ncu-rep --page raw --csv > $OUT/raw_$v.csv 2>/dev/null
  ncu -i $OUT/prof_$v.ncu-rep --page source --csv --print-source cuda,sass > $OUT/src_$v.csv 2>/dev/null
  gzip -f $OUT/src_$v.csv
  rm -f $OUT/prof_$v.ncu-rep
done
