#!/bin/bash
# A/B of library files (LIBS="name=path ..."; default: the in-tree build vs
# libmpfd_b200_head.so) per preset at 512^3, alternating REPS times; then
# optionally the GPU test suite on the in-tree build (TESTS=1)
OUT=gpurun_out/${TAG:-ab3}
mkdir -p $OUT
LIBS=${LIBS:-"head=paper_2505_20911_b200/libmpfd_b200_head.so new=paper_2505_20911_b200/libmpfd_b200.so"}
for rep in ${REPS:-1 2}; do
for kv in $LIBS; do
  v=${kv%%=*}; L=${kv#*=}
  for P in ${PRESETS:-DP SPDP HPSP}; do
    MPFD_B200_LIB=$PWD/$L timeout 600 python bench.py --precision $P --steps ${STEPS:-5} --warmup 3 --modes "" --slab-sweep "" --no-e2e --no-cpu-baseline --no-memory-table ${ARGS} > $OUT/bench_${v}_${P}_$rep.json 2> $OUT/bench_${v}_${P}_$rep.err
    python -c "import json; d=json.load(open('$OUT/bench_${v}_${P}_$rep.json')); print('$v $P', round(d['ms_per_step'],3))" || tail -3 $OUT/bench_${v}_${P}_$rep.err
  done
done
done
if [ -n "$TESTS" ]; then
  timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -x ${TESTARGS} > $OUT/pytest_gpu.log 2>&1
  tail -3 $OUT/pytest_gpu.log
fi
