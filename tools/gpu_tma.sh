#!/bin/bash
# TMA iteration: HPSP-family parity subset + A/B timing of variant libraries
OUT=gpurun_out/${TAG:-tma}
mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_decomp_ipc.py -m gpu -x -q -p no:cacheprovider -k "${PYK:-HPSP or HP}" > $OUT/pytest.log 2>&1
tail -3 $OUT/pytest.log
for v in ${VARIANTS:-base}; do
  L=paper_2505_20911_b200/libmpfd_b200_$v.so
  [ "$v" = base ] && L=paper_2505_20911_b200/libmpfd_b200.so
  for P in ${PRESETS:-HPSP}; do
    MPFD_B200_LIB=$PWD/$L timeout 600 python bench.py --precision $P --steps ${STEPS:-5} --warmup 3 --modes "" --slab-sweep "" --no-e2e --no-cpu-baseline > $OUT/bench_${v}_$P.json 2> $OUT/bench_${v}_$P.err
    python -c "import json; d=json.load(open('$OUT/bench_${v}_$P.json')); print('$v $P', round(d['ms_per_step'],2))" || tail -3 $OUT/bench_${v}_$P.err
  done
done
