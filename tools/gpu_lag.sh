#!/bin/bash
OUT=gpurun_out/${TAG:-lag}
mkdir -p $OUT
for v in lag3 c0lag3; do
  MPFD_B200_LIB=$PWD/paper_2505_20911_b200/libmpfd_b200_$v.so timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "(64_cubed or history_64 or fused_path_bitwise or 256_cubed) and (HPSP or SPDP)" > $OUT/pytest_$v.log 2>&1
  echo "$v: $(tail -1 $OUT/pytest_$v.log)"
done
for rep in 1 2; do
  for v in base lag3; do
    L=paper_2505_20911_b200/libmpfd_b200_$v.so; [ "$v" = base ] && L=paper_2505_20911_b200/libmpfd_b200.so
    MPFD_B200_LIB=$PWD/$L python bench.py --precision HPSP --steps 5 --modes "" --slab-sweep "" --no-e2e --no-cpu-baseline --no-memory-table > $OUT/b_${v}_HPSP.json 2>/dev/null
    python -c "import json; d=json.load(open('$OUT/b_${v}_HPSP.json')); print('$v HPSP', round(d['ms_per_step'],2))"
  done
  for v in base c0lag3; do
    L=paper_2505_20911_b200/libmpfd_b200_$v.so; [ "$v" = base ] && L=paper_2505_20911_b200/libmpfd_b200.so
    MPFD_B200_LIB=$PWD/$L python bench.py --precision SPDP --steps 5 --modes "" --slab-sweep "" --no-e2e --no-cpu-baseline --no-memory-table > $OUT/b_${v}_SPDP.json 2>/dev/null
    python -c "import json; d=json.load(open('$OUT/b_${v}_SPDP.json')); print('$v SPDP', round(d['ms_per_step'],2))"
  done
done
