#!/bin/bash
# one gpurun call: smoke, bench (JSON line), ncu launch list, ncu full capture
set -x
OUT=gpurun_out/${TAG:-run}
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1
timeout 900 python bench.py ${BENCH_ARGS} > $OUT/bench.json 2> $OUT/bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv \
   python bench.py --grid ${NCU_N:-256} --steps 1 --warmup 3 --modes "" --slab-sweep "" --no-e2e --no-cpu-baseline ${NCU_ARGS} > $OUT/ncu_launch_bench.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:${KREGEX:-k_resid} -s ${NCU_SKIP:-6} -c 1 \
   -o $OUT/prof python bench.py --grid ${NCU_N:-256} --steps 1 --warmup 3 --modes "" --slab-sweep "" --no-e2e --no-cpu-baseline ${NCU_ARGS} > $OUT/ncu_full.log 2>&1
ls -la $OUT
