#!/bin/bash
# full round check on one GPU: tests, smoke, bench, launch list, ncu captures
# (reports are exported to CSV on the box; the .ncu-rep files are dropped
# unless KEEP_REP=1, so gpurun_out stays under the 64 MiB copy-back limit)
OUT=gpurun_out/${TAG:-full}
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $OUT/gpu.txt
if [ -z "$NO_TESTS" ]; then
  timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > $OUT/pytest_gpu.log 2>&1
  tail -5 $OUT/pytest_gpu.log
  python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1
fi
timeout 900 python bench.py ${BENCH_ARGS} > $OUT/bench.json 2> $OUT/bench.err
cat $OUT/bench.json
# the IPC (copy-engine) transport as a 1-rank self-exchange, timed like the bench
timeout 600 python bench.py --nccl --transport ipc --precision HPSP --modes "" --slab-sweep "" --no-cpu-baseline --no-memory-table > $OUT/bench_ipc.json 2> $OUT/bench_ipc.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv \
   python bench.py --grid 256 --steps 1 --warmup 3 --modes "" --slab-sweep "" --no-e2e --no-cpu-baseline --no-memory-table --no-issue-ceiling > $OUT/ncu_launch.log 2>&1
for P in ${NCU_PRESETS:-DP SPDP HPSP}; do
  # the three substep launches of one RK step (raw page: traffic, pipes, stalls)
  timeout 600 ncu --set full --clock-control none -k regex:${KREGEX:-k_fused} -s 3 -c 3 \
     -o $OUT/prof3_$P python bench.py --grid 256 --precision $P --steps 1 --warmup 3 --modes "" --slab-sweep "" --no-e2e --no-cpu-baseline --no-memory-table --no-issue-ceiling > $OUT/ncu3_$P.log 2>&1
  ncu -i $OUT/prof3_$P.ncu-rep --page raw --csv > $OUT/raw_$P.csv 2>/dev/null
  rm -f $OUT/prof3_$P.ncu-rep
  # one launch with source correlation (SASS opcode mix, stall sites)
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:${KREGEX:-k_fused} -s 3 -c 1 \
     -o $OUT/prof_$P python bench.py --grid 256 --precision $P --steps 1 --warmup 3 --modes "" --slab-sweep "" --no-e2e --no-cpu-baseline --no-memory-table --no-issue-ceiling > $OUT/ncu_$P.log 2>&1
  ncu -i $OUT/prof_$P.ncu-rep --page raw --csv > $OUT/raw1_$P.csv 2>/dev/null
  ncu -i $OUT/prof_$P.ncu-rep --page source --csv --print-source cuda,sass > $OUT/src_$P.csv 2>/dev/null
  gzip -f $OUT/src_$P.csv
  [ -z "$KEEP_REP" ] && rm -f $OUT/prof_$P.ncu-rep
done
ls -la $OUT
