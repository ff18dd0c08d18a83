#!/bin/bash
# End-of-round measurements on one B200 (run through gpurun): bench lines of every workload, the
# ncu launch list of the default bench's timed steps, ncu --set full of the fused pass per workload.
# Outputs in gpurun_out/r02m_*; summaries are copied to profiles/ by hand (scripts/ncu_summary.py).
set -u
O=gpurun_out
python bench.py > $O/r02m_bench_default.json 2> $O/r02m_bench_default.err
for c in 1M_x_10k multifamily_boxcut powerlaw paper_table_25M; do
  python bench.py --config $c --no-cpu > $O/r02m_bench_$c.json 2> $O/r02m_bench_$c.err
done
ncu --nvtx --nvtx-include "timed_steps/" --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file $O/r02m_launches.csv python bench.py --no-gap --no-cpu --steps 3 --warmup 1 > $O/r02m_launches.log 2>&1
for spec in "100M_x_100k 100000000 2500" "1M_x_10k 1000000 2500" "multifamily_boxcut 10000000 300" "powerlaw 330000000 200" "paper_table_25M 25000000 1700"; do
  set -- $spec
  ncu --nvtx --nvtx-include "fused/" -k regex:fused --set full --import-source on --clock-control none \
      -o $O/r02m_ncu_$1 python scripts/profile_config.py $1 $2 $3 > $O/r02m_ncu_$1.log 2>&1
done
echo done
