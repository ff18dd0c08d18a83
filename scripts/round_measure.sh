#!/bin/bash
# End-of-round measurements on one B200 (run through gpurun): bench lines of every workload, the
# ncu launch list of the default bench's timed steps, ncu --set full of the fused pass per workload.
# The .ncu-rep files are summarised on the box (scripts/ncu_summary.py) and deleted, so that what
# comes back stays under gpurun's 64 MiB; outputs in gpurun_out/<tag>m_*, then scripts/collect_round.py.
#   bash scripts/round_measure.sh TAG [bench|ncu|all]
set -u
TAG=${1:-r02}; WHAT=${2:-all}; O=gpurun_out
if [ "$WHAT" = bench ] || [ "$WHAT" = all ]; then
  python bench.py > $O/${TAG}m_bench_100M_x_100k.json 2> $O/${TAG}m_bench_100M_x_100k.err
  for c in 1M_x_10k multifamily_boxcut powerlaw paper_table_25M; do
    python bench.py --config $c --no-cpu > $O/${TAG}m_bench_$c.json 2> $O/${TAG}m_bench_$c.err
  done
fi
if [ "$WHAT" = ncu ] || [ "$WHAT" = all ]; then
  ncu --nvtx --nvtx-include "timed_steps/" --metrics gpu__time_duration.sum --clock-control none --csv \
      --log-file $O/${TAG}m_launches.csv python bench.py --no-gap --no-cpu --steps 3 --warmup 1 > $O/${TAG}m_launches.log 2>&1
  for spec in "100M_x_100k 100000000 2500" "1M_x_10k 1000000 2500" "multifamily_boxcut 10000000 300" \
              "powerlaw 330000000 200" "paper_table_25M 25000000 1700"; do
    set -- $spec
    ncu --nvtx --nvtx-include "fused/" -k regex:fused --set full --import-source on --clock-control none \
        -o $O/${TAG}m_ncu_$1 python scripts/profile_config.py $1 $2 $3 > $O/${TAG}m_ncu_$1.log 2>&1
    python scripts/ncu_summary.py $O/${TAG}m_ncu_$1.ncu-rep $O/${TAG}m_ncusum_$1.txt \
        --json $O/${TAG}m_ncu_traffic.json --workload $1 > /dev/null 2>&1
    python scripts/ncu_regions.py $O/${TAG}m_ncu_$1.ncu-rep grad_impl.cuh lam:215-250 smem_helpers:360-400 \
        small_pass:1125-1228 compact_rescore:1229-1284 michelot:1285-1313 emit_overflow:1314-1340 pipeline:1455-1571 \
        > $O/${TAG}m_ncuregions_$1.txt 2>&1
    rm -f $O/${TAG}m_ncu_$1.ncu-rep
  done
fi
echo done
