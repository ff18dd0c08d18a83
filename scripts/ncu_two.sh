O=gpurun_out
for spec in "100M_x_100k 10000000 2500" "1M_x_10k 1000000 2500"; do
  set -- $spec
  ncu --nvtx --nvtx-include "fused/" -k regex:fused --set full --import-source on --clock-control none \
      -o $O/r02n_ncu_$1 python scripts/profile_config.py $1 $2 $3 > $O/r02n_ncu_$1.log 2>&1
  python scripts/ncu_summary.py $O/r02n_ncu_$1.ncu-rep $O/r02n_ncusum_$1.txt > /dev/null 2>&1
  python scripts/ncu_lines.py $O/r02n_ncu_$1.ncu-rep grad_impl.cuh > $O/r02n_nculines_$1.txt 2>&1
  rm -f $O/r02n_ncu_$1.ncu-rep
done
