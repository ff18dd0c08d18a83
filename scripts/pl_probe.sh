O=gpurun_out
python scripts/profile_config.py powerlaw 33000000 2500 > $O/r02_pl2500.txt 2>&1
ncu --nvtx --nvtx-include "fused/" -k regex:fused --set full --import-source on --clock-control none -o $O/r02p_pl python scripts/profile_config.py powerlaw 33000000 2500 > $O/r02p_pl.log 2>&1
python scripts/ncu_summary.py $O/r02p_pl.ncu-rep $O/r02p_plsum.txt > /dev/null 2>&1
python scripts/ncu_lines.py $O/r02p_pl.ncu-rep grad_impl.cuh > $O/r02p_pllines.txt 2>&1
rm -f $O/r02p_pl.ncu-rep
