cd $GRAFT_REPO_ROOT
T=/tmp/ncu_$$; mkdir -p $T
for m in 0 1; do
ncu --set full --clock-control none -k regex:dmma_tile -s 1 -c 1 -f -o $T/c$m python tools/prof_mode_c.py 512 $m > gpurun_out/ncu3m.log 2>&1
ncu -i $T/c$m.ncu-rep --page raw --csv > gpurun_out/r02e_c512_mode$m.raw.csv 2>/dev/null
python tools/ncu_brief.py $T/c$m.ncu-rep
done
