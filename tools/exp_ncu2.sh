#!/bin/bash
# one ncu --set full capture of the stencil at NLS under the given env (source page exported)
cd $GRAFT_REPO_ROOT
N="ncu --set full --clock-control none --import-source on"
T=/tmp/ncu_$$; mkdir -p $T
name=${NAME:-band_nls}
$N -k regex:kronsum_band -s 2 -c 1 -f -o $T/$name python tools/band_time.py ${CASE:-nls} reps=1 > gpurun_out/ncu2.log 2>&1
ncu -i $T/$name.ncu-rep --page raw --csv > gpurun_out/$name.raw.csv 2>/dev/null
ncu -i $T/$name.ncu-rep --page source --csv > gpurun_out/$name.src.csv 2>/dev/null
python tools/ncu_brief.py $T/$name.ncu-rep > gpurun_out/$name.brief.txt 2>&1
gzip -f gpurun_out/$name.src.csv
cat gpurun_out/$name.brief.txt
