#!/bin/bash
cd $GRAFT_REPO_ROOT
N="ncu --set full --clock-control none --import-source on"
T=/tmp/ncu_$$; mkdir -p $T
run() { name=$1; rx=$2; shift 2; $N -k regex:$rx -s 2 -c 1 -f -o $T/$name "$@" >> gpurun_out/ncu2.log 2>&1
  ncu -i $T/$name.ncu-rep --page raw --csv > gpurun_out/$name.raw.csv 2>/dev/null
  ncu -i $T/$name.ncu-rep --page source --csv > gpurun_out/$name.src.csv 2>/dev/null
  python tools/ncu_brief.py $T/$name.ncu-rep > gpurun_out/$name.brief.txt 2>&1; }
: > gpurun_out/ncu2.log
KP_BAND=${1:-v7} run ncu_band7_nls kronsum_band python tools/band_time.py nls reps=1
KP_BAND=${1:-v7} run ncu_band7_ac3d kronsum_band python tools/band_time.py ac3d reps=1
gzip -f gpurun_out/*.src.csv
tail -3 gpurun_out/ncu2.log
