#!/bin/bash
# ncu --set full captures: n=128 mode-2 product under S and B tiles; stencil v6 at NLS / AC3D
cd $GRAFT_REPO_ROOT
N="ncu --set full --clock-control none --import-source on"
T=/tmp/ncu_$$; mkdir -p $T
cap() { # name kernel-regex env... -- cmd
  name=$1; rx=$2; shift 2
  env "$@" > /dev/null 2>&1
}
run() { name=$1; rx=$2; shift 2; $N -k regex:$rx -s 1 -c 1 -f -o $T/$name "$@" >> gpurun_out/ncu1.log 2>&1
  ncu -i $T/$name.ncu-rep --page raw --csv > gpurun_out/$name.raw.csv 2>/dev/null
  ncu -i $T/$name.ncu-rep --page source --csv > gpurun_out/$name.src.csv 2>/dev/null
  python tools/ncu_brief.py $T/$name.ncu-rep > gpurun_out/$name.brief.txt 2>&1; }
: > gpurun_out/ncu1.log
KP_GEMM_BAL=0 run ncu_m2_128_S dmma_tile python tools/prof_mode.py 128 2 3
run ncu_m2_128_B dmma_tile python tools/prof_mode.py 128 2 3
run ncu_m1_128_B dmma_tile python tools/prof_mode.py 128 1 3
run ncu_band6_nls kronsum_band python tools/band_one.py nls 3
run ncu_band6_ac3d kronsum_band python tools/band_one.py ac3d 3
cp $T/ncu_band6_nls.ncu-rep gpurun_out/
gzip -f gpurun_out/*.src.csv
tail -3 gpurun_out/ncu1.log
du -sh gpurun_out
