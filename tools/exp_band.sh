#!/bin/bash
# A/B of the banded Kronecker-sum kernels (banded.cu) on one B200: bitwise
# equality of every variant on the probe cases, then the kernel alone at the
# BASELINE shapes (tools/band_time.py).  usage (on the GPU box): bash tools/exp_band.sh
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
KP_BAND=v6 python tools/band_probe.py > gpurun_out/bp_v6.txt 2>&1
for v in "KP_BAND=v2" "KP_BAND=v7" "KP_BAND=v8" "KP_BAND=v8 KP_B8_MINB=3" "KP_BAND=v8 KP_B8_YH=1"; do
  env $v python tools/band_probe.py > gpurun_out/bp_x.txt 2>&1
  cmp -s gpurun_out/bp_v6.txt gpurun_out/bp_x.txt && echo "SAME as v6: $v" || echo "DIFFERENT from v6: $v"
done
for v in "KP_BAND=v2" "KP_BAND=v6" "KP_BAND=v7" "KP_BAND=v8" "KP_BAND=v8 KP_B8_YH=1" "KP_BAND=v8 KP_B8_PF=0" \
         "KP_BAND=v8 KP_B8_MINB=3 KP_B8_BLOCKS=8" ""; do
  echo "== ${v:-defaults}"; env $v python tools/band_time.py 2>&1 | tail -3
done
