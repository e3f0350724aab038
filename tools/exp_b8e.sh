#!/bin/bash
cd $GRAFT_REPO_ROOT
KP_BAND=v6 python tools/band_probe.py > gpurun_out/bp_v6.txt 2>&1
for v in "KP_BAND=v8" "KP_BAND=v8 KP_B8_MINB=3" "KP_BAND=v8 KP_B8_YH=0"; do env $v python tools/band_probe.py > gpurun_out/bp_x.txt 2>&1; cmp gpurun_out/bp_v6.txt gpurun_out/bp_x.txt && echo "SAME $v"; done
for v in "KP_BAND=v6" "KP_BAND=v8 KP_B8_YH=0" "KP_BAND=v8" "KP_BAND=v8 KP_B8_MINB=3" "KP_BAND=v8 KP_B8_BLOCKS=8" "KP_BAND=v8 KP_B8_MINB=3 KP_B8_BLOCKS=8"  "KP_BAND=v8 KP_B8_PF=0"; do
  echo "== $v"; env $v python tools/band_time.py 2>&1 | tail -3
done
