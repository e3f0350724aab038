#!/bin/bash
cd $GRAFT_REPO_ROOT
KP_BAND=v6 python tools/band_probe.py > gpurun_out/bp_v6.txt 2>&1
for v in "KP_BAND=v7" "KP_BAND=v7 KP_B7_RY=2" "KP_BAND=v7 KP_B7_BLOCKS=1"; do env $v python tools/band_probe.py > gpurun_out/bp_x.txt 2>&1; cmp gpurun_out/bp_v6.txt gpurun_out/bp_x.txt && echo "SAME $v"; done
for v in "KP_BAND=v6" "KP_BAND=v7" "KP_BAND=v7 KP_B7_PF=0" "KP_BAND=v7 KP_B7_BLOCKS=24" "KP_BAND=v7 KP_B7_RY=2"; do
  echo "== $v"; env $v python tools/band_time.py 2>&1 | tail -3
done
KP_BAND=v7 python -m pytest tests/test_sharded_native_gpu.py -x -q 2>&1 | tail -30
