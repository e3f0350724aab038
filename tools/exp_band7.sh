#!/bin/bash
cd $GRAFT_REPO_ROOT
KP_BAND=v6 python tools/band_probe.py > gpurun_out/bp_v6.txt 2>&1
for v in "KP_BAND=v7" "KP_BAND=v7 KP_B7_RY=2" "KP_BAND=v7 KP_B7_PF=0" "KP_BAND=v7 KP_B7_BLOCKS=1" "KP_BAND=v7 KP_B7_BLOCKS=64"; do env $v python tools/band_probe.py > gpurun_out/bp_x.txt 2>&1; cmp gpurun_out/bp_v6.txt gpurun_out/bp_x.txt && echo "SAME $v"; done
tail -2 gpurun_out/bp_x.txt
for v in "KP_BAND=v6" "KP_BAND=v7" "KP_BAND=v7 KP_B7_PF=0" "KP_BAND=v7 KP_B7_PF=12" "KP_BAND=v7 KP_B7_BLOCKS=6" "KP_BAND=v7 KP_B7_BLOCKS=24" "KP_BAND=v7 KP_B7_RY=2"; do
  echo "== $v"; env $v python tools/band_time.py 2>&1 | tail -3
done
KP_BAND=v7 python -m pytest tests/test_sharded_native_gpu.py tests/test_fastpaths_gpu.py -x -q 2>&1 | tail -3
