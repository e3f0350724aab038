#!/bin/bash
# A/B of the balanced GEMM tiles (KP_GEMM_BAL) and the fused mode-0/1 kernel
set -x
cd $GRAFT_REPO_ROOT
python tools/tile_probe.py > gpurun_out/probe_default.txt 2>&1
KP_GEMM_TILE=B python tools/tile_probe.py > gpurun_out/probe_B.txt 2>&1
KP_GEMM_BAL=0 python tools/tile_probe.py > gpurun_out/probe_bal0.txt 2>&1
KP_FUSE01=0 python tools/tile_probe.py > gpurun_out/probe_nofuse.txt 2>&1
cmp gpurun_out/probe_default.txt gpurun_out/probe_B.txt && echo SAME_B
cmp gpurun_out/probe_default.txt gpurun_out/probe_bal0.txt && echo SAME_BAL0
cmp gpurun_out/probe_default.txt gpurun_out/probe_nofuse.txt && echo SAME_NOFUSE
tail -3 gpurun_out/probe_B.txt
for v in "KP_GEMM_BAL=0" "KP_GEMM_BAL=-1" "KP_FUSE01=0" "KP_FUSE01=0 KP_GEMM_BAL=0" "KP_GEMM_BAL=1" "KP_GEMM_BAL=1 KP_FUSE01=0"; do
  echo "== $v"
  env $v python tools/tucker_sweep.py 128 256 384 2>&1 | grep -v "^peak"
  env $v python tools/integrator_bench.py ac3d bru_etd 2>&1 | tail -4
done
