#!/bin/bash
cd $GRAFT_REPO_ROOT
for t in N G M L S; do echo "== KP_GEMM_TILE=$t"; KP_GEMM_TILE=$t python tools/tucker_sweep.py 256 2>&1 | grep "n=256"; done
for t in S N G M; do echo "== KP_GEMM_TILE_FUSED=$t"; KP_GEMM_TILE_FUSED=$t python tools/integrator_bench.py ac3d bru_etd bru_l2b 2>&1 | grep "steps/s"; done
