#!/bin/bash
# Round-2 final captures (one GPU): headline GEMM, n=128 tiles S vs B, stencil
# variants, and the bench command's launch list.  Outputs: gpurun_out/r02b_*.
cd $GRAFT_REPO_ROOT
N="ncu --set full --clock-control none --import-source on"
T=/tmp/ncu_$$; mkdir -p $T
: > gpurun_out/r02b_ncu.log
run() { name=$1; rx=$2; skip=$3; shift 3; $N -k regex:$rx -s $skip -c 1 -f -o $T/$name "$@" >> gpurun_out/r02b_ncu.log 2>&1
  ncu -i $T/$name.ncu-rep --page raw --csv > gpurun_out/r02b_$name.raw.csv 2>/dev/null
  python tools/ncu_brief.py $T/$name.ncu-rep > gpurun_out/r02b_$name.brief.txt 2>&1; }
run n512_mode1 dmma_tile 1 python tools/prof_mode.py 512 1 3
run n512_mode0 dmma_tile 1 python tools/prof_mode.py 512 0 3
run n128_mode2_S dmma_tile 1 python tools/prof_mode.py 128 2 3
KP_GEMM_TILE=B run n128_mode2_B dmma_tile 1 python tools/prof_mode.py 128 2 3
KP_BAND=v6 run band6_nls kronsum_band 2 python tools/band_time.py nls reps=1
KP_BAND=v7 run band7_nls kronsum_band 2 python tools/band_time.py nls reps=1
run band8_nls kronsum_band 2 python tools/band_time.py nls reps=1
run band6_ac3d kronsum_band 2 python tools/band_time.py ac3d reps=1
KP_BAND=v6 run band6_bru kronsum_band 2 python tools/band_time.py bru reps=1
# launch list of the bench command (run first without ncu)
python bench.py --steps 2 --warmup 1 --no-integrators --no-paper --no-cpu-baseline > gpurun_out/r02b_bench_short.json 2> gpurun_out/r02b_bench_short.err && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02b_launches_bench.csv \
  python bench.py --steps 2 --warmup 1 --no-integrators --no-paper --no-cpu-baseline > gpurun_out/r02b_ncu_bench.log 2>&1
for c in ac3d bru_etd nls_ee; do
  ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file gpurun_out/r02b_launches_${c}_steps.csv python tools/prof_steps.py $c 3 > /dev/null 2>&1
done
cat gpurun_out/r02b_*.brief.txt
du -sh gpurun_out
