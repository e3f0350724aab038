#!/bin/bash
cd $GRAFT_REPO_ROOT
T=/tmp/ncu_$$; mkdir -p $T
ncu --set full --clock-control none -k regex:dmma_tile -s 40 -c 8 -f -o $T/bru python tools/prof_steps.py bru_etd 3 > gpurun_out/ncu_bru.log 2>&1
ncu -i $T/bru.ncu-rep --page raw --csv > gpurun_out/ncu_bru.raw.csv 2>/dev/null
python - <<'PY'
import csv
rows=list(csv.reader(open('gpurun_out/ncu_bru.raw.csv')))
h=rows[0]
keys=["Kernel Name","launch__grid_size","gpu__time_duration.sum","sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active","dram__bytes_read.sum","dram__bytes_write.sum","smsp__issue_active.avg.pct_of_peak_sustained_active","launch__registers_per_thread","sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active"]
for r in rows[2:]:
    d=dict(zip(h,r))
    st={k.replace("smsp__pcsamp_warps_issue_stalled_",""):float(v) for k,v in d.items() if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued") and v.replace(".","",1).isdigit()}
    tot=sum(st.values()) or 1
    top=sorted(st.items(),key=lambda kv:-kv[1])[:4]
    print([d[k][:60] for k in keys], ", ".join(f"{k} {100*v/tot:.0f}%" for k,v in top))
PY
