#!/bin/bash
# Cholesky timing at several super-panel widths + launch breakdown (one gpurun call)
cd "${GRAFT_REPO_ROOT:-.}"
for W in ${WS:-4 8 16 32}; do echo W=$W; SFB_CHOL_PANEL=$W python tools/chol_ab.py 2>&1 | head -1; done
SFB_CHOL_PANEL=${WP:-8} ncu --metrics gpu__time_duration.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active --clock-control none -k regex:"chol|lower_mul" --csv python tools/chol_ab.py > gpurun_out/chol_launch.csv 2>&1
python3 - <<'PY'
import csv, collections
rows=[r for r in csv.reader(open('gpurun_out/chol_launch.csv')) if len(r)>10 and r[0].isdigit()]
t=collections.defaultdict(float); cnt=collections.Counter(); met=collections.defaultdict(lambda: collections.defaultdict(list))
for r in rows:
    name=r[4].split('(')[0]; m=r[12]
    try: v=float(r[14].replace(',',''))
    except: continue
    if m=='gpu__time_duration.sum': t[name]+=v; cnt[name]+=1
    else: met[name][m].append(v)
for k in t:
    extra=' '.join(f"{m.split('__')[1][:28]}={sum(v)/len(v):.1f}" for m,v in met[k].items())
    print(f"{k:34s} n={cnt[k]:5d} {t[k]/1e3/3:9.1f} us/run  {extra}")
PY
