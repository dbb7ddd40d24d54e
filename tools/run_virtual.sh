#!/bin/bash
# Emulated-heterogeneity scenarios, all ranks on one GPU (experiments.py --virtual); one compact line per epoch.
for sc in "$@"; do
  timeout 900 python experiments.py --virtual --scenario $sc --epochs ${EPOCHS:-8} 2>&1 | python -c "
import sys, json
for l in sys.stdin:
    try: d = json.loads(l)
    except Exception: print(l.strip()[:200]); continue
    if 'epoch' not in d or 'T_emulated' not in d: continue   # the run's summary line
    print(d['scenario'], d['epoch'], d['w'], 'frozen' if d['frozen'] else '', [round(x,3) for x in d['t_s']], 'T', round(d['T_emulated'],3), 'bound', round(d['bound'],3), 'T/bound', round(d['T_over_bound'],3))
" | tee -a gpurun_out/virtual_scenarios.txt
done
