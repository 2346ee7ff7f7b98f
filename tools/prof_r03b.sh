#!/bin/bash
# polling back-off x lead-source wait, default library
mkdir -p gpurun_out
run() { # label n jit seed fseed smooth
  for spin in 0 100 300; do for lead in 0 1; do
    echo -n "$1 spin=$spin lead=$lead  " >> gpurun_out/r03b.log
    PSCU_FLOW_SPIN_NS=$spin PSCU_FLOW_LEAD=$lead PSCU_FLOW_BSHFL=${BSHFL:-0} SMOOTH=$6 REPS=1 timeout 600 python tools/run3d.py $2 $3 $4 $5 2>&1 | grep "^{" | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); c=d['classes'].get('ilu0_apply',{})
    print('solve', round(d['solve_ms'],1), 'ilu/apply', round(c['ms']/c['n'],3), 'its', d['its'], d['coarse_its'])
" >> gpurun_out/r03b.log
  done; done
}
run c3 32 0.15 1 2 3
run c5 64 0.1 4 5 2
