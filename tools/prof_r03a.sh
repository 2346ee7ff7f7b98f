#!/bin/bash
# CTAs per SM of the small-task dataflow kernels (forward, backward): tuning builds.
mkdir -p gpurun_out
V="PSCU_FLOW_BSHFL=0;PSCU_FLOW_BSHFL=1"
for lib in c55 c44 c53 c33 c74; do
  echo "== $lib c3" >> gpurun_out/r03a.log
  PSCU_LIB=tools/libpstokes_$lib.so SMOOTH=3 REPS=0 VARIANTS="$V" timeout 600 python tools/run3d.py 32 0.15 1 2 2>&1 | grep "^{" | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); c=d['classes'].get('ilu0_apply',{})
    print('%-25s'%d['variant'], 'solve', round(d['solve_ms'],1), 'ilu/apply', round(c['ms']/c['n'],3), 'its', d['its'], d['coarse_its'])
" >> gpurun_out/r03a.log
done
for lib in c55 c44 c53 c33; do
  echo "== $lib c5" >> gpurun_out/r03a.log
  PSCU_LIB=tools/libpstokes_$lib.so SMOOTH=2 REPS=0 VARIANTS="$V" timeout 900 python tools/run3d.py 64 0.1 4 5 2>&1 | grep "^{" | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); c=d['classes'].get('ilu0_apply',{})
    print('%-25s'%d['variant'], 'solve', round(d['solve_ms'],1), 'ilu/apply', round(c['ms']/c['n'],3), 'its', d['its'], d['coarse_its'])
" >> gpurun_out/r03a.log
done
