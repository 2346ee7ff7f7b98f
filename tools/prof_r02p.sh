#!/bin/bash
# polling back-off (PSCU_FLOW_SPIN_NS) with the small-task kernel: frees issue
# slots for the folding warps on the same SM sub-partitions
mkdir -p gpurun_out
for s in 0 20 50 100 200 400; do
  echo "== spin $s" >> gpurun_out/sweep10.log
  PSCU_FLOW_SPIN_NS=$s REPS=1 timeout 300 python tools/run3d.py 32 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); c=d['classes']['ilu0_apply']; print(d['solve_ms'], c['ms']/c['n'])" >> gpurun_out/sweep10.log 2>&1
done
for s in 0 50 200; do
  echo "== spin $s" >> gpurun_out/sweep11.log
  PSCU_FLOW_SPIN_NS=$s SMOOTH=2 REPS=1 timeout 600 python tools/run3d.py 64 0.1 4 5 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); c=d['classes']['ilu0_apply']; print(d['solve_ms'], c['ms']/c['n'])" >> gpurun_out/sweep11.log 2>&1
done
