# ILU(0) apply timing of the 3D coarse level: dataflow kernel variants
for v in "PSCU_LEVEL_FLOW=1" "PSCU_LEVEL_FLOW=2"; do
  echo "== $v" >> gpurun_out/sweep4.log
  env $v REPS=1 timeout 300 python tools/run3d.py 32 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); c=d['classes']['ilu0_apply']; print(d['solve_ms'], d['its'], d['coarse_its'], c['n'], c['ms'], c['ms']/c['n'])" >> gpurun_out/sweep4.log 2>&1
done
