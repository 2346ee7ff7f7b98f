for cr in 16 8 4; do for pm in 99999999 0; do
  echo "== chain=$cr persist_min=$pm" >> gpurun_out/sweep.log
  PSCU_LEVEL_CHAIN_ROWS=$cr PSCU_LEVEL_PERSIST_MIN_ROWS=$pm REPS=1 timeout 300 python tools/run3d.py 32 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); c=d['classes']['ilu0_apply']; print(d['solve_ms'], d['its'], d['coarse_its'], c['n'], c['ms'], c['ms']/c['n'])" >> gpurun_out/sweep.log 2>&1
done; done
