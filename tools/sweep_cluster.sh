# Walker cluster-size sweep: ILU(0) apply time per level for C in {1,2,4,8}
# (both sweeps), at the 128^2 and 256^2 config-2 recipes.
for N in 128 256; do
  echo "== N=$N auto"; PSCU_DEBUG=1 timeout 300 python tools/probe_ilu.py $N 10 2>&1 | grep -E "^level|static"
  for C in 1 2 4 8; do
    echo "== N=$N C=$C"; PSCU_WALK_CLUSTER=$C timeout 300 python tools/probe_ilu.py $N 10 2>&1 | grep "^level"
  done
done
