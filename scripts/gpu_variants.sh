# Time every built variant under _variants/ with a short quick bench (phase split per variant).
cd $GRAFT_REPO_ROOT
for d in _variants/*/; do
  n=$(basename $d)
  CS_LIB_PATH=$PWD/$d/libcontactsim_b200.so timeout 600 python bench.py --steps 20 --warmup 5 --quick > gpurun_out/var_$n.log 2>&1
  echo "$n $(grep -o '"phase_ms": {[^}]*}' gpurun_out/var_$n.log)" >> gpurun_out/variants.txt
done
