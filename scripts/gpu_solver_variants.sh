# Time the solver leg (bench.py "solver") for every build under _variants/ and the default build.
cd $GRAFT_REPO_ROOT
timeout 600 python bench.py --steps 10 --warmup 3 --quick > gpurun_out/var_default.log 2>&1
echo "default $(grep -o '"solver": {[^}]*}' gpurun_out/var_default.log)" > gpurun_out/solver_variants.txt
for d in _variants/*/; do
  n=$(basename $d)
  CS_LIB_PATH=$PWD/$d/libcontactsim_b200.so timeout 600 python bench.py --steps 10 --warmup 3 --quick > gpurun_out/var_$n.log 2>&1
  echo "$n $(grep -o '"solver": {[^}]*}' gpurun_out/var_$n.log)" >> gpurun_out/solver_variants.txt
done
