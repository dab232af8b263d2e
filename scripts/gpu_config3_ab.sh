# config 3 (per-env grids: the non-uniform kernels) for the main build and every variant
cd $GRAFT_REPO_ROOT
for d in main _variants/*/; do
  n=$(basename $d)
  if [ "$d" = main ]; then L=""; else L="CS_LIB_PATH=$PWD/$d/libcontactsim_b200.so"; fi
  echo "$n $(env $L timeout 600 python scripts/bench_config3.py 2>&1 | grep -o '"ms_per_step": [0-9.]*\|"phase_ms": {[^}]*}' | tr '\n' ' ')" >> gpurun_out/c3ab.txt
done
