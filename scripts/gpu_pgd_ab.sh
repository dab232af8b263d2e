# A/B of the descent kernels: per-kernel ncu time / instructions / warps active for the
# main build and every _variants/* build (quick bench, 3 steps)
cd $GRAFT_REPO_ROOT
export PATH=/usr/local/cuda/bin:$PATH
for d in main _variants/*/; do
  n=$(basename $d)
  if [ "$d" = main ]; then L=""; else L="CS_LIB_PATH=$PWD/$d/libcontactsim_b200.so"; fi
  env $L timeout 300 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,sm__warps_active.avg.pct_of_peak_sustained_active \
      --clock-control none -k regex:${KREGEX:-k_pgd} --csv --log-file gpurun_out/l_$n.csv python bench.py --quick --steps 3 --warmup 1 > /dev/null 2>&1
done
