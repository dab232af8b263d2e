# One iteration: GPU parity suite on the in-tree build, then the quick bench for it and
# every variant under _variants/ (phase split per variant).
cd $GRAFT_REPO_ROOT
export PATH=/usr/local/cuda/bin:$PATH
rm -f gpurun_out/variants.txt
timeout 900 python -m pytest tests -m gpu -q -x --timeout 600 -p no:cacheprovider -k "${KEXPR:-}" > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/gpu_tests.log
timeout 600 python bench.py --steps 20 --warmup 5 --quick > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
echo "main $(grep -o '"ms_per_step": [0-9.]*' gpurun_out/bench.log | head -1) $(grep -o '"phase_ms": {[^}]*}' gpurun_out/bench.log)" >> gpurun_out/variants.txt
for d in _variants/*/; do
  [ -d "$d" ] || continue
  n=$(basename $d)
  CS_LIB_PATH=$PWD/$d/libcontactsim_b200.so timeout 600 python bench.py --steps 20 --warmup 5 --quick > gpurun_out/var_$n.log 2>&1
  echo "$n $(grep -o '"ms_per_step": [0-9.]*' gpurun_out/var_$n.log | head -1) $(grep -o '"phase_ms": {[^}]*}' gpurun_out/var_$n.log)" >> gpurun_out/variants.txt
done
if [ -n "$LAUNCHES" ]; then
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
    python bench.py --quick --steps 3 --warmup 1 > gpurun_out/launches_bench.log 2>&1
fi
for k in ${PROFK:-}; do
timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k -s 3 -c 1 \
    -o gpurun_out/prof_$k python bench.py --quick --steps 3 --warmup 1 > gpurun_out/prof_$k.log 2>&1
done
