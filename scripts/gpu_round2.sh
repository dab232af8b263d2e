# Round evidence: GPU suite, smoke, the default bench (e2e + CPU baseline), the reference
# arm, the launch list and ncu --set full captures of $PROFK
cd $GRAFT_REPO_ROOT
export PATH=/usr/local/cuda/bin:$PATH
timeout 1200 python -m pytest tests -m gpu -q --timeout 600 -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 900 python bench.py ${BENCH_ARGS:-} > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
timeout 1200 python bench.py --impl reference --steps ${REF_STEPS:-5} --warmup 1 > gpurun_out/bench_ref.log 2>&1; echo "ref rc=$?" >> gpurun_out/bench_ref.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
    python bench.py --quick --steps 3 --warmup 1 > gpurun_out/launches_bench.log 2>&1
for k in ${PROFK:-}; do
timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k -s 3 -c 1 \
    -o gpurun_out/prof_$k python bench.py --quick --steps 3 --warmup 1 > gpurun_out/prof_$k.log 2>&1
done
ls -la gpurun_out
