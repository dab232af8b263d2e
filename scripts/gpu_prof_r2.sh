# gpu tests (full) + ncu --set full captures of $PROFK (one launch each, after warm-up)
cd $GRAFT_REPO_ROOT
export PATH=/usr/local/cuda/bin:$PATH
if [ -z "$NOTEST" ]; then
timeout 1200 python -m pytest tests -m gpu -q --timeout 600 -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/gpu_tests.log
fi
timeout 600 python bench.py --steps 20 --warmup 5 --quick > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
for k in ${PROFK:-}; do
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$k" -s ${SKIP:-3} -c 1 \
    -o gpurun_out/prof_$k python bench.py --quick --steps 3 --warmup 1 > gpurun_out/prof_$k.log 2>&1
done
ls -la gpurun_out
