cd $GRAFT_REPO_ROOT
export PATH=/usr/local/cuda/bin:$PATH
timeout 1200 python -m pytest tests -m gpu -q --timeout 600 -p no:cacheprovider -x > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/gpu_tests.log
timeout 600 python bench.py --steps 30 --warmup 5 --quick > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
if [ -n "$PROF" ]; then
timeout 900 ncu --set full --clock-control none --import-source on -k regex:$PROF -s ${PROF_SKIP:-2} -c 1 \
    -o gpurun_out/prof_iter python bench.py --quick --steps 2 --warmup 1 > gpurun_out/prof_iter.log 2>&1
fi
