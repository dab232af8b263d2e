cd $GRAFT_REPO_ROOT
export PATH=/usr/local/cuda/bin:$PATH
timeout 900 compute-sanitizer --tool memcheck --print-limit 20 python scripts/debug_reduce.py > gpurun_out/sanitizer.log 2>&1
timeout 1200 python -m pytest tests -m gpu -q --timeout 600 -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/gpu_tests.log
timeout 600 python bench.py --steps 30 --warmup 5 --quick > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_finalize_warp -s 1 -c 1 \
    -o gpurun_out/prof_finw python bench.py --quick --steps 2 --warmup 1 > gpurun_out/prof_finw.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_reduce -s 1 -c 1 \
    -o gpurun_out/prof_red python bench.py --quick --steps 2 --warmup 1 > gpurun_out/prof_red.log 2>&1
