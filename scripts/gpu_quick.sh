cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests -m gpu -q --timeout 600 -p no:cacheprovider -x > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/gpu_tests.log
timeout 600 python bench.py --steps 30 --warmup 5 --quick > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
