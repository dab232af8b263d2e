# The other BASELINE configs (parity cases, measured beside the headline), with clock records
cd $GRAFT_REPO_ROOT
export PATH=/usr/local/cuda/bin:$PATH
timeout 900 python scripts/bench_config3.py > gpurun_out/config3.log 2>&1; echo "rc=$?" >> gpurun_out/config3.log
timeout 900 python scripts/bench_config4.py > gpurun_out/config4.log 2>&1; echo "rc=$?" >> gpurun_out/config4.log
timeout 1800 python scripts/bench_sweep.py > gpurun_out/sweep.log 2>&1; echo "rc=$?" >> gpurun_out/sweep.log
timeout 1200 python scripts/bench_sweep.py --res 64 128 256 512 --envs 32768 --steps 5 > gpurun_out/sweep_32k.log 2>&1; echo "rc=$?" >> gpurun_out/sweep_32k.log
timeout 900 python bench.py --steps 30 --warmup 5 > gpurun_out/bench_full.log 2>&1; echo "rc=$?" >> gpurun_out/bench_full.log
