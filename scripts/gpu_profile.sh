cd $GRAFT_REPO_ROOT
export PATH=/usr/local/cuda/bin:$PATH
# launch list: every kernel of a short run, device time per launch (cold, serialised)
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
    python bench.py --quick --steps 3 --warmup 1 > gpurun_out/launches_bench.log 2>&1
# full capture of the top kernels (skip the counting build + first launches)
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_faces -s 2 -c 1 \
    -o gpurun_out/prof_faces python bench.py --quick --steps 2 --warmup 1 > gpurun_out/prof_faces.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_finalize -s 1 -c 1 \
    -o gpurun_out/prof_finalize python bench.py --quick --steps 2 --warmup 1 > gpurun_out/prof_finalize.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_reduce -s 1 -c 1 \
    -o gpurun_out/prof_reduce python bench.py --quick --steps 2 --warmup 1 > gpurun_out/prof_reduce.log 2>&1
ls -la gpurun_out
