cd $GRAFT_REPO_ROOT
SPGEMM_BENCH_DEBUG=1 timeout 300 python bench.py --config 2 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_dbg.log 2>&1
tail -3 gpurun_out/bench_dbg.log | cut -c1-600
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"k_num_group|k_sym_group" -c 3 -f -o gpurun_out/c2full python tools/prof_run.py 2 1 > gpurun_out/ncu_c2.log 2>&1
tail -3 gpurun_out/ncu_c2.log
timeout 300 python tools/quick_timing.py 3 2>&1 | tail -3
