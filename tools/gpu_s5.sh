cd $GRAFT_REPO_ROOT
timeout 300 python bench.py --config 3 --steps 2 --warmup 1 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['kernels_ms'])"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_big_sym|k_big_num" -c 2 -f -o gpurun_out/c3big python tools/prof_run.py 3 1 > gpurun_out/ncu_c3.log 2>&1
tail -2 gpurun_out/ncu_c3.log
