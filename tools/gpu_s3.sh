cd $GRAFT_REPO_ROOT
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"k_num_wh|k_sym_wh" -c 2 -f -o gpurun_out/c2wh python tools/prof_run.py 2 1 > gpurun_out/ncu_c2wh.log 2>&1
tail -2 gpurun_out/ncu_c2wh.log
