cd $GRAFT_REPO_ROOT
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"k_num_group|k_sym_group" -c 3 -f -o gpurun_out/c2cc python tools/prof_run.py 2 1 > /dev/null 2>&1
ls -la gpurun_out/c2cc.ncu-rep
