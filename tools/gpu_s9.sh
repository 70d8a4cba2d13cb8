cd $GRAFT_REPO_ROOT
python tools/quick_timing.py 2 4 3 | grep cfg
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"k_num_group|k_sym_group" -c 3 python tools/prof_run.py 2 1 2>&1 | grep -E "k_num|k_sym|dram|duration" | head -20
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
