cd $GRAFT_REPO_ROOT
timeout 600 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum --clock-control none --csv --log-file gpurun_out/c3_launches.csv python tools/prof_run.py 3 1 > /dev/null 2>&1
python tools/summarize_profiles.py launches gpurun_out/c3_launches.csv gpurun_out/c3_launches.md; cat gpurun_out/c3_launches.md | head -12
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_big_sym" -c 1 -f -o gpurun_out/c3sym python tools/prof_run.py 3 1 > /dev/null 2>&1
timeout 900 ncu --section SourceCounters --section WarpStateStats --section SchedulerStats --import-source on --clock-control none -k regex:"k_big_num" -c 1 -f -o gpurun_out/c3num python tools/prof_run.py 3 1 > gpurun_out/ncu_c3num.log 2>&1
tail -2 gpurun_out/ncu_c3num.log
