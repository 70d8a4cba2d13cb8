cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -x -q -k "rmat or spill or heap" 2>&1 | tail -3
python tools/quick_timing.py 3 2>&1 | grep cfg
timeout 600 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum --clock-control none --csv --log-file gpurun_out/c3_launches.csv python tools/prof_run.py 3 1 > /dev/null 2>&1
python tools/summarize_profiles.py launches gpurun_out/c3_launches.csv gpurun_out/c3_launches.md; cat gpurun_out/c3_launches.md
