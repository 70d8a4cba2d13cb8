#!/bin/bash
# Round profile capture: bench lines for configs 1-4, the ncu launch list of the
# default bench command, and --set full captures of the dominant kernels.
cd $GRAFT_REPO_ROOT
R=${1:-r1}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/${R}_gpu.txt
for c in 2 1 4 3; do
  timeout 900 python bench.py --config $c --steps 10 --warmup 3 > gpurun_out/${R}_bench_c$c.log 2>&1
  tail -1 gpurun_out/${R}_bench_c$c.log > gpurun_out/${R}_bench_c$c.json
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/${R}_launches_config2.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_num_group|k_sym_group" -c 3 -f \
  -o gpurun_out/${R}_full_config2 python tools/prof_run.py 2 1 > /dev/null 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_num_thread|k_sym_thread" -c 2 -f \
  -o gpurun_out/${R}_full_config1 python tools/prof_run.py 1 1 > /dev/null 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_num_group|k_num_thread" -c 4 -f \
  -o gpurun_out/${R}_full_config4 python tools/prof_run.py 4 1 > /dev/null 2>&1
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:"k_big_sym" -c 1 -f \
  -o gpurun_out/${R}_full_config3_sym python tools/prof_run.py 3 1 > /dev/null 2>&1
timeout 1800 ncu --set full --import-source on --clock-control none -k regex:"k_big_num" -c 1 -f \
  -o gpurun_out/${R}_full_config3 python tools/prof_run.py 3 1 > /dev/null 2>&1
ls -la gpurun_out/
