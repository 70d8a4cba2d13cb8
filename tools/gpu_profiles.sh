#!/bin/bash
# Round profile capture (run under gpurun): bench lines for configs 1-5, the ncu
# launch lists (every kernel, serialised) of configs 1, 2 and 4, and --set full
# captures of EVERY kernel of one product of configs 1, 2, 4 and 3, summarised on
# the box (gpurun brings back <= 64 MiB: the .ncu-rep files stay there, their
# summaries and per-source-line tables come back).
cd $GRAFT_REPO_ROOT
R=${1:-r2}
mkdir -p /tmp/ncu
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/${R}_gpu.txt
lscpu > gpurun_out/${R}_lscpu.txt
if [ -z "$SKIP_BENCH" ]; then
for c in 2 1 4 3; do
  timeout 900 python bench.py --config $c --steps 10 --warmup 3 > gpurun_out/${R}_bench_c$c.log 2>&1
  tail -1 gpurun_out/${R}_bench_c$c.log > gpurun_out/${R}_bench_c$c.json
done
timeout 900 python bench.py --config 5 --rmat-scale 22 --steps 3 --warmup 3 > gpurun_out/${R}_bench_c5_s22.log 2>&1
tail -1 gpurun_out/${R}_bench_c5_s22.log > gpurun_out/${R}_bench_c5_s22.json
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/${R}_bench_reference_c2.log 2>&1
tail -1 gpurun_out/${R}_bench_reference_c2.log > gpurun_out/${R}_bench_reference_c2.json
fi
for c in 2 1 4; do
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv \
    --log-file gpurun_out/${R}_launches_config$c.csv python tools/prof_run.py $c 2 > /dev/null 2>&1
  python tools/summarize_profiles.py launches gpurun_out/${R}_launches_config$c.csv gpurun_out/${R}_launches_config$c.md > /dev/null
done
for c in 2 1 4 3; do
  T=1200; [ $c = 3 ] && T=2400
  timeout $T ncu --set full --import-source on --clock-control none -c 40 -f \
    -o /tmp/ncu/${R}_full_config$c python tools/prof_run.py $c 1 > /dev/null 2>&1
  python tools/summarize_profiles.py full /tmp/ncu/${R}_full_config$c.ncu-rep gpurun_out/ncu_config${c}_summary.json \
    gpurun_out/${R}_ncu_full_config$c.md > /dev/null
  python tools/ncu_brief.py /tmp/ncu/${R}_full_config$c.ncu-rep > gpurun_out/${R}_ncu_brief_config$c.txt 2>&1
done
for k in k_num_reuse_multi k_sym_reuse k_reuse_flags k_num_lean k_num_thread k_big_num_ord k_big_sym; do
  for c in 2 4 1 3; do
    python tools/ncu_source.py /tmp/ncu/${R}_full_config$c.ncu-rep $k 30 > gpurun_out/${R}_src_${k}_config$c.txt 2>/dev/null
    [ -s gpurun_out/${R}_src_${k}_config$c.txt ] || rm -f gpurun_out/${R}_src_${k}_config$c.txt
  done
done
du -sh gpurun_out; ls gpurun_out | grep ${R}_ | head -60
