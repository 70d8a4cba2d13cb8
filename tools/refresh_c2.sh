#!/bin/bash
# Refresh config 2's round artifacts (bench line, launch list, ncu full summary) under gpurun.
cd $GRAFT_REPO_ROOT
R=${1:-r2g}
mkdir -p /tmp/ncu
timeout 600 python bench.py --config 2 --steps 20 --warmup 3 > gpurun_out/${R}_bench_c2.log 2>&1
tail -1 gpurun_out/${R}_bench_c2.log > gpurun_out/${R}_bench_c2.json
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/${R}_bench_reference_c2.log 2>&1
tail -1 gpurun_out/${R}_bench_reference_c2.log > gpurun_out/${R}_bench_reference_c2.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv \
  --log-file gpurun_out/${R}_launches_config2.csv python tools/prof_run.py 2 2 > /dev/null 2>&1
python tools/summarize_profiles.py launches gpurun_out/${R}_launches_config2.csv gpurun_out/${R}_launches_config2.md > /dev/null
timeout 1200 ncu --set full --import-source on --clock-control none -c 40 -f \
  -o /tmp/ncu/${R}_full_config2 python tools/prof_run.py 2 1 > /dev/null 2>&1
python tools/summarize_profiles.py full /tmp/ncu/${R}_full_config2.ncu-rep gpurun_out/ncu_config2_summary.json \
  gpurun_out/${R}_ncu_full_config2.md > /dev/null
python tools/ncu_brief.py /tmp/ncu/${R}_full_config2.ncu-rep > gpurun_out/${R}_ncu_brief_config2.txt 2>&1
for k in k_num_reuse_multi k_sym_reuse k_reuse_flags; do
  python tools/ncu_source.py /tmp/ncu/${R}_full_config2.ncu-rep $k 30 > gpurun_out/${R}_src_${k}_config2.txt 2>/dev/null
done
python tools/ncu_smem_lines.py /tmp/ncu/${R}_full_config2.ncu-rep k_num_reuse_multi 15 > gpurun_out/${R}_smem_k_num_reuse_multi_config2.txt 2>/dev/null
ls gpurun_out | grep ${R}_
