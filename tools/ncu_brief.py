"""Brief of an ncu report: per kernel, the headline metrics and the top stall reasons.
  python tools/ncu_brief.py gpurun_out/x.ncu-rep"""
import csv, io, subprocess, sys

KEYS = ["Duration", "Compute (SM) Throughput", "Memory Throughput", "DRAM Throughput", "L2 Hit Rate",
        "L1/TEX Hit Rate", "Executed Ipc Active", "Achieved Occupancy", "Theoretical Occupancy",
        "Registers Per Thread", "Warp Cycles Per Issued Instruction", "Executed Instructions",
        "Dynamic Shared Memory Per Block", "Block Limit Shared Mem"]
rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[0]
ki, ni, ui, vi = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Unit"), h.index("Metric Value")
seen = {}
for r in rows[1:]:
    k = r[ki].split("(")[0] + "#" + r[0]
    if r[ni] in KEYS:
        seen.setdefault(k, {})[r[ni]] = f"{r[vi]} {r[ui]}"
for k, d in seen.items():
    print(k)
    for m in KEYS:
        if m in d:
            print(f"   {m}: {d[m]}")
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rr = list(csv.reader(io.StringIO(raw)))
hdr, units = rr[0], rr[1]
want = ["dram__bytes_read.sum", "dram__bytes_write.sum", "smsp__inst_executed.sum",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smsp__inst_executed_op_shared_atom.sum",
        "smsp__inst_executed_op_global_red.sum", "smsp__inst_executed_op_global_atom.sum",
        "lts__t_sectors.sum", "smsp__sass_inst_executed_op_shared_ld.sum", "smsp__sass_inst_executed_op_global_ld.sum"]
stall = [i for i, c in enumerate(hdr) if c.startswith("smsp__average_warp_latency_issue_stalled") or
         (c.startswith("smsp__pcsamp_warps_issue_stalled") and not c.endswith("not_issued"))]
for row in rr[2:]:
    name = row[hdr.index("Kernel Name")].split("(")[0]
    print(name, {w: f"{row[hdr.index(w)]} {units[hdr.index(w)]}" for w in want if w in hdr})
    st = sorted(((float(row[i].replace(",", "") or 0), hdr[i]) for i in stall if row[i]), reverse=True)[:8]
    for v, n in st:
        print(f"   stall {n.split('stalled_')[-1]}: {v}")
