"""Turn ncu outputs from gpurun_out/ into committed summaries under profiles/.

  python tools/summarize_profiles.py full   <rep.ncu-rep> <out.json> [<out.md>]
  python tools/summarize_profiles.py launches <launches.csv> <out.md>

'full' reads a --set full capture: per kernel (name with template args), duration,
DRAM bytes read+write per launch (the roofline 'traffic'), IPC, occupancy, cache hit
rates, top stall reasons. 'launches' reads a --metrics gpu__time_duration.sum list and
reports each kernel's share of the measured device time.
"""
import csv
import io
import json
import re
import subprocess
import sys
from collections import OrderedDict, defaultdict


def short_name(full):
    m = re.search(r"(k_\w+)(<[^(]*>)?", full)
    if not m:
        return full[:60]
    name, targs = m.group(1), m.group(2) or ""
    if targs:
        args = [a.strip().replace("(int)", "") for a in targs[1:-1].split(",")]
        keep = [a for a in args if a.isdigit()]
        last = targs[1:-1].split(",")[-1].strip().replace("(bool)", "")
        if name in ("k_sym_group", "k_num_group"):
            keep = keep[:2]
            if name == "k_num_group" and last in ("1", "true"):
                keep.append("spec")  # the speculative instance of the symbolic phase
        elif name in ("k_num_lean", "k_num_reuse", "k_num_reuse_multi", "k_num_pair"):
            keep = ["spec"] if last in ("1", "true") else []
        elif name in ("k_sym_block", "k_num_block"):
            keep = keep[:1]
        targs = "<" + ",".join(keep) + ">" if keep else ""
    return name + targs


def full(rep, out_json, out_md=None):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    kernels = OrderedDict()
    for r in data:
        d = dict(zip(hdr, r))
        name = short_name(d["Kernel Name"])
        f = lambda k: float(d[k]) if d.get(k) not in (None, "", "n/a") else None  # noqa: E731
        def unit_scale(k):
            u = units[hdr.index(k)] if k in hdr else ""
            return {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}.get(u, 1)
        dr = f("dram__bytes_read.sum")
        dw = f("dram__bytes_write.sum")
        dur = f("gpu__time_duration.sum")
        dur_unit = units[hdr.index("gpu__time_duration.sum")]
        dur_ms = dur * {"nsecond": 1e-6, "ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0, "second": 1e3, "s": 1e3}.get(dur_unit, 1e-6)
        stalls = {k.replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", ""): float(v)
                  for k, v in d.items()
                  if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio")
                  and v not in ("", "n/a")}
        top = sorted(stalls.items(), key=lambda kv: -kv[1])[:5]
        rec = {
            "duration_ms": dur_ms,
            "dram_bytes_read": dr * unit_scale("dram__bytes_read.sum") if dr is not None else None,
            "dram_bytes_write": dw * unit_scale("dram__bytes_write.sum") if dw is not None else None,
            "ipc": f("sm__inst_executed.avg.per_cycle_active"),
            "warp_instructions": f("smsp__inst_executed.sum"),
            "achieved_occupancy_pct": f("sm__warps_active.avg.pct_of_peak_sustained_active"),
            "l1_hit_pct": f("l1tex__t_sector_hit_rate.pct"),
            "l2_hit_pct": f("lts__t_sector_hit_rate.pct"),
            "registers": f("launch__registers_per_thread"),
            "smem_bank_conflicts": f("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum"),
            "shared_atomic_instructions": f("smsp__inst_executed_op_shared_atom.sum"),
            "global_red_instructions": f("smsp__inst_executed_op_global_red.sum"),
            "global_atomic_instructions": f("smsp__inst_executed_op_global_atom.sum"),
            "shared_load_instructions": f("smsp__sass_inst_executed_op_shared_ld.sum"),
            "global_load_instructions": f("smsp__sass_inst_executed_op_global_ld.sum"),
            "l2_sectors": f("lts__t_sectors.sum"),
            "top_stalls": top,
        }
        if rec["dram_bytes_read"] is not None and rec["dram_bytes_write"] is not None:
            rec["dram_bytes_per_launch"] = rec["dram_bytes_read"] + rec["dram_bytes_write"]
            rec["dram_gbs"] = rec["dram_bytes_per_launch"] / (dur_ms * 1e-3) / 1e9
        if name in kernels:  # several launches of one kernel (bins): keep each
            i = 2
            while f"{name}#{i}" in kernels:
                i += 1
            name = f"{name}#{i}"
        kernels[name] = rec
    with open(out_json, "w") as fh:
        json.dump({"source": rep, "kernels": kernels}, fh, indent=1)
    if out_md:
        with open(out_md, "w") as fh:
            fh.write(f"# ncu --set full summary ({rep.split('/')[-1]})\n\n")
            fh.write("| kernel | ms | DRAM GB (r+w) | DRAM GB/s | IPC | occ % | L1 hit % | L2 hit % | smem bank conflicts "
                     "| smem atomics (inst) | global RED (inst) | global atomics (inst) | top stalls |\n")
            fh.write("|---|---|---|---|---|---|---|---|---|---|---|---|---|\n")
            for k, r in kernels.items():
                gb = (r.get("dram_bytes_per_launch") or 0) / 1e9
                fh.write(f"| {k} | {r['duration_ms']:.3f} | {gb:.3f} | {r.get('dram_gbs', 0):.0f} | "
                         f"{(r['ipc'] or 0):.2f} | {(r['achieved_occupancy_pct'] or 0):.1f} | {(r['l1_hit_pct'] or 0):.1f} | "
                         f"{(r['l2_hit_pct'] or 0):.1f} | {r['smem_bank_conflicts']} | "
                         f"{r['shared_atomic_instructions']} | {r['global_red_instructions']} | "
                         f"{r['global_atomic_instructions']} | "
                         + ", ".join(f"{a}={b:.2f}" for a, b in r["top_stalls"]) + " |\n")
    print(json.dumps({k: {"ms": round(v["duration_ms"], 3), "dram_gb": round((v.get("dram_bytes_per_launch") or 0) / 1e9, 3)}
                      for k, v in kernels.items()}, indent=1))


def launches(csv_path, out_md):
    text = open(csv_path).read()
    start = text.find('"ID"')
    rows = list(csv.reader(io.StringIO(text[start:])))
    hdr = rows[0]
    agg = defaultdict(lambda: [0, 0.0])
    unit_of = {}
    for r in rows[1:]:
        d = dict(zip(hdr, r))
        if d.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = short_name(d["Kernel Name"])
        v = float(d["Metric Value"].replace(",", ""))
        u = d.get("Metric Unit", "nsecond")
        ms = v * {"nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0}.get(u, 1e-6)
        agg[name][0] += 1
        agg[name][1] += ms
    total = sum(v[1] for v in agg.values()) or 1
    with open(out_md, "w") as fh:
        fh.write(f"# ncu launch list ({csv_path.split('/')[-1]}): per-kernel device time, serialised & cold-cache\n\n")
        fh.write("| kernel | launches | total ms | avg ms | share |\n|---|---|---|---|---|\n")
        for k, (n, ms) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
            fh.write(f"| {k} | {n} | {ms:.3f} | {ms / n:.4f} | {ms / total * 100:.1f}% |\n")
    print(open(out_md).read())


if __name__ == "__main__":
    if sys.argv[1] == "full":
        full(sys.argv[2], sys.argv[3], sys.argv[4] if len(sys.argv) > 4 else None)
    else:
        launches(sys.argv[2], sys.argv[3])
