"""Top SASS instructions of a kernel by executed warp-instructions (ncu source page, sass view).
  python tools/ncu_sass_top.py rep.ncu-rep kernel_regex [N]"""
import csv, io, subprocess, sys
rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 60
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass", "-k", f"regex:{kern}"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hi = next(i for i, r in enumerate(rows) if r and ("Address" in r[0] or r[0] == "#"))
hdr = rows[hi]
f = lambda x: float(x) if x not in ("", "-") else 0.0  # noqa: E731
I = hdr.index("Instructions Executed")
S = hdr.index("Warp Stall Sampling (All Samples)") if "Warp Stall Sampling (All Samples)" in hdr else None
src = hdr.index("Source")
lines = [r for r in rows[hi + 1:] if len(r) == len(hdr)]
tot = sum(f(r[I]) for r in lines)
print("total", tot, "hdr", hdr[:4])
mode = sys.argv[4] if len(sys.argv) > 4 else "addr"
if mode == "addr":
    for r in lines:
        if f(r[I]) >= tot * 0.002:
            print(f"{r[0]:>8} {f(r[I]) / 1e6:9.1f}M {f(r[S]) if S else 0:7.0f}  {r[src][:90]}")
