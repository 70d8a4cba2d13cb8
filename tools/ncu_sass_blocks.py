"""Hot basic blocks of a kernel from an ncu report: runs of SASS instructions with the same
execution count, ranked by share of executed warp-instructions."""
import csv, io, subprocess, sys
rep, kern = sys.argv[1], sys.argv[2]
div = float(sys.argv[3]) if len(sys.argv) > 3 else 1.0
top = int(sys.argv[4]) if len(sys.argv) > 4 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass", "-k", f"regex:{kern}"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hi = [i for i, r in enumerate(rows) if r and r[0] == "Address"][0]
hdr = rows[hi]
data = [dict(zip(hdr, r)) for r in rows[hi + 1:] if len(r) == len(hdr) and r[0] != "Address"]
f = lambda x: float(x) if x not in ("", "-") else 0.0  # noqa: E731
I = "Instructions Executed"
tot = sum(f(d[I]) for d in data)
blocks = []
cur = None
for d in data:
    c = f(d[I])
    if cur and c == cur["c"]:
        cur["n"] += 1
        cur["ops"].append(d["Source"].strip().split()[0])
    else:
        cur = {"start": d["Address"][-5:], "n": 1, "c": c, "ops": [d["Source"].strip().split()[0]]}
        blocks.append(cur)
blocks.sort(key=lambda b: -b["c"] * b["n"])
print(f"total {tot:.3e} warp-instr, {tot / div:.1f} per unit")
for b in blocks[:top]:
    print(f"{b['start']} n={b['n']:3d} per-unit {b['c'] / div:8.2f} share {b['c'] * b['n'] / tot * 100:5.1f}%  "
          + " ".join(b["ops"][:14]))
