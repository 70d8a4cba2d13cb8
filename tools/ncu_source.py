"""Summarise an ncu report per CUDA source line: share of executed warp-instructions and
of warp-stall samples (uses --print-source cuda,sass, aggregated rows)."""
import csv, io, subprocess, sys
rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass", "-k",
                      f"regex:{kern}"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hi = next(i for i, r in enumerate(rows) if r and r[0] == "Line No")
hdr = rows[hi]
f = lambda x: float(x) if x not in ("", "-") else 0.0  # noqa: E731
lines = [r for r in rows[hi + 1:] if len(r) == len(hdr) and r[0] not in ("", "Line No")]
I, S = hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
ti = sum(f(r[I]) for r in lines) or 1
ts = sum(f(r[S]) for r in lines) or 1
print(f"{kern}: total warp-instructions {ti:.3e}, stall samples {ts:.0f}")
for r in sorted(lines, key=lambda r: -f(r[S]))[:top]:
    print(f"{r[0]:>5} inst {f(r[I]) / ti * 100:5.1f}% stall {f(r[S]) / ts * 100:5.1f}%  {r[1].strip()[:80]}")
