"""Per source line of an ncu --import-source capture: shared-memory wavefronts
(actual, ideal, excessive) and instructions -- where the bank conflicts are.
  python tools/ncu_smem_lines.py rep.ncu-rep kernel_regex [top]"""
import csv, io, subprocess, sys
rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 20
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass", "-k",
                      f"regex:{kern}"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hi = next(i for i, r in enumerate(rows) if r and r[0] == "Line No")
hdr = rows[hi]
f = lambda x: float(x) if x not in ("", "-") else 0.0  # noqa: E731
lines = [r for r in rows[hi + 1:] if len(r) == len(hdr) and r[0] not in ("", "Line No")]
W, WI, I = hdr.index("L1 Wavefronts Shared"), hdr.index("L1 Wavefronts Shared Ideal"), hdr.index("Instructions Executed")
tw = sum(f(r[W]) for r in lines) or 1
print(f"{kern}: shared wavefronts {tw:.3e}, ideal {sum(f(r[WI]) for r in lines):.3e}")
for r in sorted(lines, key=lambda r: -(f(r[W]) - f(r[WI])))[:top]:
    print(f"{r[0]:>5} wav {f(r[W]):.2e} ideal {f(r[WI]):.2e} inst {f(r[I]):.2e}  {r[1].strip()[:70]}")
