"""Config 2 timing + reuse-path row counts for a few SPGEMM_REUSE_ROWS settings (dev aid)."""
import os, subprocess, sys
for r in sys.argv[1:] or ["auto"]:
    env = dict(os.environ, SPGEMM_DEBUG_REUSE="1")
    if r != "auto":
        env["SPGEMM_REUSE_ROWS"] = r
    out = subprocess.run([sys.executable, "tools/quick_timing.py", "2"], capture_output=True, text=True, env=env)
    lines = out.stdout.strip().splitlines()[-1:] + sorted(set(out.stderr.strip().splitlines()))[-2:]
    print("rows/warp", r, *lines, sep="\n  ")
