"""A2-in-TMEM plan against the TMEM plan (LS_NO_A2T=1 in a dev build) over N2 and rank."""
import os
import subprocess
import sys

shapes = sys.argv[1] if len(sys.argv) > 1 else "256x256x256,256x512x256,256x1024x128,1024x256x64"
for R in (5, 9, 21, 41, 57):
    for env in ("", "1"):
        e = dict(os.environ, LS_LAB_ROOT=os.environ.get("LS_LAB_ROOT", "/root/repo"))
        e.pop("LS_NO_A2T", None)
        if env:
            e["LS_NO_A2T"] = env
        r = subprocess.run([sys.executable, "tools/lab/small_grid.py", "--shapes", shapes, "--R", str(R), "--reps", "20"],
                           capture_output=True, text=True, env=e)
        print(f"R={R} {'tmem' if env else 'a2t '}: " + " | ".join(ln.split(':', 1)[1].strip() for ln in r.stdout.splitlines()), flush=True)
