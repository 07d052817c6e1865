"""Runs bench.py once per value of an environment switch and prints one
summary line per run (value, ms/step, per-kernel us): A/B sweeps on the GPU box.
usage: python tools/sweep_env.py VAR v1 v2 ... [-- bench args]"""
import json
import os
import subprocess
import sys

argv = sys.argv[1:]
extra = []
if "--" in argv:
    i = argv.index("--")
    argv, extra = argv[:i], argv[i + 1:]
var, vals = argv[0], argv[1:]
for v in vals:
    env = dict(os.environ)
    if v != "unset":
        env[var] = v
    r = subprocess.run([sys.executable, "bench.py", "--no-cpu-baseline", "--e2e-steps", "1", *extra],
                       env=env, capture_output=True, text=True)
    line = [l for l in r.stdout.splitlines() if l.startswith("{")]
    if r.returncode != 0 or not line:
        print(json.dumps({var: v, "error": r.stderr[-800:]}), flush=True)
        continue
    d = json.loads(line[-1])
    ks = {k: round(x["avg_us"], 1) for k, x in d.get("kernels", {}).items()}
    print(json.dumps({var: v, "config": d["config"]["workload"], "value": d["value"], "ms": d["ms_per_step"],
                      "frac": d["roofline"]["frac"], "kernels_us": ks}), flush=True)
