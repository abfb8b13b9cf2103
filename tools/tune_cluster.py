#!/usr/bin/env python
"""Fused-MVP cluster-size sweep for one config (development tool).
Each C runs in a fresh process because plans are cached per process."""
import json, os, subprocess, sys
cfg = sys.argv[1]
cs = sys.argv[2].split(",")
for c in cs:
    env = dict(os.environ, IRL_FUSED_CLUSTER=c)
    out = subprocess.run([sys.executable, os.path.join(os.path.dirname(__file__), "sweep.py"), "--configs", cfg,
                          "--irl", "0", "--reps", "10"], env=env, capture_output=True, text=True)
    for line in out.stdout.splitlines():
        d = json.loads(line)
        f = d.get("fused", {})
        print(json.dumps({"C": c, "config": d["config"], "ms": f.get("ms"), "gbs": f.get("gbs_one_read"),
                          "plan": f.get("plan"), "err": f.get("error")}), flush=True)
    if out.returncode:
        print(out.stderr[-2000:])
