"""Same-box A/B of library variants (GPU box): bench.py once per (variant, repeat), the
variants interleaved, each run loading its library through RCP_LIB.  Prints one JSON line
per run (variant, config, ms_per_step, phases).

usage: [AB_ARGS='--rank 75'] python tools/lab/ab_bench.py CONFIG REPEATS name=path.so [...]
"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
cfg, reps = sys.argv[1], int(sys.argv[2])
variants = [a.split("=", 1) for a in sys.argv[3:]]
for r in range(reps):
    for name, so in variants:
        env = dict(os.environ, RCP_LIB=os.path.abspath(so))
        out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--config", cfg,
                              "--steps", "10", "--warmup", "3", "--no-cpu-baseline"]
                             + os.environ.get("AB_ARGS", "").split(),
                             capture_output=True, text=True, env=env, cwd=ROOT)
        line = [x for x in out.stdout.splitlines() if x.startswith("{")]
        if not line:
            print(json.dumps({"variant": name, "config": cfg, "error": out.stderr[-400:]}), flush=True)
            continue
        d = json.loads(line[-1])
        print(json.dumps({"variant": name, "config": cfg, "rep": r, "ms_per_step": d["ms_per_step"],
                          "phases": d.get("phases_ms_per_round")}), flush=True)
