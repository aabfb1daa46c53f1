"""Print ms_per_step and the per-kernel ms of a bench JSON line on stdin whose names contain the arguments."""
import json
import sys

d = json.loads(sys.stdin.read())
k = d.get("kernels_ms_per_step", {})
print(round(d["ms_per_step"], 3), {n: v for n, v in k.items() if any(a in n for a in sys.argv[1:])})
