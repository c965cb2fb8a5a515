"""Summarise an op_sweep.py JSONL: best three configurations per (level, op, kernel) and the autotuned pick."""
import json
import sys
from collections import defaultdict

rows = [json.loads(l) for l in open(sys.argv[1]) if l.startswith("{")]
best = defaultdict(list)
for r in rows:
    if "autotuned" in r:
        a = r["autotuned"]
        print(r["level"], r["op"], "autotuned:", a["kernel"], a["G"], a["U"], a["tuned_us"])
        continue
    best[(r["level"], r["op"], r["kernel"])].append(r)
for k, v in sorted(best.items()):
    v.sort(key=lambda r: r["us"])
    print(k, [(r.get("G"), r.get("U"), r["us"], r["GBps"]) for r in v[:3]])
