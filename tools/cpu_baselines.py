#!/usr/bin/env python3
"""CPU columns of BASELINE.md section 4: the reference itself (oracle/_ref, else the
port) on one core of this host, CGLS iterations/s and T x + T* y pairs/s per config.
usage: python tools/cpu_baselines.py [c1 c2 ...] > profiles/<round>_cpu_baselines.jsonl"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402

for w in (sys.argv[1:] or ["c1", "c2", "c3", "c5", "c4"]):
    d = bench.cpu_baseline(w)
    d["workload"] = w.upper()
    print(json.dumps(d), flush=True)
