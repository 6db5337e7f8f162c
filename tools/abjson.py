"""Summarise bench JSON lines from A/B runs: python tools/abjson.py gpurun_out/ab1_*.json"""
import json
import sys

for f in sys.argv[1:]:
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
    except Exception as e:  # noqa: BLE001
        print(f, "unreadable", e)
        continue
    ks = {k: round(v["ms_per_launch"], 3) for k, v in d.get("kernels", {}).items()}
    print(f, d.get("ms_per_step"), ks)
