"""Print the JSON lines from the last gpurun call's stdout tail (gpurun_out/.last_call.json)."""
import json
import os
import sys

p = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "gpurun_out", ".last_call.json")
d = json.load(open(p))
keys = sys.argv[1:]
for line in d.get("stdout_tail", "").splitlines():
    line = line.strip()
    if line.startswith("{"):
        try:
            r = json.loads(line)
        except ValueError:
            continue
        print({k: (round(r[k], 2) if isinstance(r.get(k), float) else r.get(k)) for k in keys} if keys else r)
    elif line:
        print(line)
